#!/bin/bash
# A/B step timing of two builds of the library (dev): _ab/lib_base.so vs _ab/lib_new.so,
# interleaved runs of tools/quick_time.py (miss / hit back-to-back us per step)
for r in 1 2 3; do
  for v in base new; do
    res=$(QT_NOTRACE=1 TS_LIB_PATH=$PWD/_ab/lib_$v.so timeout 120 python tools/quick_time.py ${1:-131072} 2>&1 | grep -E "^(miss|hit): [0-9]" | sed -n '3p;6p' | awk '{print $2}' | paste -sd' ')
    echo "$v miss/hit: $res"
  done
done
