#!/bin/bash
# Phase traces of several library builds (dev): _ab/lib_<name>.so for each name given.
mkdir -p gpurun_out
for v in "$@"; do
  echo "=== $v"
  TS_LIB_PATH=$PWD/_ab/lib_$v.so timeout 200 python tools/quick_time.py ${QT_N:-131072} 2>&1 | grep -E "^(miss|hit)" | grep -v "all-CTA"
done
