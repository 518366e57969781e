#!/bin/bash
# dev timing: back-to-back step time with the fused kernel ended at successive
# stop points (TS_DEBUG_FLAGS = n << 8: 15 = prologue only, 2 = after the scan; 0 = full step)
for f in 3840 256 512 768 1024 1280 1536 1792 2048 2304 2560 2816 3072 3328 0; do
  r=$(TS_DEBUG_FLAGS=$f timeout 120 python tools/quick_time.py 131072 2>&1 | grep -E "^(miss|hit): [0-9]" | sed -n '3p;6p' | awk '{print $2}' | paste -sd' ')
  echo "flags=$f stop=$((f>>8)) miss/hit us: $r"
done
