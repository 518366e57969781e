#!/bin/bash
# Phase trace + one ncu --set full capture of the fused decode kernel (miss + hit step).
mkdir -p gpurun_out
timeout 300 python tools/quick_time.py 131072 > gpurun_out/quick_time.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 2 \
  -o gpurun_out/prof_decode -f python tools/profile_decode.py 131072 > gpurun_out/ncu_full.log 2>&1
echo done
