#!/bin/bash
# GPU parity tests + phase trace + ncu full capture of a miss and a hit step (dev loop)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python tools/quick_time.py 131072 > gpurun_out/quick_time.log 2>&1
cat gpurun_out/quick_time.log
if [ "$1" == "prof" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 2 \
  -o gpurun_out/prof_decode -f python tools/profile_decode.py 131072 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
fi
