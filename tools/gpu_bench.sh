#!/bin/bash
# bench line + launch list + ncu --set full of the decode kernel (round evidence)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 2 \
  -o gpurun_out/prof_decode -f python tools/profile_decode.py 131072 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
