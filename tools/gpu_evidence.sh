#!/bin/bash
# round evidence: full GPU test suite, all bench workloads, launch list + ncu --set full of the decode kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json | cut -c1-300
for w in batched prefill; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --workload sharded --steps 20 --warmup 3 > gpurun_out/bench_sharded1.json 2> gpurun_out/bench_sharded1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 2 \
  -o gpurun_out/prof_decode -f python tools/profile_decode.py 131072 > gpurun_out/ncu_full.log 2>&1
timeout 300 python tools/quick_time.py 131072 > gpurun_out/quick_time.log 2>&1
echo done
