#!/bin/bash
# all bench workloads on one GPU (round evidence)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
cat gpurun_out/bench.json
for w in batched prefill; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -2 gpurun_out/bench_$w.err
  cat gpurun_out/bench_$w.json
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --workload sharded --steps 20 --warmup 3 > gpurun_out/bench_sharded1.json 2> gpurun_out/bench_sharded1.err; tail -3 gpurun_out/bench_sharded1.err
cat gpurun_out/bench_sharded1.json
