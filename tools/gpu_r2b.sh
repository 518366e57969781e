#!/bin/bash
# Round-2: full -m gpu suite + bench lines of every workload (evidence).
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
for w in full sharded prefill batched; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w rc=$?"
  head -c 600 gpurun_out/bench_$w.json; echo
done
