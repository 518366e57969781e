#!/bin/bash
# Evidence run: the full -m gpu suite, smoke, every bench workload, the
# reference arm, and the ncu launch list of the default bench command.
mkdir -p gpurun_out/final
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.log
tail -3 gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.log
tail -2 gpurun_out/final/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final/bench_decode.json 2> gpurun_out/final/bench_decode.err; echo "decode rc=$?"
for w in full sharded prefill batched; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/final/bench_$w.json 2> gpurun_out/final/bench_$w.err; echo "$w rc=$?"
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err; echo "reference rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches.csv \
  python bench.py --steps 6 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
for f in gpurun_out/final/bench_*.json; do echo "$f"; head -c 300 $f; echo; done
