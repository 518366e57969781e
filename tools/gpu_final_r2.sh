#!/bin/bash
# Round-2 evidence run: full -m gpu suite, smoke, every bench workload, the
# reference arm, the ncu launch list of the default bench command, ncu --set
# full of the decode kernel (miss + hit) and of the prefill kernel, phase traces.
O=${O:-gpurun_out/final3}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_decode.json 2> $O/bench_decode.err; echo "decode rc=$?"
for w in full batched prefill sharded; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > $O/bench_$w.json 2> $O/bench_$w.err; echo "$w rc=$?"
done
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "reference rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_decode.csv \
  python bench.py --steps 8 --warmup 3 --no-cpu-baseline > $O/bench_under_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 2 \
  -o $O/prof_decode -f python tools/profile_decode.py 131072 > $O/ncu_full_decode.log 2>&1; echo "ncu decode rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_tc_kernel -c 1 -o $O/prof_prefill -f \
  python bench.py --workload prefill --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full_prefill.log 2>&1; echo "ncu prefill rc=$?"
timeout 300 python tools/quick_time.py 131072 > $O/quick_time.log 2>&1
timeout 300 python tools/e2e_time.py > $O/e2e_time.log 2>&1
for f in $O/bench_*.json; do echo "$f"; head -c 400 $f; echo; done
