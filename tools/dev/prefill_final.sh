# prefill evidence after the balanced split: full -m gpu suite, bench line, launch lists, ncu --set full
O=gpurun_out/pf2
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
timeout 300 python bench.py --workload prefill --steps 20 --warmup 5 > $O/bench_prefill.json 2> $O/bench_prefill.err; echo "bench rc=$?"
for v in tc mma; do
  if [ $v == mma ]; then export TS_PREFILL_MMA_SYNC=1; else unset TS_PREFILL_MMA_SYNC; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_prefill_$v.csv \
    python bench.py --workload prefill --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
unset TS_PREFILL_MMA_SYNC
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_tc_kernel -c 1 -o $O/prof_prefill -f \
  python bench.py --workload prefill --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1; echo "ncu rc=$?"
python tools/dev/prefill_err.py > $O/err.log 2>&1; tail -1 $O/err.log
TS_PREFILL_TRACE=$O/trace.bin python tools/dev/prefill_err.py > /dev/null 2>&1; python tools/dev/ptrace_split.py $O/trace.bin > $O/trace_summary.txt 2>&1; head -1 $O/trace_summary.txt
