# dev: balanced (split) tcgen05 prefill vs one unit per CTA -- error, tests, kernel time
mkdir -p gpurun_out
timeout 120 python tools/dev/prefill_err.py > gpurun_out/ps_err.log 2>&1; echo "err rc=$?"; tail -1 gpurun_out/ps_err.log
TS_PREFILL_NO_SPLIT=1 timeout 120 python tools/dev/prefill_err.py > gpurun_out/ps_err2.log 2>&1; echo "err(no split) rc=$?"; tail -1 gpurun_out/ps_err2.log
timeout 600 python -m pytest tests -m gpu -q -x -k "prefill or chunk or config5 or wrapper" 2>&1 | tail -2
for v in split nosplit; do
  if [ $v == nosplit ]; then export TS_PREFILL_NO_SPLIT=1; else unset TS_PREFILL_NO_SPLIT; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lp_$v.csv \
    python bench.py --workload prefill --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "== $v"; python tools/summarize_ncu.py launches gpurun_out/lp_$v.csv | grep -E "prefill_tc|prep_tc"
done
unset TS_PREFILL_NO_SPLIT
timeout 300 python bench.py --workload prefill --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'])"
