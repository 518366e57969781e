# dev: fold the P.V delta every F tiles -- error and kernel time per F
for F in 1 2 4 8; do
  echo "== F=$F"; TS_PREFILL_FOLD=$F timeout 120 python tools/dev/prefill_err.py 2>&1 | tail -1
  TS_PREFILL_FOLD=$F timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lp_f$F.csv \
    python bench.py --workload prefill --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  python tools/summarize_ncu.py launches gpurun_out/lp_f$F.csv | grep -E "prefill_tc"
done
