# kernel durations (ncu launch list) of one prefill step: tcgen05 vs mma.sync
mkdir -p gpurun_out
for v in tc mma; do
  if [ $v == mma ]; then export TS_PREFILL_MMA_SYNC=1; else unset TS_PREFILL_MMA_SYNC; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_prefill_$v.csv \
    python bench.py --workload prefill --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "== $v"; python tools/summarize_ncu.py launches gpurun_out/launches_prefill_$v.csv | grep -E "prefill|decode_kernel|chunk_mean|split3|windows"
done
