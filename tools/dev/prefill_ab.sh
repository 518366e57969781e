# prefill bench: tcgen05 kernel vs the mma.sync kernel (TS_PREFILL_MMA_SYNC=1)
mkdir -p gpurun_out
for v in tc mma; do
  if [ $v == mma ]; then export TS_PREFILL_MMA_SYNC=1; else unset TS_PREFILL_MMA_SYNC; fi
  timeout 200 python bench.py --workload prefill --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['roofline'].get('tensor'))"
done
