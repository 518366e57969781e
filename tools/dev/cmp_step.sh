mkdir -p gpurun_out
for r in 1 2; do
TS_STEP=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', d['value'], d['miss_step_us'], d['hit_step_us'], d['e2e']['value'])"
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old ', d['value'], d['miss_step_us'], d['hit_step_us'], d['e2e']['value'])"
done
bash tools/ab_trace.sh new
