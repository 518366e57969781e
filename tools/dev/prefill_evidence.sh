# prefill evidence: the prefill-related GPU tests, bench line, ncu launch lists
# (tcgen05 vs mma.sync), one --set full capture of prefill_tc_kernel
mkdir -p gpurun_out/pf
timeout 900 python -m pytest tests -m gpu -q -k "prefill or chunk or config5 or select_for_chunk" > gpurun_out/pf/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pf/pytest.log
timeout 300 python bench.py --workload prefill --steps 20 --warmup 5 > gpurun_out/pf/bench_prefill.json 2> gpurun_out/pf/bench_prefill.err; echo "bench rc=$?"; head -c 600 gpurun_out/pf/bench_prefill.json; echo
bash tools/dev/prefill_ncu_ab.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_tc_kernel -c 1 -o gpurun_out/pf/prefill_tc_full \
  python bench.py --workload prefill --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/pf/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/dev/prefill_err.py > gpurun_out/pf/err.log 2>&1; cat gpurun_out/pf/err.log | tail -1
TS_PREFILL_MMA_SYNC=1 python tools/dev/prefill_err.py >> gpurun_out/pf/err.log 2>&1; tail -1 gpurun_out/pf/err.log
