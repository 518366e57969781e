# dev: the warp-specialised tcgen05 prefill -- error + per-tile trace + tests + ncu launch list
mkdir -p gpurun_out
TS_PREFILL_TRACE=gpurun_out/ptrace.bin timeout 200 python tools/dev/prefill_err.py > gpurun_out/ws_trace.log 2>&1; echo "err rc=$?"; tail -3 gpurun_out/ws_trace.log
python tools/dev/ptrace.py gpurun_out/ptrace.bin
bash tools/dev/tc_prefill.sh
bash tools/dev/prefill_ncu_ab.sh
