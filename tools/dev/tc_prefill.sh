mkdir -p gpurun_out
timeout 150 python -m pytest tests/test_gpu_parity.py tests/test_gpu_surface.py tests/test_gpu_head_vote.py -x -q -k "prefill or chunk_mean or select_for_chunk" > gpurun_out/tc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc_tests.log
tail -25 gpurun_out/tc_tests.log
timeout 150 python bench.py --workload prefill --steps 10 --warmup 3 > gpurun_out/tc_bench.json 2>gpurun_out/tc_bench.err; echo "bench rc=$?"
head -c 400 gpurun_out/tc_bench.json
