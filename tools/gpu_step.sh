#!/bin/bash
# Dev loop for the step kernel: smoke, decode parity tests, quick timing + phase trace.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
cat gpurun_out/smoke.log | tail -5
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "${PYTEST_K:-decode or config2 or zero}" > gpurun_out/pytest_step.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_step.log
tail -25 gpurun_out/pytest_step.log
QT_NOTRACE= timeout 300 python tools/quick_time.py 131072 > gpurun_out/quick_time.log 2>&1
head -12 gpurun_out/quick_time.log
