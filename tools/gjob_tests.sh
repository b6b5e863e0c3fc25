mkdir -p gpurun_out/t
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/t/pytest_gpu.log 2>&1; echo "pytest exit $?"
grep -E "passed|failed|Error|assert" gpurun_out/t/pytest_gpu.log | tail -15
