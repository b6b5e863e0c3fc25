mkdir -p gpurun_out/pt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pt" -s > gpurun_out/pt/pytest.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/pt/pytest.log
timeout 1200 python tools/convergence_probe.py 2>&1 | tee gpurun_out/pt/probe.log
