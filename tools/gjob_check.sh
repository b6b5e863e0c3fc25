# Quick GPU check (run under gpurun): gpu tests, smoke, default bench line.
mkdir -p gpurun_out/chk
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/chk/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/chk/pytest_gpu.log
tail -5 gpurun_out/chk/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk/smoke.log 2>&1; echo "smoke exit $?"; tail -3 gpurun_out/chk/smoke.log
timeout 600 python bench.py > gpurun_out/chk/bench.log 2>&1; echo "bench exit $?"; tail -c 2500 gpurun_out/chk/bench.log
