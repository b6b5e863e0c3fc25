# Round evidence job: GPU tests, smoke, default bench line, launch lists + trav captures.
mkdir -p gpurun_out/full
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/full/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/full/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full/smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/full/smoke.log
timeout 900 python bench.py > gpurun_out/full/bench.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/full/bench.log > gpurun_out/full/bench_line.json; tail -c 1500 gpurun_out/full/bench.log
bash tools/gjob_prof.sh r1c C2 C4
