mkdir -p gpurun_out/conv
timeout 900 python -m pytest tests/test_convergence.py -m gpu -x -q -s > gpurun_out/conv/pytest.log 2>&1; echo "conv pytest exit $?"; tail -12 gpurun_out/conv/pytest.log
bash tools/gjob_prof.sh r1b C2 C4
