PXG_RAY_SORT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c2_small or c4_small or c1_small" 2>&1 | tail -2
bash tools/gjob_env.sh "C2 C4" none PXG_RAY_SORT=1
