timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "traversal or occlusion or recip or pretrace or c2_small" 2>&1 | tail -2
bash tools/gjob_env.sh "C2 C4" none PXG_LEAF=2 PXG_LEAF=3
