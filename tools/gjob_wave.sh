timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -x -q -k "proxy or recip or pool or pretrace or diag" 2>&1 | tail -3
bash tools/gjob_env.sh "C2 C4" none PXG_RECIP_WAVE=0
