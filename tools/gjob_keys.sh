timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "proxy_render or pool or pretrace or diag or truncated" 2>&1 | tail -2
bash tools/gjob_ab.sh "C2 C4" default ab/libpxg_base4.so
