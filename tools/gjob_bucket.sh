timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bdpt or proxy_render or tiles" 2>&1 | tail -2
bash tools/gjob_ab.sh "C2 C4" default ab/libpxg_base5.so
