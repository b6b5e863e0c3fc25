PXG_TRACE_FUSED=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bdpt or proxy_render or tiles" 2>&1 | tail -2
bash tools/gjob_env.sh "C2 C4" none PXG_TRACE_FUSED=1
PXG_LIBRARY=$PWD/ab/libpxg_f5.so bash tools/gjob_env.sh "C2 C4" PXG_TRACE_FUSED=1
