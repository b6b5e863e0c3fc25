timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bdpt or c2_small or c4_small or caustic_box" 2>&1 | tail -2
bash tools/gjob_ab.sh "C2 C4" default ab/libpxg_gs_shade6.so ab/libpxg_base3.so
