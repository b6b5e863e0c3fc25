timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c2_small or c4_small or c1_small or caustic" 2>&1 | tail -2
bash tools/gjob_ab.sh "C2 C4" default ab/libpxg_base2.so
