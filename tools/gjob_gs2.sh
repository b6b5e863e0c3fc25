bash tools/gjob_env.sh "C2 C4" none PXG_GS_PER_SM=16 PXG_GS_PER_SM=256
PXG_LIBRARY=$PWD/ab/libpxg_base3.so bash tools/gjob_env.sh "C2 C4" none
