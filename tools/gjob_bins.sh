bash tools/gjob_ab.sh "C2 C4" default ab/libpxg_nodeq.so
bash tools/gjob_env.sh "C4" PXG_SAH_BINS=32 PXG_SAH_BINS=8
