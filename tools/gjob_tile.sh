timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tiles or traversal or c2_small or c4_small" 2>&1 | tail -3
bash tools/gjob_env.sh "C2 C3" none PXG_NODEQ=1
mkdir -p gpurun_out/c5
timeout 1200 python bench.py --config C5 --steps 4 --warmup 3 --e2e-spp 2 --no-cpu-baseline > gpurun_out/c5/bench.log 2>&1; echo "C5 bench rc=$?"; tail -c 3000 gpurun_out/c5/bench.log
