# C3/C4 probe (run under gpurun): new parity cases, then bench lines on the large configs.
mkdir -p gpurun_out/big
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c3 or c4" -s > gpurun_out/big/pytest_c34.log 2>&1; echo "pytest exit $?"
grep -E "mismatch|equal|over tol|passed|failed|Error" gpurun_out/big/pytest_c34.log | tail -30
for cfg in C3 C4; do
  timeout 900 python bench.py --config $cfg --steps 16 --warmup 8 --e2e-spp 16 --no-cpu-baseline > gpurun_out/big/bench_$cfg.log 2>&1; echo "bench $cfg exit $?"
  tail -c 2500 gpurun_out/big/bench_$cfg.log
done
