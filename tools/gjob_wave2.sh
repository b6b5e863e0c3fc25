timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "proxy or recip or pretrace" 2>&1 | tail -2
bash tools/gjob_env.sh "C4" none PXG_RECIP_WAVE=0
mkdir -p gpurun_out/wave
for w in 1 0; do
  PXG_RECIP_WAVE=$w timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/wave/l$w.csv python bench.py --config C4 --steps 8 --warmup 8 --quick > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/wave/l$w.csv 8 
done
