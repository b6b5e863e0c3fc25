# Round evidence (run under gpurun, one GPU): tests, smoke, bench lines for every config, launch
# lists and ncu --set full captures exported to CSV. Each ncu run only after the same command
# exited 0 without ncu.
O=gpurun_out/final4; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_C2.log 2>&1; echo "bench C2 exit $?"; tail -1 $O/bench_C2.log > $O/bench_C2.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.log 2>&1; echo "bench ref exit $?"; tail -1 $O/bench_ref.log
for cfg in C1 C3 C4; do
  timeout 900 python bench.py --config $cfg --steps 16 --warmup 8 --e2e-spp 16 --no-cpu-baseline > $O/bench_$cfg.log 2>&1; echo "bench $cfg exit $?"; tail -1 $O/bench_$cfg.log > $O/bench_$cfg.json
done
timeout 1200 python bench.py --config C5 --steps 4 --warmup 3 --e2e-spp 2 --no-cpu-baseline > $O/bench_C5.log 2>&1; echo "bench C5 exit $?"; tail -1 $O/bench_C5.log > $O/bench_C5.json
for cfg in C2 C4; do
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$cfg.csv \
      python bench.py --config $cfg --steps 16 --warmup 8 --quick > /dev/null 2>&1; echo "launches $cfg rc=$?"
  python tools/launch_summary.py $O/launches_$cfg.csv > $O/launch_shares_$cfg.txt 2>&1; head -12 $O/launch_shares_$cfg.txt
done
cap() {  # cfg name regex skip
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$3 --launch-skip $4 --launch-count 1 \
      -o /tmp/$1_$2 -f python bench.py --config $1 --steps 2 --warmup 8 --quick > $O/ncu_$1_$2.log 2>&1
  echo "capture $1 $2 rc=$?"
  ncu -i /tmp/$1_$2.ncu-rep --page details --csv > $O/$1_$2_details.csv 2>&1
  ncu -i /tmp/$1_$2.ncu-rep --page raw --csv > $O/$1_$2_raw.csv 2>&1
}
cap C2 trav k_trav_persistent 60
cap C4 trav k_trav_persistent 60
cap C2 recipwave k_recip_eval_wave 2
cap C4 recipwave k_recip_eval_wave 2
cap C2 connmis k_conn_mis 3
cap C2 shade k_shade 40
du -sh $O
