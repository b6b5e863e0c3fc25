# Profiling job (run under gpurun, one GPU): per config, the bench line without a profiler, the
# launch list (gpu__time_duration, serialised) and one --set full capture of the top kernel
# exported to CSV. Usage: bash tools/gjob_prof.sh TAG CFG [CFG...]
TAG=$1; shift
mkdir -p gpurun_out/prof_$TAG
for CFG in "$@"; do
  O=gpurun_out/prof_$TAG/$CFG
  mkdir -p $O
  timeout 900 python bench.py --config $CFG --steps 16 --warmup 8 --quick > $O/bench_quick.log 2>&1; rc=$?
  echo "$CFG bench rc=$rc"; tail -c 600 $O/bench_quick.log; echo
  [ $rc -ne 0 ] && continue
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
      python bench.py --config $CFG --steps 16 --warmup 8 --quick > $O/ncu_launches.log 2>&1
  echo "launches rc=$?"; python tools/launch_summary.py $O/launches.csv > $O/launch_shares.txt 2>&1; head -14 $O/launch_shares.txt
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_trav_persistent --launch-skip 60 --launch-count 1 \
      -o /tmp/trav_$CFG -f python bench.py --config $CFG --steps 2 --warmup 8 --quick > $O/ncu_trav.log 2>&1
  echo "trav capture rc=$?"
  ncu -i /tmp/trav_$CFG.ncu-rep --page raw --csv > $O/trav_raw.csv 2>&1
  ncu -i /tmp/trav_$CFG.ncu-rep --page details --csv > $O/trav_details.csv 2>&1
  ncu -i /tmp/trav_$CFG.ncu-rep --page source --csv --print-source sass > $O/trav_sass.csv 2>&1
done
du -sh gpurun_out/prof_$TAG
