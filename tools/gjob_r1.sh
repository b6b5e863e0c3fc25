# Round-1 profiling job (run under gpurun): bench line, launch list, one --set full capture
# per top kernel, exported to CSV on the box (the .ncu-rep files are large).
set -x
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench_full.log 2>&1; tail -c 3000 gpurun_out/prof/bench_full.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv python bench.py --steps 16 --warmup 8 --quick > gpurun_out/prof/ncu1.log 2>&1
cap() {  # name regex skip
  ncu --set full --clock-control none --import-source on -k regex:$2 --launch-skip $3 --launch-count 1 -o /tmp/$1 -f python bench.py --steps 2 --warmup 8 --quick > gpurun_out/prof/ncu_$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/prof/$1_raw.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/prof/$1_details.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/$1_sass.csv 2>&1
  ls -la /tmp/$1.ncu-rep
  if [ "$1" = trav ]; then cp /tmp/$1.ncu-rep gpurun_out/prof/; fi
}
cap trav k_trav_persistent 40
cap eval k_recip_eval 2
cap shade k_shade 40
# gpurun copies back at most 64 MiB
if [ $(du -sm gpurun_out | cut -f1) -gt 60 ]; then rm -f gpurun_out/prof/*_sass.csv; fi
du -sh gpurun_out/prof; ls -la gpurun_out/prof
