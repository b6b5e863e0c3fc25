# A/B job: bash tools/gjob_ab.sh "CFG..." LIB... (LIB "default" = in-tree libpxg.so); two rounds, alternating
CFGS=$1; shift
mkdir -p gpurun_out/ab
for round in 1 2; do
  for lib in "$@"; do
    for cfg in $CFGS; do
      if [ "$lib" = default ]; then unset PXG_LIBRARY; else export PXG_LIBRARY=$PWD/$lib; fi
      st=32; [ "$cfg" = C4 ] && st=16; [ "$cfg" = C3 ] && st=16
      v=$(timeout 600 python bench.py --config $cfg --steps $st --warmup 8 --quick 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" 2>&1)
      echo "round $round $cfg $lib: $v"
    done
  done
done
