# A/B job: Stage-2a CUDA graph on/off (PXG_NO_TRACE_GRAPH) and the k_conn_mis launch bounds variant
mkdir -p gpurun_out/ab
for round in 1 2; do
  for arm in graph nograph mis8; do
    for cfg in C2 C4; do
      unset PXG_LIBRARY PXG_NO_TRACE_GRAPH
      [ "$arm" = nograph ] && export PXG_NO_TRACE_GRAPH=1
      [ "$arm" = mis8 ] && export PXG_LIBRARY=$PWD/ab/libpxg_mis8.so
      st=32; [ "$cfg" = C4 ] && st=16
      v=$(timeout 600 python bench.py --config $cfg --steps $st --warmup 8 --quick 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" 2>&1)
      echo "round $round $cfg $arm: $v"
    done
  done
done
