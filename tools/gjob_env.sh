# bash tools/gjob_env.sh "CFGS" "ENV1" "ENV2" ...  (ENV e.g. PXG_LEAF=2, or "none")
CFGS=$1; shift
for round in 1 2; do
  for e in "$@"; do
    for cfg in $CFGS; do
      st=32; [ "$cfg" = C4 ] && st=16; [ "$cfg" = C3 ] && st=16
      if [ "$e" = none ]; then envs=""; else envs="$e"; fi
      v=$(env $envs timeout 600 python bench.py --config $cfg --steps $st --warmup 8 --quick 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" 2>&1)
      echo "round $round $cfg [$e]: $v"
    done
  done
done
