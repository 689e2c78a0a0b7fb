# A/B of engine options over configs: bash tools/ab.sh "<opts A>" "<opts B>" ...
# each opts string is a space-separated list of key=value; configs in $CFGS (default cfg4 cfg3 cfg5)
CFGS=${CFGS:-"cfg4 cfg3 cfg5"}
for o in "$@"; do
  args=""; for kv in $o; do args="$args --opt $kv"; done
  for c in $CFGS; do
    extra=""; [ $c = cfg5 ] && extra="--window 32 --steps 2"; [ $c = cfg5f ] && extra="--window 4 --steps 1"
    python bench.py --config $c --no-cpu --no-e2e $extra $args > gpurun_out/ab.json 2> gpurun_out/ab.err
    python -c "import json,sys; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$c', '[$o]', round(d['value'],1), round(d['roofline']['frac'],3), round(d['ms_per_step'],3))" 2>/dev/null || { echo "$c [$o] FAILED"; tail -3 gpurun_out/ab.err; }
  done
done
