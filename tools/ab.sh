# A/B of engine option sets on one box: bash tools/ab.sh "<cfgs>" "<optset> <optset> ..."
# an optset is comma-separated key=value pairs ("-" = defaults)
CFGS=${1:-"cfg4 cfg3"}
SETS=${2:-"-"}
for cfg in $CFGS; do for rep in 1 2; do for set in $SETS; do
  args=""; if [ "$set" != "-" ]; then for kv in ${set//,/ }; do args="$args --opt $kv"; done; fi
  python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu $args 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; print('$cfg $set', round(d['value']), round(d['ms_per_step'],3), round(r['achieved']), round(r['frac'],3), round(r.get('gather_ms',0),3), d.get('clocks',{}).get('sm_mhz'))"
done; done; done
