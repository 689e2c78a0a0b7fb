# A/B of engine options on one box: tools/ab_fuse.sh "<cfgs>" "<opt settings>"
CFGS=${1:-"cfg4 cfg3"}
OPTS=${2:-"fuse_gather=0 fuse_gather=1"}
for cfg in $CFGS; do for rep in 1 2; do for o in $OPTS; do
python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu --opt $o 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; print('$cfg $o', round(d['value']), round(d['ms_per_step'],3), round(r['achieved']), round(r['frac'],3), d.get('clocks',{}).get('sm_mhz'))"
done; done; done
