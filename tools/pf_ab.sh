# A/B of the fused projected-leaf pass on cfg4 / cfg3v2 / cfg4v2: bash tools/pf_ab.sh <tag> [configs]
TAG=${1:-pf}
CFGS=${2:-"cfg4 cfg4v2 cfg3v2"}
mkdir -p gpurun_out
for cfg in $CFGS; do
  python bench.py --config $cfg --no-cpu --no-e2e --steps 10 --opt proj_fuse=0 > gpurun_out/${TAG}_${cfg}_sep.json 2>&1
  for o in "pf_u=2" "pf_u=1" "pf_u=4" "pf_u=2 --opt pf_min_blocks=2"; do
    t=$(echo $o | tr -d ' -' | tr '=' '_')
    python bench.py --config $cfg --no-cpu --no-e2e --steps 10 --opt $o > gpurun_out/${TAG}_${cfg}_${t}.json 2>&1
  done
done
for f in gpurun_out/${TAG}_*.json; do echo "$f $(tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])' 2>/dev/null)"; done
