# quick A/B: separate vs fused projected leaf pass: bash tools/pf_ab2.sh <tag> [configs]
TAG=${1:-pf}
CFGS=${2:-"cfg4 cfg3v2"}
mkdir -p gpurun_out
for cfg in $CFGS; do
  python bench.py --config $cfg --no-cpu --no-e2e --steps 10 --opt proj_fuse=0 > gpurun_out/${TAG}_${cfg}_sep.json 2>&1
  python bench.py --config $cfg --no-cpu --no-e2e --steps 10 > gpurun_out/${TAG}_${cfg}_fused.json 2>&1
  python bench.py --config $cfg --no-cpu --no-e2e --steps 10 --opt pf_min_blocks=0 > gpurun_out/${TAG}_${cfg}_mb0.json 2>&1
done
for f in gpurun_out/${TAG}_*.json; do echo "$f $(tail -1 $f | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])' 2>/dev/null)"; done
