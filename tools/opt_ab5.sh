# A/B of engine options on the 28|28 configs: bash tools/opt_ab5.sh <tag> "<opt set 1>" "<opt set 2>" ...
TAG=$1; shift 1
mkdir -p gpurun_out
for cfg in cfg5 cfg5f; do
  w=16; [ $cfg = cfg5f ] && w=2
  i=0
  for set in "$@"; do
    args=""; for kv in $set; do args="$args --opt $kv"; done
    python bench.py --config $cfg --window $w --no-cpu --no-e2e --steps 2 --warmup 1 $args > gpurun_out/${TAG}_${cfg}_$i.json 2>&1
    echo "$cfg [$set] $(tail -1 gpurun_out/${TAG}_${cfg}_$i.json | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],1), d["roofline"]["classes"].get("leaf",{}).get("frac"))' 2>/dev/null)"
    i=$((i+1))
  done
done
