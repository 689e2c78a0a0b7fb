# A/B of engine options: bash tools/opt_ab.sh <tag> "<configs>" "<opt set 1>" "<opt set 2>" ...
# each opt set is a space-separated list of key=value (empty string = defaults)
TAG=$1; CFGS=$2; shift 2
mkdir -p gpurun_out
for cfg in $CFGS; do
  i=0
  for set in "$@"; do
    args=""; for kv in $set; do args="$args --opt $kv"; done
    python bench.py --config $cfg --no-cpu --no-e2e --steps 10 $args > gpurun_out/${TAG}_${cfg}_$i.json 2>&1
    echo "$cfg [$set] $(tail -1 gpurun_out/${TAG}_${cfg}_$i.json | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],3))' 2>/dev/null)"
    i=$((i+1))
  done
done
