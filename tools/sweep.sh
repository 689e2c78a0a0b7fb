# every config's bench line: bash tools/sweep.sh <tag>  -> gpurun_out/<tag>_bench_<cfg>.json
TAG=${1:-sw}
mkdir -p gpurun_out
for cfg in cfg1 cfg1v2 cfg2 cfg2v2 cfg2h cfg3 cfg3v2 cfg4 cfg4v2 cfg5 cfg5f; do
  extra=""; [ $cfg = cfg5 ] && extra="--window 64 --steps 3"; [ $cfg = cfg5f ] && extra="--window 8 --steps 2"
  python bench.py --config $cfg --no-cpu $extra > gpurun_out/${TAG}_bench_$cfg.json 2> gpurun_out/${TAG}_bench_$cfg.err
  echo "$cfg $(tail -1 gpurun_out/${TAG}_bench_$cfg.json | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]["classes"]; print(round(d["value"],1), round((d["e2e"] or {}).get("value",0),1), round(d["ms_per_step"],3), {k: round(v.get("frac",0) or 0,3) for k,v in r.items() if "frac" in v}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"])' 2>&1 | tail -1)"
done
python bench.py --config cfg4 --whole-job > gpurun_out/${TAG}_bench_cfg4_wholejob.json 2> gpurun_out/${TAG}_bench_cfg4_wholejob.err
echo "wholejob $(tail -1 gpurun_out/${TAG}_bench_cfg4_wholejob.json | cut -c1-300)"
