# cfg4 paths/s vs window: bash tools/win_ab.sh <tag>
TAG=$1
for w in 128 256 512 1024 2048; do
  python bench.py --config cfg4 --window $w --no-cpu --steps 6 > gpurun_out/${TAG}_w$w.json 2>&1
  echo "w=$w $(tail -1 gpurun_out/${TAG}_w$w.json | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["e2e"]["value"]), round(d["ms_per_step"],2), d["nodes_per_step"])' 2>/dev/null)"
done
