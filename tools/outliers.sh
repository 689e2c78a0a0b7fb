for i in 1 2 3 4 5 6; do
for mode in on off; do
  if [ $mode = off ]; then export GS_BENCH_NO_CLOCKS=1; else unset GS_BENCH_NO_CLOCKS; fi
  python bench.py --config cfg3 --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$mode', round(d['value']), round(d['ms_per_step'],3))"
done; done
