# every config's bench line into gpurun_out/bench_<cfg>.json (+ default and reference arms)
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for cfg in cfg1 cfg2 cfg2h cfg3 cfg4 cfg5 cfg5f; do
  extra=""; [ $cfg = cfg5 ] && extra="--window 64 --steps 3"; [ $cfg = cfg5f ] && extra="--window 64 --steps 3"
  python bench.py --config $cfg --no-cpu $extra > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
done
python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
