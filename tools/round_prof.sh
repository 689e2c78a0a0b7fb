# Round profile set: every config's bench line, the default line + reference arm,
# the default command's ncu launch list, and a full capture of its top pass kernel.
#   bash tools/round_prof.sh <tag>
TAG=${1:-r}
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err
python bench.py --impl reference > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
for cfg in cfg1 cfg2 cfg2h cfg3 cfg4 cfg5 cfg5f; do
  extra=""; [ $cfg = cfg5 ] && extra="--window 64 --steps 3"; [ $cfg = cfg5f ] && extra="--window 8 --steps 2"
  python bench.py --config $cfg --no-cpu $extra > gpurun_out/${TAG}_bench_$cfg.json 2> gpurun_out/${TAG}_bench_$cfg.err
done
python tools/dump_describe.py cfg4 gpurun_out/${TAG}_cfg4_describe.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__registers_per_thread \
    --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_cfg4_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu1.log 2>&1
python tools/launchmap.py gpurun_out/${TAG}_cfg4_describe.json gpurun_out/${TAG}_cfg4_launches.csv > gpurun_out/${TAG}_cfg4_launchmap.txt
TOP=$(awk 'NR==2 {print $1}' gpurun_out/${TAG}_cfg4_launchmap.txt)
ncu --set full --import-source on --clock-control none -k regex:gsj_.*_p${TOP}\$ --launch-skip 4 --launch-count 1 \
    -o gpurun_out/${TAG}_cfg4_top python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu2.log 2>&1
ncu --set full --clock-control none -k regex:gather_ --launch-skip 4 --launch-count 1 \
    -o gpurun_out/${TAG}_cfg4_gather python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu3.log 2>&1
ls -la gpurun_out/ | grep $TAG
