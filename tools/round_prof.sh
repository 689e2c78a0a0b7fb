# Round profile set for the bench default (cfg4) and the reference arm:
#   bash tools/round_prof.sh <tag>
# 1. bench line + describe (schedule hash), 2. ncu launch list of the same command,
# 3. traffic.json entry for that schedule, 4. bench line again (roofline.traffic filled),
# 5. full ncu capture of the fused leaf pass and of the top upper pass.
TAG=${1:-r}
mkdir -p gpurun_out
python bench.py --describe-out gpurun_out/${TAG}_describe.json > gpurun_out/${TAG}_bench_pre.json 2> gpurun_out/${TAG}_bench_pre.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__registers_per_thread \
    --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu1.log 2>&1
python tools/traffic.py gpurun_out/${TAG}_describe.json gpurun_out/${TAG}_launches.csv profiles/traffic.json > gpurun_out/${TAG}_traffic.log 2>&1
python tools/launchmap.py gpurun_out/${TAG}_describe.json gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launchmap.txt 2>&1
cp profiles/traffic.json gpurun_out/${TAG}_traffic.json
python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err
python bench.py --impl reference > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
ncu --set full --import-source on --clock-control none -k regex:gsj_.*_p21\$ --launch-skip 3 --launch-count 1 \
    -o gpurun_out/${TAG}_leaf python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gsj_.*_p19\$ --launch-skip 3 --launch-count 1 \
    -o gpurun_out/${TAG}_upper python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu3.log 2>&1
ls -la gpurun_out/ | grep $TAG
