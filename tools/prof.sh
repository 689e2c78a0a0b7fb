# Launch list (warm cache, serialised) + one full capture of a leaf pass kernel.
#   bash tools/prof.sh <config> <tag> [skip]
CFG=${1:-cfg4}; TAG=${2:-x}; SKIP=${3:-60}
mkdir -p gpurun_out
python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_plain.json 2>gpurun_out/${TAG}_plain.err || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__registers_per_thread \
    --clock-control none --cache-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gsj --launch-skip $SKIP --launch-count 2 \
    -o gpurun_out/${TAG}_full python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu2.log 2>&1
ls -la gpurun_out/ | grep $TAG
