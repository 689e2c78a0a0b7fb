# Full ncu capture of one launch: bash tools/prof_one.sh <config> <tag> <kernel-regex> <skip> [count]
CFG=$1; TAG=$2; RX=$3; SKIP=$4; CNT=${5:-1}
mkdir -p gpurun_out
python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_plain.json 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:$RX --launch-skip $SKIP --launch-count $CNT \
    -o gpurun_out/${TAG} python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu.log 2>&1
