# Full ncu capture of one launch under engine options: bash tools/prof_opt.sh <config> <tag> <kernel-regex> <skip> "<k=v ...>"
CFG=$1; TAG=$2; RX=$3; SKIP=$4; OPTS=$5
args=""; for kv in $OPTS; do args="$args --opt $kv"; done
mkdir -p gpurun_out
python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu $args > gpurun_out/${TAG}_plain.json 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:$RX --launch-skip $SKIP --launch-count 1 \
    -o gpurun_out/${TAG} python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu $args > gpurun_out/${TAG}_ncu.log 2>&1
