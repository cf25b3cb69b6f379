#!/bin/bash
# Run on the GPU box (via gpurun): plain bench, launch list, and one
# `ncu --set full` capture of the relaxation sweep. Outputs land in
# gpurun_out/ (scratch); summaries worth keeping are copied to profiles/.
# usage: bash tools/gpu_profile.sh <tag> [bench args...]
set -u
TAG=${1:-r01}
shift || true
ARGS=${*:-"--steps 1 --warmup 1 --no-e2e --no-cpu"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
python bench.py $ARGS > gpurun_out/${TAG}_plain.log 2>&1
echo "plain exit $?"
tail -2 gpurun_out/${TAG}_plain.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py $ARGS > gpurun_out/${TAG}_ncu_list.log 2>&1
echo "launch list exit $?"
ncu --set full --clock-control none --import-source on -k 'regex:bf_frontier|bf_pred' -c 2 \
    -o gpurun_out/${TAG}_bf python bench.py $ARGS > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full exit $?"
