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
ncu --set full --clock-control none --import-source on -k regex:bf_frontier -c 1 \
    -o gpurun_out/${TAG}_bf python bench.py $ARGS > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full exit $?"
# the pred pass writes its 34 GB output: kernel replay cannot save/restore
# it, so it is captured with application replay and the main sections only
ncu --replay-mode application --section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy \
    --section LaunchStats --section WarpStateStats --section SchedulerStats --import-source on \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum,l1tex__t_bytes.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg \
    --clock-control none -k regex:bf_pred -c 1 -o gpurun_out/${TAG}_pred python bench.py $ARGS > gpurun_out/${TAG}_ncu_pred.log 2>&1
echo "ncu pred exit $?"
