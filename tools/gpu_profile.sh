#!/bin/bash
# Run on the GPU box (via gpurun): plain bench, launch list, and one ncu
# capture of the relaxation sweep (which also runs the fused pred pass).
# Outputs land in gpurun_out/ (scratch); summaries worth keeping are copied
# to profiles/.
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
# the sweep writes the 34 GB pred output (fused a4): kernel replay cannot
# save/restore it, so the capture uses application replay with the main
# sections (throughput, memory, occupancy, warp state, per-SASS source counters)
ncu --replay-mode application --section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy \
    --section LaunchStats --section WarpStateStats --section SchedulerStats --section SourceCounters \
    --import-source on \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum,l1tex__t_bytes.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg,sm__cycles_active.min,sm__cycles_active.max \
    --clock-control none -k regex:bf_frontier -c 1 -o gpurun_out/${TAG}_bf python bench.py $ARGS > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu sweep exit $?"
