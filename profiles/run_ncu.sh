#!/bin/bash
# Profiling recipe (B200_PROFILING.md): plain run first, then the launch list,
# then one --set full capture of the top kernels.
# Usage: profiles/run_ncu.sh TAG CONFIG [KERNEL_REGEX] [SKIP] [COUNT]
TAG=${1:-r1}; CFG=${2:-5}; RE=${3:-"k_lanczos_cols|k_cg_b"}; SKIP=${4:-60}; CNT=${5:-2}
CMD="python bench.py --config $CFG --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo launches_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"$RE" -s $SKIP -c $CNT \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo full_rc=$?
