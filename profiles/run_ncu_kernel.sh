#!/bin/bash
# One --set full capture of selected kernels (after a plain run of the same command).
# Usage: profiles/run_ncu_kernel.sh TAG CONFIG REGEX SKIP COUNT
TAG=$1; CFG=$2; RE=$3; SKIP=${4:-40}; CNT=${5:-2}
CMD="python bench.py --config $CFG --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$RE" -s $SKIP -c $CNT \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo full_rc=$?
