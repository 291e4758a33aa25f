#!/bin/bash
# usage: tools/gpu_ncu.sh TAG CFG SKIP COUNT   -- plain run, launch list, and ncu --set full of k_gtrans launches [SKIP, SKIP+COUNT)
TAG=$1; CFG=$2; SKIP=$3; CNT=$4
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-check"
timeout 900 $CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1 && \
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:k_gtrans -s $SKIP -c $CNT -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "exit $?" >> gpurun_out/ncu_full_${TAG}.log
