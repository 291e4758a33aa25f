#!/bin/bash
./tools/jobs/gpu_bench.sh v3 3 5
CMD="python bench.py --config 5 --steps 1 --warmup 3 --no-check"
timeout 900 $CMD > gpurun_out/plain_c5v3.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5v3.csv $CMD > gpurun_out/ncu_launch_c5v3.log 2>&1
