#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --config 5 --steps 1 --warmup 3 --no-check"
timeout 900 $CMD > gpurun_out/plain_c5v13.log 2>&1 && \
timeout 2400 ncu --set full --import-source on --clock-control none -k regex:k_gtrans -s 8 -c 2 -o gpurun_out/prof_c5v13 $CMD > gpurun_out/ncu_full_v13.log 2>&1
echo "exit $?" >> gpurun_out/ncu_full_v13.log
