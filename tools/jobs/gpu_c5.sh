#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python bench.py --config 5 --steps 10 --warmup 3 --verbose > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo "exit $?" >> gpurun_out/bench_c5.err
timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --no-check > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv \
  python bench.py --config 3 --steps 2 --warmup 3 --no-check > gpurun_out/ncu_c3.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_c3.log
