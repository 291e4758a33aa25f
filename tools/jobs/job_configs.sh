#!/bin/bash
# bench lines for the other configs (parity-test configs; the metric's workload is config 5)
mkdir -p gpurun_out
for c in 1 1b 1c 2 3 4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/cfg_bench_c$c.json 2> gpurun_out/cfg_bench_c$c.err
done
