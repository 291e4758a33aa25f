#!/bin/bash
# One gpurun call: GPU tests, smoke, FP64 peaks, bench (configs given as args), launch list.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
./tools/bin/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
for c in "$@"; do
  timeout 1500 python bench.py --config $c --steps 10 --warmup 3 --verbose > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  echo "exit $?" >> gpurun_out/bench_c$c.err
done
