#!/bin/bash
# round 2: sector-complete reductions on/off (per-level trace), then the GPU suite subset and ncu evidence
mkdir -p gpurun_out
for v in "FDA_GT_SECTOR=0" "FDA_GT_SECTOR=1"; do
  echo "== $v" >> gpurun_out/trace_sector.log
  env $v FDA_TRACE=1 timeout 900 python bench.py --config 5 --steps 1 --warmup 3 --no-check > /dev/null 2> gpurun_out/tr.tmp
  grep "fda trace" gpurun_out/tr.tmp | tail -28 >> gpurun_out/trace_sector.log
done
FDA_GT_SECTOR=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/pytest_sector.log 2>&1; echo "exit $?" >> gpurun_out/pytest_sector.log
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_accuracy.py -q -s -p no:cacheprovider > gpurun_out/pytest_acc.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_acc.log
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --verbose > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "exit $?" >> gpurun_out/bench_c5.err
