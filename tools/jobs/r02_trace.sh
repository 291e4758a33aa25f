#!/bin/bash
# per-launch wall times of the far field (FDA_TRACE=1) for the output-accumulation variants
mkdir -p gpurun_out
for v in "FDA_GT_BULK=0" "FDA_GT_BULK=1" "FDA_GT_BULK=1 FDA_GT_WSP=32"; do
  echo "== $v" >> gpurun_out/trace.log
  env $v FDA_TRACE=1 timeout 900 python bench.py --config 5 --steps 1 --warmup 3 --no-check > /dev/null 2>> gpurun_out/trace_raw_$(echo $v | tr ' =' '__').log
  tail -40 gpurun_out/trace_raw_$(echo $v | tr ' =' '__').log >> gpurun_out/trace.log
done
timeout 900 python -m pytest tests/test_gpu_devplan.py -q -s -p no:cacheprovider > gpurun_out/pytest_devplan.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_devplan.log
