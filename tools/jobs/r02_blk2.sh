#!/bin/bash
# round 2: two-pass M2L (pass 1 T = V X stored, pass 2 target blocks in shared memory): parity, per-level trace, bench
mkdir -p gpurun_out
python -c "from paper_1311_5202_b200 import build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_m2l_block.py tests/test_gpu_parity.py -x -q -s -p no:cacheprovider > gpurun_out/pytest_parity.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_parity.log
for v in "FDA_M2L_BLOCK=1" "FDA_M2L_BLOCK=0"; do
  echo "== $v" >> gpurun_out/trace.log
  env $v FDA_TRACE=1 timeout 900 python bench.py --config 5 --steps 1 --warmup 3 --no-check --verbose > /dev/null 2> gpurun_out/trace_raw.log
  grep 'm2l blocks' gpurun_out/trace_raw.log >> gpurun_out/trace.log
  tail -20 gpurun_out/trace_raw.log >> gpurun_out/trace.log
done
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
