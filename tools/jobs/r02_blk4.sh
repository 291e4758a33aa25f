#!/bin/bash
# round 2: two-pass M2L with dedicated pass-1 (k_m2l_tv) and pass-2 (k_m2l_bu) kernels: tests, per-pass trace
mkdir -p gpurun_out
python -c "from paper_1311_5202_b200 import build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_m2l_block.py tests/test_gpu_parity.py -x -q -s -p no:cacheprovider > gpurun_out/pytest_parity.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_parity.log
FDA_TRACE=1 timeout 900 python bench.py --config 5 --steps 1 --warmup 3 --no-check > /dev/null 2> gpurun_out/trace_raw.log
grep 'm2l' gpurun_out/trace_raw.log | tail -16 > gpurun_out/trace.log
