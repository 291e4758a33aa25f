#!/bin/bash
# round 2: eps/3 with ranks rounded up to the tile height -- bench, trace, accuracy tests, then ncu evidence
mkdir -p gpurun_out
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --verbose > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "exit $?" >> gpurun_out/bench_c5.err
FDA_TRACE=1 timeout 600 python bench.py --config 5 --steps 1 --warmup 3 --no-check > /dev/null 2> gpurun_out/trace_c5.log
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_accuracy.py tests/test_gpu_table1.py -q -s -p no:cacheprovider > gpurun_out/pytest_acc.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_acc.log
./tools/jobs/r02_ncu.sh
