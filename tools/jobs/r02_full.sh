#!/bin/bash
# round 2: full GPU suite + config-5 bench (verbose plan log) + per-level trace
mkdir -p gpurun_out
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --verbose > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "exit $?" >> gpurun_out/bench_c5.err
FDA_TRACE=1 timeout 600 python bench.py --config 5 --steps 1 --warmup 3 --no-check > /dev/null 2> gpurun_out/trace_c5.log
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
