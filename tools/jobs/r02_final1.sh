#!/bin/bash
# round 2: full GPU suite, smoke, bench (verbose setup), Table-1 4.7M at 1e-8
mkdir -p gpurun_out
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --verbose > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "exit $?" >> gpurun_out/bench_c5.err
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 python tests/tools/table1.py --rows t1d 1e-8 > gpurun_out/t1d.jsonl 2> gpurun_out/t1d.err
