#!/bin/bash
# round 2: device P2 lists -- device-vs-host plan tests, parity subset, config-5 bench (setup times), Table 1 4.7M at 1e-8
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_devplan.py tests/test_gpu_parity.py tests/test_gpu_dist.py "tests/test_gpu_configs.py::test_full_oracle_hf_configs" -q -s -p no:cacheprovider > gpurun_out/pytest_lists.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_lists.log
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --verbose > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "exit $?" >> gpurun_out/bench_c5.err
./tools/jobs/r02_table1d.sh
