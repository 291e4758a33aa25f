#!/bin/bash
# round 2: device operators (fixed) + bulk-reduced (UBLKRED) translation outputs.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_bmg.py tests/test_gpu_table1.py "tests/test_gpu_configs.py::test_full_oracle_hf_configs" -q -s -x -p no:cacheprovider > gpurun_out/pytest_bulk.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_bulk.log
FDA_HOST_OPS=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_hostops.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_hostops.log
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --verbose > gpurun_out/bench_c5_bulk.json 2> gpurun_out/bench_c5_bulk.err; echo "exit $?" >> gpurun_out/bench_c5_bulk.err
FDA_GT_WSP=32 timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --no-check > gpurun_out/bench_c5_wsp32.json 2> gpurun_out/bench_c5_wsp32.err
FDA_GT_BULK=0 timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --no-check > gpurun_out/bench_c5_nobulk.json 2> gpurun_out/bench_c5_nobulk.err
timeout 600 python tests/tools/far_probe.py 2 2000 '' 'eps_lowrank=3.3e-6' 'lf_p_low=7' 'eps_lowrank=3.3e-6,lf_p_low=7' > gpurun_out/far3_c2.jsonl 2> gpurun_out/far3_c2.err
