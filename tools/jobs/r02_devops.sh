#!/bin/bash
# round 2: device-built operators -- quick GPU tests, config-5 bench with the plan log, eps-lowrank probes.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_bmg.py tests/test_gpu_table1.py "tests/test_gpu_configs.py::test_full_oracle_hf_configs" -q -s -x -p no:cacheprovider > gpurun_out/pytest_devops.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_devops.log
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --verbose > gpurun_out/bench_c5_devops.json 2> gpurun_out/bench_c5_devops.err; echo "exit $?" >> gpurun_out/bench_c5_devops.err
timeout 600 python tests/tools/far_probe.py 2 2000 '' 'eps_lowrank=3.3e-6' 'lf_p_low=7' 'eps_lowrank=3.3e-6,lf_p_low=7' > gpurun_out/far3_c2.jsonl 2> gpurun_out/far3_c2.err
timeout 900 python tests/tools/far_probe.py 5 500 '' 'eps_lowrank=3.3e-6' > gpurun_out/far3_c5.jsonl 2> gpurun_out/far3_c5.err
