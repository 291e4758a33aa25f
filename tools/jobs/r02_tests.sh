#!/bin/bash
# round 2: full GPU test suite (prints the parity numbers), far-field probes, config-5 bench.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python tests/tools/far_probe.py 2 2000 'eps_lowrank=1e-5' 'eps_lowrank=3e-6' 'eps_lowrank=3e-6,lf_p_low=8' 'eps_lowrank=1e-6,eps_internal=1e-7,lf_p_low=8' > gpurun_out/far2_c2.jsonl 2> gpurun_out/far2_c2.err
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "exit $?" >> gpurun_out/bench_c5.err
