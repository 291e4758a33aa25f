#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu_v9.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_v9.log
timeout 1200 python tests/tools/accuracy_sweep.py 1c '' 'eps_lowrank=3e-6' 'eps_lowrank=3e-5' 'eps_internal=1e-6' > gpurun_out/sweep_c1c_v9.jsonl 2> gpurun_out/sweep_c1c_v9.err
timeout 1800 python tests/tools/accuracy_sweep.py 5 '' 'eps_lowrank=3e-5' 'eps_internal=2e-6' > gpurun_out/sweep_c5_v9.jsonl 2> gpurun_out/sweep_c5_v9.err
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 > gpurun_out/bench_v9_c5.json 2> gpurun_out/bench_v9_c5.err
