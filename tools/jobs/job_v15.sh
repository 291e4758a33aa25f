#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu_v15.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_v15.log
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --verbose > gpurun_out/bench_v15_c5.json 2> gpurun_out/bench_v15_c5.err
timeout 1200 python tests/tools/accuracy_sweep.py 1c 'lf_p_low=5' > gpurun_out/sweep_c1c_v15.jsonl 2> gpurun_out/sweep_c1c_v15.err
timeout 1800 python tests/tools/accuracy_sweep.py 5 'lf_p_low=5' 'lf_p_low=5,lf_p_high=6,lf_p_switch=0.9' > gpurun_out/sweep_c5_v15.jsonl 2> gpurun_out/sweep_c5_v15.err
