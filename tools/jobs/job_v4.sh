#!/bin/bash
./tools/jobs/gpu_bench.sh v4 3 5
timeout 2400 python tests/tools/accuracy_sweep.py 5 '' 'eps_internal=1e-5' 'eps_internal=1e-5,lf_p_switch=0.7' 'eps_internal=3e-6' > gpurun_out/sweep_c5.jsonl 2> gpurun_out/sweep_c5.err
