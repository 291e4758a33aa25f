#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -s -x > gpurun_out/pytest_parity_v8.log 2>&1
timeout 1800 python tests/tools/accuracy_sweep.py 1c 'lowrank=0' 'hf_max_rows=12000' 'lf_p_high=10' 'eps_internal=1.5e-6' > gpurun_out/sweep_c1c_v8.jsonl 2> gpurun_out/sweep_c1c_v8.err
for m in atomic owned; do FDA_GT_MODE=$m timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-check > gpurun_out/bench_v8_c5_$m.json 2>&1; done
FDA_GT_MODE=atomic FDA_GT_CHUNK=256 timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-check > gpurun_out/bench_v8_c5_atomic256.json 2>&1
