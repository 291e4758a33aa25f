#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python tests/tools/accuracy_sweep.py 1c '' 'eps_internal=1e-6' 'eps_internal=2e-6' 'hf_spacing=0.2' 'lf_p_high=10' 'eps_internal=2e-6,hf_spacing=0.2' > gpurun_out/sweep_c1c.jsonl 2> gpurun_out/sweep_c1c.err
timeout 900 python -m pytest tests/test_gpu_configs.py -q -s -k "sampled" > gpurun_out/pytest_cfg_v7.log 2>&1
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-check > gpurun_out/bench_v7_c5.json 2> gpurun_out/bench_v7_c5.err
FDA_P2P=block timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-check > gpurun_out/bench_v7_c3_block.json 2>&1
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-check > gpurun_out/bench_v7_c3_warp.json 2>&1
