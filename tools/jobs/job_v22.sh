#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu_v22.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_v22.log
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 > gpurun_out/bench_v22_c5.json 2> gpurun_out/bench_v22_c5.err
FDA_P2P=v1 timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-check > gpurun_out/bench_v22_c5_p2pv1.json 2> gpurun_out/bench_v22_c5_p2pv1.err
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 > gpurun_out/bench_v22_c3.json 2> gpurun_out/bench_v22_c3.err
