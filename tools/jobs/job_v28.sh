#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu_v28.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_v28.log
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 > gpurun_out/bench_v28_c5.json 2> gpurun_out/bench_v28_c5.err
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --kernel bmg > gpurun_out/bench_v28_c5_bmg.json 2> gpurun_out/bench_v28_c5_bmg.err
