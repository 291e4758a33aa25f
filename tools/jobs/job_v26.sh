#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu_v26.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_v26.log
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 > gpurun_out/bench_v26_c5.json 2> gpurun_out/bench_v26_c5.err

timeout 600 python bench.py --config 3 --steps 10 --warmup 3 > gpurun_out/bench_v26_c3.json 2> gpurun_out/bench_v26_c3.err
CMD="python bench.py --config 5 --steps 1 --warmup 3 --no-check"
timeout 900 $CMD > gpurun_out/plain_c5v26.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum,sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed --clock-control none -s 30 -c 30 --csv --log-file gpurun_out/mem_c5v26.csv $CMD > gpurun_out/ncu_mem_v26.log 2>&1
