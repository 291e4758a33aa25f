#!/bin/bash
# item launch order experiment on config 5: M2L per-level memory metrics (cost order vs Morton order)
mkdir -p gpurun_out
./tools/bin/l2_bw > gpurun_out/l2_bw.json 2>&1
CMD="python bench.py --config 5 --steps 1 --warmup 3 --no-check"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum,sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed"
timeout 900 $CMD > gpurun_out/plain_c5v5.log 2>&1 && \
timeout 1500 ncu --metrics $M --clock-control none -k regex:k_gtrans -s 17 -c 17 --csv --log-file gpurun_out/mem_c5v5_morton.csv $CMD > gpurun_out/ncu_mem_morton.log 2>&1
FDA_ITEM_ORDER=cost timeout 1500 ncu --metrics $M --clock-control none -k regex:k_gtrans -s 17 -c 17 --csv --log-file gpurun_out/mem_c5v5_cost.csv $CMD > gpurun_out/ncu_mem_cost.log 2>&1
