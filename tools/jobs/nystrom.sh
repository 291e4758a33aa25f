#!/bin/bash
# round 2: the locally corrected Nystrom weights (f4) -- GPU parity tests, timing on config 1b's D_i pairs,
# FP64 instruction counts and pipe activity of k_nystrom_weights (ncu, after the same command exited 0)
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
timeout 1200 python -m pytest tests/test_gpu_nystrom.py -q -s -p no:cacheprovider > gpurun_out/pytest_nystrom.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_nystrom.log
timeout 600 python tools/nystrom_bench.py --config 1b > gpurun_out/nystrom_bench.jsonl 2> gpurun_out/nystrom_bench.err
timeout 600 python tools/nystrom_bench.py --config 1b --nq 12 --gamma 1e30 >> gpurun_out/nystrom_bench.jsonl 2>> gpurun_out/nystrom_bench.err
timeout 600 python tools/nystrom_bench.py --config 4 --reps 2 >> gpurun_out/nystrom_bench.jsonl 2>> gpurun_out/nystrom_bench.err
timeout 600 python tools/nystrom_bench.py --config 3 --reps 2 >> gpurun_out/nystrom_bench.jsonl 2>> gpurun_out/nystrom_bench.err && \
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:k_nystrom -c 2 --csv --log-file gpurun_out/ncu_nystrom.csv python tools/nystrom_bench.py --config 1b --reps 1 > gpurun_out/ncu_nystrom.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_nystrom.log
