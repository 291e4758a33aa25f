#!/bin/bash
# round 2: ncu evidence -- FP64 instruction counts of the ALU kernels (flop per evaluation), the launch
# list of the bench command, and a full capture of the top kernel.  Each ncu run follows the same
# command exiting 0 without ncu.
mkdir -p gpurun_out
CMD3="python bench.py --config 3 --steps 1 --warmup 3 --no-check"
CMD5="python bench.py --config 5 --steps 1 --warmup 3 --no-check"
timeout 900 $CMD3 > gpurun_out/plain_c3.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:"k_p2p|k_s2m_check|k_l2t_eval" -c 12 --csv --log-file gpurun_out/alu_counts_c3.csv $CMD3 > gpurun_out/ncu_alu.log 2>&1
echo "alu exit $?" >> gpurun_out/ncu_alu.log
timeout 900 $CMD5 > gpurun_out/plain_c5.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(gtrans|p2p|csr|s2m|l2t|permute|unpermute|xpack|xunpack)" -c 160 --csv --log-file gpurun_out/launches_c5.csv $CMD5 > gpurun_out/ncu_launch.log 2>&1
echo "launch exit $?" >> gpurun_out/ncu_launch.log
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:k_gtrans_ws -s 3 -c 1 -o gpurun_out/prof_m2l_c5 $CMD5 > gpurun_out/ncu_full.log 2>&1
echo "full exit $?" >> gpurun_out/ncu_full.log
