#!/bin/bash
# round 2: evidence of the build -- bench line (config 5, 10 steps), launch list of one apply (device time and
# DRAM bytes per launch), smoke, full GPU suite.  The ncu run follows the same command exiting 0 without ncu.
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "exit $?" >> gpurun_out/bench_c5.err
# the launch list runs the plain launches (FDA_GRAPH=0): ncu's per-node profiling of the apply's CUDA graph
# stops with LaunchFailed (profiles/r02/README.md); the kernels and their order are the same
export FDA_GRAPH=0
CMD5="python bench.py --config 5 --steps 1 --warmup 3 --no-check"
timeout 900 $CMD5 > gpurun_out/plain_c5.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(gtrans|m2l_warp|p2p|csr|s2m|l2t|leaf_s2m|leaf_l2t|permute|unpermute|xpack|xunpack)" -c 160 --csv --log-file gpurun_out/launches_c5.csv $CMD5 > gpurun_out/ncu_launch.log 2>&1
echo "launch exit $?" >> gpurun_out/ncu_launch.log
unset FDA_GRAPH
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
# the top kernel (the LF level-8 warp-task M2L launch of the first apply), once per build
K=k_m2l_warp S=3 OUT=prof_m2l8_final bash tools/jobs/ncu_m2l.sh
