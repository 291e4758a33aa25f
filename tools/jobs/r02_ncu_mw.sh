#!/bin/bash
# round 2: ncu --set full with source of the M2L launches of one apply (levels 5, 6, 7, 8 (warp-task kernel)), config 5
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
CMD="python bench.py --config 5 --steps 1 --warmup 3 --no-check"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_m2l_warp -s 0 -c 4 -o gpurun_out/prof_mw $CMD > gpurun_out/ncu_mw.log 2>&1
echo "exit $?" >> gpurun_out/ncu_mw.log
