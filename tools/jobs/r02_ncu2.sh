#!/bin/bash
# round 2: ncu --set full (with source) of the LF-level M2L launch (k_m2l_warp, 4th) and the LF->HF M2M launch
# (k_gtrans, 4th) of the first apply, config 5
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
CMD="python bench.py --config 5 --steps 1 --warmup 3 --no-check"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_m2l_warp -s 3 -c 1 -o gpurun_out/prof_m2l8b $CMD > gpurun_out/ncu2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_m2l_warp -s 0 -c 1 -o gpurun_out/prof_m2l5 $CMD >> gpurun_out/ncu2.log 2>&1
echo "exit $?" >> gpurun_out/ncu2.log
