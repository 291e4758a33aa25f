#!/bin/bash
# ncu --set full (with source) of M2L launches of the first apply at config 5: K = kernel regex, S = launches to
# skip, OUT = report name.  e.g. K=k_m2l_warp S=3 OUT=prof_m2l8 tools/jobs/ncu_m2l.sh  (the LF level-8 launch)
# The same command runs to exit 0 without ncu first.
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
CMD="python bench.py --config 5 --steps 1 --warmup 3 --no-check"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${K:-k_m2l_warp} -s ${S:-3} -c 1 -o gpurun_out/${OUT:-prof_m2l} $CMD > gpurun_out/ncu_${OUT:-prof_m2l}.log 2>&1
echo "exit $?" >> gpurun_out/ncu_${OUT:-prof_m2l}.log
