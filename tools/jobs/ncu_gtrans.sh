#!/bin/bash
# ncu --set full (with source) of one k_gtrans launch of the first apply at config 5 (M2M / L2L transitions):
# K = regex on the kernel base name (ncu matches the name without template arguments), S = launches to skip, OUT = report.
# e.g. K='^k_gtrans$' S=2 OUT=prof_m2m76  (the HF level 7 -> 6 M2M: the third k_gtrans launch of an apply).  Runs to exit 0 without ncu first.
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
CMD="python bench.py --config 5 --steps 1 --warmup 3 --no-check"
FDA_GRAPH=0 $CMD > gpurun_out/plain.log 2>&1 && \
FDA_GRAPH=0 ncu --set full --clock-control none --import-source on -k "regex:${K}" -s ${S:-0} -c 1 -o gpurun_out/${OUT:-prof_gtrans} $CMD > gpurun_out/ncu_${OUT:-prof_gtrans}.log 2>&1
echo "exit $?" >> gpurun_out/ncu_${OUT:-prof_gtrans}.log
