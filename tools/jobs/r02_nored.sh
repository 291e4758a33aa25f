#!/bin/bash
# round 2: what the FP64 output reductions cost in the translations (FDA_GT_NORED=1: none, 2: plain stores)
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
for v in "FDA_GT_NORED=0" "FDA_GT_NORED=1" "FDA_GT_NORED=2"; do
  echo "== $v" >> gpurun_out/nored.log
  env $v FDA_TRACE=1 timeout 600 python bench.py --config 5 --steps 1 --warmup 2 --no-check > /dev/null 2> gpurun_out/nored_tmp.log
  grep 'trace' gpurun_out/nored_tmp.log | tail -24 >> gpurun_out/nored.log
done
