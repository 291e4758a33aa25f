#!/bin/bash
# round 2: M2L work items cut at Morton windows of output cubes (FDA_GT_WIN), config 5 phase times
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
for v in "FDA_GT_WIN=1" "FDA_GT_WIN=16" "FDA_GT_WIN=64" "FDA_GT_WIN=256" "FDA_GT_WIN=64 FDA_ITEM_ORDER=group" "FDA_GT_WIN=1024"; do
  echo "== $v" >> gpurun_out/win.log
  env $v timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-check > gpurun_out/win_tmp.json 2>> gpurun_out/win_err.log
  python -c "import json;d=json.loads(open('gpurun_out/win_tmp.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['phases_ms'])" >> gpurun_out/win.log 2>&1
done
env FDA_GT_WIN=64 FDA_TRACE=1 timeout 600 python bench.py --config 5 --steps 1 --warmup 3 --no-check > /dev/null 2> gpurun_out/win_trace64.log
env FDA_GT_WIN=1 FDA_TRACE=1 timeout 600 python bench.py --config 5 --steps 1 --warmup 3 --no-check > /dev/null 2> gpurun_out/win_trace1.log
