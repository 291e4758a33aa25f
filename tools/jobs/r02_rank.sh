#!/bin/bash
# round 2: low-rank cut and rank round-up (R23) vs the warp-task M2L cost and the accuracy, config 5
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
for v in "FDA_RANK_ROUND=8" "FDA_RANK_ROUND=4" "FDA_RANK_ROUND=1"; do
  echo "== $v" >> gpurun_out/rank.log
  env $v timeout 600 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/rank_tmp.json 2>> gpurun_out/rank_err.log
  python -c "import json;d=json.loads(open('gpurun_out/rank_tmp.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],2), d['phases_ms']['m2l'], d['parity'], d['roofline']['frac'])" >> gpurun_out/rank.log 2>&1
done
