#!/bin/bash
# round 2: A/B of the warp-task M2L launch options at config 5, two rounds (noise), + the block-M2L test
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
timeout 600 python -m pytest tests/test_gpu_m2l_block.py -q -p no:cacheprovider > gpurun_out/pytest_blk.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_blk.log
for r in 1 2; do
for v in "FDA_M2L_X=0" "FDA_M2L_SECTOR=0" "FDA_M2L_RLIM=24 FDA_M2L_SECTOR=0" "FDA_M2L_RLIM=24"; do
  echo "== $r $v" >> gpurun_out/ab.log
  env $v timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-check > gpurun_out/ab_tmp.json 2>> gpurun_out/ab_err.log
  python -c "import json;d=json.loads(open('gpurun_out/ab_tmp.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],2), d['phases_ms']['m2l'])" >> gpurun_out/ab.log 2>&1
done
done
