#!/bin/bash
# round 2: HF M2L operators shared by the cube symmetry -- equality test, config 5 phase times and trace
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
timeout 900 python -m pytest tests/test_gpu_m2l_share.py -q -s -p no:cacheprovider > gpurun_out/pytest_share.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_share.log
for v in "FDA_M2L_NOSHARE=0" "FDA_M2L_NOSHARE=1"; do
  echo "== $v" >> gpurun_out/share.log
  env $v timeout 600 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/share_tmp.json 2>> gpurun_out/share_err.log
  python -c "import json;d=json.loads(open('gpurun_out/share_tmp.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['phases_ms'], d['parity'], d['plan'], d['setup_s'])" >> gpurun_out/share.log 2>&1
done
env FDA_TRACE=1 timeout 600 python bench.py --config 5 --steps 1 --warmup 3 --no-check > /dev/null 2> gpurun_out/share_trace.log
