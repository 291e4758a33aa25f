#!/bin/bash
# round 2: warp-task low-rank M2L kernel (m2l_warp.cu) -- equality test, full parity tests, config 5 times
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
timeout 900 python -m pytest tests/test_gpu_m2l_warp.py tests/test_gpu_parity.py -q -s -p no:cacheprovider -x > gpurun_out/pytest_warp.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_warp.log
for v in "FDA_M2L_WARP=1" "FDA_M2L_WARP=0" "FDA_M2L_WARP=1 FDA_GT_CHUNK=4096"; do
  echo "== $v" >> gpurun_out/warp.log
  env $v timeout 600 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/warp_tmp.json 2>> gpurun_out/warp_err.log
  python -c "import json;d=json.loads(open('gpurun_out/warp_tmp.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['phases_ms'], d['parity'], d['roofline'])" >> gpurun_out/warp.log 2>&1
done
env FDA_TRACE=1 timeout 600 python bench.py --config 5 --steps 1 --warmup 3 --no-check > /dev/null 2> gpurun_out/warp_trace.log
