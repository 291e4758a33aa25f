#!/bin/bash
# round 2: warp-task M2L v2 (predicated x loads, integer row bound, 3M sums staged) -- tests + config 5 times
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bmg.py tests/test_gpu_m2l_warp.py -q -s -p no:cacheprovider -x > gpurun_out/pytest_gtpf.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gtpf.log
for v in "FDA_X=0"; do
  echo "== $v" >> gpurun_out/gtpf.log
  env $v timeout 600 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/warp_tmp.json 2>> gpurun_out/warp_err.log
  python -c "import json;d=json.loads(open('gpurun_out/warp_tmp.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['phases_ms'], d['parity'], d['roofline'])" >> gpurun_out/gtpf.log 2>&1
done
env FDA_TRACE=1 timeout 600 python bench.py --config 5 --steps 1 --warmup 3 --no-check > /dev/null 2> gpurun_out/gtpf_trace.log
