#!/bin/bash
# A/B of plan / launch options at one config: one bench line per variant (phase times, parity, roofline),
# optionally GPU tests first and a per-launch trace (FDA_TRACE) of one variant at the end.
#   tools/jobs/ab.sh NAME CONFIG "VAR=1 X=2" "VAR=0" ...        (env variants; "FDA_X=0" = the defaults)
#   TESTS="tests/test_gpu_m2l_warp.py tests/test_gpu_parity.py" TRACE="FDA_X=0" tools/jobs/ab.sh ...
# Outputs gpurun_out/NAME.log (one line per variant), NAME_trace.log, pytest_NAME.log.
NAME=$1; CFG=$2; shift 2
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest $TESTS -q -s -p no:cacheprovider -x > gpurun_out/pytest_$NAME.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_$NAME.log
fi
for v in "$@"; do
  echo "== $v" >> gpurun_out/$NAME.log
  env $v timeout 900 python bench.py --config $CFG --steps 5 --warmup 3 > gpurun_out/${NAME}_tmp.json 2>> gpurun_out/${NAME}_err.log
  python -c "import json;d=json.loads(open('gpurun_out/${NAME}_tmp.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['phases_ms'], d['parity'], d['roofline'])" >> gpurun_out/$NAME.log 2>&1
done
if [ -n "$TRACE" ]; then
  env $TRACE FDA_TRACE=1 timeout 900 python bench.py --config $CFG --steps 1 --warmup 3 --no-check > /dev/null 2> gpurun_out/${NAME}_trace.log
fi
