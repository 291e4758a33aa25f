#!/bin/bash
# usage: tools/gpu_bench.sh TAG cfg [cfg...]   -- GPU tests, smoke, then bench per config (outputs in gpurun_out/)
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
for c in "$@"; do
  timeout 1500 python bench.py --config $c --steps 10 --warmup 3 --verbose > gpurun_out/bench_${TAG}_c$c.json 2> gpurun_out/bench_${TAG}_c$c.err
  echo "exit $?" >> gpurun_out/bench_${TAG}_c$c.err
done
