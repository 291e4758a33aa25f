#!/bin/bash
# round 2: owned-output items (plain read-modify-write, no atomics) with large Morton windows vs atomic items;
# FP64 atomic throughput microbenchmark
mkdir -p gpurun_out
./tools/bin/l2_atomic_bw > gpurun_out/l2_atomic_bw.jsonl 2>&1
for v in "FDA_GT_MODE=atomic" "FDA_GT_MODE=owned FDA_GT_SLABS=148" "FDA_GT_MODE=owned FDA_GT_SLABS=296" "FDA_GT_MODE=owned FDA_GT_SLABS=592" "FDA_GT_MODE=owned FDA_GT_SLABS=1184"; do
  echo "== $v" >> gpurun_out/trace_owned.log
  env $v FDA_TRACE=1 timeout 900 python bench.py --config 5 --steps 1 --warmup 1 --no-check > /dev/null 2> gpurun_out/tr.tmp
  grep "fda trace" gpurun_out/tr.tmp | tail -28 >> gpurun_out/trace_owned.log
done
