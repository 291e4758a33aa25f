#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_v17.log 2>&1; echo "exit $?" >> gpurun_out/pytest_v17.log
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-check > gpurun_out/bench_v17_$tag.json 2> gpurun_out/bench_v17_$tag.err; }
run default A=1
run ct1_4 FDA_GT_CT1=4
run ct1_1 FDA_GT_CT1=1
run ct2_bal FDA_GT_CT2=-1
run chunk512 FDA_GT_CHUNK=512
run chunk128 FDA_GT_CHUNK=128
