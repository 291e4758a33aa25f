#!/bin/bash
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-check > gpurun_out/bench_v27_$tag.json 2> gpurun_out/bench_v27_$tag.err; }
run default A=1
run ct2_2 FDA_GT_CT2=2
run ct2_1 FDA_GT_CT2=1
