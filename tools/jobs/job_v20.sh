#!/bin/bash
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-check > gpurun_out/bench_v20_$tag.json 2> gpurun_out/bench_v20_$tag.err; }
run default A=1
run chunk512 FDA_GT_CHUNK=512
run chunk1024 FDA_GT_CHUNK=1024
run smem74 FDA_GT_SMEM_KB=74
run smem150 FDA_GT_SMEM_KB=150
