#!/bin/bash
# round 2: setup-time breakdown of the device lists; which HF wedge misses at eps = 1e-8 on the 4.7M point set
mkdir -p gpurun_out
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --verbose --no-check > gpurun_out/bench_c5_setup.json 2> gpurun_out/bench_c5_setup.err
timeout 1200 python tests/tools/table1.py --rows t1d 1e-8 > gpurun_out/t1d.jsonl 2> gpurun_out/t1d.err
