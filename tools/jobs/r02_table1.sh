#!/bin/bash
# round 2: Table 1 on the GPU -- original / reduced / improved at eps 1e-4, 1e-6, 1e-8, all four point sets
mkdir -p gpurun_out
timeout 3000 python tests/tools/table1.py 1e-4 1e-6 1e-8 > gpurun_out/table1_r02.jsonl 2> gpurun_out/table1_r02.err
echo "exit $?" >> gpurun_out/table1_r02.err
