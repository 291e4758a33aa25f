#!/bin/bash
# round 2: the Table-1 4.7M row at eps = 1e-8 (after the eps-dependent HF sample size)
mkdir -p gpurun_out
timeout 2400 python tests/tools/table1.py --rows t1d 1e-8 > gpurun_out/table1_t1d_1e8.jsonl 2> gpurun_out/table1_t1d_1e8.err
echo "exit $?" >> gpurun_out/table1_t1d_1e8.err
