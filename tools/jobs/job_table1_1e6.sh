#!/bin/bash
mkdir -p gpurun_out
timeout 2700 python tests/tools/table1.py 1e-6 > gpurun_out/table1_1e-6.jsonl 2> gpurun_out/table1_1e-6.err
echo "exit $?" >> gpurun_out/table1_1e-6.err
