#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_table1.py tests/test_gpu_bmg.py tests/test_gpu_parity.py -q -s > gpurun_out/pytest_gpu_v29.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_v29.log
timeout 2400 python tests/tools/table1.py 1e-4 > gpurun_out/table1_v29.jsonl 2> gpurun_out/table1_v29.err
