#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_table1.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_v32.log 2>&1; echo "exit $?" >> gpurun_out/pytest_v32.log
timeout 2400 python tests/tools/table1.py 1e-6 > gpurun_out/table1_1e-6b.jsonl 2> gpurun_out/table1_1e-6b.err
