#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gmres.py -q -s > gpurun_out/pytest_gpu_v30.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_v30.log
