#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/final3_pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/final3_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/final3_smoke.log
