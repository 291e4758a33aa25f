#!/bin/bash
# low-rank LF -> HF transitions (FDA_M2M_LR): GPU test, plan log (ranks) and A/B at config 5
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
timeout 900 python -m pytest tests/test_gpu_m2m_lowrank.py tests/test_gpu_graph.py -q -s -p no:cacheprovider > gpurun_out/pytest_m2mlr.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_m2mlr.log
FDA_M2M_LR=0.1 timeout 600 python tools/plan_probe.py 5 1 2>&1 | grep -E 'm2m/l2l|ERR|^t ' > gpurun_out/m2mlr_plan_c5.log
bash tools/jobs/ab.sh m2mlr_c5 5 "FDA_M2M_LR=0" "FDA_M2M_LR=1" "FDA_M2M_LR=0.1" "FDA_M2M_LR=0.3"
