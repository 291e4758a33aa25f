#!/bin/bash
# k_gtrans stage-2 column tiles per warp unit (FDA_GT_CT2; 0 = default P/8, -1 = balance rule) at config 5, with
# per-launch traces of the M2M / L2L levels
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
bash tools/jobs/ab.sh ct2_c5 5 "FDA_GT_CT2=0" "FDA_GT_CT2=-1" "FDA_GT_CT2=2" "FDA_GT_CT2=1"
for v in 0 -1 2 1; do echo "== FDA_GT_CT2=$v"; FDA_GT_CT2=$v FDA_TRACE=1 timeout 600 python bench.py --config 5 --steps 1 --warmup 1 --no-check 2>&1 >/dev/null | grep -E 'm2m|l2l' | tail -8; done > gpurun_out/ct2_trace_c5.log
