#!/bin/bash
# round 2: two-pass M2L: per-pass trace at config 5, ncu full of the L8 pass 1 (k_gtrans tstore) and pass 2 (k_m2l_bu)
mkdir -p gpurun_out
python -c "from paper_1311_5202_b200 import build as b; b.build()" > gpurun_out/build.log 2>&1
FDA_TRACE=1 timeout 900 python bench.py --config 5 --steps 1 --warmup 3 --no-check > /dev/null 2> gpurun_out/trace_raw.log
grep 'm2l' gpurun_out/trace_raw.log | tail -12 > gpurun_out/trace.log
timeout 900 ncu --set full --import-source on -k regex:k_m2l_bu --launch-skip 3 --launch-count 1 -o gpurun_out/ncu_bu_l8 python bench.py --config 5 --steps 1 --warmup 1 --no-check > gpurun_out/ncu_bu.log 2>&1
timeout 900 ncu --set full --import-source on -k regex:k_gtrans --launch-skip 9 --launch-count 1 -o gpurun_out/ncu_p1_l8 python bench.py --config 5 --steps 1 --warmup 1 --no-check > gpurun_out/ncu_p1.log 2>&1
