#!/bin/bash
# re-entry probe: plan log (rank histograms) + per-launch trace at config 5, bench lines at configs 3 and 5
mkdir -p gpurun_out
python -c "import paper_1311_5202_b200.fda" || exit 1
timeout 600 python tools/plan_probe.py 5 1 > gpurun_out/probe_c5.log 2>&1
FDA_TRACE=1 timeout 600 python bench.py --config 5 --steps 1 --warmup 3 --no-check > /dev/null 2> gpurun_out/trace_c5.log
timeout 600 python bench.py --config 3 --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
