#!/bin/bash
# Final round-1 evidence: GPU tests, smoke, the default bench line, the reference arm, the ncu launch
# list of the default bench command, and one ncu --set full capture of the top kernel.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/final2_pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/final2_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/final2_smoke.log
timeout 900 python bench.py > gpurun_out/final2_bench.json 2> gpurun_out/final2_bench.err; echo "exit $?" >> gpurun_out/final2_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/final2_bench_ref.json 2> gpurun_out/final2_bench_ref.err
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final2_launches.csv python bench.py > gpurun_out/final2_ncu_launch.log 2>&1; echo "exit $?" >> gpurun_out/final2_ncu_launch.log
CMD="python bench.py --config 5 --steps 1 --warmup 3 --no-check"
timeout 900 $CMD > gpurun_out/final2_plain.log 2>&1 && \
timeout 2400 ncu --set full --import-source on --clock-control none -k regex:k_gtrans_ws -s 3 -c 1 -o gpurun_out/final2_prof $CMD > gpurun_out/final2_ncu_full.log 2>&1
echo "exit $?" >> gpurun_out/final2_ncu_full.log
