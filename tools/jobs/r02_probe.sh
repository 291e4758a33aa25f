#!/bin/bash
# round 2, first GPU call: FP64 peaks with a clock record, GPU test suite, far-field probes.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
python tools/fp64_peak.py 10 > gpurun_out/fp64_peak_r02.json 2> gpurun_out/fp64_peak.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python tests/tools/far_probe.py 2 2000 '' 'lf_p_low=8' 'lf_p_low=10' 'eps_internal=1e-8' 'leaf_size=120' 'lowrank=0' > gpurun_out/far_c2.jsonl 2> gpurun_out/far_c2.err
for c in 1b 3 4; do timeout 600 python tests/tools/far_probe.py $c 2000 '' > gpurun_out/far_c$c.jsonl 2> gpurun_out/far_c$c.err; done
