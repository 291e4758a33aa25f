#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python tests/tools/eps_probe.py 1e-6 '' 'lf_p_low=8,lf_p_high=10' 'lf_p_low=10,lf_p_high=12' 'hf_spacing=0.15' 'lf_p_low=10,lf_p_high=12,hf_spacing=0.15' 'hf_max_rows=12000' > gpurun_out/eps_probe.jsonl 2> gpurun_out/eps_probe.err
