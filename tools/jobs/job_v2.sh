./tools/jobs/gpu_bench.sh v2 3 5
timeout 1200 python tests/tools/accuracy_sweep.py 3 '' 'eps_internal=1e-5' 'lf_p_switch=0.7' 'eps_internal=3e-6,lf_p_switch=0.7' 'eps_internal=1e-5,lf_p_switch=0.7' > gpurun_out/sweep_c3.jsonl 2> gpurun_out/sweep_c3.err
