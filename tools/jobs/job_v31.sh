#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python tests/tools/solve.py 5 1e-4 > gpurun_out/solve_c5.json 2> gpurun_out/solve_c5.err
