#!/bin/bash
# compute-sanitizer memcheck over the smoke apply (config 1) and a small HF plan (one tool per call)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python -c "
import __graft_entry__ as g; g.smoke()
import numpy as np, torch, synth
from paper_1311_5202_b200 import fda
p = synth.make_problem('x', k=50.0, nu=16)
h = fda.fda_plan_create(p.x, p.n, p.w, p.k, p.alpha, p.eps)
phi = torch.from_numpy(synth.random_phi(p.N, 1).view(np.float64)).cuda(); out = torch.empty_like(phi)
fda.fda_apply(h, phi, out); torch.cuda.synchronize(); fda.fda_plan_destroy(h)
h = fda.fda_plan_create(p.x, p.n, p.w, p.k, p.alpha, p.eps, fda.fda_options_default(kernel=fda.FDA_KERNEL_BMG))
fda.fda_apply(h, phi, out); torch.cuda.synchronize(); fda.fda_plan_destroy(h)
print('memcheck run done')
" > gpurun_out/memcheck.log 2>&1
echo "exit $?" >> gpurun_out/memcheck.log
