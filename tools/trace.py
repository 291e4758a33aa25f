"""Per-launch trace of one apply (FDA_TRACE=1): python tools/trace.py <config>"""
import os
import sys
import time

os.environ["FDA_TRACE"] = "1"
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1311_5202_b200 import fda  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "3"
extra = dict(a.split("=") for a in sys.argv[2:])
extra = {k: (float(v) if "." in v or "e" in v else int(v)) for k, v in extra.items()}
p = synth.make_problem(cfg)
t0 = time.time()
h = fda.fda_plan_create(torch.from_numpy(p.x).cuda(), torch.from_numpy(p.n).cuda(), torch.from_numpy(p.w).cuda(),
                        p.k, p.alpha, p.eps, fda.fda_options_default(verbose=1, **extra))
print("plan", time.time() - t0, flush=True)
print(fda.fda_plan_log(h), flush=True)
phi = torch.from_numpy(synth.random_phi(p.N, 1).view(np.float64)).cuda()
out = torch.empty_like(phi)
for it in range(2):
    print("---- apply", it, flush=True)
    fda.fda_apply(h, phi, out)
    torch.cuda.synchronize()
print(fda.fda_plan_stats(h))
