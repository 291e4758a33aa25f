"""Plan-creation probe (diagnostics): python tools/plan_probe.py <config> [verbose=1]; prints the plan log and stats
(FDA_DEBUG=1 reports failing CUDA call sites)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1311_5202_b200 import fda  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "4"
verbose = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = synth.make_problem(cfg)
print("N", p.N, "k", p.k, flush=True)
fr, tot = torch.cuda.mem_get_info()
print("free GB", fr / 1e9, flush=True)
t0 = time.time()
try:
    h = fda.fda_plan_create(torch.from_numpy(p.x).cuda(), torch.from_numpy(p.n).cuda(), torch.from_numpy(p.w).cuda(),
                            p.k, p.alpha, p.eps, fda.fda_options_default(verbose=verbose))
    print(fda.fda_plan_log(h))
    print(fda.fda_plan_stats(h))
    fda.fda_plan_destroy(h)
except Exception as e:  # noqa: BLE001
    print("ERR", e)
print("t", time.time() - t0)
