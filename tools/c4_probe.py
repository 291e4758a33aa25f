import sys, time
sys.path.insert(0, '.')
import numpy as np, torch, synth
from paper_1311_5202_b200 import fda
p = synth.make_problem("4")
print("N", p.N, "k", p.k, flush=True)
fr, tot = torch.cuda.mem_get_info(); print("free GB", fr/1e9, flush=True)
t0=time.time()
try:
    h = fda.fda_plan_create(torch.from_numpy(p.x).cuda(), torch.from_numpy(p.n).cuda(), torch.from_numpy(p.w).cuda(), p.k, p.alpha, p.eps, fda.fda_options_default(verbose=int(sys.argv[1]) if len(sys.argv) > 1 else 1))
    print(fda.fda_plan_log(h)); print(fda.fda_plan_stats(h)); fda.fda_plan_destroy(h)
except Exception as e:
    print("ERR", e)
print("t", time.time()-t0)
