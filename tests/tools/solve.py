"""Time a GMRES solve at a benchmark config on the GPU (solver plumbing around the apply; SURVEY §8(f)
row 3).  python tests/tools/solve.py [config] [tol]  -> one JSON line: applies, seconds per
iteration (apply + Krylov work), final residual, oracle residual on 200 rows.  The paper's context
figure: 250 s per GMRES iteration for its 4M-point submarine on one CPU core."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1311_5202_b200 import fda  # noqa: E402
from paper_1311_5202_b200.gmres import gmres  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "5"
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-4
p = synth.make_problem(cfg)
csr = p.correction(seed=2024)
b = np.exp(1j * p.k * (p.x @ np.array([0.0, 0.6, 0.8])))
dev = torch.device("cuda", 0)
plan = fda.Plan(torch.from_numpy(p.x).to(dev), torch.from_numpy(p.n).to(dev), torch.from_numpy(p.w).to(dev),
                p.k, p.alpha, p.eps)
plan.set_correction(csr[0], csr[1], csr[2].view(np.float64))
db = torch.from_numpy(b).to(dev)
torch.cuda.synchronize()
t0 = time.time()
x, hist, napply = gmres(plan.h, db, tol=tol, restart=30, maxiter=400)
torch.cuda.synchronize()
dt = time.time() - t0
plan.close()
rows = synth.sample_rows(p.N, 200, 3)
xs = x.cpu().numpy()
res = oracle.rel_l2(oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, xs, rows=rows, csr=csr), b[rows])
print(json.dumps({"config": cfg, "N": p.N, "tol": tol, "applies": napply, "seconds": dt,
                  "s_per_apply": dt / napply, "final_residual": hist[-1], "oracle_residual_200_rows": res}))
