"""Far-field accuracy probe on a benchmark config (BM_H operator), per plan-option variant.

    python tests/tools/far_probe.py CONFIG ROWS 'opt=v,opt=v' ...     (one JSON line per variant)

For each variant: relative l2 of the full apply and of the far field alone
 on ROWS seeded rows, for a random density (Re, Im U(-1,1),
PAPER.md:889-890) and for the smooth plane-wave density phi = e^{ik d.x}
(PAPER.md:1043-1048), against the CPU oracle."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1311_5202_b200 import fda  # noqa: E402


def parse(v):
    kw = {}
    for item in filter(None, v.split(",")):
        k, x = item.split("=")
        kw[k] = float(x) if any(c in x for c in ".e") else int(x)
    return kw


cfg, nrows = sys.argv[1], int(sys.argv[2])
p = synth.make_problem(cfg)
csr = p.correction(seed=2024)
rows = synth.sample_rows(p.N, nrows, 7)
dens = {"random": synth.random_phi(p.N, 2025), "planewave": synth.plane_wave(p.x, p.k, (0.0, 0.6, 0.8))}
refs = {nm: oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, rows=rows, csr=csr) for nm, phi in dens.items()}
dev = torch.device("cuda", 0)
for v in sys.argv[3:] or [""]:
    h = fda.fda_plan_create(torch.from_numpy(p.x).to(dev), torch.from_numpy(p.n).to(dev),
                            torch.from_numpy(p.w).to(dev), p.k, p.alpha, p.eps, fda.fda_options_default(**parse(v)))
    fda.fda_plan_set_correction(h, csr[0], csr[1], csr[2].view(np.float64))
    res = {"config": cfg, "N": p.N, "variant": v}
    for nm, phi in dens.items():
        d_phi = torch.from_numpy(phi.view(np.float64).copy()).to(dev)
        d_out = torch.empty_like(d_phi)
        fda.fda_apply(h, d_phi, d_out)
        got = d_out.cpu().numpy().view(np.complex128)[rows].copy()
        fda.fda_apply_phases(h, fda.FDA_PHASE_NEAR | fda.FDA_PHASE_CORR, d_phi, d_out)
        near = d_out.cpu().numpy().view(np.complex128)[rows].copy()
        ref = refs[nm]
        res[nm] = {"rel_l2": oracle.rel_l2(got, ref), "far_rel_l2": oracle.rel_l2(got - near, ref - near),
                   "far_over_near": float(np.linalg.norm(ref - near) / np.linalg.norm(near)),
                   "max_row_rel": float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))}
    res["apply_ms"] = sum(fda.fda_apply_timed(h, fda.FDA_PHASE_ALL, d_phi, d_out).values())
    fda.fda_plan_destroy(h)
    print(json.dumps(res), flush=True)
