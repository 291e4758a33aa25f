"""Which plan parameter caps the accuracy below eps = 1e-4?  Table-1 kernel on the cube-sphere t1 / t1b
point sets at a given eps with option variants; eps_a on 400 targets against the oracle.
    python tests/tools/eps_probe.py EPS 'opt=v,opt=v' ...        (one JSON line per variant)"""
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


eps = float(sys.argv[1])
for m, k in ((32, 8 * np.pi), (64, 16 * np.pi)):
    x, n, w, _, _ = synth.quadrature_cloud(synth.cube_sphere(m))
    N = x.shape[0]
    q = synth.random_phi(N, 31)
    rows = synth.sample_rows(N, 400, 5)
    ref = oracle.apply_rows(x, n, np.ones(N), k, 1j / k, q, rows=rows, kind=oracle.KIND_T1)
    d_q = torch.from_numpy(q.view(np.float64).copy()).cuda()
    d_p = torch.empty_like(d_q)
    for v in sys.argv[2:] or [""]:
        h = fda.fda_plan_create(x, n, np.ones(N), k, 1j / k, eps,
                                fda.fda_options_default(kernel=fda.FDA_KERNEL_T1, **parse(v)))
        fda.fda_apply(h, d_q, d_p)
        ms = sum(fda.fda_apply_timed(h, fda.FDA_PHASE_ALL, d_q, d_p).values())
        got = d_p.cpu().numpy().view(np.complex128)
        fda.fda_plan_destroy(h)
        print(json.dumps({"N": N, "eps": eps, "variant": v, "eps_a": oracle.rel_l2(got[rows], ref), "apply_ms": ms}),
              flush=True)
