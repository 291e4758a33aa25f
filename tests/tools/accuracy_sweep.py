"""Accuracy / speed trade-off of the plan knobs on one config (GPU):

    python tools/accuracy_sweep.py CFG 'eps_internal=1e-5' 'lf_p_switch=0.7' ...

Each argument is one variant (comma-separated option=value list; '' = defaults).  For each:
plan setup time, apply ms (CUDA events, median of 5), rel l2 and far-only rel l2 against the
oracle on 2000 seeded rows.  Prints one JSON line per variant.
"""
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


def parse(v):
    kw = {}
    for item in filter(None, v.split(",")):
        k, x = item.split("=")
        kw[k] = float(x) if any(c in x for c in ".e") else int(x)
    return kw


def main():
    cfg = sys.argv[1]
    variants = sys.argv[2:] or [""]
    p = synth.make_problem(cfg)
    csr = p.correction(seed=2024)
    phi = synth.random_phi(p.N, 2025)
    rows = synth.sample_rows(p.N, 2000, 7)
    ref = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, rows=rows, csr=csr)
    dev = torch.device("cuda", 0)
    d_phi = torch.from_numpy(phi.view(np.float64)).to(dev)
    d_out = torch.empty_like(d_phi)
    for v in variants:
        kw = parse(v)
        t0 = time.time()
        h = fda.fda_plan_create(torch.from_numpy(p.x).to(dev), torch.from_numpy(p.n).to(dev),
                                torch.from_numpy(p.w).to(dev), p.k, p.alpha, p.eps,
                                fda.fda_options_default(verbose=1, **kw))
        fda.fda_plan_set_correction(h, csr[0], csr[1], csr[2].view(np.float64))
        t_plan = time.time() - t0
        fda.fda_apply(h, d_phi, d_out)
        got = d_out.cpu().numpy().view(np.complex128).copy()
        fda.fda_apply_phases(h, fda.FDA_PHASE_NEAR | fda.FDA_PHASE_CORR, d_phi, d_out)
        near = d_out.cpu().numpy().view(np.complex128)[rows].copy()
        ms = []
        phases = None
        for _ in range(5):
            ph = fda.fda_apply_timed(h, fda.FDA_PHASE_ALL, d_phi, d_out)
            ms.append(sum(ph.values()))
            phases = ph
        st = fda.fda_plan_stats(h)
        log = fda.fda_plan_log(h)
        fda.fda_plan_destroy(h)
        rel = float(np.linalg.norm(got[rows] - ref) / np.linalg.norm(ref))
        far = float(np.linalg.norm(got[rows] - ref) / np.linalg.norm(ref - near))
        print(json.dumps({"cfg": cfg, "variant": v, "plan_s": round(t_plan, 1), "apply_ms": float(np.median(ms)),
                          "rel_l2": rel, "far_rel_l2": far, "phases": {k: round(x, 3) for k, x in phases.items()},
                          "device_gb": st["device_bytes"] / 1e9, "m2l_gflop": st["flops_m2l"] / 1e9}), flush=True)
        print(log, file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()
