"""GPU diagnostics: far-field error of plan variants against the oracle (dev tool).

    python tools/diag.py [config] [variant ...]
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1311_5202_b200 import fda  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run(h, phi, mask=None):
    d = dev(phi.view(np.float64))
    o = torch.empty_like(d)
    if mask is None:
        fda.fda_apply(h, d, o)
    else:
        fda.fda_apply_phases(h, mask, d, o)
    torch.cuda.synchronize()
    return o.cpu().numpy().view(np.complex128)


VARIANTS = {
    "default": {},
    "nolowrank": {"lowrank": 0},
    "p8": {"lf_p_low": 8},
    "leaf150": {"leaf_size": 150},
    "leaf150nolr": {"leaf_size": 150, "lowrank": 0},
    "eps1e-7": {"eps_internal": 1e-7},
    "eps1e-7nolr": {"eps_internal": 1e-7, "lowrank": 0},
    "eps1e-6": {"eps_internal": 1e-6},
    "p10": {"lf_p_high": 10},
    "p10eps1e-6": {"lf_p_high": 10, "eps_internal": 1e-6},
    "rows12k": {"hf_max_rows": 12000},
    "sp02": {"hf_spacing": 0.2},
}


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "1"
    names = sys.argv[2:] or list(VARIANTS)
    if cfg.startswith("nu"):
        nu, k = cfg[2:].split("k")
        p = synth.make_problem("x", k=float(k), nu=int(nu))
    else:
        p = synth.make_problem(cfg)
    phi = synth.random_phi(p.N, 5)
    t0 = time.time()
    ref = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi)
    print(f"N={p.N} k={p.k} oracle {time.time() - t0:.1f}s", flush=True)
    for nm in names:
        kw = dict(VARIANTS[nm])
        kw["verbose"] = 1
        opt = fda.fda_options_default(**kw)
        t0 = time.time()
        h = fda.fda_plan_create(dev(p.x), dev(p.n), dev(p.w), p.k, p.alpha, 1e-4, opt)
        tp = time.time() - t0
        got = run(h, phi)
        near = run(h, phi, fda.FDA_PHASE_NEAR)
        ms = fda.fda_apply_timed(h, fda.FDA_PHASE_ALL, dev(phi.view(np.float64)), dev(np.zeros(2 * p.N)))
        st = fda.fda_plan_stats(h)
        lg = fda.fda_plan_log(h)
        fda.fda_plan_destroy(h)
        err = oracle.rel_l2(got, ref)
        ferr = oracle.rel_l2(got - near, ref - near)
        print(f"[{nm}] plan {tp:.1f}s rel {err:.3e} far {ferr:.3e} ms " +
              json.dumps({k: round(v, 3) for k, v in ms.items()}), flush=True)
        print(lg, flush=True)


if __name__ == "__main__":
    main()
