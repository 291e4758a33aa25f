"""Table 1 of the paper on the GPU.

    python tests/tools/table1.py [eps ...]          (default eps = 1e-4)

For each Table-1 point set (cube-sphere, N = 73,728 * 4^j, k = 8 pi 2^j, ~20 points per wavelength)
and each eps: the summation p_i = sum_{j != i} [G + alpha dG/dn_y] q_j (eq_sum, alpha = i/k, random
q with mean 0, unit weights) by the FDA apply in "improved" mode (reduced + low-rank M2L, the
default) and with the low-rank step off (lowrank = 0: reduced dense K~; our reduction is not
optional, so this is not the paper's "original"); eps_a at N_t = 200 random targets against the
oracle's direct sum.  Prints one JSON line per (row, mode); times are CUDA-event
phase times of one apply on this B200 (the paper's are single-core CPU seconds: context only).
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

ROWS = [("t1", 32, 8 * np.pi), ("t1b", 64, 16 * np.pi), ("t1c", 128, 32 * np.pi), ("t1d", 256, 64 * np.pi)]


def main():
    eps_list = [float(a) for a in sys.argv[1:]] or [1e-4]
    dev = torch.device("cuda", 0)
    for name, m, k in ROWS:
        x, n, w, hmax, smp = synth.quadrature_cloud(synth.cube_sphere(m))
        N = x.shape[0]
        ones = np.ones(N)
        alpha = 1j / k
        q = synth.random_phi(N, 31)
        rows = synth.sample_rows(N, 200, 5)
        ref = oracle.apply_rows(x, n, ones, k, alpha, q, rows=rows, kind=oracle.KIND_T1)
        d_q = torch.from_numpy(q.view(np.float64).copy()).to(dev)
        d_p = torch.empty_like(d_q)
        for eps in eps_list:
            for mode, lowrank in (("improved", 1), ("no-lowrank", 0)):
                t0 = time.time()
                h = fda.fda_plan_create(torch.from_numpy(x).to(dev), torch.from_numpy(n).to(dev),
                                        torch.from_numpy(ones).to(dev), k, alpha, eps,
                                        fda.fda_options_default(kernel=fda.FDA_KERNEL_T1, lowrank=lowrank))
                t_plan = time.time() - t0
                fda.fda_apply(h, d_q, d_p)
                ph = None
                for _ in range(3):
                    ph = fda.fda_apply_timed(h, fda.FDA_PHASE_ALL, d_q, d_p)
                got = d_p.cpu().numpy().view(np.complex128)
                st = fda.fda_plan_stats(h)
                fda.fda_plan_destroy(h)
                print(json.dumps({"row": name, "N": N, "k": k, "eps": eps, "mode": mode,
                                  "eps_a": oracle.rel_l2(got[rows], ref), "apply_ms": sum(ph.values()),
                                  "m2l_ms": ph["m2l"], "up_ms": ph["s2m"] + ph["m2m"], "plan_s": round(t_plan, 1),
                                  "device_gb": st["device_bytes"] / 1e9, "m2l_gflop": st["flops_m2l"] / 1e9}),
                      flush=True)


if __name__ == "__main__":
    main()
