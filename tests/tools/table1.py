"""Table 1 of the paper on the GPU.

    python tests/tools/table1.py [eps ...]          (default eps = 1e-4)

For each Table-1 point set (cube-sphere, N = 73,728 * 4^j, k = 8 pi 2^j, ~20 points per wavelength)
and each eps: the summation p_i = sum_{j != i} [G + alpha dG/dn_y] q_j (eq_sum, alpha = i/k, random
q with mean 0, unit weights) by the FDA apply in the paper's three settings: "original" (unreduced
equivalent-density expansions, dense M2L: fda_options.original = 1, R24), "reduced" (SVD-
reduced basis, dense K~: lowrank = 0) and "improved" (reduced + low-rank M2L, the default); eps_a at
N_t = 200 random targets against the oracle's direct sum and the device memory of the
plan (Table 1's M column).  One JSON line per (row, eps, mode); times are CUDA-event phase times of one
apply on this B200 (the paper's are single-core CPU seconds: context only).

    python tests/tools/table1.py [--rows t1,t1b,...] eps ...
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
    args = sys.argv[1:]
    rows_sel = None
    if args and args[0] == "--rows":
        rows_sel = set(args[1].split(","))
        args = args[2:]
    eps_list = [float(a) for a in args] or [1e-4]
    dev = torch.device("cuda", 0)
    for name, m, k in ROWS:
        if rows_sel and name not in rows_sel:
            continue
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
            for mode, lowrank, orig in (("original", 0, 1), ("reduced", 0, 0), ("improved", 1, 0)):
                t0 = time.time()
                torch.cuda.synchronize()
                mem0 = torch.cuda.mem_get_info()[0]
                h = fda.fda_plan_create(torch.from_numpy(x).to(dev), torch.from_numpy(n).to(dev),
                                        torch.from_numpy(ones).to(dev), k, alpha, eps,
                                        fda.fda_options_default(kernel=fda.FDA_KERNEL_T1, lowrank=lowrank,
                                                                original=orig))
                t_plan = time.time() - t0
                torch.cuda.synchronize()
                plan_mem = (mem0 - torch.cuda.mem_get_info()[0]) / 1e9
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
                                  "device_gb": st["device_bytes"] / 1e9, "m2l_gflop": st["flops_m2l"] / 1e9,
                                  "plan_mem_gb": plan_mem}),
                      flush=True)


if __name__ == "__main__":
    main()
