"""Time fda_nystrom_weights on every non-self (field point, element) pair of the local
regions D_i of a synthetic sphere: device-resident inputs and outputs, wall clock around the synchronising call.

    python tools/nystrom_bench.py [--config 1b] [--reps 5]
Prints one JSON line: pairs, pairs per second, ms per call."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1311_5202_b200 import fda  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="1b")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--nq", type=int, default=0)
    ap.add_argument("--theta", type=float, default=0.0)
    ap.add_argument("--gamma", type=float, default=0.0)
    a = ap.parse_args()
    p = synth.make_problem(a.config)
    ptr, idx = synth.local_regions(p.samples, p.hmax, p.x)
    ts = np.repeat(np.arange(p.N, dtype=np.int64), np.diff(ptr))
    es = idx.astype(np.int64)
    keep = es != ts // 6
    ts, es = np.ascontiguousarray(ts[keep]), np.ascontiguousarray(es[keep])
    rp = synth.rule_points()
    dev = torch.device("cuda", 0)
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in
         dict(nodes=p.nodes, xi=rp[:, :2], wref=0.5 * rp[:, 2], x=p.x, n=p.n, ts=ts, es=es).items()}
    out = torch.zeros(ts.shape[0], 12, dtype=torch.float64, device=dev)
    dl = torch.zeros_like(out)
    times = []
    for _ in range(a.reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fda.fda_nystrom_weights(fda.FDA_KERNEL_BMH, p.k, p.alpha, d["nodes"], d["xi"], d["wref"], d["x"], d["n"],
                                d["ts"], d["es"], out, dl, nq=a.nq, theta=a.theta, gamma=a.gamma)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    t = min(times[1:])
    print(json.dumps({"config": a.config, "N": p.N, "pairs": int(ts.shape[0]), "pairs_per_point": ts.shape[0] / p.N,
                      "ms": 1e3 * t, "Mpairs_per_s": ts.shape[0] / t / 1e6, "nq": a.nq or 8, "gamma": a.gamma or 0.05, "theta": a.theta or 0.5,
                      "checksum": float(out.abs().sum().item())}))


if __name__ == "__main__":
    main()
