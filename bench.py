"""Benchmark: FDA Burton-Miller apply (BASELINE.json metric) on synthetic sphere / spheroid workloads.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl fda|reference]

One step = one full apply out = H phi (all §8(a) hot-path rows: permute, P2P,
correction SpMV, S2M, M2M, M2L, L2L, L2T, unpermute) through the C ABI, plus the
NCCL all-reduce that assembles the result when N > 1.  Prints ONE JSON line on
rank 0.  The plan (tree, lists, operators) is built once, outside the timed
region, and its setup time is reported separately.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "FDA apply sec and Mpoints/s at kD=1000, N=4M; frac of FP64/HBM roofline"
UNIT = "Mpoints/s"
WORKLOADS = {
    "1": "unit sphere N=3072 kD=10 (configs[0])",
    "2": "sphere D=2 N=196608 kD=1 (configs[1])",
    "3": "sphere D=2 N=397488 kD=100 (configs[2])",
    "4": "prolate spheroid 10:1:1 N=999600 kD=400 (configs[3])",
    "5": "sphere D=2 N=4009008 kD=1000 eps=1e-4 (configs[4], the metric's workload)",
}


def fp64_peaks(sm_mhz: float):
    """FP64 roofline peaks {"alu": DFMA, "tensor": DMMA} in TFLOP/s: measured on this pool's B200 by
    tools/fp64_peak.py (profiles/fp64_peak_r02.json, with its clock record; MEASURED_PEAKS.json has no FP64
    figure), else derived from the unit counts 148 SM x 64 FP64 FMA/clk x 2 flop x clock."""
    p = os.path.join(ROOT, "profiles", "fp64_peak_r02.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        src = "measured (tools/fp64_peak.py, profiles/fp64_peak_r02.json)"
        return {"alu": d["dfma_tflops"], "tensor": d["dmma_tflops"]}, src
    v = 148 * 64 * 2 * sm_mhz * 1e6 / 1e12
    return {"alu": v, "tensor": v}, "derived: 148 SM x 64 FP64 FMA/clk x 2 x sm_max_mhz"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            c = [x.strip() for x in line.split(",")]
            if len(c) < 9:
                continue
            try:
                sm.append(float(c[1]))
                mx.append(float(c[2]))
            except ValueError:
                continue
            for nm, v in zip(names, c[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


class stdout_to_stderr:
    """Send fd 1 to stderr while NCCL initialises (it may print its version on stdout); the bench's one JSON
    line goes to the real stdout."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)
        return False


def make_inputs(cfg: str, seed: int = 2024):
    p = synth.make_problem(cfg)
    csr = p.correction(seed=seed)
    phi = synth.random_phi(p.N, seed + 1)
    return p, csr, phi


def run_reference(args, rank, world):
    """Reference arm: the CPU oracle as it stands, on this host's cores, bounded sample of rows per step."""
    import oracle
    if rank != 0:
        return
    p, csr, phi = make_inputs(args.config)
    nrow = args.ref_rows
    rows_all = synth.sample_rows(p.N, nrow * (args.warmup + args.steps), 99)
    for w in range(args.warmup):
        oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, rows=rows_all[w * nrow:(w + 1) * nrow], csr=csr)
    t = []
    for s in range(args.steps):
        r = rows_all[(args.warmup + s) * nrow:(args.warmup + s + 1) * nrow]
        t0 = time.perf_counter()
        oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, rows=r, csr=csr)
        t.append(time.perf_counter() - t0)
    sec = float(np.sum(t))
    value = nrow * args.steps / sec / 1e6
    cores = oracle.num_threads()
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS.get(args.config, args.config), "N": p.N, "k": p.k, "eps": p.eps,
                       "rows_per_step": nrow},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{nrow} seeded rows of the {p.N}-point operator per step (direct O(N) sum per row + CSR row)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="5")
    ap.add_argument("--impl", default="fda", choices=["fda", "reference"])
    ap.add_argument("--kernel", default="bmh", choices=["bmh", "bmg"],
                    help="operator: Burton-Miller H (the metric's) or G (SURVEY §8(f) row 1)")
    ap.add_argument("--check-rows", type=int, default=2000)
    ap.add_argument("--ref-rows", type=int, default=200)
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="use the library's NCCL data plane (fda_plan_create_dist) even on one rank (tests the path)")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_1311_5202_b200 import fda

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    use_dist = world > 1 or args.dist
    quiet = stdout_to_stderr()
    quiet.__enter__()
    if use_dist:
        for key_, v_ in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29511"), ("RANK", "0"), ("WORLD_SIZE", "1")):
            os.environ.setdefault(key_, v_)
        dist.init_process_group("nccl", device_id=dev)
    t0 = time.time()
    p, csr, phi = make_inputs(args.config)
    t_gen = time.time() - t0
    t0 = time.time()
    kernel = fda.FDA_KERNEL_BMG if args.kernel == "bmg" else fda.FDA_KERNEL_BMH
    opt = fda.fda_options_default(verbose=1 if args.verbose else 0, kernel=kernel)
    pts, nrm, wts = (torch.from_numpy(a).to(dev) for a in (p.x, p.n, p.w))
    if use_dist:
        # the library's own data plane: NCCL communicator inside libfda, partial-expansion
        # exchange + output all-gather inside fda_apply; the process group only distributes the NCCL id
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(fda.fda_nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        h = fda.fda_plan_create_dist(pts, nrm, wts, p.k, p.alpha, p.eps, bytes(uid.cpu().numpy()), rank, world, opt)
    else:
        h = fda.fda_plan_create(pts, nrm, wts, p.k, p.alpha, p.eps, opt)
    torch.cuda.synchronize()
    t_create = time.time() - t0
    # the correction CSR (24.5 GB at config 5) comes from pageable host memory: its upload is the caller's
    # input transfer, reported apart from the plan build
    fda.fda_plan_set_correction(h, csr[0], csr[1], csr[2].view(np.float64))
    torch.cuda.synchronize()
    t_plan = time.time() - t0
    stream = torch.cuda.current_stream(dev)
    fda.fda_plan_set_stream(h, stream.cuda_stream)
    st = fda.fda_plan_stats(h)
    if args.verbose and rank == 0:
        print(fda.fda_plan_log(h), file=sys.stderr)
    d_phi = torch.from_numpy(phi.view(np.float64)).to(dev)
    d_out = torch.empty_like(d_phi)
    N = p.N

    def step():
        fda.fda_apply(h, d_phi, d_out)     # multi-GPU: exchange + output all-gather inside (full out on every rank)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    quiet.__exit__(None, None, None)
    # ---- timed region (device time, CUDA events on the launching stream)
    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches_step = launches_per_step(h)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = N / (ms * 1e-3) / 1e6
    # ---- per-phase CUDA-event times (separate applies after the timed region; phases serialised)
    phases = {}
    for _ in range(args.steps):
        for key, v in fda.fda_apply_timed(h, fda.FDA_PHASE_ALL, d_phi, d_out).items():
            phases[key] = phases.get(key, 0.0) + v
    torch.cuda.synchronize()

    # ---- end to end through the public API with HOST buffers (pinned), copies inside the timed region
    h_phi = torch.from_numpy(phi.view(np.float64)).pin_memory()
    h_out = torch.empty_like(h_phi).pin_memory()
    fda.fda_apply(h, h_phi, h_out)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fda.fda_apply(h, h_phi, h_out)
    e2e_s = (time.perf_counter() - t0) / args.steps
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    # ---- parity at full size on seeded sampled rows (oracle, outside the timed region; rank 0)
    parity = None
    cpu_baseline = None
    if not args.no_check:      # the applies are collective on every rank; the oracle runs on rank 0
        fda.fda_apply(h, d_phi, d_out)
        got = d_out.cpu().numpy().view(np.complex128).copy()
        fda.fda_apply_phases(h, fda.FDA_PHASE_NEAR | fda.FDA_PHASE_CORR, d_phi, d_out)
        near = d_out.cpu().numpy().view(np.complex128).copy()
    if rank == 0 and not args.no_check:
        import oracle
        rows = synth.sample_rows(N, args.check_rows, 7)
        t0 = time.perf_counter()
        ref = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, rows=rows, csr=csr,
                                kind=oracle.KIND_BMG if args.kernel == "bmg" else oracle.KIND_BMH)
        t_or = time.perf_counter() - t0
        rel = float(np.linalg.norm(got[rows] - ref) / np.linalg.norm(ref))
        far = float(np.linalg.norm((got[rows] - near[rows]) - (ref - near[rows])) / np.linalg.norm(ref - near[rows]))
        parity = {"rows": int(rows.shape[0]), "rel_l2": rel, "far_rel_l2": far, "tol": 1e-4, "pass": rel <= 1e-4}
        cpu_v = rows.shape[0] / t_or / 1e6
        cpu_baseline = {"value": cpu_v, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                        "sample": f"{rows.shape[0]} seeded rows of the full N={N} operator (direct sum + CSR), "
                                  f"{t_or:.1f} s"}

    # ---- roofline of the dominant phase
    pk, pk_kind = measured_peaks()
    sm_mhz = clk.get("sm_mhz") or pk.get("sm_max_mhz", 1965.0)
    per = {k_: v / args.steps for k_, v in phases.items()}
    flops = {"p2p": st["flops_p2p"], "m2l": st["flops_m2l"], "m2m": st["flops_m2m"], "l2l": st["flops_l2l"],
             "s2m": st["flops_s2m"], "l2t": st["flops_l2t"]}
    dom = max(per, key=lambda k_: per[k_]) if per else "m2l"
    traffic = None
    tp = os.path.join(ROOT, "profiles", "r02", "traffic.json")
    if not os.path.exists(tp):
        tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"config{args.config}", {}).get(dom)
    peak64, peak_src = fp64_peaks(pk.get("sm_max_mhz", 1965.0))
    # bound of each phase: the translations run on the FP64 tensor pipe (DMMA), P2P / surface
    # evaluations on the FP64 ALU (sincos, rsqrt, DFMA), the correction SpMV on HBM
    bound = {"m2l": "tensor", "m2m": "tensor", "l2l": "tensor", "p2p": "alu", "s2m": "alu", "l2t": "alu"}

    # stored leaf S2M / L2T matrices: those phases are one HBM read of the matrices
    hbm_bytes = {"csr": st["bytes_csr"], "s2m": st.get("bytes_s2m", 0.0), "l2t": st.get("bytes_l2t", 0.0)}

    def phase_roof(ph):
        if hbm_bytes.get(ph, 0.0) > 0:
            a = hbm_bytes[ph] / (per[ph] * 1e-3) / 1e9
            return {"bound": "hbm", "achieved": a, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": a / pk["hbm_gbs"],
                    "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({pk_kind})"}
        a = flops.get(ph, 0.0) / (per[ph] * 1e-3) / 1e12
        b = bound.get(ph, "alu")
        return {"bound": b, "achieved": a, "peak": peak64[b], "unit": "TFLOP/s", "frac": a / peak64[b],
                "peak_source": f"FP64 {'DMMA' if b == 'tensor' else 'DFMA'} peak, {peak_src}"}

    roof = dict(phase_roof(dom), traffic=traffic, kernel=dom)
    roof_phases = {ph: {k_: (round(v, 4) if isinstance(v, float) else v) for k_, v in phase_roof(ph).items()
                        if k_ in ("bound", "achieved", "frac")}
                   for ph in ("p2p", "csr", "s2m", "m2m", "m2l", "l2l", "l2t") if per.get(ph, 0) > 0}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "apply_s": ms * 1e-3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": WORKLOADS.get(args.config, args.config), "operator": args.kernel.upper(),
                           "parallelism": "single GPU" if not use_dist else
                           f"{world} Morton leaf range(s), libfda NCCL partial-expansion exchange + output all-gather",
                           "N": N, "k": p.k, "kD": p.k * float(np.ptp(p.x, axis=0).max()),
                           "eps": p.eps, "alpha": "i/k", "csr_nnz": int(st["csr_nnz"]),
                           "l2": "inputs larger than L2 (correction CSR %.1f GB)" % (st["csr_nnz"] * 20 / 1e9)},
                "e2e": {"value": N / e2e_s / 1e6, "unit": UNIT, "h2d_bytes_per_step": int(N * 16),
                        "d2h_bytes_per_step": int(N * 16)},
                "gpu_launches": None, "roofline": roof, "roofline_phases": roof_phases,
                "cpu_baseline": cpu_baseline, "clocks": clk,
                "phases_ms": {k_: round(v, 4) for k_, v in per.items()}, "parity": parity,
                "setup_s": {"inputs": round(t_gen, 2), "plan": round(t_plan, 2),
                            "plan_create": round(t_create, 2), "set_correction": round(t_plan - t_create, 2), "tree": st["setup_tree_s"],
                            "lists": st["setup_lists_s"], "ops": st["setup_ops_s"], "upload": st["setup_upload_s"]},
                "plan": {k_: st[k_] for k_ in ("nleaves", "nlevels", "lmin", "p2p_point_pairs", "m2l_pairs",
                                               "m2l_groups", "m2l_lowrank_groups", "m2l_ops", "out_slots", "in_slots",
                                               "device_bytes", "s2m_evals", "l2t_evals", "xchg_send_bytes",
                                               "xchg_recv_bytes")}}
        line["gpu_launches"] = launches_step * args.steps
        print(json.dumps(line), flush=True)
    fda.fda_plan_destroy(h)
    if use_dist:
        dist.destroy_process_group()


def launches_per_step(h):
    """Kernels the library launches per apply (from the plan structure)."""
    from paper_1311_5202_b200 import fda
    return fda.fda_plan_launches(h)


if __name__ == "__main__":
    main()
