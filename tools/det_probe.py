import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1311_5202_b200 import fda
name = sys.argv[1] if len(sys.argv) > 1 else "1b"
p = synth.make_problem(name)
csr = p.correction(seed=3)
phi = synth.random_phi(p.N, 5)
h = fda.fda_plan_create(p.x, p.n, p.w, p.k, p.alpha, p.eps)
fda.fda_plan_set_correction(h, csr[0], csr[1], csr[2].view(np.float64))
d_phi = torch.from_numpy(phi.view(np.float64).copy()).cuda()
outs = []
for i in range(4):
    d_out = torch.empty_like(d_phi)
    fda.fda_apply(h, d_phi, d_out)
    torch.cuda.synchronize()
    outs.append(d_out.cpu().numpy().copy())
ph = fda.fda_apply_timed(h, fda.FDA_PHASE_ALL, d_phi, d_out)
fda.fda_plan_destroy(h)
same = [bool(np.array_equal(outs[0], o)) for o in outs[1:]]
md = max(float(np.max(np.abs(outs[0] - o))) for o in outs[1:])
np.save(f"/tmp/det_{os.environ.get('TAG','x')}.npy", outs[0])
print({"env": {k: v for k, v in os.environ.items() if k.startswith("FDA_")}, "N": p.N, "bit_identical": same, "max_abs_diff": md,
       "ms": sum(ph.values()), "phases": {k: round(v, 3) for k, v in ph.items()}})
