import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import synth
from paper_1311_5202_b200 import fda
name = sys.argv[1]
t0 = time.time()
p = synth.make_problem(name)
print("N", p.N, "gen", time.time()-t0, flush=True)
opt = fda.fda_options_default(host_only=1)
h = fda.fda_plan_create(p.x, p.n, p.w, p.k, p.alpha, p.eps, opt)
print("plan", time.time()-t0, flush=True)
ml, mt, ms = fda.fda_plan_export_m2l(h)
fda.fda_plan_destroy(h)
np.savez(f"/tmp/st/m2l_{name}.npz", ml=ml, mt=mt, ms=ms)
for l in np.unique(ml):
    sel = ml == l
    t = mt[sel]; s = ms[sel]
    off = s - t
    # morton key of target
    def spread(v):
        v = v.astype(np.uint64) & np.uint64(0x1fffff)
        r = np.zeros_like(v)
        for b in range(21):
            r |= ((v >> np.uint64(b)) & np.uint64(1)) << np.uint64(3*b)
        return r
    key = (spread(t[:,0]) << np.uint64(2)) | (spread(t[:,1]) << np.uint64(1)) | spread(t[:,2])
    ukey, tid = np.unique(key, return_inverse=True)
    ntgt = len(ukey)
    offk = ((off[:,0]+64)*128 + (off[:,1]+64))*128 + (off[:,2]+64)
    print(f"level {l}: pairs {sel.sum()} targets {ntgt} pairs/target {sel.sum()/ntgt:.1f} offsets {len(np.unique(offk))}")
    for B in (32, 48, 64, 96, 128):
        blk = tid // B
        u = np.unique(blk.astype(np.int64) * 10**7 + offk)
        nch = len(u)
        print(f"   B={B}: (block,offset) groups {nch}, pairs per group {sel.sum()/nch:.1f}")
