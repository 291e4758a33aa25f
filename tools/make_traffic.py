"""profiles/traffic.json from an ncu metric capture of one apply (tools/job_*.sh mem_*.csv):
DRAM bytes (read + write) per apply, summed over the launches of each phase, in launch order of
api.cu's apply: permute, p2p, csr, s2m (check + product per LF level), m2m (per transition),
m2l (per level), l2l (per transition), l2t (product + evaluation per LF level), unpermute.

    python tools/make_traffic.py gpurun_out/mem_c5v11.csv config5 NLF NTRANS NM2L
(NLF LF leaf levels, NTRANS transitions, NM2L M2L levels of the plan; config 5: 2 4 5)
"""
import csv
import json
import os
import sys


def main():
    path, key, nlf, ntr, nm2l = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hdr]
    per = {}
    order = []
    for r in rows[hdr + 1:]:
        i = int(r[h.index("ID")])
        if i not in per:
            order.append(i)
            per[i] = {"name": r[h.index("Kernel Name")]}
        per[i][r[h.index("Metric Name")]] = float(r[h.index("Metric Value")])
    # find the start of an apply: k_permute_scale
    start = next(j for j, i in enumerate(order) if per[i]["name"].startswith("k_permute_scale"))
    seq = ["permute", "p2p", "csr"] + ["s2m"] * (2 * nlf) + ["m2m"] * ntr + ["m2l"] * nm2l + ["l2l"] * ntr + \
          ["l2t"] * (2 * nlf) + ["unpermute"]
    out = {}
    # consecutive applies launch the same sequence: read it cyclically from the first k_permute_scale
    # (the capture must hold at least one apply's worth of launches)
    n = len(seq)
    assert len(order) >= n, "capture shorter than one apply"
    base = [order[start + j] if start + j < len(order) else order[start + j - n] for j in range(n)]
    for ph, i in zip(seq, base):
        d = per[i]
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        out[ph] = out.get(ph, 0.0) + b
    tp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    allt = json.load(open(tp)) if os.path.exists(tp) else {}
    allt[key] = {k: int(v) for k, v in out.items()}
    allt["_about"] = ("DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per apply and phase, summed over the "
                      "phase's launches, from ncu metric captures (tools/make_traffic.py)")
    json.dump(allt, open(tp, "w"), indent=1)
    print(json.dumps(allt[key]))


if __name__ == "__main__":
    main()
