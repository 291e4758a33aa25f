"""profiles/r02/traffic.json from an ncu launch list of the bench command (tools/jobs/r02_ncu.sh,
`-k regex:"k_(gtrans|m2l_warp|p2p|csr|s2m|l2t|leaf_s2m|leaf_l2t|permute|unpermute|xpack|xunpack)"`, metrics gpu__time_duration.sum and
dram__bytes_{read,write}.sum): DRAM bytes (read + write) per apply, summed over the launches of each
phase of the second apply in the list.  Launch order of api.cu's apply: permute, p2p, csr, then per LF
leaf level (S2M check + product), the M2M transitions, the M2L launches (one or two per level), the
L2L transitions, per LF leaf level (L2T product + evaluation), unpermute.

    python tools/make_traffic.py gpurun_out/launches_c5.csv config5 NLF NTRANS [out.json]
(NLF: LF leaf levels of the plan, NTRANS: transitions; config 5: 2 5)
"""
import csv
import json
import os
import sys


def main():
    path, key, nlf, ntr = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    out = sys.argv[5] if len(sys.argv) > 5 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                                "profiles", "r02", "traffic.json")
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hdr]
    per, order = {}, []
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        i = int(r[h.index("ID")])
        if i not in per:
            order.append(i)
            per[i] = {"name": r[h.index("Kernel Name")]}
        per[i][r[h.index("Metric Name")]] = float(r[h.index("Metric Value")])
    starts = [j for j, i in enumerate(order) if "k_permute_scale" in per[i]["name"]]
    a, b = starts[1], (starts[2] if len(starts) > 2 else len(order))
    ids = order[a:b]
    # stored leaf matrices (k_leaf_s2m / k_leaf_l2t): one launch per LF leaf level each; else two (surface
    # evaluation + product)
    per_lf = 1 if any("k_leaf_s2m" in per[i]["name"] for i in ids) else 2
    # the near field (P2P, correction) runs on a side stream / graph branch: its launches may sit anywhere
    # between the permute and the unpermute, so they are told apart by name; the far field keeps its order
    def near_phase(i):
        nm = per[i]["name"]
        return "p2p" if "k_p2p" in nm else "csr" if "k_csr" in nm else None
    near = [(near_phase(i), i) for i in ids if near_phase(i)]
    far = [i for i in ids if not near_phase(i)]
    nm2l = len(far) - 2 - 2 * per_lf * nlf - 2 * ntr
    seq = ["permute"] + ["s2m"] * (per_lf * nlf) + ["m2m"] * ntr + ["m2l"] * nm2l + ["l2l"] * ntr + \
          ["l2t"] * (per_lf * nlf) + ["unpermute"]
    assert len(seq) == len(far), (len(seq), len(far))
    res = {}
    for ph, i in list(zip(seq, far)) + near:
        d = per[i]
        res.setdefault(ph, {"dram_bytes": 0.0, "ms": 0.0, "launches": 0})
        res[ph]["dram_bytes"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        res[ph]["ms"] += d.get("gpu__time_duration.sum", 0) / 1e6
        res[ph]["launches"] += 1
    tot = sum(v["ms"] for v in res.values())
    for v in res.values():
        v["share"] = v["ms"] / tot
    data = json.load(open(out)) if os.path.exists(out) else {}
    data[key] = {ph: v["dram_bytes"] for ph, v in res.items()}
    data[key + "_detail"] = res
    os.makedirs(os.path.dirname(out), exist_ok=True)
    json.dump(data, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
