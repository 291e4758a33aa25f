"""profiles/r02/table1.md rows from the JSON lines of tests/tools/table1.py, next to the paper's Table 1
(`tab_improve`: single-core CPU seconds and MB -- context, not a target).

    python tools/table1_md.py gpurun_out/table1.jsonl > rows.md
"""
import json
import sys

# (eps, N) -> T_M2L orig, impr (s); T_up orig, impr (s); eps_a orig, impr; M orig, impr (MB)
PAPER = {
    (1e-4, 73728): (10, 4, 5, 3, 4.86e-5, 5.88e-5, 310, 158),
    (1e-4, 294912): (44, 17, 17, 10, 7.30e-5, 1.31e-4, 735, 441),
    (1e-4, 1179648): (218, 94, 103, 58, 1.15e-4, 2.33e-4, 1993, 1338),
    (1e-4, 4718592): (966, 383, 458, 214, 2.00e-4, 3.70e-4, 6818, 5053),
    (1e-6, 73728): (33, 11, 12, 7, 2.97e-7, 9.33e-7, 1010, 471),
    (1e-6, 294912): (154, 55, 59, 36, 7.75e-7, 2.72e-6, 2186, 1189),
    (1e-6, 1179648): (631, 235, 218, 145, 1.30e-6, 3.83e-6, 4744, 2941),
    (1e-6, 4718592): (2937, 1145, 1153, 742, 3.26e-6, 1.06e-5, 13938, 9764),
    (1e-8, 73728): (93, 29, 24, 16, 2.39e-8, 2.79e-8, 2644, 1156),
    (1e-8, 294912): (421, 137, 119, 84, 4.93e-8, 1.11e-7, 5154, 2684),
    (1e-8, 1179648): (1806, 602, 563, 384, 7.12e-8, 7.27e-8, 10147, 5944),
    (1e-8, 4718592): (7721, 2527, 2478, 1586, 1.71e-7, 2.55e-7, 26860, 18121),
}


def main():
    recs = {}
    for line in open(sys.argv[1]):
        line = line.strip()
        if line.startswith("{"):
            d = json.loads(line)
            recs[(d["eps"], d["N"], d["mode"])] = d
    print("| ε | N | k | T_M2L ms orig / red / impr (paper s orig / impr) | M2L orig/impr (paper) | T_up ms orig / impr "
          "(paper s) | ε_a orig / impr (paper orig / impr) | M GB orig / impr (paper MB) | apply ms impr |")
    print("|---|---|---|---|---|---|---|---|---|")
    for (eps, N), p in PAPER.items():
        o, r, i = (recs.get((eps, N, m)) for m in ("original", "reduced", "improved"))
        if not (o and r and i):
            have = [m for m in ("original", "reduced", "improved") if recs.get((eps, N, m))]
            print(f"| {eps:g} | {N:,} | | not run ({', '.join(have) or 'no mode'} measured) | | | | | |")
            continue
        print(f"| {eps:g} | {N:,} | {o['k']:.4g} | {o['m2l_ms']:.1f} / {r['m2l_ms']:.1f} / {i['m2l_ms']:.1f} ({p[0]} / {p[1]}) "
              f"| {o['m2l_ms'] / i['m2l_ms']:.1f}x ({p[0] / p[1]:.1f}x) | {o['up_ms']:.1f} / {i['up_ms']:.1f} ({p[2]} / {p[3]}) "
              f"| {o['eps_a']:.2e} / {i['eps_a']:.2e} ({p[4]:.2e} / {p[5]:.2e}) "
              f"| {o['device_gb']:.2f} / {i['device_gb']:.2f} ({p[6]} / {p[7]}) | {i['apply_ms']:.1f} |")


if __name__ == "__main__":
    main()
