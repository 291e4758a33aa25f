"""Summarise an ncu report (--set full) into a small markdown table for profiles/.

    python tools/ncu_summary.py gpurun_out/prof_X.ncu-rep "label for each kernel id, comma separated" > profiles/...md

Per profiled kernel: duration, DRAM bytes (read + write), DRAM / L2 / L1 throughput, L2 hit rate,
FP64 tensor-pipe and FP64 pipe utilisation, issue-slot use, occupancy, registers, top stall reasons
and the source lines with the most warp-stall samples.
"""
import csv
import io
import subprocess
import sys


def ncu(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def num(v):
    try:
        return float(v)
    except (TypeError, ValueError):
        return None


def main():
    rep = sys.argv[1]
    labels = sys.argv[2].split(",") if len(sys.argv) > 2 else []
    raw = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    hdr, units = raw[0], raw[1]
    want = [("gpu__time_duration.sum", "duration"),
            ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
            ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
            ("lts__t_sector_hit_rate.pct", "L2 hit %"),
            ("sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", "FP64 tensor %"),
            ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
            ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 cycles %"),
            ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
            ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
            ("launch__registers_per_thread", "regs"),
            ("launch__grid_size", "grid"),
            ("launch__shared_mem_per_block_dynamic", "dyn smem")]
    print("| id | kernel | " + " | ".join(w[1] for w in want) + " | top stalls |")
    print("|" + "---|" * (len(want) + 3))
    for r in raw[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        kid = d.get("ID", "?")
        lab = labels[int(kid)] if kid.isdigit() and int(kid) < len(labels) else d.get("Kernel Name", "")[:30]
        cells = []
        for key, _ in want:
            v = d.get(key, "")
            cells.append(f"{v} {u.get(key, '')}".strip())
        st = [(k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), num(v))
              for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_") and
              k.endswith("_per_issue_active.ratio") and num(v)]
        st.sort(key=lambda kv: -kv[1])
        cells.append(", ".join(f"{k} {v:.1f}" for k, v in st[:4]))
        print(f"| {kid} | {lab} | " + " | ".join(cells) + " |")
    # hottest source lines of each kernel
    for i, lab in enumerate(labels or ["kernel"]):
        txt = ncu([rep, "--page", "source", "--csv", "--print-source=cuda,sass", "--kernel-id", f":::{i}"])
        rows = list(csv.reader(io.StringIO(txt)))
        if len(rows) < 4:
            continue
        h = rows[2]
        if "Warp Stall Sampling (All Samples)" not in h:
            continue
        k = h.index("Warp Stall Sampling (All Samples)")
        lines = [x for x in rows[3:] if x and x[0] not in ("", "Line No") and len(x) > k and num(x[k])]
        tot = sum(num(x[k]) for x in lines) or 1.0
        lines.sort(key=lambda x: -num(x[k]))
        print(f"\n**{lab}** — source lines by warp-stall samples:\n")
        for x in lines[:8]:
            print(f"- line {x[0]}: {100 * num(x[k]) / tot:.1f}% `{x[1].strip()[:90]}`")


if __name__ == "__main__":
    main()
