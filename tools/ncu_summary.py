"""Key numbers of one ncu --set full capture (first kernel in the report) as
JSON: duration, DRAM bytes, issue/warp activity, FP64 pipe, stall reasons per
issue, and the source lines with the most warp-stall samples.
usage: python tools/ncu_summary.py REPORT.ncu-rep [top_lines]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, top=15):
    raw = ncu_csv(rep, "--page", "raw")
    h, units, v = raw[0], raw[1], raw[2]
    res = {"report": rep.split("/")[-1], "kernel": v[h.index("Kernel Name")][:120]}
    for k in KEYS:
        if k in h:
            res[k] = f"{v[h.index(k)]} {units[h.index(k)]}".strip()
    res["stalls_per_issue"] = {
        k.split("issue_stalled_")[1].split("_per_issue")[0]: float(x)
        for k, x in zip(h, v)
        if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")
        and x not in ("", "0") and float(x) > 0.05}
    src = ncu_csv(rep, "--page", "source", "--print-source", "cuda,sass")
    lines, tot = [], 0
    for r in src[3:]:
        if len(r) < 8 or r[2] != "-":
            continue
        try:
            s, i = int(r[4]), int(r[7])
        except ValueError:
            continue
        tot += s
        lines.append((s, i, r[0], r[1].strip()[:100]))
    lines.sort(reverse=True)
    res["top_lines"] = [{"line": ln, "samples_pct": round(100 * s / max(tot, 1), 1),
                         "source": t} for s, i, ln, t in lines[:top]]
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 15)
