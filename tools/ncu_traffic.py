"""Per-launch DRAM traffic and headline counters from `ncu --set full` captures
(`ncu -i <rep> --page raw --csv`), written as the JSON bench.py reads for the
roofline `traffic` field.

usage: python tools/ncu_traffic.py OUT.json CONFIG=REP.ncu-rep [CONFIG=REP ...]"""
import csv
import io
import json
import subprocess
import sys

FIELDS = {
    "gpu__time_duration.sum": "gpu__time_duration_us",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__inst_executed.sum": "warp_instructions",
}
SCALE = {"ms": 1e3, "us": 1.0, "ns": 1e-3, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def launches(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[head.index("Kernel Name")][:60]}
        for k, name in FIELDS.items():
            if k not in head:
                continue
            i = head.index(k)
            v = float(r[i].replace(",", "")) if r[i] else 0.0
            d[name] = v * SCALE.get(units[i], 1.0) if name.endswith(("_us", "_bytes")) else v
        res.append(d)
    return res


def main(out, *pairs):
    doc = {}
    for p in pairs:
        cfg, rep = p.split("=", 1)
        ls = launches(rep)
        per = sum(l["dram_read_bytes"] + l["dram_write_bytes"] for l in ls) / max(len(ls), 1)
        doc[cfg] = {"dram_bytes_per_launch": per,
                    "source": f"ncu --set full --clock-control none, {ls[0]['kernel']}, "
                              f"bench.py --config {cfg} (L2 flushed between iterations)",
                    "launches": ls}
    json.dump(doc, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
