"""Summarises ncu reports (--set full) into markdown + a traffic JSON for bench.py.

  python tools/ncu_summary.py out.md traffic.json rep1.ncu-rep [rep2.ncu-rep ...]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem throughput % of peak"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "long-scoreboard"),
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          ",".join(m for m, _ in METRICS)], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    h, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {"kernel": row[h.index("Kernel Name")], "id": row[h.index("ID")]}
        for m, _ in METRICS:
            if m in h:
                i = h.index(m)
                d[m] = (row[i], units[i])
        res.append(d)
    return res


def to_bytes(v, unit):
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)


def main():
    md, tj, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    lines = ["| report | kernel | " + " | ".join(n for _, n in METRICS) + " |",
             "|" + "---|" * (len(METRICS) + 2)]
    traffic = {}
    for rep in reps:
        for d in rows(rep):
            name = d["kernel"].split("(")[0][:70]
            cells = []
            for m, _ in METRICS:
                v = d.get(m)
                cells.append(f"{v[0]} {v[1]}".strip() if v else "")
            lines.append(f"| {rep.split('/')[-1]} | `{name}` | " + " | ".join(cells) + " |")
            if "dram__bytes_read.sum" in d:
                rd = to_bytes(*d["dram__bytes_read.sum"])
                wr = to_bytes(*d["dram__bytes_write.sum"])
                traffic.setdefault(name, []).append(rd + wr)
    with open(md, "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(tj, "w") as f:
        json.dump({k: sum(v) / len(v) for k, v in traffic.items()}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
