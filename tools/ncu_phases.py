"""Per-phase warp-stall breakdown of one kernel in an ncu report (source page, SASS view): the
instruction stream is cut at block / cluster barriers and each region's stall samples are
summed by reason.   python tools/ncu_phases.py report.ncu-rep [kernel-substring]"""
import csv
import subprocess
import sys

REASONS = ["stall_long_sb", "stall_short_sb", "stall_mio", "stall_lg", "stall_math", "stall_wait", "stall_barrier",
           "stall_membar", "stall_not_selected", "stall_selected", "stall_branch_resolving", "stall_dispatch",
           "stall_no_inst", "stall_drain", "stall_misc", "stall_sleep", "stall_tex"]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] +
                         (["-k", sys.argv[2]] if len(sys.argv) > 2 else []), capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, data = rows[1], rows[2:]
    ix = {r: hdr.index(r) for r in REASONS if r in hdr}
    iS, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    total = sum(int(r[iS]) for r in data if r[iS].isdigit())
    acc = {r: 0 for r in ix}
    n = 0
    start = 0
    for k, r in enumerate(data):
        for name, i in ix.items():
            acc[name] += int(r[i]) if r[i].isdigit() else 0
        n += int(r[iS]) if r[iS].isdigit() else 0
        src = r[iSrc].strip()
        if ("BAR.SYNC" in src or "UCGABAR_WAIT" in src or k == len(data) - 1) and n:
            top = sorted(acc.items(), key=lambda kv: -kv[1])[:4]
            print(f"[{start:5d}-{k:5d}] {n:5d} samples ({100.0 * n / total:4.1f}%)  " +
                  "  ".join(f"{a[6:]} {b}" for a, b in top if b))
            acc = {r: 0 for r in ix}
            n = 0
            start = k + 1
    print("total", total)


if __name__ == "__main__":
    main()
