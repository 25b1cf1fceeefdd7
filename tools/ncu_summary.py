"""Per-kernel summary of an ncu --set full report (ncu -i ... --page details --csv):
duration, throughputs, occupancy, issue statistics and the top warp-stall reasons.

usage: python tools/ncu_summary.py report.ncu-rep > summary.md
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ("Duration", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "No Eligible", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Executed Instructions", "Grid Size", "Block Size")


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(path):
    det = list(csv.reader(io.StringIO(run([path, "--page", "details", "--csv"]))))
    h = det[0]
    ki, ii = h.index("Kernel Name"), h.index("ID")
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = collections.OrderedDict()
    for r in det[1:]:
        d = per.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("void ", "")})
        if r[mi] in KEYS:
            d[r[mi]] = "%s %s" % (r[vi], r[ui])
    raw = list(csv.reader(io.StringIO(run([path, "--page", "raw", "--csv"]))))
    rh = raw[0]
    stalls = {}
    for row in raw[2:]:
        kid = row[rh.index("ID")]
        st = []
        for n, x in zip(rh, row):
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
                try:
                    st.append((float(x), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1.0
        stalls[kid] = ", ".join("%s %.0f%%" % (n, 100 * v / tot) for v, n in sorted(st)[::-1][:5])
    for kid, d in per.items():
        print("### `%s` (ID %s)\n" % (d["name"], kid))
        print("| metric | value |\n|---|---|")
        for k in KEYS:
            if k in d:
                print("| %s | %s |" % (k, d[k]))
        print("| top stall reasons (PC samples) | %s |\n" % stalls.get(kid, ""))


if __name__ == "__main__":
    main(sys.argv[1])
