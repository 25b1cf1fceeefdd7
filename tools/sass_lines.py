"""Attribute ncu per-instruction metrics (source page, SASS) to CUDA source lines using the
line table of the same cubin (nvdisasm --print-line-info).

usage: python tools/sass_lines.py ncu_source_sass.csv nvdisasm_lineinfo.txt KERNEL_SUBSTR
"""
import collections
import csv
import re
import sys


def line_table(path, kernel):
    cur_fn, line, table = None, None, {}
    for raw in open(path):
        m = re.match(r"\s*\.text\.(\S+):", raw)
        if m:
            cur_fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', raw)
        if m:
            line = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(\S.*?);", raw)
        if m and cur_fn and kernel in cur_fn:
            table[int(m.group(1), 16)] = (line, m.group(2).strip())
    return table


def main(csv_path, li_path, kernel):
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r)
    h = rows[hi]
    data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0].startswith("0x")]
    ai, si, ie = (h.index("Address"), h.index("Warp Stall Sampling (All Samples)"),
                  h.index("Instructions Executed"))
    base = int(data[0][ai], 16)
    table = line_table(li_path, kernel)
    per_line = collections.defaultdict(lambda: [0.0, 0.0])
    tot_s = tot_i = 0.0
    for r in data:
        off = int(r[ai], 16) - base
        ln = table.get(off, (("?", 0), ""))[0]
        s, n = float(r[si] or 0), float(r[ie] or 0)
        per_line[ln][0] += s
        per_line[ln][1] += n
        tot_s += s
        tot_i += n
    print("samples %.0f  warp-instructions %.0f" % (tot_s, tot_i))
    for ln, (s, n) in sorted(per_line.items(), key=lambda x: -x[1][0])[:40]:
        print("%-24s stall %5.1f%%  instr %5.1f%%" % ("%s:%d" % ln, 100 * s / tot_s, 100 * n / tot_i))


if __name__ == "__main__":
    main(*sys.argv[1:4])
