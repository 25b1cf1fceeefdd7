"""Summarise an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_*]) of one
ALS round into a markdown table: per kernel count, total time, share, DRAM bytes.

usage: python tools/launch_table.py launches.csv > profiles/rNN_launches.md
"""
import collections
import csv
import sys

MTTKRP = ("hash_insert", "rep_flag", "rep_compact", "lookup_kernel", "finalize_counts",
          "item_count", "item_fill", "cta_hist", "cta_prefix", "rows_hit", "cta_scatter",
          "bucket_offsets", "bucket_scatter", "bucket_rows", "spmm_packed", "spmm_group", "row_count",
          "scatter_kernel", "big_hist", "big_colprefix", "big_offsets", "big_rows",
          "mttkrp_init", "tile_hist", "pair_scatter", "pair_count", "pair_emit", "tile_bounds",
          "tile_entries", "tile_chunks", "chunk_rows", "tile_rowscan", "chunk_write", "spmm_fix",
          "sample_fiber", "fiber_start", "ordered_w2")


def short(name):
    n = name.split("(")[0].replace("<unnamed>::", "").replace("void ", "")
    return n[:48]


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ii, ki, mi, vi = (h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"),
                      h.index("Metric Value"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        d = per.setdefault(int(r[ii]), {"name": short(r[ki])})
        d[r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.OrderedDict()
    for d in per.values():
        a = agg.setdefault(d["name"], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0) / 1e3
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print("| kernel | launches | total µs | share | DRAM MB (rd+wr) |")
    print("|---|---:|---:|---:|---:|")
    for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
        print("| `%s` | %d | %.1f | %.1f%% | %.1f |" % (n, c, t, 100 * t / tot, b / 1e6))
    print("\nTotal: %.1f µs over %d launches (serialised, cold-cache per launch)." % (tot, len(per)))
    mt = [(n, a) for n, a in agg.items() if any(n.startswith(m) or m in n for m in MTTKRP)]
    mt_t = sum(a[1] for _, a in mt)
    mt_b = sum(a[2] for _, a in mt)
    # (one launch per walk at R <= 64; above, an inner-levels launch and a leaf-level launch)
    walks = sum(v[0] for k, v in agg.items() if k.startswith("walk_runs_kernel") and not k.endswith(", 2>"))
    solves = max(agg.get("lookup_kernel", [0])[0], 1)
    print("\nSampled-MTTKRP pipeline kernels (%s): %.1f µs, %.1f MB DRAM over %d solves -> "
          "%.1f MB DRAM traffic per rcp_sampled_mttkrp call." %
          (", ".join(sorted(set(n.split("<")[0] for n, _ in mt))), mt_t, mt_b / 1e6, solves,
           mt_b / solves / 1e6))
    print("STS walks: %d launches." % walks)


if __name__ == "__main__":
    main(sys.argv[1])
