"""Structure of the sampled MTTKRP operands in a real round (design input, GPU box):
distinct fibers, fiber lengths, rows hit, entries per row, and how many (row tile, fiber)
pairs a row-tiled traversal would visit.  Writes gpurun_out/mttkrp_stats.json."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2210_05105_b200 import _lib  # noqa: E402
from paper_2210_05105_b200.engine import make_local_cluster  # noqa: E402

cfg = os.environ.get("CFG", "c3")
sampler = os.environ.get("SAMPLER", "sts")
dev = torch.device("cuda", 0)
_lib.load()
c, idx, vals = bench.make_tensor(cfg, 0, dev)
cl = make_local_cluster(c["dims"], idx, vals, c["R"], c["J"], sampler, 0)
me = cl.ranks[0]
res = []
orig = me.mttkrp


def hook(k):
    st = me.stores[k]
    key = torch.zeros(me.J, dtype=torch.int64, device=dev)
    for m in range(me.N):
        if m != k:
            key += me.X[m] * int(st.strides[m])
    u, cnt = torch.unique(key, return_counts=True)
    c_ = torch.searchsorted(st.keys, u)
    c_ = c_.clamp(max=st.n_cols - 1)
    hit = st.keys[c_] == u
    lo = torch.where(hit, st.colptr[c_], torch.zeros_like(c_))
    ln = torch.where(hit, st.colptr[c_ + 1] - st.colptr[c_], torch.zeros_like(c_))
    nnz_d = int(ln.sum())
    fid = torch.repeat_interleave(torch.arange(u.numel(), device=dev), ln)
    off = torch.cumsum(ln, 0) - ln
    pos = torch.repeat_interleave(lo - off, ln) + torch.arange(nnz_d, device=dev)
    rows = st.rows[pos].long()
    rh = torch.bincount(rows, minlength=st.n_rows)
    d = {"mode": k, "n_rows": st.n_rows, "n_cols": st.n_cols, "store_nnz": st.nnz,
         "S_d": int(u.numel()), "S_ne": int(hit.sum()), "nnz_d": nnz_d,
         "nnz_m": int((ln * cnt).sum()), "rows_hit": int((rh > 0).sum()),
         "fiber_len_pct": [int(x) for x in torch.quantile(ln[hit].double(), torch.tensor(
             [0.5, 0.9, 0.99, 1.0], dtype=torch.float64, device=dev)).long()],
         "row_cnt_pct": [int(x) for x in torch.quantile(rh.double(), torch.tensor(
             [0.5, 0.9, 0.99, 1.0], dtype=torch.float64, device=dev)).long()],
         "top_rows_share": [float(torch.topk(rh, t).values.sum()) / max(nnz_d, 1)
                            for t in (1, 16, 256)],
         "top_fibers_share": [float(torch.topk(ln, min(t, ln.numel())).values.sum()) / max(nnz_d, 1)
                              for t in (1, 16, 256, 4096)],
         "mult_pct": [int(x) for x in torch.quantile(cnt.double(), torch.tensor(
             [0.5, 0.9, 0.99, 1.0], dtype=torch.float64, device=dev)).long()]}
    pairs = {}
    for T in (64, 256, 512, 1024, 4096):
        nt = (st.n_rows + T - 1) // T
        pairs[str(T)] = int(torch.unique(fid * nt + rows // T).numel())
    d["tile_fiber_pairs"] = pairs
    for T in (8, 16, 32):
        nt = (st.n_rows + T - 1) // T
        pairs[str(T)] = int(torch.unique(fid * nt + rows // T).numel())
    # rows relabelled by descending entry count: how dense are row tiles of the head?
    order = torch.argsort(rh, descending=True)
    rank = torch.empty_like(order)
    rank[order] = torch.arange(order.numel(), device=dev)
    rr = rank[rows]
    ranked = {}
    for T in (8, 16):
        nt = (st.n_rows + T - 1) // T
        tile = rr // T
        pk = torch.unique(fid * nt + tile)
        ptile = torch.bincount(pk % nt, minlength=nt)      # fibers touching each ranked tile
        etile = torch.bincount(tile, minlength=nt)         # entries in each ranked tile
        cum_e = torch.cumsum(etile, 0).double() / max(nnz_d, 1)
        cum_p = torch.cumsum(ptile, 0).double()
        pts = []
        for frac in (0.25, 0.5, 0.75, 0.9, 1.0):
            t_ = int(torch.searchsorted(cum_e, torch.tensor([frac - 1e-12], dtype=torch.float64, device=dev)))
            t_ = min(t_, nt - 1)
            # dense-block density of the first t_+1 ranked tiles: entries / (T * fibers)
            pts.append({"entry_frac": frac, "tiles": t_ + 1, "pairs": int(cum_p[t_]),
                        "density": float(cum_e[t_] * nnz_d / (T * cum_p[t_]))})
        ranked[str(T)] = pts
    d["ranked_tiles"] = ranked
    # a dense head block: the nh most-hit rows x every sampled fiber
    srt = torch.sort(rh, descending=True).values.double()
    cs = torch.cumsum(srt, 0)
    d["dense_head"] = [{"rows": nh, "entry_frac": float(cs[min(nh, cs.numel()) - 1]) / max(nnz_d, 1),
                        "density": float(cs[min(nh, cs.numel()) - 1]) / (nh * max(int(hit.sum()), 1))}
                       for nh in (128, 256, 512, 1024, 2048, 4096)]
    # 2-D dense block: the nh most-hit rows (ranked by the STORE's row counts, a static
    # choice) x the nf longest sampled fibers
    srh = torch.bincount(st.rows.long(), minlength=st.n_rows)
    sorder = torch.argsort(srh, descending=True)
    srank = torch.empty_like(sorder)
    srank[sorder] = torch.arange(sorder.numel(), device=dev)
    er = srank[rows]
    forder = torch.argsort(ln, descending=True)
    frank = torch.empty_like(forder)
    frank[forder] = torch.arange(forder.numel(), device=dev)
    ef = frank[fid]
    blk = []
    for nh in (256, 512, 1024, 2048, 4096, 8192):
        for nf in (1024, 2048, 4096, 8192, 1 << 30):
            inb = int(((er < nh) & (ef < nf)).sum())
            nfe = min(nf, int(hit.sum()))
            blk.append({"rows": nh, "fibers": nfe, "entry_frac": inb / max(nnz_d, 1),
                        "density": inb / (min(nh, st.n_rows) * max(nfe, 1))})
    d["dense_block_static_rows"] = blk
    res.append(d)
    return orig(k)


for rnd in range(1, 4):
    cl.round(rnd)
me.mttkrp = hook
cl.round(4)
torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/mttkrp_stats_%s_%s.json" % (cfg, sampler), "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res, indent=1))
