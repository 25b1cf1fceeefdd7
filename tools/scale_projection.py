"""Projected accumulator-stationary scaling from ONE GPU (design input for SURVEY.md 8(e)).

Only one B200 is available to this build, so the N-GPU step time cannot be measured.
This tool measures what one GPU can: it runs the real engine with P virtual ranks
(`LocalComm`, the same kernels and the same per-rank shards an N-GPU run uses), times
every rank's device work between two collectives with CUDA events (the ranks run one
after another on the GPU, each with the whole device, as on its own GPU), and adds up the
bulk-synchronous critical path:

    T_P = sum over segments (max over ranks of the rank's device time in the segment)
          + modelled collective time (NOT measured: bytes / bus bandwidth + latency)

A segment is the work between two consecutive collectives of a solve (STS: one exchange
per constant mode, the column-norm all-gather, the block-Gram all-gather).  Work the
engine runs on side streams at P = 1 (sketched Gram + pseudo-inverse under the MTTKRP,
tree builds under the chain pseudo-inverse) is serialised here so that its time is clean,
reported separately, and counted as hidden when it is shorter than the work it overlaps.

Output: gpurun_out/scale_projection_<cfg>_<sampler>.json with, per P: per-phase max and
mean over ranks, load imbalance (max/mean of the sampled-MTTKRP time and of the distinct
gathered nonzeros), the projected round time and the projected parallel efficiency
T_1 / (P T_P).  The numbers are a projection, not a bench value.

    CFG=c3 SAMPLER=sts PLIST=1,2,4,8 python tools/scale_projection.py
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2210_05105_b200 import _lib  # noqa: E402
from paper_2210_05105_b200.engine import make_local_cluster  # noqa: E402

# modelled interconnect (NVLink 5 / NVSwitch, NCCL): stated, not measured
BUS_GBS = float(os.environ.get("BUS_GBS", "350"))     # all-reduce / all-gather bus bandwidth
LAT_US = float(os.environ.get("LAT_US", "15"))        # per-collective launch + sync latency

RANK_METHODS = ("prefetch_trees", "prefetch_gm", "chain", "sts_mode", "fold_urow", "arls_draw", "arls_fold",
                "weights", "sketched_system", "mttkrp", "update", "renormalize", "block_gram",
                "set_gram", "build_tree", "arls_local")
SIDE = ("sketched_system", "prefetch_trees", "prefetch_gm")   # overlapped work at P = 1 (side streams)


class Recorder:
    def __init__(self):
        self.log = []   # ("call", rank, name, ev0, ev1) | ("coll", name, bytes, ev0, ev1)

    def wrap_rank(self, r):
        for name in RANK_METHODS:
            fn = getattr(r, name, None)
            if fn is None:
                continue

            def make(fn=fn, name=name, rank=r.rank):
                def timed(*a, **k):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    out = fn(*a, **k)
                    e1.record()
                    self.log.append(("call", rank, name, e0, e1))
                    return out
                return timed
            setattr(r, name, make())

    def wrap_exchange(self, cl):
        """The per-rank packing/unpacking around the STS exchange (eager torch ops)."""
        fn = cl._exchange_walk

        def timed(*a):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(*a)
            e1.record()
            self.log.append(("xchg", e0, e1))
        cl._exchange_walk = timed

    def wrap_comm(self, comm):
        for name in ("all_gather", "all_gather_v", "all_reduce_sum"):
            fn = getattr(comm, name)

            def make(fn=fn, name=name):
                def timed(local, *a):
                    nbytes = sum(int(x.numel()) * x.element_size() for x in local
                                 if hasattr(x, "numel")) // max(len(local), 1)
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    out = fn(local, *a)
                    e1.record()
                    self.log.append(("coll", name, nbytes, e0, e1))
                    return out
                return timed
            setattr(comm, name, make())


def coll_model_us(name, nbytes, P):
    """Ring/NVLS-style cost model: per-rank payload `nbytes`."""
    if P == 1:
        return 0.0
    if name == "all_reduce_sum":
        vol = 2.0 * (P - 1) / P * nbytes
    else:   # all-gather(-v): every rank receives (P - 1) payloads
        vol = (P - 1) * nbytes
    return LAT_US + vol / (BUS_GBS * 1e3)


def analyse(log, P, rounds):
    """Critical path over the segments between collectives."""
    torch.cuda.synchronize()
    seg = [dict() for _ in range(1)]   # rank -> {name: ms}
    segs = [seg[0]]
    colls = []
    pack_ms = tracked = 0.0
    for rec in log:
        if rec[0] == "xchg":   # appended after its collective: the rest is P ranks' packing
            pack_ms += max(rec[1].elapsed_time(rec[2]) - colls[-1][2], 0.0) / P
            continue
        if rec[0] == "coll":
            _, name, nbytes, e0, e1 = rec
            colls.append((name, nbytes, e0.elapsed_time(e1)))
            segs.append(dict())
        else:
            _, rank, name, e0, e1 = rec
            d = segs[-1].setdefault(rank, {})
            d[name] = d.get(name, 0.0) + e0.elapsed_time(e1)
            tracked += e0.elapsed_time(e1)
    tracked += sum(c[2] for c in colls)
    crit = serial = pack_ms
    hidden = 0.0
    phase_max, phase_sum = {}, {}
    for s in segs:
        if not s:
            continue
        per_rank_main, per_rank_all = [], []
        for rank in range(P):
            d = s.get(rank, {})
            side = sum(v for k, v in d.items() if k in SIDE)
            main = sum(v for k, v in d.items() if k not in SIDE)
            # side-stream work hides under the main-stream work of its segment
            per_rank_main.append(max(main, side))
            per_rank_all.append(main + side)
        crit += max(per_rank_main)
        serial += max(per_rank_all)
        hidden += max(per_rank_all) - max(per_rank_main)
        names = set(k for d in s.values() for k in d)
        for nme in names:
            vals = [s.get(r, {}).get(nme, 0.0) for r in range(P)]
            phase_max[nme] = phase_max.get(nme, 0.0) + max(vals)
            phase_sum[nme] = phase_sum.get(nme, 0.0) + sum(vals) / P
    comm_us = sum(coll_model_us(n, b, P) for n, b, _ in colls)
    comm_bytes = sum(b for _, b, _ in colls)
    return {
        "compute_ms_per_round": crit / rounds,
        "compute_no_overlap_ms_per_round": serial / rounds,
        "hidden_side_stream_ms_per_round": hidden / rounds,
        "modelled_comm_ms_per_round": comm_us / 1e3 / rounds,
        "exchange_pack_unpack_ms_per_round_per_rank": pack_ms / rounds,
        "tracked_device_ms_per_round_all_ranks": tracked / rounds,
        "collectives_per_round": len(colls) / rounds,
        "comm_payload_bytes_per_rank_per_round": comm_bytes / rounds,
        "projected_ms_per_round": (crit + comm_us / 1e3) / rounds,
        "phase_ms_per_round_max_over_ranks": {k: round(v / rounds, 4) for k, v in sorted(phase_max.items())},
        "phase_ms_per_round_mean_over_ranks": {k: round(v / rounds, 4) for k, v in sorted(phase_sum.items())},
    }


def main():
    cfg = os.environ.get("CFG", "c3")
    sampler = os.environ.get("SAMPLER", "sts")
    plist = [int(x) for x in os.environ.get("PLIST", "1,2,4,8").split(",")]
    rounds = int(os.environ.get("ROUNDS", "3"))
    rank_override = os.environ.get("RANK_R")
    # LEAF: STS leaf rows for every rank (P virtual ranks share one GPU's memory: C4's
    # default trees, sized for a GPU per rank, do not fit eight times)
    leaf = int(os.environ["LEAF"]) if os.environ.get("LEAF") else None
    dev = torch.device("cuda", 0)
    _lib.load()
    c, idx, vals = bench.make_tensor(cfg, 0, dev)
    R = int(rank_override) if rank_override else c["R"]
    out = {"config": cfg, "sampler": sampler, "rank": R, "samples_J": c["J"],
           "dims": list(c["dims"]), "row_blocks": "nnz-balanced (P > 1)", "sts_leaf_rows": leaf,
           "model": {"bus_GBps": BUS_GBS, "latency_us_per_collective": LAT_US,
                     "note": "collective time is modelled, not measured (one GPU available)"},
           "method": "P virtual ranks (LocalComm) on one B200, eager launches; per-rank device "
                     "time between collectives from CUDA events; T_P = sum over segments of "
                     "the max over ranks + modelled collectives",
           "points": []}
    t1 = None
    for P in plist:
        t0 = time.perf_counter()
        cl = make_local_cluster(c["dims"], idx, vals, R, c["J"], sampler, 0, P=P,
                                balance="nnz" if P > 1 else "rows", leaf=leaf)
        if P == plist[-1]:
            idx = vals = None   # the COO is not needed once the last cluster holds its stores
            torch.cuda.empty_cache()
        torch.cuda.synchronize()
        setup = time.perf_counter() - t0
        for rnd in range(1, 4):
            cl.round(rnd)
        torch.cuda.synchronize()
        # the same P ranks' rounds replayed from a CUDA graph (no host launch gaps): the
        # ratio to the eager wall time says how much of the event-bracketed times below is
        # launch latency that a replayed N-GPU round does not pay
        graph_ms = None
        rnd0 = 4
        if os.environ.get("GRAPH", "1") == "1" and cl.graph_ok():
            cl.round_graph(rnd0)
            torch.cuda.synchronize()
            g0 = torch.cuda.Event(enable_timing=True)
            g1 = torch.cuda.Event(enable_timing=True)
            g0.record()
            for rnd in range(rnd0 + 1, rnd0 + 1 + rounds):
                cl.round_graph(rnd)
            g1.record()
            torch.cuda.synchronize()
            cl.check("graph rounds")
            graph_ms = g0.elapsed_time(g1) / rounds
            rnd0 += 1 + rounds
            for r in cl.ranks:   # back to host-side keys for the eager rounds below
                r.dkeys = None
                r.gperm = None
        # serialise the side streams: clean per-call timings, overlap credited in analyse()
        cl._side = torch.cuda.current_stream()
        for r in cl.ranks:
            r._tree_stream = torch.cuda.current_stream()
        cl.round(rnd0)
        rnd0 += 1
        torch.cuda.synchronize()
        rec = Recorder()
        for r in cl.ranks:
            rec.wrap_rank(r)
        rec.wrap_comm(cl.comm)
        if P > 1 and sampler == "sts":
            rec.wrap_exchange(cl)
        stats0 = [r.stats.clone() for r in cl.ranks]
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for rnd in range(rnd0, rnd0 + rounds):
            cl.round(rnd, check=False)
        e1.record()
        torch.cuda.synchronize()
        cl.check("projection rounds")
        a = analyse(rec.log, P, rounds)
        st = [(r.stats - s0).cpu().tolist() for r, s0 in zip(cl.ranks, stats0)]
        nnz_d = [s[2] / rounds for s in st]
        nnz_m = [s[3] / rounds for s in st]
        mt = []
        for rank in range(P):
            mt.append(sum(x[3].elapsed_time(x[4]) for x in rec.log
                          if x[0] == "call" and x[1] == rank and x[2] == "mttkrp") / rounds)
        a.update({
            "P": P, "setup_s": round(setup, 1),
            "one_gpu_wall_ms_per_round_all_ranks_serial": e0.elapsed_time(e1) / rounds,
            "one_gpu_graph_replay_ms_per_round_all_ranks": graph_ms,
            "distinct_nnz_per_round_per_rank": nnz_d,
            "sampled_nnz_per_round_total": sum(nnz_m),
            "mttkrp_ms_per_round_per_rank": [round(x, 4) for x in mt],
            "imbalance_mttkrp_time_max_over_mean": max(mt) / (sum(mt) / P) if sum(mt) else None,
            "imbalance_distinct_nnz_max_over_mean": max(nnz_d) / (sum(nnz_d) / P) if sum(nnz_d) else None,
            "store_nnz_per_rank": [[int(s.nnz) for s in r.stores] for r in cl.ranks],
            "peak_mem_GB": round(torch.cuda.max_memory_allocated() / 1e9, 1),
        })
        if P == 1:
            t1 = a["projected_ms_per_round"]
        if t1:
            a["projected_speedup_vs_P1"] = t1 / a["projected_ms_per_round"]
            a["projected_parallel_efficiency"] = t1 / (P * a["projected_ms_per_round"])
            a["projected_sampled_nnz_per_s"] = sum(nnz_m) / (a["projected_ms_per_round"] / 1e3)
        out["points"].append(a)
        print("P=%d eager wall %.2f graph wall %s | projected %.3f ms/round (compute %.3f + comm %.3f), mttkrp imbalance %.2f, eff %s"
              % (P, a["one_gpu_wall_ms_per_round_all_ranks_serial"],
                 "%.2f" % graph_ms if graph_ms else "n/a",
                 a["projected_ms_per_round"], a["compute_ms_per_round"],
                 a["modelled_comm_ms_per_round"], a["imbalance_mttkrp_time_max_over_mean"] or 0,
                 "%.2f" % a["projected_parallel_efficiency"] if t1 else "n/a"), flush=True)
        del cl, rec
        import gc
        from paper_2210_05105_b200 import ops as _ops
        _ops._OPS.clear()   # per-device workspaces (the MTTKRP's is sized by the largest shard)
        gc.collect()
        torch.cuda.empty_cache()
    os.makedirs("gpurun_out", exist_ok=True)
    tag = "%s_%s%s" % (cfg, sampler, "_r%d" % R if rank_override else "")
    with open("gpurun_out/scale_projection_%s.json" % tag, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
