"""Benchmark: sampled-MTTKRP nonzeros/s and ALS rounds/s of the leverage-sampled ALS hot
path on B200 (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--sampler sts]
    python bench.py --impl reference ...     # reference CPU implementation (oracle port)

A step is one ALS round (N mode solves: sample -> weights -> sketched Gram -> sampled
MTTKRP -> update -> renormalise -> rebuild) over the synthetic tensor of the named
config, all inputs resident in HBM.  `value` = sampled nonzeros iterated by the MTTKRP
(with sample multiplicity -- the reference's csr.nnz and the paper's "nonzeros iterated",
PAPER.md:1527-1529) per second of round time, summed over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "sampled-MTTKRP nnz/s"
L2_GATHER_GBS = 15765.0   # measured: 2^26 random 400-B rows of a 7 MB table, profiles/r01_l2_gather.json
UNIT = "nnz/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--sampler", default="sts", choices=["sts", "arls-lev"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-samples", type=int, default=0)
    ap.add_argument("--leaf", type=int, default=None, help="STS tree leaf rows (default: engine)")
    ap.add_argument("--balance", default="auto", choices=["auto", "rows", "nnz"],
                    help="row blocks: reference equal-row cuts, or nnz-balanced cuts "
                         "(auto: nnz when more than one GPU)")
    ap.add_argument("--rank", type=int, default=None, help="CP rank (default: the config's)")
    ap.add_argument("--eager", action="store_true",
                    help="launch every kernel from the host (default: replay STS rounds from a "
                         "CUDA graph when the cluster allows it)")
    ap.add_argument("--samples", type=int, default=None, help="J (default: the config's)")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._th = None

    def start(self):
        def run():
            q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "--query-gpu=" + q, "--format=csv,noheader,nounits",
                                          "-i", str(self.index)], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._th = threading.Thread(target=run, daemon=True)
        self._th.start()

    def stop(self):
        self._stop.set()
        if self._th:
            self._th.join(timeout=6)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ workload
def make_tensor(cfg_name, seed, dev, rank_grid=None):
    """Synthetic tensor of the named config on `dev` (torch tensors), reference
    load-balancing permutation applied (ref tensor.py:207-210).  rank_grid=(grid, rank):
    device-generated configs keep only that rank's accumulator-stationary blocks."""
    import torch
    from paper_2210_05105_b200 import rng, synth
    c = synth.CONFIGS[cfg_name]
    perm_of = lambda j, d: rng.permutation(rng.stream_key(seed, rng.TENSOR_PERM, j), d)  # noqa: E731
    if c["kind"] == "zipf_device":   # C4/C5: generated, deduplicated and permuted on the GPU
        perms = [perm_of(j, d) for j, d in enumerate(c["dims"])]
        keep = None
        if rank_grid is not None:
            g, p = rank_grid
            keep = [g.block_range(j, p) for j in range(len(c["dims"]))]
        chunks = synth.zipf_chunks(c["dims"], c["draws"], c["s"], seed=seed, values=c["values"],
                                   sigma=c.get("sigma", 1.0), parts=c["parts"], device=dev,
                                   perms=perms, log=lambda m: print(m, file=sys.stderr, flush=True),
                                   keep=keep)
        return c, chunks, None
    if c["kind"] == "planted":
        idx, vals = synth.planted_c1(seed=seed)
        return c, torch.as_tensor(idx, device=dev), torch.as_tensor(vals, device=dev)
    idx, vals = synth.zipf_tensor(c["dims"], c["nnz"], c["s"], seed=seed, values=c["values"],
                                  sigma=c.get("sigma", 1.0), device=dev)
    idx, _ = synth.permute(idx, c["dims"], seed, perm_of)
    return c, idx, vals


def traffic_bytes(args):
    """DRAM bytes (read + write) per rcp_sampled_mttkrp call measured by ncu for this
    workload (profiles/traffic.json, committed with the profile it came from), else None."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                               "traffic.json")) as f:
            return json.load(f)["entries"].get("%s/%s" % (args.config, args.sampler))
    except (OSError, ValueError, KeyError):
        return None


def peaks():
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def flush_l2(buf):
    buf.add_(1.0)


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    from paper_2210_05105_b200 import _lib
    from paper_2210_05105_b200.engine import (Cluster, LocalComm, RankState, make_local_cluster)
    from paper_2210_05105_b200.grid import optimal_grid
    from paper_2210_05105_b200.linalg import init_factors

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # RCP_SPMD=1 runs the torch.distributed (NCCL) code path even at world size 1 (a check
    # of the multi-GPU plumbing on a single GPU)
    spmd = world > 1 or os.environ.get("RCP_SPMD") == "1"
    # RCP_BENCH_BACKEND=gloo with RCP_BENCH_ONE_GPU=1: a functional check of the multi-rank
    # flow on a one-GPU box (every rank on cuda:0, collectives staged through the host; no
    # kernel waits on another process).  Its timings are not bench values.
    backend = os.environ.get("RCP_BENCH_BACKEND", "nccl")
    if os.environ.get("RCP_BENCH_ONE_GPU") == "1":
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    _lib.load()
    if spmd:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    t_setup = time.perf_counter()
    balance = args.balance if args.balance != "auto" else ("nnz" if world > 1 else "rows")
    rank_grid = None
    from paper_2210_05105_b200 import synth as _synth
    cdef = _synth.CONFIGS[args.config]
    if spmd and cdef["kind"] == "zipf_device":
        # per-rank ingest: the grid first (nnz cuts from the expected Zipf row weights), then
        # every rank generates the tensor and keeps only its own blocks
        from paper_2210_05105_b200 import rng as _rng
        from paper_2210_05105_b200.grid import ProcessorGrid, optimal_grid
        rw = None
        if balance == "nnz":
            perms = [_rng.permutation(_rng.stream_key(args.seed, _rng.TENSOR_PERM, j), d)
                     for j, d in enumerate(cdef["dims"])]
            rw = _synth.zipf_expected_row_weights(cdef["dims"], cdef["s"], perms)
        rank_grid = (optimal_grid(cdef["dims"], world, row_weights=rw), rank)
    c, idx, vals = make_tensor(args.config, args.seed, dev, rank_grid=rank_grid)
    dims = c["dims"]
    R = args.rank or c["R"]
    J = args.samples or c["J"]
    N = len(dims)
    nnz = sum(int(ch[0].shape[0]) for ch in idx) if isinstance(idx, list) else int(idx.shape[0])
    t_gen = time.perf_counter() - t_setup
    if spmd:
        from paper_2210_05105_b200.dist import make_spmd_cluster
        cl = make_spmd_cluster(dims, idx, vals, R, J, args.sampler, args.seed, leaf=args.leaf,
                               balance=balance, grid=rank_grid[0] if rank_grid else None)
    else:
        cl = make_local_cluster(dims, idx, vals, R, J, args.sampler, args.seed, leaf=args.leaf,
                                balance=balance)
    del idx, vals
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    print("setup %.1f s (generate %.1f s), nnz %d, peak %.1f GB, resident %.1f GB" % (
        setup_s, t_gen, nnz, torch.cuda.max_memory_allocated() / 1e9,
        torch.cuda.memory_allocated() / 1e9), file=sys.stderr, flush=True)
    me = cl.ranks[0]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev).view(torch.float64)  # 256 MB > L2

    # per-step events: whole round, and the sampled-MTTKRP calls inside it
    mt_events = []
    orig = me.mttkrp

    def timed_mttkrp(k):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        out = orig(k)
        e.record()
        mt_events.append((s, e))
        return out
    use_graph = (not args.eager) and cl.graph_ok()
    # events cannot time calls inside a replayed graph: with graphs, the MTTKRP call
    # durations come from eager rounds of the same kernels after the timed region
    me.mttkrp = orig if use_graph else timed_mttkrp
    rnd = 0
    for w in range(args.warmup):
        rnd += 1
        if use_graph and w > 0:   # the first warm-up round sizes every workspace eagerly
            cl.round_graph(rnd)
            torch.cuda.synchronize()
            cl.check("in warm-up round %d" % rnd)
        else:
            cl.round(rnd)
    torch.cuda.synchronize()
    mt_events.clear()
    # factor state entering the first timed round: the e2e leg replays the same rounds
    from paper_2210_05105_b200.als import AlsSession
    snap = AlsSession(cl).pinned_factors()
    first_timed = rnd + 1
    stats0 = me.stats.clone()
    if spmd:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local_rank)
    clocks.start()
    lib = _lib.lib()
    launches0 = lib.rcp_launch_count()
    step_ms = []
    for _ in range(args.steps):
        flush_l2(flush)
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        rnd += 1
        s.record()
        if use_graph:
            cl.round_graph(rnd)
        else:
            cl.round(rnd, check=False)
        e.record()
        e.synchronize()
        step_ms.append(s.elapsed_time(e))
    torch.cuda.synchronize()
    clk = clocks.stop()
    print("step ms: " + " ".join("%.2f" % x for x in step_ms), file=sys.stderr, flush=True)
    launches = lib.rcp_launch_count() - launches0
    if use_graph:   # replayed kernels do not pass through the host-side launch counter
        launches += cl.graph_kernels * args.steps
    cl.check("in timed rounds")
    st = (me.stats - stats0).cpu().numpy().astype(np.int64)
    if use_graph:
        me.mttkrp = timed_mttkrp
        mt_events.clear()
        s1 = me.stats.clone()
        for _ in range(args.steps):
            flush_l2(flush)
            rnd += 1
            cl.round(rnd, check=False)
        torch.cuda.synchronize()
        st_mt = (me.stats - s1).cpu().numpy().astype(np.int64)
    else:
        st_mt = st
    mt_ms = sum(a.elapsed_time(b) for a, b in mt_events)
    n_launch = len(mt_events)
    # one extra (untimed) round with device phase markers for the breakdown
    cl.phase_events = []
    me.mttkrp = orig
    rnd += 1
    cl.round(rnd, check=False)
    torch.cuda.synchronize()
    phases = {k: round(v, 4) for k, v in cl.phase_breakdown().items()}
    cl.phase_events = None
    t_total = sum(step_ms) / 1e3
    if spmd:
        import torch.distributed as dist
        tt = torch.tensor([t_total, float(st[3]), float(st[2])], dtype=torch.float64, device=dev)
        gathered = [torch.zeros_like(tt) for _ in range(world)]
        dist.all_gather(gathered, tt)
        t_total = max(float(g[0]) for g in gathered)
        nnz_m = sum(float(g[1]) for g in gathered)
        nnz_d = sum(float(g[2]) for g in gathered)
    else:
        nnz_m, nnz_d = float(st[3]), float(st[2])
    K = args.steps
    value = nnz_m / t_total
    hbm, peak_kind = peaks()
    # algorithmic bytes of the sampled MTTKRP:
    #   12 nnz_d + 16 S_d + 8R S_ne + 8R rows_hit  per solve, summed over the timed solves
    B = 12.0 * st_mt[2] + 16.0 * st_mt[0] + 8.0 * R * st_mt[1] + 8.0 * R * st_mt[4]
    achieved = (B / (mt_ms / 1e3)) / 1e9 if mt_ms > 0 else 0.0
    e2e = measure_e2e(cl, args, first_timed, snap, float(st[3]))
    if spmd:
        import torch.distributed as dist
        tt = torch.tensor([e2e.pop("_dt"), e2e.pop("_nnz")], dtype=torch.float64, device=dev)
        gathered = [torch.zeros_like(tt) for _ in range(world)]
        dist.all_gather(gathered, tt)
        dt_max = max(float(g[0]) for g in gathered)
        e2e["value"] = sum(float(g[1]) for g in gathered) / dt_max
        e2e["ms_per_step"] = dt_max / e2e["steps"] * 1e3
    else:
        e2e.pop("_dt")
        e2e.pop("_nnz")
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": sum(step_ms) / K, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "%s %s R=%d J=%d dims=%s nnz=%d" % (args.config, args.sampler, R, J,
                                                                 "x".join(map(str, dims)), nnz),
                   "sampler": args.sampler, "rank": R, "samples_J": J, "modes": N,
                   "parallelism": "as%d" % world, "row_blocks": balance, "l2": "256 MB flush between timed rounds "
                   "(outside the round events); stores %.1f GB > L2" % (
                       sum(s.bytes() for s in me.stores) / 1e9),
                   "setup_s": round(setup_s, 1), "generate_s": round(t_gen, 1),
                   "launch": "cuda-graph replay of the round" if use_graph else "eager",
                   **({"functional_check": "backend %s, every rank on cuda:0: not a bench value" % backend}
                      if backend != "nccl" else {})},
        "rounds_per_s": K / t_total,
        "distinct_nnz_per_s": nnz_d / t_total,
        "sampled_nnz_per_round": nnz_m / K,
        "distinct_nnz_per_round": nnz_d / K,
        "roofline": {"kernel": "rcp_sampled_mttkrp (dedup+lookup+transpose+segmented SpMM)",
                     "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic_bytes(args), "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": B / max(n_launch, 1),
                     "avg_launch_ms": mt_ms / max(n_launch, 1), "launches": n_launch,
                     "share_of_step": mt_ms / max(sum(step_ms), 1e-9),
                     # the bound the segmented SpMM actually meets: every distinct gathered
                     # entry pulls its scaled KRP row (8R bytes) from L2; peak = random 400-B
                     # row gathers measured on B200 (tools/lab/run_lab.py LABMODE=gather)
                     "l2_gather": {"bytes_per_launch": 8.0 * R * st_mt[2] / max(n_launch, 1),
                                   "achieved": (8.0 * R * st_mt[2] / (mt_ms / 1e3)) / 1e9
                                   if mt_ms > 0 else 0.0,
                                   "peak": L2_GATHER_GBS, "unit": "GB/s",
                                   "frac": ((8.0 * R * st_mt[2] / (mt_ms / 1e3)) / 1e9) / L2_GATHER_GBS
                                   if mt_ms > 0 else 0.0},
                     "launch_timing": "eager rounds after the timed region" if use_graph
                     else "inside the timed rounds"},
        "clocks": clk,
        "gpu_launches": int(launches),
        "phases_ms_per_round": phases,
    }
    if e2e is not None:
        out["e2e"] = e2e
    if c["kind"] == "zipf_device":
        out["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                               "sample": "not run: the reference keeps ~64 B per nonzero per mode "
                                         "on the host (>300 GB at this size, SURVEY.md 8(d))"}
    elif rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline(args, cl, c)
        except Exception as ex:  # reported, never fatal
            out["cpu_baseline"] = {"value": None, "error": repr(ex)[:200]}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if spmd:
        import torch.distributed as dist
        dist.destroy_process_group()


def measure_e2e(cl, args, first, snap, timed_nnz):
    """Same metric through the public host-buffer API, over the SAME rounds as the timed
    region: step 0 uploads the factor state that entered the first timed round (pinned
    host snapshot), each later step uploads the factors the previous step downloaded
    (ping-pong between two pinned sets), so every step rebuilds the sampler state from
    host memory, runs the round with the timed region's round id and reads the updated
    factors and sigma back (AlsSession.step_host).  The rounds are deterministic, so the
    sampled-nonzero count equals the timed region's (`same_rounds` says whether it did)."""
    import torch
    from paper_2210_05105_b200.als import AlsSession
    sess = AlsSession(cl)
    bufs = [sess.pinned_factors(), sess.pinned_factors()]
    steps = args.steps
    me = cl.ranks[0]
    graph = not args.eager
    sess.step_host(snap, bufs[0], first)   # eager: sizes every workspace
    for b in bufs:                         # one graph per output set
        sess.step_host(snap, b, first, graph=graph)
    torch.cuda.synchronize()
    st0 = me.stats.clone()
    t0 = time.perf_counter()
    for s in range(steps):
        src = snap if s == 0 else bufs[(s - 1) % 2]
        sess.step_host(src, bufs[s % 2], first + s, graph=graph)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = (me.stats - st0).cpu().numpy()
    return {"value": float(st[3]) / dt, "unit": UNIT,
            "h2d_bytes_per_step": int(sum(h.numel() * 8 for h in snap)),
            "d2h_bytes_per_step": int(sum(h.numel() * 8 for h in bufs[0]) + 8 * me.R),
            "steps": steps, "ms_per_step": dt / steps * 1e3, "_dt": dt, "_nnz": float(st[3]),
            "same_rounds": bool(float(st[3]) == timed_nnz),
            "api": "AlsSession.step_host (pinned host factors in, factors + sigma out; the "
                   "timed region's rounds replayed from its entry state)" +
                   (", round replayed from a CUDA graph" if graph and cl.graph_ok() else "")}


# ------------------------------------------------------------------ CPU arms
def cpu_baseline(args, cl, c, samples=None):
    """Oracle port (numpy, oracle/) timed on this host on a bounded sample of the same
    workload: one mode-k solve's gather + downsampled MTTKRP (the dominant CPU phase)
    for the first `samples` draws of a real device batch of the last solved mode."""
    import torch
    from oracle import randcp_oracle as O
    me = cl.ranks[0]
    k = me.N - 1
    samples = samples or args.cpu_samples or min(2048, cl.J)
    st = me.stores[k]
    # host copy of the mode-k store in the oracle's own layout (built untimed)
    t0 = time.perf_counter()
    ostore = oracle_store_from_device(st)
    build_s = time.perf_counter() - t0
    X = me.X.T.contiguous().cpu().numpy()[:samples]
    H = me.H.cpu().numpy()[:samples]
    w = me.w.cpu().numpy()[:samples]
    workers = os.cpu_count() or 1
    t0 = time.perf_counter()
    csr = O.sampled_csr(ostore, X, k)
    out = O.sketched_mttkrp(csr, H, w, workers=workers)
    dt = time.perf_counter() - t0
    # parity on the benchmarked batch (untimed): the fused GPU MTTKRP of the same samples
    dev = me.X.device
    Xd = me.X[:, :samples].contiguous()
    gout = torch.empty((st.n_rows, me.R), dtype=torch.float64, device=dev)
    gst = torch.zeros(8, dtype=torch.int64, device=dev)
    me.ops.sampled_mttkrp(st, Xd, k, me.H[:samples].contiguous(), me.w[:samples].contiguous(),
                          gout, gst)
    got = gout.cpu().numpy()
    parity = {"samples": int(samples), "mode": int(k),
              "max_rel_err": float(np.abs(got - out).max() / max(np.abs(out).max(), 1e-300)),
              "gathered_nnz_gpu": int(gst[3]), "gathered_nnz_oracle": int(csr.nnz),
              "bar": "max_rel_err <= 1e-9, equal gathered nonzeros"}
    parity["ok"] = bool(parity["max_rel_err"] <= 1e-9 and
                        parity["gathered_nnz_gpu"] == parity["gathered_nnz_oracle"])
    del out, gout
    return {"value": csr.nnz / dt, "unit": UNIT, "cores": workers, "kind": "port",
            "parity": parity, "host": host_info(),
            "sample": "oracle gather_sampled_nonzeros_to_csr + downsampled_mttkrp, mode %d of %s, "
                      "first %d of J=%d samples of a device STS/ARLS batch; %d nnz iterated in %.2f s "
                      "(store conversion %.1f s untimed)" % (k, args.config, samples, cl.J, csr.nnz,
                                                             dt, build_s)}


class _HostStore:
    """Oracle-shaped view (skeys/col_order/idx-rows/vals) of a device store."""


def oracle_store_from_device(st):
    keys = st.keys.cpu().numpy()
    colptr = st.colptr.cpu().numpy()
    rows = st.rows.cpu().numpy().astype(np.int64) + st.row_lo
    vals = st.vals.cpu().numpy()
    s = _HostStore()
    s.j = st.mode
    s.dims = st.dims
    s.lo = st.row_lo
    s.hi = st.row_hi
    s.skeys = np.repeat(keys, np.diff(colptr))
    s.col_order = np.arange(vals.size, dtype=np.int64)
    s.idx = np.zeros((vals.size, len(st.dims)), dtype=np.int64)
    s.idx[:, st.mode] = rows
    s.vals = vals
    s.n_rows = st.row_hi - st.row_lo
    s.find = lambda q: (np.searchsorted(s.skeys, q, side="left"),
                        np.searchsorted(s.skeys, q, side="right"))
    return s


def host_info():
    """CPU model, cores, RAM, numpy and BLAS versions of this host."""
    info = {"cpu_count": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        with open("/proc/meminfo") as f:
            kb = int(f.readline().split()[1])
        info["ram_gb"] = round(kb / 2 ** 20, 1)
    except (OSError, ValueError, IndexError):
        pass
    info["numpy"] = np.__version__
    try:
        from threadpoolctl import threadpool_info
        info["blas"] = ["%s %s (%s threads)" % (p.get("internal_api"), p.get("version"),
                                                p.get("num_threads"))
                        for p in threadpool_info() if p.get("user_api") == "blas"]
    except Exception:   # pragma: no cover - informational only
        pass
    info["threads_env"] = {k: os.environ[k] for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS")
                           if k in os.environ}
    return info


def reference_tensor(args, c):
    """The workload's tensor for the reference arm, without this repo's CUDA library:
    the same seeded Zipf draws (torch, on the GPU when present, else the host) and the
    reference's own permutation streams (numpy Philox, ref rng.py:26-32, tensor.py:207-210)
    through the oracle."""
    import torch
    from oracle import randcp_oracle as O
    from paper_2210_05105_b200 import synth
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    if c["kind"] == "planted":
        idx, vals = synth.planted_c1(seed=args.seed)
        return np.asarray(idx), np.asarray(vals)
    idx, vals = synth.zipf_tensor(c["dims"], c["nnz"], c["s"], seed=args.seed, values=c["values"],
                                  sigma=c.get("sigma", 1.0), device=dev)
    idx = idx.cpu().numpy()
    vals = vals.cpu().numpy()
    for j, d in enumerate(c["dims"]):
        perm = O.stream(args.seed, O.P_TENSOR_PERM, j).permutation(d)
        idx[:, j] = perm[idx[:, j]]
    return idx, vals


def run_reference(args):
    """`--impl reference`: the reference's own algorithm (the oracle port, numpy on all
    host cores; the reference is pure Python, so nothing compiles into oracle/_ref) on the
    same config and metric.  Each step is one ALS round over all N modes restricted to a
    bounded number of samples per solve: sampler + gather + downsampled MTTKRP + sketched
    solve timed (ref schedules.py:227-258), factor update + sampler-state rebuild untimed.
    It never loads this repo's CUDA library: state comes from the reference's init_factors
    on the host."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import randcp_oracle as O
    from paper_2210_05105_b200 import synth
    c = synth.CONFIGS[args.config]
    if c["kind"] == "zipf_device":
        print(json.dumps({"impl": "reference", "metric": METRIC, "unit": UNIT,
                          "unavailable": "the reference's host working set at %s (~64 B per nonzero "
                          "per mode, >300 GB) exceeds the host; SURVEY.md 8(d)" % args.config}),
              flush=True)
        return
    dims = c["dims"]
    R = args.rank or c["R"]
    J = args.samples or c["J"]
    N = len(dims)
    samples = args.cpu_samples or min(J, 1024)
    workers = os.cpu_count() or 1
    t0 = time.perf_counter()
    idx, vals = reference_tensor(args, c)
    gen_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    stores = [O.Store(dims, idx, vals, k) for k in range(N)]
    factors, _ = O.init_factors(dims, R, args.seed)
    factors = [np.array(U) for U in factors]

    def rebuild(j):
        blocks = [[factors[j]]]
        grams[j] = O.gram_blocks(blocks[0])
        if args.sampler == "sts":
            state[j] = O.tree_build(blocks[0], [0])
        else:
            state[j] = O.lev_build(blocks[0], [0])

    grams = [None] * N
    state = [None] * N
    for j in range(N):
        rebuild(j)
    setup = time.perf_counter() - t0
    total_nnz, total_t = 0, 0.0
    for step in range(args.warmup + args.steps):
        rnd = 1 + step
        for k in range(N):
            ts = time.perf_counter()
            if args.sampler == "sts":
                cp = O.sym_pinv(O.hadamard_chain(grams, skip=k))
                b = O.tree_sample(state, k, samples, cp, grams, [[U] for U in factors], args.seed, rnd)
            else:
                b = O.lev_sample(state, k, samples, factors, args.seed, rnd)
            w = O.weights_for(b.prob, samples)
            csr = O.sampled_csr(stores[k], b.X, k)
            out = O.sketched_mttkrp(csr, b.H, w, workers=workers)
            Hw = b.H * w[:, None]
            newU = out @ O.sym_pinv(Hw.T @ Hw)
            dt = time.perf_counter() - ts
            if step >= args.warmup:
                total_nnz += csr.nnz
                total_t += dt
            norms = np.sqrt((newU * newU).sum(axis=0))     # ref als.py:129-138 (untimed)
            norms[norms == 0] = 1.0
            factors[k] = newU / norms
            rebuild(k)
    value = total_nnz / total_t
    hi = host_info()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_t / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "%s %s R=%d J=%d dims=%s nnz=%d" % (
                           args.config, args.sampler, R, J, "x".join(map(str, dims)), len(vals)),
                       "sampler": args.sampler, "rank": R, "samples_J": J, "modes": N,
                       "parallelism": "host"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                             "sample": "each step = one round over all %d modes with %d of J=%d "
                                       "samples per solve (sampler + gather + downsampled MTTKRP + "
                                       "sketched solve timed; factor update and sampler rebuild "
                                       "untimed), from the reference's init_factors; tensor "
                                       "generation %.0f s and the reference's per-mode store build "
                                       "%.0f s untimed" % (N, samples, J, gen_s, setup),
                             "host": hi},
            "host": hi,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
