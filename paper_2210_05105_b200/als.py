"""ALS driver -- drop-in for ref als.py (AlsConfig, DecompResult, run_als, run_trials),
running the device-resident engine (engine.py).

Only sketched solves on the accumulator-stationary schedule are in scope (the hot path);
`sampler="exact"` or `schedule="tensor-stationary"` raise ScheduleError.  With
`procs = P > 1` in a single process the P ranks are simulated on the current GPU (same
partition and random streams as the reference's simulated grid); real multi-GPU runs go
through `dist.run_distributed` (one process per GPU, NCCL).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .coo import ModePermutations, permute_modes
from .device import require_cuda, to_dev, to_host, torch
from .engine import PHASES, make_local_cluster
from .grid import ProcessorGrid, optimal_grid
from .linalg import init_factors
from .schedules import ScheduleError

SAMPLERS = ("exact", "arls-lev", "sts")
SCHEDULES = ("tensor-stationary", "accumulator-stationary")


@dataclass
class AlsConfig:
    """(ref als.py:27-62) -- same fields and validation."""
    rank: int
    rounds: int
    tensor_path: str = None
    sampler: str = "exact"
    samples: int = 0
    schedule: str = "tensor-stationary"
    grid_dims: tuple = None
    procs: int = 1
    seed: int = 0
    trial: int = 0
    fit_every: int = 5
    log_transform: bool = False
    dedup: bool = True
    permute: bool = True
    workers: int = 1
    leaf_block_size: int = None
    record_samples: bool = False
    compute_fits: bool = True

    def validate(self):
        if self.rank < 1:
            raise ValueError("rank must be >= 1")
        if self.rounds < 1:
            raise ValueError("rounds must be >= 1")
        if self.sampler not in SAMPLERS:
            raise ValueError("sampler must be one of %s" % (SAMPLERS,))
        if self.schedule not in SCHEDULES:
            raise ValueError("schedule must be one of %s" % (SCHEDULES,))
        if self.sampler != "exact" and self.samples < 1:
            raise ValueError("samples must be >= 1 for sketched solves")
        if self.schedule == "accumulator-stationary" and self.sampler == "exact":
            raise ScheduleError("accumulator-stationary schedule requires a sampler")
        if self.fit_every < 1:
            raise ValueError("fit_every must be >= 1")


@dataclass
class DecompResult:
    factors: list
    sigma: np.ndarray
    fit_history: list
    running_max: list
    final_fit: float
    ledger: object
    timings: dict
    config: AlsConfig
    grid_dims: tuple
    stored_nnz: int
    sample_log: list = field(default_factory=list)
    stats: dict = field(default_factory=dict)

    def summary(self) -> str:
        c = self.config
        lines = ["config rank=%d rounds=%d sampler=%s samples=%d schedule=%s grid=%s seed=%d "
                 "trial=%d" % (c.rank, c.rounds, c.sampler, c.samples, c.schedule,
                               "x".join(str(d) for d in self.grid_dims), c.seed, c.trial),
                 "stored_nnz %d" % self.stored_nnz]
        for (r, f), m in zip(self.fit_history, self.running_max):
            lines.append("fit round=%d fit=%.6f running_max=%.6f" % (r, f, m))
        lines.append("final_fit %.6f" % self.final_fit)
        for phase, secs in sorted(self.timings.items()):
            lines.append("time %s %.3f" % (phase, secs))
        for key, val in sorted(self.stats.items()):
            lines.append("stat %s %d" % (key, val))
        return "\n".join(lines)


def build_grid(dims, cfg: AlsConfig) -> ProcessorGrid:
    if cfg.grid_dims is not None:
        return ProcessorGrid(dims, cfg.grid_dims)
    return optimal_grid(dims, cfg.procs)


def _check_supported(cfg):
    if cfg.schedule != "accumulator-stationary":
        raise ScheduleError("only the accumulator-stationary schedule is part of this build")


def run_als(cfg: AlsConfig, tensor=None, perms=None, grid=None, partition=None,
            fit_mat=None, timed_phases=False) -> DecompResult:
    """One ALS trial (ref als.py:141-218) on the device engine."""
    cfg.validate()
    _check_supported(cfg)
    if tensor is None:   # (ref als.py:148-154)
        if cfg.tensor_path is None:
            raise ValueError("no tensor given and no tensor_path configured")
        from .tensorio import load_frostt
        tensor = load_frostt(cfg.tensor_path, log_transform=cfg.log_transform, dedup=cfg.dedup)
        if cfg.permute:
            tensor, perms = permute_modes(tensor, cfg.seed)
    timings = {"load": 0.0, "fit": 0.0}
    t0 = time.perf_counter()
    dev = require_cuda()
    t = torch()
    if perms is None:
        perms = ModePermutations.identity(tensor.dims)
    if grid is None:
        grid = build_grid(tensor.dims, cfg)
    idx = to_dev(tensor.idx, dev, t.int64)
    vals = to_dev(tensor.vals, dev, t.float64)
    factors0, sigma0 = init_factors(tensor.dims, cfg.rank, cfg.seed, cfg.trial)
    cl = make_local_cluster(tensor.dims, idx, vals, cfg.rank, cfg.samples, cfg.sampler, cfg.seed,
                            grid_dims=grid.grid_dims, leaf=cfg.leaf_block_size, factors=factors0)
    del idx, vals
    t.cuda.synchronize()
    timings["load"] = time.perf_counter() - t0
    cl.timed = timed_phases
    N = tensor.mode_count
    fit_history, running_max, sample_log = [], [], []
    best = -np.inf
    sigma = sigma0
    for rnd in range(1, cfg.rounds + 1):
        for k in range(N):
            cl.solve(k, rnd, check=True)
            cl.check("after round %d mode %d solve" % (rnd, k))
            if cfg.record_samples:
                sample_log.append(to_host(cl.ranks[0].X.T.contiguous()))
        sigma = to_host(cl.ranks[0].sigma).copy()
        if cfg.compute_fits and (rnd % cfg.fit_every == 0 or rnd == cfg.rounds):
            tf = time.perf_counter()
            f = cl.fit()
            best = max(best, f)
            fit_history.append((rnd, f))
            running_max.append(best)
            timings["fit"] += time.perf_counter() - tf
    final_fit = fit_history[-1][1] if fit_history else float("nan")
    full = gather_factors(cl)
    factors_out = [perms.unpermute_factor(full[j], j) for j in range(N)]
    timings.update({p: cl.timings[p] for p in PHASES})
    st = np.zeros(8, dtype=np.int64)
    for r in cl.ranks:
        st += to_host(r.stats)
    stats = dict(distinct_samples=int(st[0]), nonempty_samples=int(st[1]),
                 sampled_nnz_distinct=int(st[2]), sampled_nnz=int(st[3]))
    stored = sum(s.nnz for r in cl.ranks for s in r.stores)
    return DecompResult(factors_out, sigma, fit_history, running_max, final_fit, None, timings,
                        cfg, grid.grid_dims, stored, sample_log, stats)


def gather_factors(cl):
    """Assemble full factor matrices (host) from the rank blocks."""
    r0 = cl.ranks[0]
    out = []
    for j in range(r0.N):
        U = np.zeros((r0.dims[j], r0.R))
        for r in cl.ranks:
            U[r.lo[j]:r.lo[j] + r.n[j]] = to_host(r.U[j])
        out.append(U)
    return out


class AlsSession:
    """Host-buffer round API over a device cluster (single process): the factor matrices
    live on the host between calls, as in a host-driven reference loop."""

    def __init__(self, cluster):
        self.cl = cluster
        self.sigma = None
        self.copy = None   # copy stream for the host transfers

    def pinned_factors(self):
        t = torch()
        out = []
        for U in self.cl.ranks[0].U:
            h = t.empty(U.shape, dtype=t.float64, pin_memory=True)
            h.copy_(U)
            out.append(h)
        return out

    def step_host(self, factors_in, factors_out, rnd, graph=False):
        """Upload factors (pinned host) -> rebuild sampler state -> one ALS round ->
        download the updated factors and sigma.  Transfers run on a copy stream: mode j's
        upload overlaps the rebuild of the modes before it, and factor k's download
        overlaps the solves after k.  graph=True replays the round (with its downloads)
        from a CUDA graph when the cluster allows it (Cluster.graph_ok); one graph is
        captured per `factors_out` buffer set (the downloads are part of the graph), so a
        caller may ping-pong between two sets."""
        t = torch()
        r0 = self.cl.ranks[0]
        if len(self.cl.ranks) != 1:
            raise ValueError("step_host drives one rank per process (P=1 or SPMD)")
        main = t.cuda.current_stream()
        if self.copy is None:
            self.copy = t.cuda.Stream(device=main.device)
        self.copy.wait_stream(main)   # previous users of the factor buffers are done
        ups = []
        with t.cuda.stream(self.copy):
            for j, h in enumerate(factors_in):
                r0.U[j].copy_(h, non_blocking=True)
                ev = t.cuda.Event()
                ev.record()
                ups.append(ev)
        for j in range(r0.N):
            main.wait_event(ups[j])
            self.cl.rebuild(j)

        def download(k):
            ev = t.cuda.Event()
            ev.record()
            self.copy.wait_event(ev)
            with t.cuda.stream(self.copy):
                factors_out[k].copy_(r0.U[k], non_blocking=True)

        if graph and self.cl.graph_ok():
            self.cl.round_graph(rnd, on_solved=download, join=(self.copy,),
                               tag="step_host:%x" % factors_out[0].data_ptr())
        else:
            self.cl.round(rnd, check=False, on_solved=download)
        self.sigma = r0.sigma.to("cpu", non_blocking=True)
        main.wait_stream(self.copy)
        main.synchronize()
        self.cl.check("in AlsSession.step_host")
        return factors_out


def run_trials(cfg: AlsConfig, trials: int, tensor=None):
    """Mean-of-trials harness with shared tensor (ref als.py:221-237): the tensor is
    loaded (and permuted) once."""
    cfg.validate()
    perms = None
    if tensor is None and cfg.tensor_path is not None:
        from .tensorio import load_frostt
        tensor = load_frostt(cfg.tensor_path, log_transform=cfg.log_transform, dedup=cfg.dedup)
        if cfg.permute:
            tensor, perms = permute_modes(tensor, cfg.seed)
    results = []
    for tr in range(trials):
        trial_cfg = AlsConfig(**{**cfg.__dict__, "trial": tr})
        results.append(run_als(trial_cfg, tensor=tensor, perms=perms))
    return results
