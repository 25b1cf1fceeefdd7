"""Seeded synthetic sparse tensors for the BASELINE.json configurations.

The reference benchmarks on FROSTT tensors (Uber, Amazon, Reddit; PAPER.md
Table 3) that are not available here; BASELINE.json names seeded synthetic
stand-ins with those shapes.  All generators are deterministic functions of
(config, seed):

* ``planted_c1`` -- C1, the CPU-runnable oracle case: 200k distinct uniform
  coordinates in 2000x1500x1000 carrying a planted rank-8 CP model with
  U(0,1) factors plus N(0, (0.01 std)^2) noise.  Pure numpy (small).
* ``zipf_tensor`` -- C2..C5: per-mode finite-support Zipf(s) indices,
  P(i) ~ (i+1)^-s, drawn by inverse CDF from a host-built fp64 table;
  duplicates are summed (ref tensor.py:72-83 semantics) and the first
  ``target`` distinct coordinates in draw order are kept.  Runs with torch
  on whatever device is given (CUDA on the GPU box), with the uniform
  stream derived from a splitmix64 counter hash so CPU and CUDA agree.

Afterwards ``permute`` applies the reference's load-balancing permutation
semantics (ref tensor.py:182-210): one seeded random bijection per mode.
"""

from __future__ import annotations

import math

import numpy as np

CONFIGS = {
    "c1": dict(dims=(2000, 1500, 1000), nnz=200_000, R=8, J=4096, rounds=10,
               samplers=("arls-lev", "sts"), kind="planted"),
    "c2": dict(dims=(183, 24, 1140, 1717), nnz=3_300_000, R=25, J=65536, rounds=20,
               samplers=("sts",), kind="zipf", s=1.1, values="lognormal", sigma=1.0),
    "c3": dict(dims=(12092, 9184, 28818), nnz=77_000_000, R=50, J=65536, rounds=1,
               samplers=("arls-lev", "sts"), kind="zipf", s=1.05, values="lognormal", sigma=1.0),
    # C4/C5: built on the device (zipf_chunks) from a fixed number of draws (the expected
    # count reaching the target distinct cells); the actual
    # post-dedup nonzero count is reported.
    "c4": dict(dims=(4_800_000, 1_800_000, 1_800_000), nnz=1_700_000_000, R=50, J=65536,
               rounds=1, samplers=("arls-lev", "sts"), kind="zipf_device", s=1.2,
               values="lognormal", sigma=1.5, draws=5_830_000_000, parts=16),
    "c5": dict(dims=(8_200_000, 177_000, 8_100_000), nnz=4_700_000_000, R=100, J=131072,
               rounds=1, samplers=("sts",), kind="zipf_device", s=1.1, values="log1p_poisson",
               draws=9_120_000_000, parts=32),
    # C5's shape, rank and sample count at one eighth of its draws: the share of the tensor
    # one of eight GPUs holds, sized for a single B200 (C5 itself needs 169 GB of stores);
    # exercises the R = 100, J = 131072, 8M-row paths at scale
    "c5s": dict(dims=(8_200_000, 177_000, 8_100_000), nnz=780_000_000, R=100, J=131072,
                rounds=1, samplers=("sts",), kind="zipf_device", s=1.1, values="log1p_poisson",
                draws=1_140_000_000, parts=8),
}


def planted_c1(seed=0, dims=(2000, 1500, 1000), nnz=200_000, R=8, noise=0.01):
    """C1: distinct uniform coordinates + planted rank-R model + Gaussian noise."""
    gen = np.random.default_rng(seed)
    cells = int(np.prod(dims))
    keep = np.empty(0, dtype=np.int64)
    while keep.size < nnz:
        draw = gen.integers(0, cells, size=2 * nnz, dtype=np.int64)
        pool = np.concatenate([keep, draw])
        _, first = np.unique(pool, return_index=True)
        keep = pool[np.sort(first)]
    keep = keep[:nnz]
    idx = np.stack(np.unravel_index(keep, dims), axis=1).astype(np.int64)
    fac = [gen.random((d, R)) for d in dims]
    v = np.ones((nnz, R))
    for m, F in enumerate(fac):
        v *= F[idx[:, m]]
    vals = v.sum(axis=1)
    vals = vals + gen.normal(0.0, noise * vals.std(), size=nnz)
    return idx, vals


def small_random(dims, nnz, seed):
    """Tiny random tensor with distinct coordinates and N(0,1) values (tests)."""
    gen = np.random.default_rng(seed)
    idx = np.stack([gen.integers(0, d, nnz * 3) for d in dims], axis=1)
    idx = np.unique(idx, axis=0)
    idx = idx[gen.permutation(idx.shape[0])[:nnz]]
    return idx.astype(np.int64), gen.standard_normal(idx.shape[0])


# ---------------------------------------------------------------------------
# Zipf generators (torch; identical streams on CPU and CUDA)
# ---------------------------------------------------------------------------
_M64 = (1 << 64) - 1


def _u64_to_i64(x):
    x &= _M64
    return x - (1 << 64) if x >= (1 << 63) else x


def _splitmix_uniform(torch, base, n, salt, device):
    """n doubles in [0,1) from splitmix64(base + salt*2^40 + i), computed with int64 ops."""
    i = torch.arange(n, dtype=torch.int64, device=device)
    z = i + _u64_to_i64(base * 0x9E3779B97F4A7C15 + salt * (1 << 40))
    z = z * _u64_to_i64(0x9E3779B97F4A7C15)

    def lsr(t, s):  # logical right shift on int64
        return (t >> s) & ((1 << (64 - s)) - 1)

    z = (z ^ lsr(z, 30)) * _u64_to_i64(0xBF58476D1CE4E5B9)
    z = (z ^ lsr(z, 27)) * _u64_to_i64(0x94D049BB133111EB)
    z = z ^ lsr(z, 31)
    return lsr(z, 11).to(torch.float64) * (1.0 / 9007199254740992.0)


def zipf_cdf(n, s):
    """Host fp64 CDF of finite Zipf(s) over [0, n): P(i) ~ (i+1)^-s."""
    w = np.arange(1, n + 1, dtype=np.float64) ** (-float(s))
    c = np.cumsum(w)
    return c / c[-1]


def zipf_tensor(dims, target, s, seed=0, values="lognormal", sigma=1.0, device="cpu",
                batch=None):
    """Draw Zipf coordinates until >= target distinct; keep the first target distinct
    (draw order); sum per-occurrence values over duplicates.  Returns torch tensors
    (idx int64 [nnz, N], vals float64 [nnz]) on `device`."""
    import torch
    dims = tuple(int(d) for d in dims)
    N = len(dims)
    strides = [1] * N
    for m in range(N - 2, -1, -1):
        strides[m] = strides[m + 1] * dims[m + 1]
    if strides[0] * dims[0] >= (1 << 63):
        raise ValueError("linear cell ids exceed int64; use a uint64 path")
    cdfs = [torch.as_tensor(zipf_cdf(d, s), device=device) for d in dims]
    batch = int(batch or max(target, 1 << 20))
    keys_all, vals_all, first_all = [], [], []
    drawn = 0
    uniq = None
    rnd = 0
    while True:
        lin = torch.zeros(batch, dtype=torch.int64, device=device)
        for m in range(N):
            u = _splitmix_uniform(torch, seed * 1000 + rnd, batch, m + 1, device)
            ix = torch.searchsorted(cdfs[m], u, right=True).clamp_(max=dims[m] - 1)
            lin += ix * strides[m]
        u1 = _splitmix_uniform(torch, seed * 1000 + rnd, batch, 101, device)
        if values == "lognormal":
            u2 = _splitmix_uniform(torch, seed * 1000 + rnd, batch, 102, device)
            z = torch.sqrt(-2.0 * torch.log1p(-u1)) * torch.cos(2.0 * math.pi * u2)
            v = torch.exp(sigma * z)
        elif values == "log1p_poisson":
            v = _poisson3(torch, u1)
        else:
            raise ValueError(values)
        keys_all.append(lin)
        vals_all.append(v)
        first_all.append(torch.arange(drawn, drawn + batch, dtype=torch.int64, device=device))
        drawn += batch
        rnd += 1
        keys = torch.cat(keys_all)
        uniq = torch.unique(keys)
        if uniq.numel() >= target:
            break
    keys = torch.cat(keys_all)
    vals = torch.cat(vals_all)
    pos = torch.cat(first_all)
    del keys_all, vals_all, first_all
    uk, inv = torch.unique(keys, return_inverse=True)
    first = torch.full((uk.numel(),), drawn, dtype=torch.int64, device=device)
    first.scatter_reduce_(0, inv, pos, reduce="amin")
    total = torch.zeros(uk.numel(), dtype=torch.float64, device=device)
    total.index_add_(0, inv, vals)
    order = torch.argsort(first)[:target]
    order, _ = torch.sort(order)            # canonical: ascending linear cell id
    lin = uk[order]
    v = total[order]
    if values == "log1p_poisson":
        v = torch.log1p(v)
    idx = torch.empty((lin.numel(), N), dtype=torch.int64, device=device)
    rem = lin
    for m in range(N):
        idx[:, m] = rem // strides[m]
        rem = rem % strides[m]
    return idx, v


def zipf_expected_row_weights(dims, s, perms=None):
    """Expected share of draws per (permuted) row of every mode: the finite Zipf(s) pmf
    moved through the mode permutation (row perm[i] carries the weight of i).  Used to cut
    nnz-balanced row blocks before a rank ingests only its own blocks (the exact counts
    need the whole tensor)."""
    out = []
    for j, d in enumerate(dims):
        w = np.arange(1, int(d) + 1, dtype=np.float64) ** (-float(s))
        if perms is not None:
            pw = np.empty_like(w)
            pw[np.asarray(perms[j], dtype=np.int64)] = w
            w = pw
        out.append(w / w.sum())
    return out


def zipf_chunks(dims, draws, s, seed=0, values="lognormal", sigma=1.0, parts=16,
                chunk_bits=28, device=None, perms=None, log=None, keep=None):
    """Device ingest for C4/C5 (ingest.cu): `draws` Zipf draws of the splitmix stream of
    `zipf_tensor` (chunks of 2^chunk_bits draws), duplicates summed in draw order, all
    distinct cells kept.  One pass over the draw sequence per hash partition of the cell
    space keeps the working set at ~draws/parts cells; a cell's draws are summed in
    ascending value order (reproducible).  Coordinates are mapped through
    `perms` (the reference's per-mode load-balancing permutations, ref tensor.py:207-210).
    Returns a list of (idx int32 [n, N], vals fp64 [n]) CUDA tensors, one per partition.
    keep: optional per-mode (lo, hi) row ranges -- each partition then keeps only the cells
    with at least one mode index inside its range (a rank's accumulator-stationary blocks,
    ref matricization.py:187-198), so a rank never holds the whole tensor."""
    import torch
    from .ops import ops_for
    dev = torch.device(device) if device is not None else torch.device("cuda", 0)
    ops = ops_for(dev)
    dims = tuple(int(d) for d in dims)
    N = len(dims)
    part_bits = int(round(math.log2(parts)))
    if (1 << part_bits) != parts:
        raise ValueError("parts must be a power of two")
    cdfs = [torch.as_tensor(zipf_cdf(d, s), device=dev) for d in dims]
    guides = [torch.empty(d, dtype=torch.int32, device=dev) for d in dims]
    for c, g in zip(cdfs, guides):
        ops.zipf_guide(c, g)
    pdev = None
    if perms is not None:
        pdev = [torch.as_tensor(np.asarray(p, dtype=np.int32), device=dev) for p in perms]
    vkind = {"lognormal": 0, "log1p_poisson": 1}[values]
    step = 1 << 30
    chunks = []
    for p in range(parts):
        cap = int(draws / parts * 1.25) + (1 << 20)
        while True:
            keys = torch.empty(cap, dtype=torch.int64, device=dev)
            vals = torch.empty(cap, dtype=torch.float64, device=dev)
            cnt = torch.zeros(1, dtype=torch.int64, device=dev)
            for d0 in range(0, int(draws), step):
                ops.zipf_draws(dims, cdfs, guides, seed, chunk_bits, d0, min(int(draws), d0 + step),
                               vkind, sigma, part_bits if parts > 1 else 0, p, keys, vals, cnt)
            n = int(cnt.item())
            if n <= cap:
                ops.status.check("in zipf_draws")
                break
            ops.status.reset()
            del keys, vals
            cap = n + (1 << 20)
        # the draws' buffer order depends on the atomic append order; ordering each cell's
        # draws by value (non-negative doubles sort as their bit patterns) makes the sums
        # reproducible
        sv, order = torch.sort(vals[:n])
        keys = keys[:n][order]
        del vals, order
        sk, order = torch.sort(keys, stable=True)
        del keys
        sv = sv[order]
        del order
        flag = torch.empty(n, dtype=torch.int32, device=dev)
        ops.run_flags(sk, flag)
        starts = torch.nonzero(flag).squeeze(1)
        del flag
        nc = int(starts.numel())
        idx = torch.empty((nc, N), dtype=torch.int32, device=dev)
        v = torch.empty(nc, dtype=torch.float64, device=dev)
        ops.cells(sk, sv, starts, dims, pdev, values == "log1p_poisson", idx, v)
        del sk, sv, starts
        if keep is not None:
            sel = torch.zeros(nc, dtype=torch.bool, device=dev)
            for j, (lo, hi) in enumerate(keep):
                col = idx[:, j]
                sel |= (col >= int(lo)) & (col < int(hi))
            idx, v = idx[sel].contiguous(), v[sel].contiguous()
            del sel
        chunks.append((idx, v))
        if log:
            log("partition %d/%d: %d draws -> %d cells%s" % (
                p + 1, parts, n, nc, "" if keep is None else " (%d kept)" % idx.shape[0]))
    return chunks


def _poisson3(torch, u):
    """Poisson(3) counts by inverse CDF on a uniform."""
    lam = 3.0
    p = math.exp(-lam)
    cdf = [p]
    for k in range(1, 40):
        p = p * lam / k
        cdf.append(cdf[-1] + p)
    table = torch.as_tensor(np.array(cdf), device=u.device)
    return torch.searchsorted(table, u, right=True).to(torch.float64)


def permute(idx, dims, seed, perm_of):
    """Apply one bijection per mode: idx'[:, j] = perm_j[idx[:, j]] (ref tensor.py:182-210).
    ``perm_of(j, d)`` returns the mode-j permutation (numpy int64 array)."""
    out = idx.copy() if isinstance(idx, np.ndarray) else idx.clone()
    perms = []
    for j, d in enumerate(dims):
        p = perm_of(j, d)
        perms.append(p)
        if isinstance(idx, np.ndarray):
            out[:, j] = p[idx[:, j]]
        else:
            import torch
            pt = torch.as_tensor(p, device=idx.device)
            out[:, j] = pt[idx[:, j]]
    return out, perms
