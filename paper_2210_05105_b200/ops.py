"""Typed wrappers over the C ABI taking torch CUDA tensors (stream = torch's current
stream).  One `Ops` object per device owns the status word and reusable workspaces."""

from __future__ import annotations

import numpy as np

from . import _lib
from .device import Status, empty, ptr, stream_handle, torch

CUTOFF = 1e-10   # ref linalg.py:16


def _key_args(key):
    """(key0, key1, d_key): a host key pair, or a device tensor of two words (int64 view of
    the uint64 key) read by the kernel itself (graph-replayed rounds)."""
    if hasattr(key, "data_ptr"):
        return 0, 0, key.data_ptr()
    return int(key[0]), int(key[1]), None


class Ops:
    def __init__(self, dev):
        self.dev = dev
        self.status = Status(dev)
        self._ws = {}
        self.lib = _lib.lib()

    # ------------------------------------------------------------------ workspace
    def ws(self, name, nbytes):
        t = torch()
        nbytes = max(int(nbytes), 256)
        buf = self._ws.get(name)
        if buf is None or buf.numel() < nbytes:
            buf = empty(nbytes, t.uint8, self.dev)
            self._ws[name] = buf
        return buf

    def _c(self, name, *args):
        rc = getattr(self.lib, name)(*args)
        if rc != _lib.OK:
            _lib.check(rc, name)

    # ------------------------------------------------------------------- dense
    def gram(self, U, scale=None, out=None):
        t = torch()
        n, R = U.shape
        if out is None:
            out = empty((R, R), t.float64, self.dev)
        w = self.ws("gram", self.lib.rcp_gram_ws_bytes(n, R))
        self._c("rcp_gram", ptr(U), ptr(scale), n, R, ptr(out), ptr(w), stream_handle())
        return out

    def pinv(self, G, n_chain=0, skip=-1, cutoff=CUTOFF, out=None, chain_out=None):
        t = torch()
        R = G.shape[-1]
        if out is None:
            out = empty((R, R), t.float64, self.dev)
        self._c("rcp_pinv", ptr(G), int(n_chain), int(skip), int(R), float(cutoff),
                ptr(chain_out), ptr(out), self.status.ptr, stream_handle())
        return out

    def update(self, M, B, out, colsq):
        n, R = M.shape
        w = self.ws("update", self.lib.rcp_update_ws_bytes(n, R))
        self._c("rcp_update", ptr(M), n, R, ptr(B), ptr(out), ptr(colsq), ptr(w),
                self.status.ptr, stream_handle())

    def renormalize(self, U, colsq, sigma):
        n, R = U.shape
        self._c("rcp_renormalize", ptr(U), n, R, ptr(colsq), ptr(sigma), stream_handle())

    def weights(self, pmp, prob, w):
        N, J = pmp.shape
        self._c("rcp_weights", ptr(pmp), N, J, ptr(prob), ptr(w), self.status.ptr,
                stream_handle())

    def ordered_sum(self, parts, out):
        """out = parts[0] + parts[1] + ... (left to right) for a stacked (P, ...) tensor."""
        P = parts.shape[0]
        self._c("rcp_ordered_sum", ptr(parts), P, parts[0].numel(), ptr(out), stream_handle())
        return out

    def hadamard_rows(self, H, urow, init):
        J, R = H.shape
        self._c("rcp_hadamard_rows", ptr(H), ptr(urow), J, R, 1 if init else 0, stream_handle())

    # -------------------------------------------------------------------- ARLS
    def arls_build(self, U, Gp, dist, cdf, mass):
        n, R = U.shape
        w = self.ws("arls", self.lib.rcp_arls_build_ws_bytes(n, R))
        self._c("rcp_arls_build", ptr(U), n, R, ptr(Gp), ptr(dist), ptr(cdf), ptr(mass), ptr(w),
                stream_handle())

    def arls_draw(self, cdf, dist, row_lo, ratio, total_mass, key, q, offset, rows_out,
                  prob_out, U=None, urow_out=None):
        n = cdf.shape[0]
        R = U.shape[1] if U is not None else 0
        k0, k1, dk = _key_args(key)
        self._c("rcp_arls_draw", ptr(cdf), ptr(dist), n, int(row_lo), float(ratio),
                ptr(total_mass), k0, k1, dk, int(q), int(offset), ptr(rows_out),
                ptr(prob_out), ptr(U), R, ptr(urow_out), self.status.ptr, stream_handle())

    def batch_fold(self, perm, rows, prob, U, u_row_lo, urows, first, Xi, pmp_i, H):
        J, R = H.shape
        self._c("rcp_batch_fold", ptr(perm), ptr(rows), ptr(prob), J, ptr(U), int(u_row_lo),
                ptr(urows), R, 1 if first else 0, ptr(Xi), ptr(pmp_i), ptr(H), stream_handle())

    # --------------------------------------------------------------------- STS
    def sts_depth(self, n, leaf):
        return int(self.lib.rcp_sts_depth(int(n), int(leaf)))

    def sts_build(self, U, leaf, tree=None):
        t = torch()
        n, R = U.shape
        nd = int(self.lib.rcp_sts_tree_doubles(n, int(leaf), R))
        if tree is None or tree.numel() < nd:
            tree = empty(max(nd, 1), t.float64, self.dev)
        self._c("rcp_sts_build", ptr(U), n, R, int(leaf), ptr(tree), stream_handle())
        return tree

    def sts_cond(self, chain_pinv, grams, i, k, out):
        N, R = grams.shape[0], grams.shape[1]
        self._c("rcp_sts_cond", ptr(chain_pinv), ptr(grams), N, int(i), int(k), R, ptr(out),
                stream_handle())

    def sts_walk_ws(self, J, n, leaf, R, ws=None, owned=False):
        """The walk workspace: the device-wide one, or with owned=True a caller-owned buffer
        (`ws`, allocated when None and grown when too small; several rank states share one
        device object, and a prefetched conditioning pass must not be overwritten by
        another rank's)."""
        need = int(self.lib.rcp_sts_walk_ws_bytes(int(J), int(n), int(leaf), int(R)))
        if not owned:
            return self.ws("sts_walk", need)
        if ws is None or ws.numel() < need:
            ws = empty(need, torch().uint8, self.dev)
        return ws

    def sts_walk_gm(self, tree, n, leaf, M, J, ws):
        """The walk's conditioning pass into `ws` (see rcp_sts_walk_gm)."""
        R = M.shape[0]
        self._c("rcp_sts_walk_gm", ptr(tree), int(n), R, int(leaf), ptr(M), int(J), ptr(ws),
                ws.numel(), stream_handle())

    def sts_walk(self, tree, U, leaf, row_lo, M, H_in, J, key, override, rin, sel, sel_value,
                 Xi, pmp_i, resid, hkey=None, key_bits=64, H_out=None, ws=None, gm_ready=False):
        n, R = U.shape
        w = ws if ws is not None else self.sts_walk_ws(J, n, leaf, R)
        k0, k1, dk = _key_args(key)
        self._c("rcp_sts_walk_prepared" if gm_ready else "rcp_sts_walk", ptr(tree), ptr(U), n, R,
                int(leaf), int(row_lo), ptr(M),
                ptr(H_in), ptr(hkey), int(key_bits), int(J), k0, k1, dk, ptr(override), ptr(rin),
                ptr(sel),
                int(sel_value), ptr(Xi), ptr(pmp_i), ptr(resid), ptr(H_out), ptr(w), w.numel(),
                self.status.ptr, stream_handle())

    def sts_flat_draw(self, cdf, dist, row_lo, mass, key, J, Xi, pmp_i):
        n = cdf.shape[0]
        k0, k1, dk = _key_args(key)
        self._c("rcp_sts_flat_draw", ptr(cdf), ptr(dist), n, int(row_lo), ptr(mass), k0, k1, dk,
                int(J), ptr(Xi), ptr(pmp_i), self.status.ptr, stream_handle())

    def fold_rows(self, out, U, row_lo, Xi, init, sel=None, sel_value=0):
        n, R = U.shape
        J = Xi.shape[0]
        self._c("rcp_fold_rows", ptr(out), ptr(U), n, R, int(row_lo), ptr(Xi), J,
                1 if init else 0, ptr(sel), int(sel_value), stream_handle())

    def row_keys(self, X, strides, out):
        N, J = X.shape
        st = np.ascontiguousarray(strides, dtype=np.int64)
        self._c("rcp_row_keys", ptr(X), N, J, st.ctypes.data, ptr(out), stream_handle())

    def walk_key(self, X, dims, k, i, out):
        """Mixed-radix key of the modes already sampled before constant mode i
        (modes < i, excluding k) and the number of low bits that hold it; (None, 64) for
        the first constant mode."""
        prev = [m for m in range(i) if m != k]
        if not prev:
            return None, 64
        strides = [0] * len(dims)
        span = 1
        for m in prev:
            strides[m] = span
            span *= int(dims[m])
        if span >= (1 << 63):
            raise ValueError("walk grouping key overflows int64")
        self.row_keys(X, strides, out)
        return out, max(1, int(span).bit_length())

    def sts_rank_walk(self, node_grams, depth, P, leaf_rank, M, H, J, key, override, owner,
                      r_out, pmp_i):
        R = M.shape[0]
        k0, k1, dk = _key_args(key)
        self._c("rcp_sts_rank_walk", ptr(node_grams), int(depth), int(P), ptr(leaf_rank),
                ptr(M), ptr(H), int(J), R, k0, k1, dk, ptr(override), ptr(owner),
                ptr(r_out), ptr(pmp_i), self.status.ptr, stream_handle())

    def sts_rank_tree(self, block_grams, order, tree=None):
        """Packed rank tree of P block Grams (P x R x R, summed pairwise up the levels)."""
        t = torch()
        P, R = block_grams.shape[0], block_grams.shape[1]
        nd = int(self.lib.rcp_sts_rank_tree_doubles(P, R))
        if tree is None or tree.numel() < nd:
            tree = t.zeros(nd, dtype=t.float64, device=self.dev)
        self._c("rcp_sts_rank_tree", ptr(block_grams), ptr(order), P, R, ptr(tree), stream_handle())
        return tree

    def sts_rank_walk_grouped(self, rank_tree, P, leaf_rank, M, H_in, J, key, override, owner,
                              r_out, pmp_i, hkey=None, key_bits=64):
        R = M.shape[0]
        k0, k1, dk = _key_args(key)
        if H_in is None and hkey is None and P <= 1024:   # one group: H = ones for every sample
            self._c("rcp_sts_rank_walk_ones", ptr(rank_tree), int(P), ptr(leaf_rank), R, ptr(M),
                    int(J), k0, k1, dk, ptr(override), ptr(owner), ptr(r_out), ptr(pmp_i),
                    self.status.ptr, stream_handle())
            return
        w = self.ws("sts_rank_walk", self.lib.rcp_sts_rank_walk_ws_bytes(int(J), int(P), R))
        self._c("rcp_sts_rank_walk_grouped", ptr(rank_tree), int(P), ptr(leaf_rank), R, ptr(M),
                ptr(H_in), ptr(hkey), int(key_bits), int(J), k0, k1, dk, ptr(override), ptr(owner),
                ptr(r_out), ptr(pmp_i), ptr(w), w.numel(), self.status.ptr, stream_handle())

    def sts_flat_local(self, cdf, dist, row_lo, mass, rin, sel, sel_value, J, Xi, pmp_i, resid):
        n = cdf.shape[0]
        self._c("rcp_sts_flat_local", ptr(cdf), ptr(dist), n, int(row_lo), ptr(mass), ptr(rin),
                ptr(sel), int(sel_value), int(J), ptr(Xi), ptr(pmp_i), ptr(resid), self.status.ptr,
                stream_handle())

    def exchange_pack(self, Xi, pmp_i, resid, U, row_lo, owner, rank, buf):
        n, R = U.shape
        J = Xi.shape[0]
        self._c("rcp_exchange_pack", ptr(Xi), ptr(pmp_i), ptr(resid), ptr(U), n, int(row_lo),
                ptr(owner), int(rank), J, R, ptr(buf), stream_handle())

    def exchange_unpack(self, buf, init, Xi, pmp_i, resid, H):
        J, R = H.shape
        self._c("rcp_exchange_unpack", ptr(buf), J, R, 1 if init else 0, ptr(Xi), ptr(pmp_i),
                ptr(resid), ptr(H), stream_handle())

    # ------------------------------------------------------------------ MTTKRP
    def mttkrp_ws(self, J, cap, n_rows, R):
        return self.ws("mttkrp", self.lib.rcp_mttkrp_ws_bytes(int(J), int(cap), int(n_rows), int(R)))

    def sampled_mttkrp(self, store, X, k, H, w, out, stats, cap=None, need=False):
        """need=True: synchronise and return (gathered entries this call required, entry
        capacity of the workspace it ran with); it overflowed iff the first exceeds the
        second (then it processed nothing and raised the capacity flag)."""
        N, J = X.shape
        R = H.shape[1]
        cap = store.nnz if cap is None else cap
        ws = self.mttkrp_ws(J, cap, store.n_rows, R)
        strides = np.ascontiguousarray(store.strides, dtype=np.int64)
        self._c("rcp_sampled_mttkrp", ptr(store.keys), ptr(store.colptr), store.n_cols,
                ptr(store.rows), ptr(store.vals), store.n_rows, ptr(X), N, J, int(k),
                strides.ctypes.data, ptr(H), ptr(w), R, ptr(out), ptr(stats), ptr(ws),
                ws.numel(), self.status.ptr, stream_handle())
        if need:   # (entries required, entry capacity of the workspace used)
            lay = np.zeros(14, dtype=np.int64)
            self._c("rcp_mttkrp_layout", int(J), store.n_rows, R, ws.numel(), lay.ctypes.data)
            o = int(lay[12])
            return int(ws[o + 8:o + 16].view(torch().int64).item()), int(lay[13])

    def fiber_lookup(self, store, X, k, lo, counts):
        N, J = X.shape
        strides = np.ascontiguousarray(store.strides, dtype=np.int64)
        self._c("rcp_fiber_lookup", ptr(store.keys), store.n_cols, ptr(store.colptr), ptr(X), N,
                J, int(k), strides.ctypes.data, ptr(lo), ptr(counts), stream_handle())

    def fiber_expand(self, lo, off, store, row_out, col_out, val_out):
        J = lo.shape[0]
        self._c("rcp_fiber_expand", ptr(lo), ptr(off), J, ptr(store.rows), ptr(store.vals),
                ptr(row_out), ptr(col_out), ptr(val_out), stream_handle())

    def csr_spmm(self, row_ptr, col, val, H, scale, out):
        n_rows = row_ptr.shape[0] - 1
        R = H.shape[1]
        self._c("rcp_csr_spmm", ptr(row_ptr), n_rows, ptr(col), ptr(val), ptr(H), ptr(scale), R,
                ptr(out), stream_handle())

    # ------------------------------------------------------------- exact fit (F1)
    @staticmethod
    def _factor_arrays(factors, los, N):
        import ctypes as C
        U = (C.c_void_p * N)(*[C.c_void_p(ptr(f)) if f is not None else None for f in factors])
        lo = np.ascontiguousarray([int(x) for x in los], dtype=np.int64)
        return U, lo

    def fit_cross(self, store, factors, los, Uk, sigma, out):
        """out[0] = sum over the store's entries of v <sigma (.) prod_m U_m[i_m], U_k[row]>."""
        N = len(store.dims)
        R = Uk.shape[1]
        U, lo = self._factor_arrays(factors, los, N)
        dims = np.ascontiguousarray(store.dims, dtype=np.int64)
        strides = np.ascontiguousarray([max(int(x), 1) for x in store.strides], dtype=np.int64)
        w = self.ws("fit", self.lib.rcp_fit_ws_bytes(store.nnz))
        self._c("rcp_fit_cross", ptr(store.keys), ptr(store.colptr), store.n_cols, ptr(store.rows),
                ptr(store.vals), store.nnz, N, int(store.mode), dims.ctypes.data,
                strides.ctypes.data, U, lo.ctypes.data, ptr(Uk), R, ptr(sigma), ptr(out), ptr(w),
                w.numel(), stream_handle())
        return out

    def sum_squares(self, v, out):
        n = v.numel()
        w = self.ws("fit", self.lib.rcp_fit_ws_bytes(n))
        self._c("rcp_sum_squares", ptr(v), n, ptr(out), ptr(w), w.numel(), stream_handle())
        return out

    def model_norm(self, grams, sigma, out):
        N, R = grams.shape[0], grams.shape[1]
        self._c("rcp_model_norm", ptr(grams), N, R, ptr(sigma), ptr(out), stream_handle())
        return out

    def exact_mttkrp(self, store, factors, los, out):
        N = len(store.dims)
        R = out.shape[1]
        U, lo = self._factor_arrays(factors, los, N)
        dims = np.ascontiguousarray(store.dims, dtype=np.int64)
        strides = np.ascontiguousarray([max(int(x), 1) for x in store.strides], dtype=np.int64)
        self._c("rcp_exact_mttkrp", ptr(store.keys), ptr(store.colptr), store.n_cols,
                ptr(store.rows), ptr(store.vals), store.nnz, store.n_rows, N, int(store.mode),
                dims.ctypes.data, strides.ctypes.data, U, lo.ctypes.data, R, ptr(out),
                stream_handle())
        return out

    # ------------------------------------------------------------- device ingest (F2)
    def zipf_guide(self, cdf, guide):
        self._c("rcp_zipf_guide", ptr(cdf), cdf.numel(), guide.numel(), ptr(guide),
                stream_handle())

    def zipf_draws(self, dims, cdfs, guides, seed, chunk_bits, d0, d1, value_kind, sigma,
                   part_bits, part, keys, vals, count):
        import ctypes as C
        N = len(dims)
        hd = np.ascontiguousarray(dims, dtype=np.int64)
        hc = (C.c_void_p * N)(*[C.c_void_p(ptr(c)) for c in cdfs])
        hg = (C.c_void_p * N)(*[C.c_void_p(ptr(g)) for g in guides])
        hG = np.ascontiguousarray([g.numel() for g in guides], dtype=np.int64)
        self._c("rcp_zipf_draws", N, hd.ctypes.data, hc, hg, hG.ctypes.data, int(seed),
                int(chunk_bits), int(d0), int(d1), int(value_kind), float(sigma), int(part_bits),
                int(part), ptr(keys), ptr(vals), ptr(count), keys.numel(), self.status.ptr,
                stream_handle())

    def order_by_key_row(self, key, row, key_max, row_max):
        """Positions in (key, row) order, stable (key None: by row alone).  The workspace is
        released after the call: store builds order up to 10^8 entries at a time."""
        t = torch()
        n = row.numel()
        order = empty(n, t.int64, self.dev)
        if n == 0:
            return order
        nb = self.lib.rcp_sort_ws_bytes(n)
        w = empty(nb, t.uint8, self.dev)
        self._c("rcp_order_by_key_row", ptr(key) if key is not None else None, ptr(row), n,
                int(key_max), int(row_max), ptr(order), ptr(w), nb, stream_handle())
        return order

    def run_flags(self, sorted_keys, flag):
        self._c("rcp_run_flags", ptr(sorted_keys), sorted_keys.numel(), ptr(flag),
                stream_handle())

    def cells(self, sorted_keys, svals, starts, dims, perms, log1p_vals, idx_out, val_out):
        import ctypes as C
        N = len(dims)
        hd = np.ascontiguousarray(dims, dtype=np.int64)
        hp = (C.c_void_p * N)(*[C.c_void_p(ptr(p)) if p is not None else None
                                for p in (perms or [None] * N)])
        self._c("rcp_cells", ptr(sorted_keys), ptr(svals), ptr(starts), starts.numel(),
                sorted_keys.numel(), N, hd.ctypes.data, hp, int(bool(log1p_vals)), ptr(idx_out),
                ptr(val_out), stream_handle())


_OPS = {}


def ops_for(dev) -> Ops:
    key = str(dev)
    o = _OPS.get(key)
    if o is None:
        o = Ops(dev)
        _OPS[key] = o
    return o
