"""ctypes binding of librandcp_b200.so (the C ABI declared in include/randcp_b200.h).

The product path has no CPU fallback: importing a compute entry point without the built
library, or calling one without a CUDA device, raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librandcp_b200.so")

OK = 0
ST_DEGENERATE = 1
ST_ZERO_PROB = 2
ST_ASYMMETRIC = 4
ST_ZERO_MASS = 8
ST_NONFINITE = 16
ST_CAPACITY = 32
ST_TIMEOUT = 64

_vp = C.c_void_p
_i64 = C.c_int64
_u64 = C.c_uint64
_i32 = C.c_int
_f64 = C.c_double
_sz = C.c_size_t

# name -> (restype, argtypes)
_SIGS = {
    "rcp_version": (C.c_char_p, []),
    "rcp_last_error": (C.c_char_p, []),
    "rcp_device_sms": (_i32, []),
    "rcp_launch_count": (_i64, []),
    "rcp_stream_key": (_i32, [_u64, _u64, _vp, _i32, _vp]),
    "rcp_uniform_host": (_i32, [_vp, _i64, _i64, _vp]),
    "rcp_permutation_host": (_i32, [_vp, _i64, _vp]),
    "rcp_permutations_host": (_i32, [_vp, _i32, _i64, _vp, _i32]),
    "rcp_uniform": (_i32, [_u64, _u64, _i64, _i64, _vp, _vp]),
    "rcp_gram_ws_bytes": (_sz, [_i64, _i32]),
    "rcp_gram": (_i32, [_vp, _vp, _i64, _i32, _vp, _vp, _vp]),
    "rcp_pinv": (_i32, [_vp, _i32, _i32, _i32, _f64, _vp, _vp, _vp, _vp]),
    "rcp_update_ws_bytes": (_sz, [_i64, _i32]),
    "rcp_update": (_i32, [_vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rcp_renormalize": (_i32, [_vp, _i64, _i32, _vp, _vp, _vp]),
    "rcp_arls_build_ws_bytes": (_sz, [_i64, _i32]),
    "rcp_arls_build": (_i32, [_vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rcp_arls_draw": (_i32, [_vp, _vp, _i64, _i64, _f64, _vp, _u64, _u64, _vp, _i64, _i64, _vp,
                             _vp, _vp, _i32, _vp, _vp, _vp]),
    "rcp_batch_fold": (_i32, [_vp, _vp, _vp, _i64, _vp, _i64, _vp, _i32, _i32, _vp, _vp, _vp,
                              _vp]),
    "rcp_sts_depth": (_i32, [_i64, _i32]),
    "rcp_sts_tree_doubles": (_sz, [_i64, _i32, _i32]),
    "rcp_sts_cond": (_i32, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "rcp_sts_rank_walk": (_i32, [_vp, _i32, _i32, _vp, _vp, _vp, _i64, _i32, _u64, _u64, _vp,
                                 _vp, _vp, _vp, _vp, _vp, _vp]),
    "rcp_sts_rank_tree_doubles": (_sz, [_i32, _i32]),
    "rcp_sts_rank_tree": (_i32, [_vp, _vp, _i32, _i32, _vp, _vp]),
    "rcp_sts_rank_walk_ws_bytes": (_sz, [_i64, _i32, _i32]),
    "rcp_sts_rank_walk_grouped": (_i32, [_vp, _i32, _vp, _i32, _vp, _vp, _vp, _i32, _i64, _u64,
                                         _u64, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _vp]),
    "rcp_sts_rank_walk_ones": (_i32, [_vp, _i32, _vp, _i32, _vp, _i64, _u64, _u64, _vp, _vp, _vp, _vp,
                                      _vp, _vp, _vp]),
    "rcp_sts_flat_local": (_i32, [_vp, _vp, _i64, _i64, _vp, _vp, _vp, _i32, _i64, _vp, _vp, _vp,
                                  _vp, _vp]),
    "rcp_exchange_pack": (_i32, [_vp, _vp, _vp, _vp, _i64, _i64, _vp, _i32, _i64, _i32, _vp, _vp]),
    "rcp_exchange_unpack": (_i32, [_vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "rcp_sts_build": (_i32, [_vp, _i64, _i32, _i32, _vp, _vp]),
    "rcp_sts_walk_ws_bytes": (_sz, [_i64, _i64, _i32, _i32]),
    "rcp_sts_walk": (_i32, [_vp, _vp, _i64, _i32, _i32, _i64, _vp, _vp, _vp, _i32, _i64, _u64, _u64,
                            _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _vp]),
    "rcp_sts_walk_prepared": (_i32, [_vp, _vp, _i64, _i32, _i32, _i64, _vp, _vp, _vp, _i32, _i64,
                                     _u64, _u64, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp,
                                     _sz, _vp, _vp]),
    "rcp_sts_walk_gm": (_i32, [_vp, _i64, _i32, _i32, _vp, _i64, _vp, _sz, _vp]),
    "rcp_fold_rows": (_i32, [_vp, _vp, _i64, _i32, _i64, _vp, _i64, _i32, _vp, _i32, _vp]),
    "rcp_row_keys": (_i32, [_vp, _i32, _i64, _vp, _vp, _vp]),
    "rcp_sts_flat_draw": (_i32, [_vp, _vp, _i64, _i64, _vp, _u64, _u64, _vp, _i64, _vp, _vp, _vp,
                                 _vp]),
    "rcp_hadamard_rows": (_i32, [_vp, _vp, _i64, _i32, _i32, _vp]),
    "rcp_ordered_sum": (_i32, [_vp, _i32, _i64, _vp, _vp]),
    "rcp_weights": (_i32, [_vp, _i32, _i64, _vp, _vp, _vp, _vp]),
    "rcp_mttkrp_ws_bytes": (_sz, [_i64, _i64, _i64, _i32]),
    "rcp_mttkrp_layout": (_i32, [_i64, _i64, _i32, _sz, _vp]),
    "rcp_set_mttkrp_mode": (_i32, [_i32]),
    "rcp_sampled_mttkrp": (_i32, [_vp, _vp, _i64, _vp, _vp, _i64, _vp, _i32, _i64, _i32, _vp,
                                  _vp, _vp, _i32, _vp, _vp, _vp, _sz, _vp, _vp]),
    "rcp_fiber_lookup": (_i32, [_vp, _i64, _vp, _vp, _i32, _i64, _i32, _vp, _vp, _vp, _vp]),
    "rcp_fiber_expand": (_i32, [_vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rcp_csr_spmm": (_i32, [_vp, _i64, _vp, _vp, _vp, _vp, _i32, _vp, _vp]),
    "rcp_fit_ws_bytes": (_sz, [_i64]),
    "rcp_fit_cross": (_i32, [_vp, _vp, _i64, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp,
                             _i32, _vp, _vp, _vp, _sz, _vp]),
    "rcp_sum_squares": (_i32, [_vp, _i64, _vp, _vp, _sz, _vp]),
    "rcp_model_norm": (_i32, [_vp, _i32, _i32, _vp, _vp, _vp]),
    "rcp_zipf_guide": (_i32, [_vp, _i64, _i64, _vp, _vp]),
    "rcp_zipf_draws": (_i32, [_i32, _vp, _vp, _vp, _vp, _u64, _i32, _i64, _i64, _i32, _f64, _i32,
                              _i64, _vp, _vp, _vp, _i64, _vp, _vp]),
    "rcp_sort_ws_bytes": (_sz, [_i64]),
    "rcp_order_by_key_row": (_i32, [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _sz, _vp]),
    "rcp_run_flags": (_i32, [_vp, _i64, _vp, _vp]),
    "rcp_cells": (_i32, [_vp, _vp, _vp, _i64, _i64, _i32, _vp, _vp, _i32, _vp, _vp, _vp]),
    "rcp_exact_mttkrp": (_i32, [_vp, _vp, _i64, _vp, _vp, _i64, _i64, _i32, _i32, _vp, _vp, _vp,
                                _vp, _i32, _vp, _vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


class LibraryMissing(RuntimeError):
    pass


def load(path=None):
    """Load and bind the library (no GPU needed to load).  RCP_LIB overrides the in-tree
    path (A/B runs of library variants, tools/lab/ab_bench.py)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("RCP_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise LibraryMissing("librandcp_b200.so not built (run __graft_entry__.build() or "
                             "python paper_2210_05105_b200/build.py): %s" % path)
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    return _lib if _lib is not None else load()


def check(rc, what=""):
    if rc != OK:
        msg = lib().rcp_last_error().decode(errors="replace")
        raise RuntimeError("randcp_b200 %s failed (rc=%d): %s" % (what, rc, msg))


def call(name, *args):
    rc = getattr(lib(), name)(*args)
    check(rc, name)
    return rc
