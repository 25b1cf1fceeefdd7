"""C-ABI library: loads without a GPU, exports every symbol include/randcp_b200.h
declares, and its host-side random-stream code reproduces the reference's numpy streams
bit for bit (golden vectors from the reference)."""

import os
import re

import numpy as np
import pytest

from conftest import REPO, golden
from paper_2210_05105_b200 import _lib, rng


def header_functions():
    src = open(os.path.join(REPO, "include", "randcp_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rcp_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_header_symbols():
    lib = _lib.load()
    declared = header_functions()
    assert declared, "no functions parsed from header"
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.EXPORTED)
    assert lib.rcp_version().decode().startswith("randcp_b200")


def test_no_gpu_reports_zero_sms_without_crashing():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert _lib.load().rcp_device_sms() == 0


def test_stream_keys_draws_permutations_match_reference():
    g = golden("rng.npz")
    for row, key, draws in zip(g["ctx"], g["keys"], g["draws"]):
        seed, purpose, n = int(row[0]), int(row[1]), int(row[2])
        ctx = [int(v) for v in row[3:3 + n]]
        k = rng.stream_key(seed, purpose, *ctx)
        assert k == (int(key[0]), int(key[1]))
        assert np.array_equal(rng.uniforms_host(k, 13), draws)
        assert np.array_equal(rng.uniforms_host(k, 5, first=8), draws[8:13])
    s, p, *ctx = [int(v) for v in g["perm_ctx"]]
    k = rng.stream_key(s, p, *ctx)
    for J in (1, 2, 7, 1000, 4096):
        assert np.array_equal(rng.permutation(k, J), g["perm_%d" % J])


@pytest.mark.parametrize("seed,purpose,ctx", [(0, 5, (4, 2, 1)), (99, 3, (1, 0, 2, 5)),
                                               (2 ** 63 + 11, 4, (7, 1, 0)), (5, 2, ())])
def test_streams_match_numpy_live(seed, purpose, ctx):
    ss = np.random.SeedSequence(entropy=seed, spawn_key=(purpose,) + ctx)
    gen = np.random.Generator(np.random.Philox(ss))
    k = rng.stream_key(seed, purpose, *ctx)
    assert k == tuple(int(v) for v in ss.generate_state(2, np.uint64))
    assert np.array_equal(rng.uniforms_host(k, 257), gen.random(257))
    gen2 = np.random.Generator(np.random.Philox(np.random.SeedSequence(entropy=seed,
                                                                       spawn_key=(purpose,) + ctx)))
    assert np.array_equal(rng.permutation(k, 3001), gen2.permutation(3001))


def test_product_path_refuses_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2210_05105_b200 import gram
    with pytest.raises(RuntimeError, match="CUDA"):
        gram(np.eye(3))


def test_mttkrp_workspace_holds_requested_capacity():
    """rcp_mttkrp_ws_bytes(J, cap, ...) must yield a layout whose entry capacity is >= cap
    (host-only layout arithmetic; a short capacity silently dropped gathered nonzeros)."""
    lib = _lib.load()
    lay = np.zeros(14, dtype=np.int64)
    for J in (1, 7, 256, 65536):
        for cap in (0, 1, 5, 60, 63, 64, 65, 1000, 12345, 10 ** 6):
            for n in (1, 5, 30000, 60000):
                for R in (1, 6, 50, 128):
                    b = lib.rcp_mttkrp_ws_bytes(J, cap, n, R)
                    assert lib.rcp_mttkrp_layout(J, n, R, b, lay.ctypes.data) == 0
                    assert lay[13] >= cap, (J, cap, n, R, lay[13])
