"""FROSTT parsing, duplicate summing and result files (host side, no GPU), against the
reference's semantics (ref tensor.py:72-149,213-225, cli.py:93-104)."""

import numpy as np
import pytest

from paper_2210_05105_b200.coo import BoundsError
from paper_2210_05105_b200.tensorio import (ParseError, load_frostt, read_matrix,
                                            sum_duplicates, write_matrix)


def write(tmp_path, text, name="t.tns"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_load_frostt_dedup_and_log(tmp_path):
    path = write(tmp_path, "# comment\n1 1 1 2.0\n2 3 1 1.5\n\n1 1 1 0.5\n2 1 2 3.0\n")
    t = load_frostt(path)
    assert t.dims == (2, 3, 2)
    assert np.array_equal(t.idx, [[0, 0, 0], [1, 0, 1], [1, 2, 0]])
    assert np.allclose(t.vals, [2.5, 3.0, 1.5])
    tl = load_frostt(path, log_transform=True)
    assert np.allclose(tl.vals, np.log1p([2.5, 3.0, 1.5]))
    raw = load_frostt(path, dedup=False)
    assert raw.nnz == 4 and raw.idx[2].tolist() == [0, 0, 0]
    assert load_frostt(path, dims=(5, 5, 5)).dims == (5, 5, 5)


@pytest.mark.parametrize("text,err", [
    ("", ParseError), ("# only\n", ParseError), ("1 1 2.0\n", ParseError),
    ("1 1 1 2.0\n1 1 x 1.0\n", ParseError), ("1 1.5 1 2.0\n", ParseError),
    ("0 1 1 2.0\n", BoundsError), ("1 2 3 4 1.0\n1 1 1 1.0\n", ParseError)])
def test_load_frostt_errors(tmp_path, text, err):
    with pytest.raises(err):
        load_frostt(write(tmp_path, text))


def test_load_frostt_declared_dims(tmp_path):
    path = write(tmp_path, "3 1 1 1.0\n")
    with pytest.raises(BoundsError):
        load_frostt(path, dims=(2, 2, 2))
    with pytest.raises(ParseError):
        load_frostt(path, dims=(3, 3))


def test_sum_duplicates_order_and_sums():
    rs = np.random.default_rng(0)
    idx = rs.integers(0, 3, size=(200, 3))
    vals = rs.standard_normal(200)
    u, s = sum_duplicates(idx, vals)
    keys = [tuple(r) for r in u]
    assert keys == sorted(set(map(tuple, idx)))
    for k, v in zip(keys, s):
        assert np.isclose(v, vals[(idx == k).all(axis=1)].sum())
    e_idx, e_vals = sum_duplicates(np.zeros((0, 3), dtype=np.int64), np.zeros(0))
    assert e_idx.shape == (0, 3) and e_vals.size == 0


def test_matrix_file_roundtrip(tmp_path):
    M = np.arange(12.0).reshape(4, 3)
    write_matrix(str(tmp_path / "m.bin"), M)
    assert np.array_equal(read_matrix(str(tmp_path / "m.bin")), M)
    write_matrix(str(tmp_path / "v.bin"), np.array([1.0, 2.0]))
    assert read_matrix(str(tmp_path / "v.bin")).shape == (2, 1)
    raw = (tmp_path / "m.bin").read_bytes()
    assert np.frombuffer(raw[:16], dtype="<i8").tolist() == [4, 3]
    (tmp_path / "bad.bin").write_bytes(raw[:40])
    with pytest.raises(ParseError):
        read_matrix(str(tmp_path / "bad.bin"))
