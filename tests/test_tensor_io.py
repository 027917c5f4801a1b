"""CPDT binary / text COO files (reference tensor_io.py), pinned to files the
reference's own writers produced (tests/golden/make_golden.py io_fixtures)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from paper_1409_2383_b200 import tensor_io as io


def test_reads_reference_files_and_round_trips(tmp_path):
    g = load_golden("io.npz")
    t = io.read_binary(os.path.join(GOLDEN, "small.cpdt"))
    assert np.array_equal(t.values, g["dense"])
    c = io.read_coo(os.path.join(GOLDEN, "small4.coo"))
    assert c.dims == tuple(g["coo_dims"]) and np.array_equal(c.indices, g["coo_idx"])
    assert np.array_equal(c.vals, g["coo_vals"])
    assert isinstance(io.read_tensor(os.path.join(GOLDEN, "small.cpdt")), type(t))
    # our writers produce byte-identical files
    io.write_tensor(t, tmp_path / "a.cpdt")
    io.write_tensor(c, tmp_path / "b.coo")
    assert (tmp_path / "a.cpdt").read_bytes() == open(os.path.join(GOLDEN, "small.cpdt"), "rb").read()
    assert (tmp_path / "b.coo").read_text() == open(os.path.join(GOLDEN, "small4.coo")).read()


def test_bad_files_rejected(tmp_path):
    (tmp_path / "bad.cpdt").write_bytes(b"XXXX\x03\x00\x00\x00")
    with pytest.raises(ValueError, match="bad magic"):
        io.read_binary(tmp_path / "bad.cpdt")
    data = open(os.path.join(GOLDEN, "small.cpdt"), "rb").read()
    (tmp_path / "cut.cpdt").write_bytes(data[:-8])
    with pytest.raises(ValueError, match="truncated"):
        io.read_binary(tmp_path / "cut.cpdt")
    (tmp_path / "bad.coo").write_text("nodims 2 2 2\n")
    with pytest.raises(ValueError):
        io.read_coo(tmp_path / "bad.coo")


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_binary_streams_into_hbm(tmp_path, dtype):
    """Chunked pinned-buffer upload (chunks smaller than the payload) equals
    the host read; fp32 conversion happens on the device."""
    import torch

    rng = np.random.default_rng(8)
    x = rng.random((37, 29, 23))
    io.write_binary(x, tmp_path / "x.cpdt")
    t = io.read_binary(tmp_path / "x.cpdt", device="cuda", dtype=dtype, chunk_bytes=8 * 1000)
    assert t.values.is_cuda and tuple(t.values.shape) == x.shape
    assert np.array_equal(t.values.cpu().numpy(), x.astype(dtype))
    assert t.values.dtype == (torch.float32 if dtype == np.float32 else torch.float64)
