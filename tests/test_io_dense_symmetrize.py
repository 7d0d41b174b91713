"""§8(f) rows: BCSS file I/O (reference format, straight to device), the dense
GPU baseline and blocked symmetrization.  The functions are torch-generic, so
the same checks run on CPU tensors here and on CUDA tensors under -m gpu."""

import itertools

import numpy as np
import pytest
import torch

import paper_1301_7744_b200 as bs
from conftest import GOLDEN
from oracle import bcss_oracle as orc
from paper_1301_7744_b200 import dense, io

DEVICES = ["cpu", pytest.param("cuda", marks=pytest.mark.gpu)]


def test_bcss_file_bytes_match_reference(tmp_path):
    d = np.load(GOLDEN / "bcss_file.npz")
    m, n, b = (int(v) for v in d["dims"])
    path = tmp_path / "t.bcss"
    io.save_bcss(bs.BcssTensor(m, n, b, payload=d["A"]), path)
    assert path.read_bytes() == d["raw"].tobytes()  # byte-identical to blocksym.save_bcss
    back = io.load_bcss(path)
    assert back.order == m and back.n == n and back.b == b
    assert np.array_equal(back.payload, d["A"])


def test_bcss_file_errors(tmp_path):
    bad = tmp_path / "bad.bcss"
    bad.write_bytes(b"NOPE" + bytes(20))
    with pytest.raises(ValueError):
        io.load_bcss(bad)
    d = np.load(GOLDEN / "bcss_file.npz")
    trunc = tmp_path / "trunc.bcss"
    trunc.write_bytes(d["raw"].tobytes()[:-8])
    with pytest.raises(ValueError):
        io.load_bcss(trunc)


@pytest.mark.gpu
def test_bcss_file_device_round_trip(tmp_path):
    d = np.load(GOLDEN / "sttsm_rbcss_m4_n12_b4.npz")
    path = tmp_path / "a.bcss"
    io.save_bcss(bs.BcssTensor(4, 12, 4, payload=d["A"]), path)
    pay, m, n, b = io.load_bcss_device(path, chunk_bytes=4096)  # many chunks
    assert (m, n, b) == (4, 12, 4)
    assert np.array_equal(pay.cpu().numpy(), d["A"])
    out = tmp_path / "b.bcss"
    io.save_bcss_device(pay, m, n, b, out, chunk_bytes=4096)
    assert out.read_bytes() == path.read_bytes()


@pytest.mark.parametrize("device", DEVICES)
def test_bcss_to_dense_matches_decompress(device):
    for case in ("sttsm_small_m3_n6_p6_ba3_bc3", "sttsm_rbcss_m4_n12_b4", "sttsm_small_m5_n8_p8_ba4_bc4"):
        d = np.load(GOLDEN / f"{case}.npz")
        m, n, p, ba, bc = (int(v) for v in d["dims"])
        got = dense.bcss_to_dense_device(torch.from_numpy(d["A"]).to(device), m, n, ba).cpu().numpy()
        assert np.array_equal(got, orc.unpack_dense(d["A"], m, n, ba))


@pytest.mark.parametrize("device", DEVICES)
def test_dense_baseline_matches_reference(device):
    """sttsm_dense_ttm on the device == reference C (golden) within fp64 rounding."""
    for case in ("sttsm_config1", "sttsm_small_m3_n6_p4_ba3_bc2", "sttsm_small_m5_n6_p6_ba3_bc3"):
        d = np.load(GOLDEN / f"{case}.npz")
        m, n, p, ba, bc = (int(v) for v in d["dims"])
        a_dense = dense.bcss_to_dense_device(torch.from_numpy(d["A"]).to(device), m, n, ba)
        c = dense.sttsm_dense_ttm_device(a_dense, torch.from_numpy(d["X"]).to(device)).cpu().numpy()
        want = orc.unpack_dense(d["C"], m, p, bc)
        assert orc.rel_frobenius(c, want) <= 1e-13
    assert dense.dense_flops(3, 4, 2) == 448  # reference anchor, tests/test_costs.py:95-96


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["sttsm_rbcss_m4_n12_b4", "sttsm_rbcss_m5_n8_b2", "sttsm_rbcss_m3_n32_b8",
                                  "sttsm_small_m6_n8_p8_ba4_bc4"])
def test_symmetrize_makes_c_exactly_symmetric(case):
    """The native blocked symmetrization (csrc/symmetrize.cu): exact symmetry
    (every orbit one value), and a change within rounding of the reference's
    output (its diagonal blocks are symmetric to ~1 ulp)."""
    device = "cuda"
    d = np.load(GOLDEN / f"{case}.npz")
    m, n, p, ba, bc = (int(v) for v in d["dims"])
    c = torch.from_numpy(d["C"].copy()).to(device)
    before = orc.unpack_dense(d["C"], m, p, bc)
    dense.symmetrize_bcss_device(c, m, p, bc)
    after = orc.unpack_dense(c.cpu().numpy(), m, p, bc)
    asym = lambda t: max(np.max(np.abs(t - np.transpose(t, q))) for q in itertools.permutations(range(m)))
    assert asym(after) == 0.0
    assert orc.rel_frobenius(after, before) <= 1e-14
