"""The CPU oracle (oracle/) pinned against vectors produced by the reference
itself (tests/golden/make_golden.py imports rsvdkit 0.1.0)."""

import hashlib
import json
import os

import numpy as np
import pytest

import rsvd_oracle as o
from conftest import GOLDEN


def _g(name):
    return np.load(os.path.join(GOLDEN, name))


def test_gauss_fill_bitwise_against_reference():
    g = _g("gauss_fill.npz")
    for count in (1, 2, 7, 100, 1001):
        out, st = o.gauss_fill(count, 987654321)
        assert np.array_equal(out, g[f"fill_{count}"])
        assert st == int(g[f"state_{count}"][0])


def test_pi_c1_and_fill_stream():
    g = _g("gauss_fill.npz")
    meta = json.load(open(os.path.join(GOLDEN, "meta.json")))
    pi = o.gaussian(1000, 20, o.SeededRng(0))
    assert np.array_equal(pi.ravel()[:64], g["pi_c1_head"])
    assert hashlib.sha256(pi.tobytes()).hexdigest() == meta["pi_c1_sha256"]
    fill = o.SeededRng(o.QR_FILL_SEED).normal_fill(4096)
    assert np.array_equal(fill, g["qr_fill_head"])


def test_kernel_kats():
    k = _g("kernels.npz")
    assert np.max(np.abs(o.mm_naive(k["mm_a"], k["mm_b"]) - k["mm_c"])) == 0.0
    rows, cols = k["sp_shape"]
    nt = o.spmm_nt(rows, k["sp_indptr"], k["sp_col"], k["sp_val"], k["sp_bx"])
    assert np.array_equal(nt, k["sp_nt"])
    t = o.spmm_t(rows, cols, k["sp_indptr"], k["sp_col"], k["sp_val"], k["sp_by"])
    assert np.array_equal(t, k["sp_t"])
    m, v = k["jac_in"].copy(), np.eye(12)
    off, sweeps, conv = o.jacobi_sweeps(m, v, 1e-14, 50)
    assert conv and sweeps == int(k["jac_sweeps"][0])
    assert np.array_equal(np.diag(m), k["jac_diag"])
    assert np.array_equal(v, k["jac_v"])
    vals, vecs = o.symmetric_eig(k["jac_in"])
    assert np.array_equal(vals, k["eig_vals"]) and np.array_equal(vecs, k["eig_vecs"])


def _cases():
    c = _g("cases.npz")
    names = sorted({key.split("__")[0] for key in c.files})
    return c, names


@pytest.mark.parametrize("name", _cases()[1])
def test_small_cases_match_reference(name):
    c, _ = _cases()
    cfg = json.loads(str(c[f"{name}__cfg"]))
    if f"{name}__A" in c.files:
        op = o.DenseOp(c[f"{name}__A"], mm=o.mm_naive)
    else:
        rows, cols = c[f"{name}__csr_shape"]
        op = o.CsrOp(rows, cols, c[f"{name}__csr_indptr"], c[f"{name}__csr_col"], c[f"{name}__csr_val"])
        op.mm = o.mm_naive
    r = o.factorize(op, cfg["k"], cfg["variant"], q=cfg["q"], p=cfg["p"], seed=cfg["seed"], every=cfg["every"])
    sig = c[f"{name}__sigma"]
    assert r.q_used == int(c[f"{name}__q_used"])
    assert np.max(np.abs(r.sigma - sig)) <= 1e-12 * max(1.0, sig.max())
    assert np.max(np.abs(r.Z - c[f"{name}__Z"])) <= 1e-8


def test_c1_regenerated_bitwise_and_reference_outputs():
    g = _g("c1.npz")
    meta = json.load(open(os.path.join(GOLDEN, "meta.json")))
    A = o.synth_matrix(2000, 1000, 1.0 / np.arange(1, 1001), seed=0)
    assert hashlib.sha256(A.tobytes()).hexdigest() == meta["c1"]["A_sha256"]
    r = o.factorize(o.DenseOp(A), 20, "bk", q=8, seed=0)
    assert r.q_used == 9 and r.basis_width == 200
    assert np.max(np.abs(r.sigma - g["sigma"]) / g["sigma"]) < 1e-13
    cap = o.captured_variance(A, r.Z)
    assert np.max(np.abs(cap - g["captured"]) / g["captured"]) < 1e-12
    # the reference's sigma equals the true spectrum 1/i
    assert np.max(np.abs(g["sigma"] - 1.0 / np.arange(1, 21)) * np.arange(1, 21)) < 1e-13
    assert abs(o.spectral_error_exact(A, r.Z) - g["spectral_exact"][0]) < 1e-13
