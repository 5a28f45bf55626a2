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


def _ref_kernels():
    """The reference's own compiled kernel module, built by oracle/build_ref.sh
    from the sources under /root/reference into oracle/_ref (git-ignored; it
    travels to the GPU box with the snapshot). None when it was never built."""
    import importlib.util
    import sysconfig

    here = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
    path = os.path.join(here, "_kernels" + sysconfig.get_config_var("EXT_SUFFIX"))
    if not os.path.exists(path):
        return None
    spec = importlib.util.spec_from_file_location("_kernels", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_oracle_kernels_bitwise_against_compiled_reference(seed):
    """oracle/kernels_oracle.c against the reference's compiled _kernels module
    (backend.py:39-43 binds exactly these five functions) on fresh random
    inputs, beyond the committed fixtures: Gaussian stream, mm, spmm_nt / spmm_t
    and the Jacobi sweeps, all bitwise."""
    ref = _ref_kernels()
    if ref is None:
        pytest.skip("oracle/_ref not built (no /root/reference on this machine)")
    rng = np.random.default_rng(seed)
    for count in (3, 64, 1001):
        state = int(rng.integers(1, 2 ** 62))
        a, sa = o.gauss_fill(count, state)
        b, sb = ref.gauss_fill(count, state)
        assert np.array_equal(a, np.asarray(b)) and int(sa) == int(sb)
    m, k, n = 37, 29, 11
    A = rng.standard_normal((m, k))
    B = rng.standard_normal((k, n))
    assert np.array_equal(o.mm_naive(A, B), np.asarray(ref.mm(A, B)))
    rows, cols = 40, 31
    dense = rng.standard_normal((rows, cols)) * (rng.random((rows, cols)) < 0.2)
    dense[7] = 0.0  # an empty row
    indptr = np.zeros(rows + 1, dtype=np.int64)
    indptr[1:] = np.cumsum((dense != 0).sum(1))
    r, c = np.nonzero(dense)
    col = c.astype(np.int64)
    val = dense[r, c].astype(np.float64)
    X = rng.standard_normal((cols, 5))
    Y = rng.standard_normal((rows, 5))
    assert np.array_equal(o.spmm_nt(rows, indptr, col, val, X), np.asarray(ref.spmm_nt(rows, indptr, col, val, X)))
    assert np.array_equal(o.spmm_t(rows, cols, indptr, col, val, Y),
                          np.asarray(ref.spmm_t(rows, cols, indptr, col, val, Y)))
    w = 24
    S = rng.standard_normal((w, w))
    S = 0.5 * (S + S.T)
    M1, V1 = S.copy(), np.eye(w)
    M2, V2 = S.copy(), np.eye(w)
    r1 = o.jacobi_sweeps(M1, V1, 1e-14, 50)
    r2 = ref.jacobi_sweeps(M2, V2, 1e-14, 50)
    assert np.array_equal(M1, M2) and np.array_equal(V1, V2)
    assert float(r1[0]) == float(r2[0]) and int(r1[1]) == int(r2[1]) and bool(r1[2]) == bool(r2[2])
