"""TEST INFRASTRUCTURE ONLY — CPU oracle for the randomized block-Krylov path.

A numpy restatement of the reference algorithm (rsvdkit 0.1.0) on the
north_star path, used as the parity checker by tests/, by
``__graft_entry__.smoke()`` and by bench.py's ``cpu_baseline`` /
``--impl reference`` legs. The product package never imports this module.

Each function cites the reference file:line it follows (paths relative to
pkg/src/rsvdkit/). The scalar kernels (Gaussian fill, Jacobi sweeps, naive
mm, CSR products) come from ``kernels_oracle.c`` (built to
``oracle/liboracle.so``); dense products default to numpy/BLAS exactly as the
reference's python backend does (_kernels_py.py:48-49).

Pinned against the reference itself: tests/golden/ holds vectors produced by
importing the reference (tests/golden/make_golden.py) and
tests/test_oracle.py checks this module against them.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force=False):
    """Compile kernels_oracle.c with the reference's flags (setup.py:15-19),
    plus -fopenmp for the row/column-sliced CSR loops (bitwise identical)."""
    src = os.path.join(_HERE, "kernels_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        import subprocess

        subprocess.check_call(
            ["gcc", "-O3", "-ffp-contract=off", "-fno-builtin-sin", "-fno-builtin-cos", "-fopenmp",
             "-shared", "-fPIC", "-o", _LIB_PATH, src, "-lm"]
        )
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, u64, dp, ip = ctypes.c_int64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
        L.oracle_gauss_fill.argtypes = [i64, u64, dp]
        L.oracle_gauss_fill.restype = u64
        L.oracle_mm.argtypes = [i64, i64, i64, dp, dp, dp]
        L.oracle_spmm_nt.argtypes = [i64, i64, ip, ip, dp, dp, dp]
        L.oracle_spmm_t.argtypes = [i64, i64, i64, ip, ip, dp, dp, dp]
        L.oracle_jacobi_sweeps.argtypes = [i64, dp, dp, ctypes.c_double, ctypes.c_int, dp, ctypes.POINTER(ctypes.c_int)]
        L.oracle_jacobi_sweeps.restype = ctypes.c_int
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


# ---------------------------------------------------------------- kernels
def gauss_fill(count, state):
    """_kernels.pyx:31-53 — (normals, new_state)."""
    out = np.empty(int(count), dtype=np.float64)
    new = lib().oracle_gauss_fill(int(count), ctypes.c_uint64(int(state) & ((1 << 64) - 1)), _dp(out))
    return out, int(new)


def mm_naive(a, b):
    """_kernels.pyx:56-71 — i-l-j loop, fixed summation order."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    c = np.empty((a.shape[0], b.shape[1]))
    lib().oracle_mm(a.shape[0], a.shape[1], b.shape[1], _dp(a), _dp(b), _dp(c))
    return c


def mm_blas(a, b):
    """_kernels_py.py:48-49 — numpy/BLAS product."""
    return np.ascontiguousarray(a) @ np.ascontiguousarray(b)


def spmm_nt(nrows, indptr, col, val, b):
    """_kernels.pyx:74-92."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int64)
    val = np.ascontiguousarray(val, dtype=np.float64)
    out = np.empty((int(nrows), b.shape[1]))
    lib().oracle_spmm_nt(int(nrows), b.shape[1], _ip(indptr), _ip(col), _dp(val), _dp(b), _dp(out))
    return out


def spmm_t(nrows, ncols, indptr, col, val, b):
    """_kernels.pyx:95-113."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int64)
    val = np.ascontiguousarray(val, dtype=np.float64)
    out = np.empty((int(ncols), b.shape[1]))
    lib().oracle_spmm_t(int(nrows), int(ncols), b.shape[1], _ip(indptr), _ip(col), _dp(val), _dp(b), _dp(out))
    return out


def jacobi_sweeps(m_, v_, tol, max_sweeps):
    """_kernels.pyx:127-192 — in place on m_ and v_ (C-contiguous float64)."""
    assert m_.flags.c_contiguous and v_.flags.c_contiguous
    off = ctypes.c_double()
    sw = ctypes.c_int()
    conv = lib().oracle_jacobi_sweeps(m_.shape[0], _dp(m_), _dp(v_), float(tol), int(max_sweeps),
                                      ctypes.byref(off), ctypes.byref(sw))
    return off.value, sw.value, bool(conv)


# ---------------------------------------------------------------- rng
class SeededRng:
    """matrix.py:38-70 — SplitMix64 + Box-Muller stream."""

    def __init__(self, seed):
        self.seed = int(seed)
        self._state = int(seed)

    def normal_fill(self, count):
        out, self._state = gauss_fill(count, self._state)
        return out


def gaussian(rows, cols, rng):
    """matrix.py:266-276 — row-major fill."""
    return rng.normal_fill(rows * cols).reshape(rows, cols)


# ---------------------------------------------------------------- factor
QR_FILL_SEED = 0x5EED_F111_0C0F_FEE5  # factor.py:40
DEFICIENCY_RTOL = 1e-12  # factor.py:41
DEFAULT_JACOBI_TOL = 1e-14  # factor.py:34
JACOBI_MAX_SWEEPS = 50  # factor.py:35


class ConvergenceError(RuntimeError):
    def __init__(self, message, residual=None):
        super().__init__(message)
        self.residual = residual


def mgs(arr, fill_rng=None):
    """factor.py:79-118 — CGS2 per column with fill-stream replacement.

    Also returns the list of replaced column indices (diagnostic only)."""
    n, m = arr.shape
    if n < m:
        raise ValueError("qr_orthonormalize requires rows >= cols")
    if fill_rng is None:
        fill_rng = SeededRng(QR_FILL_SEED)
    q = np.empty((n, m), dtype=np.float64)
    replaced = []

    def orth(v, j):
        for _ in range(2):
            if j:
                h = q[:, :j]
                v = v - h @ (h.T @ v)
        return v

    for j in range(m):
        col = np.array(arr[:, j], dtype=np.float64)
        ref = float(np.linalg.norm(col))
        v = orth(col, j)
        nv = float(np.linalg.norm(v))
        if nv <= DEFICIENCY_RTOL * ref:
            replaced.append(j)
            for _ in range(100):
                g = fill_rng.normal_fill(n)
                gn = float(np.linalg.norm(g))
                v = orth(g, j)
                nv = float(np.linalg.norm(v))
                if nv > 1e-6 * gn:
                    break
            else:
                raise ConvergenceError("could not find an independent replacement column", residual=nv)
        q[:, j] = v / nv
    mgs.last_replaced = replaced
    return q


def symmetric_eig(m, tol=DEFAULT_JACOBI_TOL, max_sweeps=JACOBI_MAX_SWEEPS):
    """factor.py:132-166 — Jacobi, eigenvalues descending (stable)."""
    arr = np.asarray(m, dtype=np.float64)
    n = arr.shape[0]
    work = np.ascontiguousarray(0.5 * (arr + arr.T))
    vecs = np.ascontiguousarray(np.eye(n))
    off, sweeps, conv = jacobi_sweeps(work, vecs, tol, max_sweeps)
    if not conv:
        raise ConvergenceError(f"Jacobi did not converge in {max_sweeps} sweeps", residual=off)
    vals = np.diag(work).copy()
    order = np.argsort(-vals, kind="stable")
    symmetric_eig.last_sweeps = sweeps
    return vals[order], vecs[:, order]


# ---------------------------------------------------------------- rsvd
def round_up_odd(q):
    return q if q % 2 == 1 else q + 1  # rsvd.py:52-53


def resolve_q(variant, q, d=None):
    """rsvd.py:151-162 (explicit-q branch): BK bumps even q >= 1 to odd."""
    if variant == "sketch":
        return 0
    q = int(q)
    if variant == "bk" and q >= 1:
        q = round_up_odd(q)
    return q


def canonicalize_signs(z):
    """rsvd.py:192-197."""
    for j in range(z.shape[1]):
        idx = int(np.argmax(np.abs(z[:, j])))
        if z[idx, j] < 0:
            z[:, j] = -z[:, j]
    return z


class DenseOp:
    """matrix.py:195-257 (dense branch): A @ X and A^T @ Y with a cached A^T."""

    def __init__(self, a, mm=mm_blas):
        self.a = np.ascontiguousarray(a, dtype=np.float64)
        self.at = None
        self.mm = mm
        self.shape = self.a.shape

    def apply(self, x):
        return self.mm(self.a, np.ascontiguousarray(x, dtype=np.float64))

    def apply_transpose(self, y):
        if self.at is None:
            self.at = np.ascontiguousarray(self.a.T)
        return self.mm(self.at, np.ascontiguousarray(y, dtype=np.float64))


class CsrOp:
    """matrix.py:227-247 (sparse branch)."""

    def __init__(self, rows, cols, indptr, col, val):
        self.shape = (int(rows), int(cols))
        self.indptr = np.asarray(indptr, dtype=np.int64)
        self.col = np.asarray(col, dtype=np.int64)
        self.val = np.asarray(val, dtype=np.float64)
        self.mm = mm_blas

    def apply(self, x):
        return spmm_nt(self.shape[0], self.indptr, self.col, self.val, x)

    def apply_transpose(self, y):
        return spmm_t(self.shape[0], self.shape[1], self.indptr, self.col, self.val, y)


def post_process(op, q, k):
    """rsvd.py:200-221 — M = Q^T A A^T Q, Jacobi eig, Z = Q U_k, signs."""
    if q.shape[1] < k:
        raise ValueError("Q must have at least k columns")
    qt = np.ascontiguousarray(q.T)
    gram = op.mm(qt, q)
    if float(np.max(np.abs(gram - np.eye(q.shape[1])))) > 1e-8:
        raise ValueError("Q must have orthonormal columns")
    m = op.mm(qt, op.apply(op.apply_transpose(q)))
    vals, vecs = symmetric_eig(0.5 * (m + m.T))
    top = np.ascontiguousarray(vecs[:, :k])
    z = canonicalize_signs(op.mm(q, top))
    sigma = np.sqrt(np.clip(vals[:k], 0.0, None))
    return z, sigma


def sketch_basis(op, p, rng):
    """rsvd.py:224-226."""
    pi = gaussian(op.shape[1], p, rng)
    return mgs(op.apply(pi))


def si_basis(op, p, q, every, rng):
    """rsvd.py:229-241."""
    if q == 0:
        return sketch_basis(op, p, rng)
    pi = gaussian(op.shape[1], p, rng)
    b = op.apply(pi)
    orthonormal = False
    for t in range(1, q + 1):
        b = op.apply(op.apply_transpose(b))
        orthonormal = False
        if every and t % every == 0:
            b = mgs(b)
            orthonormal = True
    return b if orthonormal else mgs(b)


def bk_basis(op, p, q, rng):
    """rsvd.py:244-260 — returns (Q, q_used, blocks)."""
    n, d = op.shape
    if p > n:
        raise ValueError("block width p exceeds n; no Krylov block fits")
    n_blocks = min(q + 1, max(1, min(n, d) // p))
    b = sketch_basis(op, p, rng)
    if n_blocks == 1:
        return b, 0
    blocks = [b]
    for _ in range(1, n_blocks):
        b = mgs(op.apply(op.apply_transpose(b)))
        blocks.append(b)
    return mgs(np.hstack(blocks)), n_blocks - 1


@dataclass
class OracleResult:
    Z: np.ndarray
    sigma: np.ndarray
    q_used: int
    basis_width: int
    replaced: list


def factorize(op, k, variant, q=None, p=None, seed=0, every=1):
    """rsvd.py:263-290 — the whole path on one operator."""
    n, d = op.shape
    if k > min(n, d):
        raise ValueError("k must not exceed min(n, d)")
    p = k if p is None else int(p)
    qe = resolve_q(variant, q if q is not None else 0, d)
    rng = SeededRng(seed)
    if variant == "si":
        basis = si_basis(op, p, qe, every, rng)
        q_used = qe
    elif variant == "bk":
        basis, q_used = bk_basis(op, p, qe, rng)
    else:
        basis = sketch_basis(op, p, rng)
        q_used = 0
    replaced = list(getattr(mgs, "last_replaced", []))
    z, sigma = post_process(op, basis, k)
    return OracleResult(z, sigma, q_used, basis.shape[1], replaced)


# ---------------------------------------------------------------- metrics
def captured_variance(a_dense_or_op, z):
    """metrics.py:136 — ||A^T z_i||^2 per column."""
    if isinstance(a_dense_or_op, np.ndarray):
        w = a_dense_or_op.T @ z
    else:
        w = a_dense_or_op.apply_transpose(z)
    return np.sum(w * w, axis=0)


def spectral_norm_est(apply, apply_t, d, tol=1e-9, max_iters=20000, seed=0):
    """factor.py:217-253 — power iteration, returns the best estimate."""
    rng = SeededRng(seed)
    v = rng.normal_fill(d).reshape(d, 1)
    nv = float(np.linalg.norm(v))
    if nv == 0.0:
        return 0.0
    v /= nv
    best, prev = 0.0, None
    for _ in range(int(max_iters)):
        w = apply(v)
        est = float(np.linalg.norm(w))
        best = max(best, est)
        if est == 0.0:
            return 0.0
        if prev is not None and abs(est - prev) <= tol * est:
            break
        prev = est
        v = apply_t(w / est)
        nv = float(np.linalg.norm(v))
        if nv == 0.0:
            break
        v /= nv
    return best


def spectral_error(a, z, seeds=(101, 202, 303), tol=1e-9, max_iters=20000):
    """metrics.py:65-81, 102-122 — ||(I - Z Z^T) A||_2 by restarted power iteration."""
    def proj(y):
        return y - z @ (z.T @ y)

    return max(
        spectral_norm_est(lambda x: proj(a @ x), lambda y: a.T @ proj(y), a.shape[1], tol, max_iters, s)
        for s in seeds
    )


def spectral_error_exact(a, z):
    """Exact ||A - Z Z^T A||_2 by LAPACK."""
    r = a - z @ (z.T @ a)
    return float(np.linalg.norm(r, 2))


# ---------------------------------------------------------------- inputs
def synth_matrix(n, d, spectrum, seed=0, mm=mm_naive):
    """synth.py:59-74 (without the oracle self-check): A = U diag(s) V^T."""
    spectrum = np.asarray(spectrum, dtype=np.float64)
    m = spectrum.size
    rng = SeededRng(seed)
    u = mgs(gaussian(n, m, rng))
    v = mgs(gaussian(d, m, rng))
    return mm(u * spectrum[None, :], np.ascontiguousarray(v.T))
