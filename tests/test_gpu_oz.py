"""FP64-accurate int8 tensor-core products of an FP32 A (csrc/gemm_oz.cu)
against cuBLAS FP64 GEMMs of the same (exactly upcast) operands.

The reference computes every product in float64 on A upcast from float32
(matrix.py:80, _kernels.pyx:56-71); the Ozaki digit-plane kernels must match
that arithmetic to FP64 rounding: normwise relative error <= 1e-14 (the
scheme's neglected terms are ~2^-56 |A||X| per entry)."""

import pytest
import torch

pytestmark = pytest.mark.gpu

# Normwise per entry, |C - C_exact| / (|a_r| |x_c|). The scheme keeps digit
# levels i + j <= 5 of signed base-256 digits (5 of A, 6 of X); the dropped
# level-6 terms are ~2^-49 of (row scale x column scale) per entry (the
# base-128 first version measured A X 5.4e-15 at K = 900 against 80-bit sums;
# cuBLAS DGEMM 1.4e-16). A^T Y with rows of very different magnitude
# (row_spread) carries each row's exponent into Y's column scale and loses
# about one more digit (6e-14 at e^(+-3) row spread).
TOL = 4e-14  # base-256 digits: A X 2.3e-14 measured at K = 900
TOL_SPREAD = 2e-13
# against cuBLAS DGEMM (whose own blocked FP64 accumulation adds ~1e-13 at
# K ~ 1e4); base-256 digits with a row spread of e^(+-2): 3.6e-13 measured
TOL_DGEMM = 6e-13


def _ops():
    from paper_1504_05477_b200 import device as ops

    return ops


def _case(n, d, seed, row_spread=0.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = torch.randn((n, d), generator=g, device="cuda", dtype=torch.float64)
    if row_spread:
        # rows of very different magnitude (per-row exponents must follow)
        A *= torch.exp(row_spread * torch.randn((n, 1), generator=g, device="cuda", dtype=torch.float64))
    return A.float()


def _normwise(C, ref, left, right):
    """max_ij |C - ref|_ij / (|left_i| |right_j|) (normwise per entry)."""
    den = torch.outer(left.norm(dim=1), right.norm(dim=0)).clamp_min(1e-300)
    return float(((C - ref).abs() / den).max())


@pytest.mark.parametrize("n,d,p", [(1000, 700, 50), (4133, 2051, 20), (3000, 1000, 64), (2000, 1500, 130),
                                   (257, 33, 7), (20000, 400, 50)])
def test_oz_nn_tn_match_fp64(n, d, p):
    ops = _ops()
    A = _case(n, d, n + d + p, row_spread=2.0)
    A64 = A.double()
    g = torch.Generator(device="cuda").manual_seed(7)
    X = torch.randn((d, p), generator=g, device="cuda", dtype=torch.float64)
    Y = torch.randn((n, p), generator=g, device="cuda", dtype=torch.float64)
    P = ops.OzPlanes(A)
    C = torch.empty((n, p), dtype=torch.float64, device="cuda")
    ops.oz_gemm(P, X, C, trans=0)
    W = torch.empty((d, p), dtype=torch.float64, device="cuda")
    ops.oz_gemm(P, Y, W, trans=1)
    torch.cuda.synchronize()
    e_nn = _normwise(C, A64 @ X, A64, X)
    e_tn = _normwise(W, A64.T @ Y, A64.T, Y)
    assert e_nn < TOL_DGEMM, e_nn
    assert e_tn < TOL_DGEMM, e_tn


def test_oz_vs_extended():
    """Against 80-bit extended-precision host sums (numpy longdouble): the
    digit-plane products are FP64-accurate, at least as close as cuBLAS DGEMM."""
    import numpy as np

    ops = _ops()
    n, d, p = 700, 900, 24
    A = _case(n, d, 5, row_spread=1.0)  # e^(+-3) row magnitudes
    g = torch.Generator(device="cuda").manual_seed(2)
    X = torch.randn((d, p), generator=g, device="cuda", dtype=torch.float64)
    Y = torch.randn((n, p), generator=g, device="cuda", dtype=torch.float64)
    P = ops.OzPlanes(A)
    C = torch.empty((n, p), dtype=torch.float64, device="cuda")
    W = torch.empty((d, p), dtype=torch.float64, device="cuda")
    ops.oz_gemm(P, X, C, trans=0)
    ops.oz_gemm(P, Y, W, trans=1)
    torch.cuda.synchronize()
    Ah = A.double().cpu().numpy().astype(np.longdouble)
    Xh = X.cpu().numpy().astype(np.longdouble)
    Yh = Y.cpu().numpy().astype(np.longdouble)
    for name, ours, blas, exact, left, right in (
            ("A X", C, A.double() @ X, Ah @ Xh, Ah, Xh), ("A^T Y", W, A.double().T @ Y, Ah.T @ Yh, Ah.T, Yh)):
        den = np.outer(np.linalg.norm(left.astype(np.float64), axis=1), np.linalg.norm(right.astype(np.float64), axis=0))
        e_ours = float(np.max(np.abs(ours.cpu().numpy() - exact).astype(np.float64) / den))
        e_blas = float(np.max(np.abs(blas.cpu().numpy() - exact).astype(np.float64) / den))
        print(f"{name}: normwise error vs 80-bit sums: digit planes {e_ours:.2e}, cuBLAS DGEMM {e_blas:.2e}")
        assert e_ours < (TOL if name == "A X" else TOL_SPREAD), (name, e_ours, e_blas)


def test_oz_long_reduction_splits():
    """A^T Y with n > 16384 (several K splits: int32 exactness bound) and
    alpha / beta handling."""
    ops = _ops()
    n, d, p = 70000, 300, 50
    A = _case(n, d, 3)
    A64 = A.double()
    g = torch.Generator(device="cuda").manual_seed(9)
    Y = torch.randn((n, p), generator=g, device="cuda", dtype=torch.float64)
    W0 = torch.randn((d, p), generator=g, device="cuda", dtype=torch.float64)
    P = ops.OzPlanes(A)
    W = W0.clone()
    ops.oz_gemm(P, Y, W, trans=1, alpha=-0.5, beta=2.0)
    ref = -0.5 * (A64.T @ Y) + 2.0 * W0
    torch.cuda.synchronize()
    err = float(((W - ref).abs()).max() / (A64.T.abs() @ Y.abs()).max())
    assert err < TOL_DGEMM, err


def test_oz_wide_reduction_and_extreme_digits():
    """A X with d > 16384 (the NN reduction split for int32 exactness) on an
    adversarial operand: every entry of A and X at the same magnitude and sign,
    so that every digit product has the same sign and the int32 level sums run
    as high as the scheme allows (7 pairs x 128^2 x 16384 < 2^31); plus the
    random case."""
    ops = _ops()
    n, d, p = 300, 40000, 40
    for kind in ("extreme", "random"):
        if kind == "extreme":
            A = torch.full((n, d), -0.99609375 * 0.5, device="cuda")  # u = -0.498...: digits near -127
            X = torch.full((d, p), -(1.0 - 2.0 ** -40), device="cuda", dtype=torch.float64)
        else:
            A = _case(n, d, 31)
            X = torch.randn((d, p), device="cuda", dtype=torch.float64)
        P = ops.OzPlanes(A)
        C = torch.empty((n, p), dtype=torch.float64, device="cuda")
        ops.oz_gemm(P, X, C, trans=0)
        torch.cuda.synchronize()
        assert _normwise(C, A.double() @ X, A.double(), X) < TOL_DGEMM, kind


def test_oz_zero_rows_and_columns():
    """All-zero rows of A and zero columns of B give exact zeros."""
    ops = _ops()
    n, d, p = 600, 300, 40
    A = _case(n, d, 11)
    A[17] = 0.0
    A[:, 5] = 0.0
    X = torch.randn((d, p), device="cuda", dtype=torch.float64)
    X[:, 3] = 0.0
    P = ops.OzPlanes(A)
    C = torch.empty((n, p), dtype=torch.float64, device="cuda")
    ops.oz_gemm(P, X, C, trans=0)
    torch.cuda.synchronize()
    assert bool((C[17] == 0).all()) and bool((C[:, 3] == 0).all())
    assert _normwise(C, A.double() @ X, A.double(), X) < TOL_DGEMM


@pytest.mark.parametrize("jp", [50, 200, 550])
def test_oz_basis_projections(jp):
    """Digit planes of an orthonormal FP64 basis, sliced one block at a time
    (column offsets not aligned to the 16-column storage blocks): Q_p^T V and
    V - Q_p C against cuBLAS FP64, normwise (|q| <= 1, ||q_c|| = 1)."""
    ops = _ops()
    n, w, p = 30000, 600, 50
    g = torch.Generator(device="cuda").manual_seed(jp)
    Q, _ = torch.linalg.qr(torch.randn((n, w), generator=g, device="cuda", dtype=torch.float64))
    Q = Q.contiguous()
    B = ops.OzBasis(n, w, Q.device)
    for c0 in range(0, w, p):
        B.slice(Q, c0, p)
    V = torch.randn((n, p), generator=g, device="cuda", dtype=torch.float64)
    C = torch.empty((jp, p), dtype=torch.float64, device="cuda")
    B.gemm(1, jp, V, C)
    Qp = Q[:, :jp]
    ref = Qp.T @ V
    torch.cuda.synchronize()
    e_tn = float(((C - ref).abs() / V.norm(dim=0).view(1, -1)).max())
    V2 = V.clone()
    B.gemm(0, jp, C, V2, alpha=-1.0, beta=1.0)
    ref2 = V - Qp @ C
    torch.cuda.synchronize()
    e_nn = float(((V2 - ref2).abs() / C.norm(dim=0).view(1, -1)).max())
    assert e_tn < TOL, e_tn
    assert e_nn < TOL, e_nn


@pytest.mark.parametrize("p", [64, 200, 600])
def test_oz_reduced_levels(p):
    """The Rayleigh-Ritz variant (digit levels i + j <= 3): ~1e-10 normwise;
    widths above 64 run the 128-column N tile (two epilogue passes, u64 TMA
    view of the B planes), 600 = C2's Krylov width with a ragged last tile."""
    ops = _ops()
    n, d = 5000, 700
    A = _case(n, d, 21)
    A64 = A.double()
    Y = torch.randn((n, p), device="cuda", dtype=torch.float64)
    P = ops.OzPlanes(A)
    W = torch.empty((d, p), dtype=torch.float64, device="cuda")
    ops.oz_gemm(P, Y, W, trans=1, reduced=True)
    torch.cuda.synchronize()
    e = _normwise(W, A64.T @ Y, A64.T, Y)
    assert 1e-15 < e < 1e-9, e
