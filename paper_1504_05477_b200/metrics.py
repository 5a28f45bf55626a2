"""GPU parity metrics: the reference's per-vector
captured variance and restarted power-iteration spectral error, evaluated
with the device product kernels.

    captured_variance(A, Z)      ||A^T z_i||^2 per column   (metrics.py:136)
    spectral_error(A, Z)         ||A - Z Z^T A||_2 estimate  (metrics.py:102-122,
                                 spectral_norm_est / spectral_norm_max_restarts,
                                 factor.py:217-261)
    spectral_error_ratio(A, Z, sigma_k1), per_vector_errors(A, Z, sigma)

The estimator follows the reference step for step on the deflated operator
x -> (I - Z Z^T) A x (metrics.py:65-81): start v = SeededRng(seed).normal_fill(d)
normalised; w = op(v), est = ||w||, best = max(best, est); stop when
|est - prev| <= tol * est; v = op^T(w / est), normalised. The three seeded
starts (101, 202, 303) run batched as three columns of one block (one pass
over A per iteration serves all three); a start that meets its stopping rule
is frozen, so each column's result equals its own sequential run. At C2 one
iteration reads the 2 GB A twice (~0.8 ms), where the reference's CPU
estimator reads a 4 GB FP64 copy twice per start.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device as ops
from .krylov import rows_buffer
from .matrix import SeededRng

SPECTRAL_TOL = 1e-9           # metrics.py:36
SPECTRAL_MAX_ITERS = 20000    # metrics.py:37
RESTART_SEEDS = (101, 202, 303)  # metrics.py:38


def _operator(A, precision="auto"):
    """A device operator for A (an already-built DenseDeviceOp / CsrDeviceOp
    is used as is, so a sweep uploads its input once)."""
    from .operators import CsrDeviceOp, DenseDeviceOp
    from .rsvd import make_operator

    if isinstance(A, (DenseDeviceOp, CsrDeviceOp)):
        return A
    return make_operator(A, precision=precision)


def _as_device_z(Z, op):
    from .matrix import DenseMatrix

    z = Z.data if isinstance(Z, DenseMatrix) else Z
    if not isinstance(z, torch.Tensor):
        z = torch.from_numpy(np.ascontiguousarray(z))
    z = z.to(device=op.device)
    n, k = z.shape
    out = rows_buffer(n, k, op.dtype, op.device)
    out.copy_(z.to(op.dtype))
    return out


def captured_variance(A, Z, precision="auto"):
    """||A^T z_i||^2 for every column of Z (metrics.py:136), FP64 result."""
    op = _operator(A, precision)
    z = _as_device_z(Z, op)
    d = op.shape[1]
    W = torch.empty((d, z.shape[1]), dtype=torch.float64, device=op.device)
    op.apply_t(z, W)
    out = torch.empty(z.shape[1], dtype=torch.float64, device=op.device)
    ops.colreduce(W, True, out)
    return out.cpu().numpy()


class _Deflated:
    """x -> (I - Z Z^T) A x and its transpose (metrics.py:65-81)."""

    def __init__(self, op, z):
        self.op, self.z = op, z
        self.n, self.d = op.local_rows, op.shape[1]
        self.dtype, self.device = op.dtype, op.device

    def _project_off(self, y):
        c = torch.empty((self.z.shape[1], y.shape[1]), dtype=self.dtype, device=self.device)
        ops.gemm_tn(self.z, y, c)
        ops.gemm_nn(self.z, c, y, alpha=-1.0, beta=1.0)
        return y

    def apply(self, x):
        y = rows_buffer(self.n, x.shape[1], self.dtype, self.device)
        self.op.apply(x, y)
        return self._project_off(y)

    def apply_t(self, x):
        x = self._project_off(x.clone())
        out = rows_buffer(self.d, x.shape[1], self.dtype, self.device)
        self.op.apply_t(x, out)
        return out


def _colnorms(x):
    out = torch.empty(x.shape[1], dtype=torch.float64, device=x.device)
    ops.colreduce(x, True, out)
    return out.sqrt()


class _Plain:
    """x -> A x and its transpose: the estimator's operator interface over a
    device operator without deflation (spectral_norm_est on A itself)."""

    def __init__(self, op):
        self.op = op
        self.n, self.d = op.local_rows, op.shape[1]
        self.dtype, self.device = op.dtype, op.device

    def apply(self, x):
        y = rows_buffer(self.n, x.shape[1], self.dtype, self.device)
        return self.op.apply(x, y)

    def apply_t(self, x):
        out = rows_buffer(self.d, x.shape[1], self.dtype, self.device)
        return self.op.apply_t(x, out)


def spectral_norm_batched(defl, seeds=RESTART_SEEDS, tol=SPECTRAL_TOL, max_iters=SPECTRAL_MAX_ITERS, starts=None):
    """The reference's spectral_norm_est for each seed, batched as columns.
    Returns (best per seed, iterations per seed). ``starts``: d x m start
    vectors instead of SeededRng(seed).normal_fill(d) per seed."""
    if tol <= 0:
        raise ValueError("tol must be positive")
    d = defl.d
    V = np.stack([SeededRng(s).normal_fill(d) for s in seeds], axis=1) if starts is None else np.asarray(starts)
    m = V.shape[1]
    v = rows_buffer(d, m, defl.dtype, defl.device)
    v.copy_(torch.from_numpy(V).to(defl.device, defl.dtype))
    nv = _colnorms(v).cpu().numpy()
    best = np.zeros(m)
    prev = np.full(m, np.nan)
    active = nv > 0.0
    iters = np.zeros(m, dtype=np.int64)
    scale = torch.from_numpy(np.where(active, 1.0 / np.where(nv > 0, nv, 1.0), 0.0)).to(defl.device)
    v.mul_(scale.to(defl.dtype))
    for _ in range(int(max_iters)):
        if not active.any():
            break
        w = defl.apply(v)
        est = _colnorms(w).cpu().numpy()
        iters += active
        upd = active & (est > best)
        best[upd] = est[upd]
        zero = active & (est == 0.0)
        best[zero] = 0.0
        conv = active & ~np.isnan(prev) & (np.abs(est - prev) <= tol * est)
        active &= ~(zero | conv)
        prev = np.where(active, est, prev)
        if not active.any():
            break
        sc = torch.from_numpy(np.where(active, 1.0 / np.where(est > 0, est, 1.0), 0.0)).to(defl.device)
        v = defl.apply_t(w.mul_(sc.to(defl.dtype)))
        nv = _colnorms(v).cpu().numpy()
        active &= nv > 0.0
        sc = torch.from_numpy(np.where(active, 1.0 / np.where(nv > 0, nv, 1.0), 0.0)).to(defl.device)
        v.mul_(sc.to(defl.dtype))
    return best, iters


def spectral_error(A, Z, seeds=RESTART_SEEDS, tol=SPECTRAL_TOL, max_iters=SPECTRAL_MAX_ITERS, precision="auto"):
    """||A - Z Z^T A||_2 by the reference's restarted power estimate (max over
    the seeded starts, metrics.py:116-121)."""
    op = _operator(A, precision)
    best, _ = spectral_norm_batched(_Deflated(op, _as_device_z(Z, op)), seeds, tol, max_iters)
    return float(best.max())


def _sv(oracle):
    """Oracle singular values: the reference passes its SvdResult
    (``.singular_values``, factor.py:59-76); a plain descending array works too.
    Values past the oracle's rank read as 0 (metrics.py:50-52)."""
    return np.asarray(getattr(oracle, "singular_values", oracle), dtype=np.float64).reshape(-1)


def _ncols(Z):
    from .matrix import DenseMatrix

    z = Z.data if isinstance(Z, DenseMatrix) else Z
    return int(z.shape[1])


def spectral_error_ratio(A, Z, oracle, **kw):
    """metrics.py:102-122: ||A - Z Z^T A||_2 over sigma_{k+1}; 1.0 for exact
    rank. ``oracle``: the reference's oracle object / its singular values, or
    sigma_{k+1} itself as a scalar."""
    op = _operator(A, kw.get("precision", "auto"))
    check_orthonormal(Z, op.device)
    sigma_k1 = float(oracle) if np.isscalar(oracle) else _sig(_sv(oracle), _ncols(Z))
    if sigma_k1 == 0.0:
        return 1.0
    return spectral_error(op, Z, **kw) / sigma_k1


def per_vector_errors(A, Z, oracle, precision="auto"):
    """metrics.py:125-142: |sigma_i^2 - ||A^T z_i||^2| / sigma_{k+1}^2 against
    the oracle's singular values; absolute errors when sigma_{k+1} = 0."""
    op = _operator(A, precision)
    check_orthonormal(Z, op.device)
    cap = captured_variance(op, Z, precision)
    k = cap.shape[0]
    sigma = _sv(oracle)
    true_sq = np.array([_sig(sigma, i) ** 2 for i in range(k)])
    errs = np.abs(true_sq - cap)
    denom = _sig(sigma, k) ** 2
    return errs if denom == 0.0 else errs / denom


def error_function(A, Z, l, oracle, precision="auto"):
    """metrics.py:145-158: Frobenius shortfall of the rank-l prefix of Z against
    the optimal one, sum_{i<=l} sigma_i^2 - ||Z_l^T A||_F^2."""
    from .matrix import DenseMatrix

    z = Z.data if isinstance(Z, DenseMatrix) else Z
    if l > z.shape[1]:
        raise ValueError("l exceeds the number of columns of Z")
    if l == 0:
        return 0.0
    sigma = _sv(oracle)
    captured = float(np.sum(captured_variance(A, z[:, :l], precision)))
    return float(np.sum(np.array([_sig(sigma, i) ** 2 for i in range(l)]))) - captured


# ---------------------------------------------------------------------------
# the full error report (metrics.py:32-38, 65-99, 184-252): Frobenius ratio,
# spectral ratio, per-vector errors, against oracle singular values

Z_ORTHO_TOL = 1e-8        # metrics.py:38
EXACT_RANK_RTOL = 1e-14   # metrics.py:37


def frobenius_sq(A, precision="auto"):
    """||A||_F^2 in FP64 (MatrixOperator.frobenius_sq)."""
    op = _operator(A, precision)
    parts = [op.val.view(-1, 1)] if op.is_sparse else [op.A]
    if op.is_sparse and op.hot is not None:  # hybrid operator: cold CSR + dense hot panel
        parts.append(op.hot["panel"])
    total = 0.0
    for x in parts:
        if x.numel():
            cols = torch.empty(x.shape[1], dtype=torch.float64, device=op.device)
            ops.colreduce(x, True, cols)
            total += float(cols.sum().item())
    return total


def check_orthonormal(Z, device):
    """metrics.py:41-45: ValueError if max |Z^T Z - I| > 1e-8 (FP64 Gram of
    the FP64 Z, whatever precision the operator runs in)."""
    from .matrix import DenseMatrix

    z = Z.data if isinstance(Z, DenseMatrix) else Z
    if not isinstance(z, torch.Tensor):
        z = torch.from_numpy(np.ascontiguousarray(z))
    z = z.to(device=device, dtype=torch.float64).contiguous()
    g = ops.gram(z)
    err = float(ops.ortho_error(g).item())
    if err > Z_ORTHO_TOL:
        raise ValueError(f"Z is not orthonormal (max deviation {err:.3e})")


def _tail_sq(sigma, k):
    return float(np.sum(sigma[k:] ** 2)) if k < sigma.shape[0] else 0.0


def _sig(sigma, i):
    return float(sigma[i]) if i < sigma.shape[0] else 0.0


def frob_error_ratio(A, Z, sigma, precision="auto"):
    """metrics.py:84-99: ||A - Z Z^T A||_F / ||A - A_k||_F through
    ||A||_F^2 - ||Z^T A||_F^2; exact-rank inputs report 1.0."""
    op = _operator(A, precision)
    check_orthonormal(Z, op.device)
    z = _as_device_z(Z, op)
    sigma = _sv(sigma)
    k = z.shape[1]
    fro_sq = frobenius_sq(op)
    captured = float(np.sum(captured_variance(op, z)))
    num_sq = max(fro_sq - captured, 0.0)
    tail = _tail_sq(sigma, k)
    if np.sqrt(tail) < EXACT_RANK_RTOL * np.sqrt(fro_sq):
        return 1.0
    return float(np.sqrt(num_sq / tail))


@dataclass(frozen=True)
class AdditiveSpectralCheck:
    """metrics.py:160-168 -- outcome of the additive Frobenius-to-spectral
    transfer property."""

    passed: bool
    eta: float
    spectral_sq: float
    bound: float
    slack: float


def additive_spectral_check(A, B, k, oracle):
    """metrics.py:171-200: ||A - B||_2^2 <= sigma_{k+1}^2 + eta (+ 1e-8 sigma_1^2)
    with eta the Frobenius excess of B over the best rank-k error; B must have
    numerical rank at most k (1e-7 relative). Both spectral norms come from the
    desk-scale oracle SVD (computed on the GPU, factor.dense_svd_reference)."""
    from .factor import dense_svd_reference
    from .matrix import DenseMatrix, as_dense_array, as_operator

    op = as_operator(A)
    b = as_dense_array(as_operator(B).densify())
    sv_b = dense_svd_reference(DenseMatrix(b)).singular_values
    if len(sv_b) > k and sv_b[0] > 0 and sv_b[k] >= 1e-7 * sv_b[0]:
        raise ValueError(f"B has numerical rank above {k}")
    diff = op.densify().data - b
    sigma = _sv(oracle)
    eta = float(np.sum(diff ** 2)) - _tail_sq(sigma, k)
    diff_sv = dense_svd_reference(DenseMatrix(diff)).singular_values
    spectral_sq = float(diff_sv[0] ** 2) if len(diff_sv) else 0.0
    bound = _sig(sigma, k) ** 2 + eta + 1e-8 * _sig(sigma, 0) ** 2
    return AdditiveSpectralCheck(passed=spectral_sq <= bound, eta=eta, spectral_sq=spectral_sq, bound=bound,
                                 slack=bound - spectral_sq)


@dataclass(frozen=True)
class ErrorReport:
    """metrics.py:184-216 — the three measures for one run."""

    frob_ratio: float
    spectral_ratio: float
    per_vector: np.ndarray
    per_vector_max: float
    exact_rank: bool
    absolute_per_vector: bool
    k: int
    q: int | None = None
    variant: str | None = None
    seed: int | None = None

    def __post_init__(self):
        pv = np.array(self.per_vector, dtype=np.float64, copy=True)
        pv.setflags(write=False)
        object.__setattr__(self, "per_vector", pv)
        if self.per_vector_max != (float(np.max(pv)) if pv.size else 0.0):
            raise ValueError("per_vector_max must equal max(per_vector)")


def compute_error_report(A, Z, sigma, q=None, variant=None, seed=None, precision="auto"):
    """metrics.py:236-252 on the GPU, A uploaded once: frob and spectral
    ratios, per-vector errors against the oracle singular values `sigma`."""
    op = _operator(A, precision)
    check_orthonormal(Z, op.device)
    z = _as_device_z(Z, op)
    sigma = _sv(sigma)
    k = z.shape[1]
    pv = per_vector_errors(op, z, sigma)
    fro_sq = frobenius_sq(op)
    sk = _sig(sigma, k)
    spec = 1.0 if sk == 0.0 else spectral_error(op, z) / sk
    if variant is not None:
        variant = getattr(variant, "value", str(variant))
    return ErrorReport(
        frob_ratio=frob_error_ratio(op, Z, sigma),
        spectral_ratio=spec,
        per_vector=pv,
        per_vector_max=float(np.max(pv)) if pv.size else 0.0,
        exact_rank=bool(np.sqrt(_tail_sq(sigma, k)) < EXACT_RANK_RTOL * np.sqrt(fro_sq)),
        absolute_per_vector=sk == 0.0,
        k=k, q=q, variant=variant, seed=seed,
    )
