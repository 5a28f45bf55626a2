"""TEST DOUBLE: a torch-CPU FP64 implementation of the device-op interface
that krylov.py drives (paper_1504_05477_b200/device.py). Used only by the CPU
tests to exercise the orchestration and the row-sharded (gloo) logic without
a GPU. The product never imports it."""

import numpy as np
import torch

import rsvd_oracle as o

_G = 0x9E3779B97F4A7C15
_M = (1 << 64) - 1


def _off(pred):
    return pred is not None and int(pred.reshape(-1)[0]) == 0


class SplitPlanes:
    """CPU double of device.SplitPlanes: no planes, nothing ever described."""

    @classmethod
    def get(cls, rows, cols, device):
        return cls()

    @classmethod
    def peek(cls, device):
        return None

    def describes(self, t):
        return False

    def invalidate(self):
        pass

    def split(self, B, pred=None):
        pass


def gemm_nn(A, B, C, alpha=1.0, beta=0.0, row_sub=None, algo=0, pred=None, emit=None):
    if _off(pred):
        return C
    r = A.double() @ B.double()
    if row_sub is not None:
        r = r - row_sub.view(1, -1)
    r = alpha * r
    if beta != 0.0:
        r = r + beta * C.double()
    C.copy_(r.to(C.dtype))
    return C


def gemm_tn(A, B, C, alpha=1.0, beta=0.0, mu=None, colsum_b=None, algo=0, pred=None, b_planes=None):
    if _off(pred):
        return C
    r = A.double().T @ B.double()
    if mu is not None:
        r = r - mu.view(-1, 1) * colsum_b.view(1, -1)
    r = alpha * r
    if beta != 0.0:
        r = r + beta * C.double()
    C.copy_(r.to(C.dtype))
    return C


def gram(V, out=None, algo=0, pred=None, b_planes=None):
    if out is None:
        out = torch.empty((V.shape[1], V.shape[1]), dtype=torch.float64)
    return gemm_tn(V, V, out, pred=pred)


def colreduce(X, square=True, out=None):
    r = (X.double() ** 2).sum(0) if square else X.double().sum(0)
    if out is None:
        return r
    out.copy_(r)
    return out


def mask_cols(X, keep, pred=None):
    if _off(pred):
        return X
    X[:, keep == 0] = 0
    return X


def chol_deflate(G, ref2, tau2, T, mask, ndef, running=None, active=None, pred=None):
    if _off(pred):
        return
    g = G.numpy().copy()
    p = g.shape[0]
    S = np.triu(g)
    R = np.zeros((p, p))
    m = np.zeros(p, dtype=np.int32)
    orig = np.diag(g).copy()
    for j in range(p):
        d = S[j, j]
        r = ref2[j].item() if ref2 is not None else orig[j]
        act = int(active[j]) if active is not None else 1
        if not act or not (d > tau2 * r) or not (d > 0):
            m[j] = 1 if act else 2
            R[j, j] = 1.0
            continue
        rjj = np.sqrt(d)
        R[j, j] = rjj
        R[j, j + 1:] = S[j, j + 1:] / rjj
        S[j + 1:, j + 1:] -= np.outer(R[j, j + 1:], R[j, j + 1:])
    Tn = np.linalg.inv(R)
    Tn = np.triu(Tn)
    for j in np.nonzero(m)[0]:
        Tn[:, j] = 0
        Tn[j, :] = 0
    m[m == 2] = 0
    T.copy_(torch.from_numpy(Tn))
    mask.copy_(torch.from_numpy(m))
    base = int(running[0]) if running is not None else 0
    ndef[0] = int(m.sum())
    ndef[1] = base
    if running is not None:
        running[0] = base + int(m.sum())


def insert_fill(X, mask, ndef, seed, row_offset=0, n_total=None, pred=None):
    if _off(pred):
        return
    n, p = X.shape
    n_total = n if n_total is None else n_total
    if int(ndef[0]) == 0:
        return
    rank = int(ndef[1])
    for j in range(p):
        if int(mask[j]):
            state = (seed + 2 * ((n_total + 1) // 2) * rank * _G) & _M
            vec, _ = o.gauss_fill(n_total, state)
            X[:, j] = torch.from_numpy(vec[row_offset: row_offset + n]).to(X.dtype)
            rank += 1


def jacobi_sweeps(M, V, tol, max_sweeps, info=None, off=None):
    m = np.ascontiguousarray(M.numpy())
    v = np.ascontiguousarray(V.numpy())
    offv, sweeps, conv = o.jacobi_sweeps(m, v, tol, max_sweeps)
    M.copy_(torch.from_numpy(m))
    V.copy_(torch.from_numpy(v))
    return torch.tensor([int(conv), sweeps, 0, 0], dtype=torch.int32), torch.tensor([offv])


def syev_topk(M, k, evals=None, evecs=None, info=None):
    vals, vecs = o.symmetric_eig(M.numpy())
    return (torch.from_numpy(vals[:k].copy()), torch.from_numpy(np.ascontiguousarray(vecs[:, :k])),
            torch.tensor([1, 0, 0, 0], dtype=torch.int32))


def eig_select(M, V, k, evals=None, evecs=None):
    d = torch.diagonal(M).numpy()
    order = np.argsort(-d, kind="stable")[:k]
    return torch.from_numpy(d[order].copy()), V[:, torch.from_numpy(order)].clone()


def canonicalize_signs(X):
    x = X.numpy()
    o.canonicalize_signs(x)
    return X


def col_absargmax(X, row_offset=0):
    n, k = X.shape
    if n == 0:
        return torch.zeros(k, dtype=torch.float64), torch.full((k,), np.iinfo(np.int64).max, dtype=torch.int64)
    idx = torch.from_numpy(np.argmax(np.abs(X.numpy()), axis=0))
    val = X.gather(0, idx.view(1, -1)).view(-1).double()
    return val, idx + row_offset


def flip_by_sign(X, sign_val):
    X[:, sign_val < 0] *= -1
    return X


def convert(src, dst, pred=None):
    if _off(pred):
        return dst
    dst.copy_(src.to(dst.dtype))
    return dst


def sqrt_clip(x, out=None):
    r = torch.sqrt(torch.clamp(x, min=0.0))
    if out is None:
        return r
    out.copy_(r)
    return out


def ortho_error(G, out=None):
    e = (G - torch.eye(G.shape[0], dtype=G.dtype)).abs().max().view(1)
    if out is not None:
        out.copy_(e)
        return out
    return e


class CpuDenseOp:
    def __init__(self, A, n_total=None, row_offset=0, mu=None):
        self.A = A
        self.local_rows = A.shape[0]
        self.n_total = A.shape[0] if n_total is None else n_total
        self.row_offset = row_offset
        self.shape = (self.n_total, A.shape[1])
        self.dtype = A.dtype
        self.device = A.device
        self.mu = mu

    def apply(self, X, out):
        rs = None
        if self.mu is not None:
            rs = (self.mu.view(1, -1) @ X.double()).view(-1)
        return gemm_nn(self.A, X.to(self.A.dtype), out, row_sub=rs)

    def apply_t(self, Y, out):
        cs = Y.double().sum(0) if self.mu is not None else None
        return gemm_tn(self.A, Y.to(self.A.dtype), out, mu=self.mu, colsum_b=cs)


class cond_section:
    """No graph capture on the CPU path: the section runs inline (its ops keep
    their own predicates), as device.cond_section does outside capture."""

    def __init__(self, flag, enabled=True):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False
