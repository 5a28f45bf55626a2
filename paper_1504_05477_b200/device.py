"""Device layer: torch CUDA tensors in, C-ABI kernel launches out.

torch provides device memory, the current stream and (for multi-GPU) the
NCCL communicator; every FLOP of the path runs in librsvd_b200.so. All calls
are stream-ordered on ``torch.cuda.current_stream()`` and never synchronise,
so a whole factorization can be captured in a CUDA graph.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import F32, F64, GEMM_AUTO, check

_TDT = {torch.float32: F32, torch.float64: F64}


def lib():
    return _lib.load()


def dcode(t):
    try:
        return _TDT[t.dtype]
    except KeyError:
        raise ValueError(f"unsupported dtype {t.dtype}") from None


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _ld(t):
    assert t.dim() == 2 and (t.stride(1) == 1 or t.shape[1] <= 1), "row-major 2-D tensor required"
    return max(t.stride(0), t.shape[1]) if t.shape[0] > 1 else max(t.shape[1], 1)


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


_BODY_STREAMS = {}
_WS_ALIAS = {}  # conditional-body stream -> the stream it was opened from


class cond_section:
    """``with cond_section(flag): ...`` — a device-decided section. Under CUDA
    graph capture the section becomes an IF node on ``*flag != 0`` (csrc/
    graph_cond.cu) and its launches go to the node's body; eagerly it runs
    inline (its kernels keep their own ``pred`` checks, so both behave the
    same). The section must not allocate memory (graph body restriction)."""

    def __init__(self, flag, enabled=True):
        self.flag = flag
        self.enabled = enabled
        self.body = None
        self.ctx = None

    def __enter__(self):
        if not self.enabled or not torch.cuda.is_current_stream_capturing():
            return self
        dev = self.flag.device
        body = _BODY_STREAMS.get(dev)
        if body is None:
            body = _BODY_STREAMS[dev] = torch.cuda.Stream(device=dev)
        opened = ctypes.c_int32(0)
        check(lib().rsvd_cond_begin(_stream(), _ptr(self.flag), ctypes.c_void_p(body.cuda_stream),
                                         ctypes.byref(opened)), "cond_begin")
        if opened.value:
            # the body's launches run in the parent stream's order: they share its workspace
            _WS_ALIAS[body.cuda_stream] = torch.cuda.current_stream(dev).cuda_stream
            self.body = body
            self.ctx = torch.cuda.stream(body)
            self.ctx.__enter__()
        return self

    def __exit__(self, *exc):
        if self.body is not None:
            self.ctx.__exit__(*exc)
            check(lib().rsvd_cond_end(ctypes.c_void_p(self.body.cuda_stream)), "cond_end")
            self.body = None
        return False


class _Workspace:
    """One growing scratch buffer per (device, stream). Safe because every
    user of a buffer runs in stream order on that stream (threads driving
    separate streams -- e.g. virtual row shards -- get separate buffers).

    Grow-only: a superseded buffer is kept referenced for the life of the
    process, never handed back to torch's caching allocator. A CUDA graph
    captured earlier (rsvd.GraphedFactorization, the public API's graph
    cache) has the old address baked into its kernel parameters; an eager
    call that grows the scratch in between must not let that memory be
    reused by live tensors before the next replay."""

    def __init__(self):
        self.buf = {}
        self.retired = []

    def get(self, nbytes, device):
        dev = torch.device(device)
        sp = torch.cuda.current_stream(dev).cuda_stream
        key = (dev.index, _WS_ALIAS.get(sp, sp))
        b = self.buf.get(key)
        if b is None or b.numel() < nbytes:
            if b is not None:
                self.retired.append(b)
            b = torch.empty(max(int(nbytes), 1 << 20), dtype=torch.uint8, device=device)
            self.buf[key] = b
        return b

    def reserve(self, nbytes, device):
        self.get(nbytes, device)


WS = _Workspace()


class SplitPlanes:
    """hi / lo split planes of an FP32 block as the B operand of the tcgen05
    3xTF32 TN products (rsvd_split_planes layout), with the identity of the
    block they currently describe. ``gemm_nn(..., emit=planes)`` fills them
    from the product's epilogue; ``gemm_tn(..., b_planes=planes)`` uses them
    when they describe its B (no k_split_b pass over B). One buffer per
    (device, stream), grown on demand (SplitPlanes.get)."""

    _cache = {}

    def __init__(self, nbytes, device):
        self.buf = torch.empty(int(nbytes), dtype=torch.uint8, device=device)
        self.key = None

    @classmethod
    def get(cls, rows, cols, device):
        dev = torch.device(device)
        sp = torch.cuda.current_stream(dev).cuda_stream
        k = (dev.index, _WS_ALIAS.get(sp, sp))
        need = int(lib().rsvd_split_planes_bytes(int(rows), int(cols)))
        cur = cls._cache.get(k)
        if cur is None or cur.buf.numel() < need:
            old = cur
            cur = cls._cache[k] = cls(need, dev)
            if old is not None:  # captured graphs may still point into the old buffer
                cur._retired = getattr(old, "_retired", []) + [old.buf]
        return cur

    @classmethod
    def peek(cls, device):
        """The current stream's buffer if one exists (no allocation)."""
        dev = torch.device(device)
        sp = torch.cuda.current_stream(dev).cuda_stream
        return cls._cache.get((dev.index, _WS_ALIAS.get(sp, sp)))

    @staticmethod
    def ident(t):
        return (t.data_ptr(), tuple(t.shape), t.stride(0))

    def describes(self, t):
        return self.key is not None and self.key == self.ident(t)

    def invalidate(self):
        self.key = None

    def split(self, B, pred=None):
        """Cut B's planes with the standalone kernel (device-predicated by ``pred``)."""
        K, N = B.shape
        check(lib().rsvd_split_planes(K, N, _ptr(B), _ld(B), _ptr(self.buf), self.buf.numel(), _ptr(pred), _stream()),
              "split_planes")
        self.key = self.ident(B)


def gemm_nn(A, B, C, alpha=1.0, beta=0.0, row_sub=None, algo=GEMM_AUTO, pred=None, emit=None):
    m, k = A.shape
    k2, n = B.shape
    assert k == k2 and C.shape == (m, n), (A.shape, B.shape, C.shape)
    assert A.dtype == B.dtype == C.dtype
    if emit is not None and A.dtype == torch.float32 and algo == GEMM_AUTO:
        # FP32 product that also leaves C's split planes behind (for a following TN
        # product with B = C). A device-predicated product (pred) leaves the planes
        # as they were when it is skipped: the caller orders its emits accordingly.
        done = ctypes.c_int32(0)
        check(lib().rsvd_gemm_nn_f32_emit(m, n, k, float(alpha), _ptr(A), _ld(A), _ptr(B), _ld(B), float(beta), _ptr(C),
                                          _ld(C), _ptr(row_sub), _ptr(emit.buf), emit.buf.numel(),
                                          ctypes.byref(done), _ptr(pred), _stream()), "gemm_nn_emit")
        emit.key = emit.ident(C) if done.value else None
        return C
    check(lib().rsvd_gemm_nn(dcode(A), m, n, k, float(alpha), _ptr(A), _ld(A), _ptr(B), _ld(B),
                             float(beta), _ptr(C), _ld(C), _ptr(row_sub), int(algo), _ptr(pred), _stream()),
          "gemm_nn")
    return C


def gemm_tn(A, B, C, alpha=1.0, beta=0.0, mu=None, colsum_b=None, algo=GEMM_AUTO, pred=None, b_planes=None):
    """C (k x n) = alpha (A^T B - mu colsum_b^T) + beta C, A m x k, B m x n.
    ``b_planes``: SplitPlanes that may describe B (then B is not read at all)."""
    m, k = A.shape
    m2, n = B.shape
    assert m == m2 and C.shape == (k, n), (A.shape, B.shape, C.shape)
    assert A.dtype == B.dtype
    L = lib()
    nbytes = L.rsvd_gemm_tn_ws_bytes(dcode(A), m, n, k, int(algo))
    ws = WS.get(nbytes, A.device)
    if (b_planes is not None and A.dtype == torch.float32 and algo == GEMM_AUTO and b_planes.describes(B)
            and L.rsvd_gemm_tn_f32_planes_ok(m, n, k, _ptr(A), _ld(A))):
        check(L.rsvd_gemm_tn_f32_planes(dcode(C), m, n, k, float(alpha), _ptr(A), _ld(A), _ptr(b_planes.buf),
                                        b_planes.buf.numel(), float(beta), _ptr(C), _ld(C), _ptr(mu), _ptr(colsum_b),
                                        _ptr(ws), ws.numel(), _ptr(pred), _stream()), "gemm_tn_planes")
        return C
    check(L.rsvd_gemm_tn(dcode(A), dcode(C), m, n, k, float(alpha), _ptr(A), _ld(A), _ptr(B), _ld(B),
                         float(beta), _ptr(C), _ld(C), _ptr(mu), _ptr(colsum_b), _ptr(ws), ws.numel(),
                         int(algo), _ptr(pred), _stream()), "gemm_tn")
    return C


class OzPlanes:
    """FP32 A cut once into signed base-256 digit planes (int8) + per-row exponents for
    the FP64-accurate int8 tensor-core products (csrc/gemm_oz.cu)."""

    def __init__(self, A):
        assert A.dtype == torch.float32 and A.dim() == 2 and A.stride(1) == 1
        n, d = A.shape
        L = lib()
        self.n, self.d = n, d
        self.planes = torch.empty(int(L.rsvd_oz_planes_bytes(n, d)), dtype=torch.int8, device=A.device)
        self.row_exp = torch.empty(n, dtype=torch.int32, device=A.device)
        self.refresh(A)

    def refresh(self, A):
        """Re-cut the planes from A (same shape), stream-ordered."""
        check(lib().rsvd_oz_prepare(self.n, self.d, _ptr(A), _ld(A), _ptr(self.planes), _ptr(self.row_exp),
                                    _stream()), "oz_prepare")
        return self

    def refresh_rows(self, A, r0, nr):
        """Re-cut rows [r0, r0 + nr) only (r0 a multiple of 32): a row panel of
        a matrix that is still being uploaded."""
        check(lib().rsvd_oz_prepare_rows(self.n, self.d, int(r0), int(nr), _ptr(A), _ld(A), _ptr(self.planes),
                                         _ptr(self.row_exp), _stream()), "oz_prepare_rows")
        return self


def oz_gemm(P, B, C, trans, alpha=1.0, beta=0.0, pred=None, reduced=False):
    """trans=0: C (n x p) = alpha A B + beta C; trans=1: C (d x p) = alpha A^T B
    + beta C; A given by its digit planes P, B and C FP64. ``reduced``: ~1e-10
    relative accuracy (10 digit-pair GEMMs instead of 20)."""
    assert B.dtype == torch.float64 and C.dtype == torch.float64
    p = B.shape[1]
    assert B.shape[0] == (P.n if trans else P.d) and C.shape == ((P.d if trans else P.n), p), (B.shape, C.shape)
    L = lib()
    nbytes = L.rsvd_oz_gemm_ws_bytes(int(trans), P.n, P.d, p)
    ws = WS.get(nbytes, B.device)
    check(L.rsvd_oz_gemm(int(trans) + (2 if reduced else 0), P.n, P.d, p, float(alpha), _ptr(P.planes), _ptr(P.row_exp),
                         _ptr(B), _ld(B), float(beta), _ptr(C), _ld(C), _ptr(ws), ws.numel(), _ptr(pred),
                         _stream()), "oz_gemm")
    return C


class OzBasis:
    """Digit planes of an orthonormal FP64 basis Q (n x w) for FP64-accurate
    int8 tensor-core projections against its final prefix Q[:, :jp]
    (csrc/gemm_oz.cu). Blocks are sliced in as they become final."""

    def __init__(self, n, w, device):
        L = lib()
        self.n, self.w = n, w
        self.rows_alloc = -(-n // 128) * 128
        self.cols_alloc = -(-w // 128) * 128
        self.nplanes = int(L.rsvd_oz_basis_planes())
        self.planes = torch.zeros(int(L.rsvd_oz_basis_bytes(n, w)), dtype=torch.int8, device=device)
        self.col_exp = torch.zeros(w, dtype=torch.int32, device=device)

    def slice(self, Q, c0, ncols):
        """Digit planes of Q[:, c0:c0 + ncols] (Q = the full n x w basis)."""
        assert Q.dtype == torch.float64 and Q.shape == (self.n, self.w)
        L = lib()
        ws = WS.get(L.rsvd_oz_basis_ws_bytes(int(ncols)), Q.device)
        check(L.rsvd_oz_basis_slice(self.n, self.w, _ptr(Q), _ld(Q), int(c0), int(ncols), _ptr(self.planes),
                                    _ptr(self.col_exp), _ptr(ws), ws.numel(), _stream()), "oz_basis_slice")

    def gemm(self, trans, jp, B, C, alpha=1.0, beta=0.0, pred=None):
        """trans=1: C (jp x p) = alpha Q_p^T B + beta C (B n x p);
        trans=0: C (n x p) = alpha Q_p B + beta C (B jp x p); Q_p = Q[:, :jp]."""
        p = B.shape[1]
        L = lib()
        nbytes = L.rsvd_oz_gemm_ws_bytes(int(trans), self.n, int(jp), p)
        ws = WS.get(nbytes, B.device)
        check(L.rsvd_oz_gemm_planes(int(trans), self.n, int(jp), p, float(alpha), _ptr(self.planes), self.nplanes,
                                    self.rows_alloc, self.cols_alloc, _ptr(self.col_exp), 1, _ptr(B), _ld(B),
                                    float(beta), _ptr(C), _ld(C), _ptr(ws), ws.numel(), _ptr(pred), _stream()),
              "oz_gemm_planes")
        return C


def gram(V, out=None, algo=GEMM_AUTO, pred=None, b_planes=None):
    """FP64 Gram V^T V."""
    p = V.shape[1]
    if out is None:
        out = torch.empty((p, p), dtype=torch.float64, device=V.device)
    return gemm_tn(V, V, out, algo=algo, pred=pred, b_planes=b_planes)


def colreduce(X, square=True, out=None):
    n, p = X.shape
    if out is None:
        out = torch.empty(p, dtype=torch.float64, device=X.device)
    L = lib()
    ws = WS.get(L.rsvd_colreduce_ws_bytes(n, p), X.device)
    check(L.rsvd_colreduce(dcode(X), 1 if square else 0, n, p, _ptr(X), _ld(X), _ptr(out), _ptr(ws),
                           ws.numel(), _stream()), "colreduce")
    return out


def chol_deflate(G, ref2, tau2, T, mask, ndef, running=None, active=None, pred=None):
    p = G.shape[0]
    L = lib()
    ws = WS.get(L.rsvd_chol_deflate_ws_bytes(p), G.device)
    check(L.rsvd_chol_deflate(p, _ptr(G), _ld(G), _ptr(ref2), float(tau2), _ptr(T), _ld(T), _ptr(mask),
                              _ptr(ndef), _ptr(running), _ptr(active), _ptr(ws), ws.numel(), _ptr(pred),
                              _stream()), "chol_deflate")


def mask_cols(X, keep, pred=None):
    n, p = X.shape
    check(lib().rsvd_mask_cols(dcode(X), n, p, _ptr(X), _ld(X), _ptr(keep), _ptr(pred), _stream()), "mask_cols")
    return X


def insert_fill(X, mask, ndef, seed, row_offset=0, n_total=None, pred=None):
    n, p = X.shape
    n_total = n if n_total is None else int(n_total)
    check(lib().rsvd_insert_fill(dcode(X), n, p, _ptr(X), _ld(X), _ptr(mask), _ptr(ndef),
                                 ctypes.c_uint64(int(seed)), int(row_offset), n_total, _ptr(pred), _stream()),
          "insert_fill")


def fill_stream(n, nvec, seed, device):
    out = torch.empty((nvec, n), dtype=torch.float64, device=device)
    check(lib().rsvd_fill_stream(n, nvec, ctypes.c_uint64(int(seed)), _ptr(out), _stream()), "fill_stream")
    return out


def jacobi_sweeps(M, V, tol, max_sweeps, info=None, off=None):
    """In place on M (diagonalised) and V (accumulated rotations).
    Returns device tensors (info[int32: converged, sweeps, _], off[f64])."""
    n = M.shape[0]
    if info is None:
        info = torch.zeros(4, dtype=torch.int32, device=M.device)
    if off is None:
        off = torch.zeros(1, dtype=torch.float64, device=M.device)
    L = lib()
    ws = WS.get(L.rsvd_jacobi_ws_bytes(n), M.device)
    check(L.rsvd_jacobi_sweeps(n, _ptr(M), _ld(M), _ptr(V), _ld(V), float(tol), int(max_sweeps), _ptr(info),
                               _ptr(off), _ptr(ws), ws.numel(), _stream()), "jacobi_sweeps")
    return info, off


def eig_select(M, V, k, evals=None, evecs=None):
    w = M.shape[0]
    if evals is None:
        evals = torch.empty(k, dtype=torch.float64, device=M.device)
    if evecs is None:
        evecs = torch.empty((w, k), dtype=torch.float64, device=M.device)
    order = torch.empty(max(k, 1), dtype=torch.int32, device=M.device)
    check(lib().rsvd_eig_select(w, _ptr(M), _ld(M), _ptr(V), _ld(V), k, _ptr(evals), _ptr(evecs),
                                _ld(evecs) if k > 0 else 1, _ptr(order), _stream()), "eig_select")
    return evals, evecs


def syev_topk(M, k, evals=None, evecs=None, info=None, values_only=False):
    """Top-k eigenpairs of symmetric M (descending). Returns device tensors
    (evals[k], evecs[w x k] or None with values_only, info[int32: ok, _])."""
    w = M.shape[0]
    if evals is None:
        evals = torch.empty(k, dtype=torch.float64, device=M.device)
    if evecs is None and not values_only:
        evecs = torch.empty((w, k), dtype=torch.float64, device=M.device)
    if info is None:
        info = torch.zeros(4, dtype=torch.int32, device=M.device)
    L = lib()
    ws = WS.get(L.rsvd_syev_topk_ws_bytes(w, k), M.device)
    check(L.rsvd_syev_topk(w, _ptr(M), _ld(M), k, _ptr(evals), _ptr(evecs), k if evecs is None else _ld(evecs),
                           _ptr(info), _ptr(ws),
                           ws.numel(), _stream()), "syev_topk")
    return evals, evecs, info


def canonicalize_signs(X):
    n, k = X.shape
    L = lib()
    ws = WS.get(L.rsvd_colreduce_ws_bytes(n, k), X.device)
    check(L.rsvd_canonicalize_signs(dcode(X), n, k, _ptr(X), _ld(X), _ptr(ws), ws.numel(), _stream()),
          "canonicalize_signs")
    return X


def col_absargmax(X, row_offset=0):
    n, k = X.shape
    val = torch.empty(k, dtype=torch.float64, device=X.device)
    idx = torch.empty(k, dtype=torch.int64, device=X.device)
    L = lib()
    ws = WS.get(L.rsvd_colreduce_ws_bytes(max(n, 1), k), X.device)
    check(L.rsvd_col_absargmax(dcode(X), n, k, _ptr(X), _ld(X), int(row_offset), _ptr(val), _ptr(idx),
                               _ptr(ws), ws.numel(), _stream()), "col_absargmax")
    return val, idx


def flip_by_sign(X, sign_val):
    n, k = X.shape
    check(lib().rsvd_flip_by_sign(dcode(X), n, k, _ptr(X), _ld(X), _ptr(sign_val), _stream()), "flip_by_sign")
    return X


def convert(src, dst, pred=None):
    assert src.shape == dst.shape
    r, c = src.shape
    check(lib().rsvd_convert(dcode(src), dcode(dst), r, c, _ptr(src), _ld(src), _ptr(dst), _ld(dst), _ptr(pred),
                             _stream()), "convert")
    return dst


def gather_rows(idx, src, dst):
    """dst[i, :] = src[idx[i], :] (idx int64 on the device)."""
    check(lib().rsvd_gather_rows(dcode(src), idx.numel(), src.shape[1], _ptr(idx), _ptr(src), _ld(src), _ptr(dst),
                                 _ld(dst), _stream()), "gather_rows")
    return dst


def scatter_rows(idx, src, dst):
    """dst[idx[i], :] = src[i, :]."""
    check(lib().rsvd_scatter_rows(dcode(src), idx.numel(), src.shape[1], _ptr(idx), _ptr(src), _ld(src), _ptr(dst),
                                  _ld(dst), _stream()), "scatter_rows")
    return dst


def sqrt_clip(x, out=None):
    if out is None:
        out = torch.empty_like(x)
    check(lib().rsvd_sqrt_clip(x.numel(), _ptr(x), _ptr(out), _stream()), "sqrt_clip")
    return out


def ortho_error(G, out=None):
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=G.device)
    check(lib().rsvd_ortho_error(G.shape[0], _ptr(G), _ld(G), _ptr(out), _stream()), "ortho_error")
    return out


def spmm_csr(indptr, col, val, ncols, B, C, alpha=1.0, beta=0.0):
    nrows = indptr.numel() - 1
    idx64 = 1 if indptr.dtype == torch.int64 else 0
    assert col.dtype == indptr.dtype and val.dtype == B.dtype == C.dtype
    nb = B.shape[1]
    check(lib().rsvd_spmm_csr(dcode(val), idx64, nrows, ncols, nb, _ptr(indptr), _ptr(col), _ptr(val),
                              _ptr(B), _ld(B), float(alpha), float(beta), _ptr(C), _ld(C), _stream()),
          "spmm_csr")
    return C


class SpmmPlan:
    """Row-split plan of a CSR matrix for rsvd_spmm_csr_plan (built once per
    operator): rows longer than `chunk` nonzeros are cut into chunks whose
    partial sums are added in chunk order."""

    def __init__(self, indptr, chunk=512):
        dev = indptr.device
        n = indptr.numel() - 1
        ip = indptr.to(torch.int64)
        lens = ip[1:] - ip[:-1]
        nch = torch.clamp((lens + chunk - 1) // chunk, min=1)  # an empty row still writes beta * C
        total = int(nch.sum())  # host sync: plan construction is setup, not the hot loop
        crow = torch.repeat_interleave(torch.arange(n, device=dev), nch)
        first = torch.cumsum(nch, 0) - nch
        k_in_row = torch.arange(total, device=dev) - first[crow]
        self.lo = (ip[crow] + k_in_row * chunk).contiguous()
        self.hi = torch.minimum(self.lo + chunk, ip[crow + 1]).contiguous()
        self.row = crow.to(torch.int32).contiguous()
        split = nch > 1
        split_chunk = split[crow]
        nslots = int(split_chunk.sum())
        self.slot = torch.full((total,), -1, dtype=torch.int32, device=dev)
        self.slot[split_chunk] = torch.arange(nslots, dtype=torch.int32, device=dev)
        self.split_row = torch.nonzero(split).flatten().to(torch.int32).contiguous()
        counts = nch[split]
        self.split_beg = torch.zeros(self.split_row.numel() + 1, dtype=torch.int64, device=dev)
        self.split_beg[1:] = torch.cumsum(counts, 0)
        self.nchunks, self.nsplit, self.nslots, self.nrows = total, self.split_row.numel(), nslots, n


def spmm_csr_plan(plan, col, val, B, C, alpha=1.0, beta=0.0):
    """C = alpha A B + beta C through the load-balanced kernel (rsvd_spmm_csr_plan)."""
    idx64 = 1 if col.dtype == torch.int64 else 0
    assert val.dtype == B.dtype == C.dtype
    nb = B.shape[1]
    ws = WS.get(max(1, plan.nslots * min(nb, 256) * B.element_size()), B.device) if plan.nsplit else None
    check(lib().rsvd_spmm_csr_plan(dcode(val), idx64, plan.nrows, nb, _ptr(col), _ptr(val), _ptr(B), _ld(B),
                                   float(alpha), float(beta), _ptr(C), _ld(C), plan.nchunks, _ptr(plan.lo),
                                   _ptr(plan.hi), _ptr(plan.row), _ptr(plan.slot), plan.nsplit, _ptr(plan.split_row),
                                   _ptr(plan.split_beg), _ptr(ws), 0 if ws is None else ws.numel(), _stream()),
          "spmm_csr_plan")
    return C


class SpmmNnzPlan:
    """Nonzero-balanced plan of a CSR matrix for rsvd_spmm_nnz_plan (built
    once per operator): work units of `chunk` consecutive nonzeros; a row cut
    by a unit boundary gets one workspace slot per unit it touches (consecutive
    slot numbers), summed in order afterwards."""

    CHUNK = int(__import__("os").environ.get("RSVD_SPMM_CHUNK", "1024"))

    def __init__(self, indptr, chunk=None):
        chunk = int(chunk or self.CHUNK)
        dev = indptr.device
        ip = indptr.to(torch.int64)
        n = ip.numel() - 1
        nnz = int(ip[-1])  # host sync: plan construction is setup, not the hot loop
        lens = ip[1:] - ip[:-1]
        self.chunk, self.nnz, self.nrows = chunk, nnz, n
        self.rowid = torch.repeat_interleave(torch.arange(n, device=dev, dtype=torch.int32), lens).contiguous()
        nch = -(-nnz // chunk)
        e0 = torch.arange(nch, device=dev, dtype=torch.int64) * chunk
        e1 = torch.clamp(e0 + chunk, max=nnz)
        if nch:
            fr = self.rowid[e0].to(torch.int64)
            lr = self.rowid[e1 - 1].to(torch.int64)
            head = (ip[fr] < e0) | (ip[fr + 1] > e1)
            tail = (lr != fr) & (ip[lr + 1] > e1)
            flags = torch.stack([head, tail], 1).flatten()
            ids = torch.cumsum(flags.to(torch.int64), 0) - 1
            slot = torch.where(flags, ids, torch.full_like(ids, -1)).to(torch.int32).view(nch, 2)
            self.head_slot = slot[:, 0].contiguous()
            self.tail_slot = slot[:, 1].contiguous()
            prow = torch.stack([fr, lr], 1).flatten()[flags]
            self.nslots = int(prow.numel())
            srow, counts = torch.unique_consecutive(prow, return_counts=True)
            self.split_row = srow.to(torch.int32).contiguous()
            self.split_beg = torch.zeros(srow.numel() + 1, dtype=torch.int64, device=dev)
            self.split_beg[1:] = torch.cumsum(counts, 0)
        else:
            self.head_slot = self.tail_slot = torch.empty(0, dtype=torch.int32, device=dev)
            self.split_row = torch.empty(0, dtype=torch.int32, device=dev)
            self.split_beg = torch.zeros(1, dtype=torch.int64, device=dev)
            self.nslots = 0
        self.nsplit = int(self.split_row.numel())
        self.empty_rows = torch.nonzero(lens == 0).flatten().to(torch.int32).contiguous()

    @staticmethod
    def eligible(col, val, B, C):
        nb = B.shape[1]
        return (val.dtype == torch.float32 and col.dtype == torch.int32 and B.dtype == C.dtype == torch.float32
                and nb <= 128 and nb % 4 == 0 and _ld(B) % 4 == 0 and _ld(C) % 4 == 0
                and B.data_ptr() % 16 == 0 and C.data_ptr() % 16 == 0)


def spmm_nnz_plan(plan, col, val, B, C, alpha=1.0, beta=0.0):
    """C = alpha A B + beta C through the nonzero-balanced kernel (rsvd_spmm_nnz_plan)."""
    nb = B.shape[1]
    ws = WS.get(max(16, plan.nslots * nb * 4), B.device) if plan.nslots else None
    check(lib().rsvd_spmm_nnz_plan(plan.nnz, plan.chunk, nb, _ptr(col), _ptr(val), _ptr(plan.rowid), _ptr(B), _ld(B),
                                   float(alpha), float(beta), _ptr(C), _ld(C), _ptr(plan.head_slot),
                                   _ptr(plan.tail_slot), plan.nsplit, _ptr(plan.split_row), _ptr(plan.split_beg),
                                   plan.empty_rows.numel(), _ptr(plan.empty_rows), _ptr(ws),
                                   0 if ws is None else ws.numel(), _stream()), "spmm_nnz_plan")
    return C


def spmm_slab(slab, X, C):
    """C += A_slab X (slab = dict(ptr, idx, val, cols): the slab tier of the hybrid CSR product)."""
    assert X.dtype == C.dtype == torch.float32
    nrows = slab["ptr"].numel() - 1
    check(lib().rsvd_spmm_slab(nrows, X.shape[1], _ptr(slab["ptr"]), _ptr(slab["idx"]), _ptr(slab["val"]),
                               _ptr(slab["cols"]), slab["cols"].numel(), _ptr(X), _ld(X), _ptr(C), _ld(C),
                               _stream()), "spmm_slab")
    return C


def csr_transpose(indptr, col, val, nrows, ncols):
    """Device CSR of A^T (stable in row order). The stable column sort that
    orders the nonzeros is torch plumbing done once per operator."""
    nnz = col.numel()
    perm = torch.sort(col.to(torch.int64), stable=True).indices
    tptr = torch.empty(ncols + 1, dtype=indptr.dtype, device=col.device)
    tcol = torch.empty(nnz, dtype=col.dtype, device=col.device)
    tval = torch.empty(nnz, dtype=val.dtype, device=col.device)
    idx64 = 1 if indptr.dtype == torch.int64 else 0
    check(lib().rsvd_csr_transpose(dcode(val), idx64, nrows, ncols, nnz, _ptr(indptr), _ptr(col), _ptr(val),
                                   _ptr(perm), _ptr(tptr), _ptr(tcol), _ptr(tval), _stream()), "csr_transpose")
    return tptr, tcol, tval


def gauss_fill_host(count, state):
    """Host Gaussian stream through the C ABI (bit-identical to the reference)."""
    import numpy as np

    out = np.empty(int(count), dtype=np.float64)
    new = ctypes.c_uint64(0)
    check(lib().rsvd_gauss_fill(int(count), ctypes.c_uint64(int(state) & ((1 << 64) - 1)),
                                out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(new)), "gauss_fill")
    return out, int(new.value)
