"""Device orchestration of the north_star path: Krylov chain, blocked
orthonormalization, Rayleigh-Ritz.

Reference call stack (rsvd.py:263-290):
    _run -> _bk_basis / _si_basis / _sketch_basis (rsvd.py:224-260)
         -> _mgs per block and on hstack(blocks) (factor.py:79-118)
         -> post_process (rsvd.py:200-221) -> symmetric_eig (factor.py:132-166)

B200 restructuring:
  * every n-side block (Y, b_j, Q, Z) lives in HBM in the work precision;
    A is read in place for both A X and A^T Y (no cached A^T copy,
    matrix.py:245-247);
  * _mgs's column loop (BLAS-2, factor.py:100-117) becomes a blocked
    BCGS2 + CholeskyQR2 with deficiency deflation (``orth_block``): GEMMs
    for the projections, an FP64 Gram, a single-CTA column-ordered Cholesky
    that applies the reference's "residual small relative to the column's
    original norm" test and replaces deficient columns from the reference's
    fill stream, generated on the device;
  * post_process's two passes over A at width w (rsvd.py:216) become one:
    W = A^T Q, M = W^T W (the same matrix, Q^T A A^T Q);
  * nothing here synchronises with the host; the whole call is one stream.

Row sharding (multi-GPU): every reduction over the row dimension n (A^T Y,
Grams, projections Q^T V, W = A^T Q, column sums) is followed by
``comm.allreduce``; small matrices are replicated and computed identically
on every rank (deterministic kernels => identical decisions).
"""

from __future__ import annotations

import os

import torch

QR_FILL_SEED = 0x5EED_F111_0C0F_FEE5  # factor.py:40
JACOBI_TOL = 1e-14  # factor.py:34
JACOBI_MAX_SWEEPS = 50  # factor.py:35
# Deflation thresholds on the residual norm relative to the original column
# norm (the reference's is 1e-12 on exact CGS2 residuals, factor.py:41,105;
# a Gram-based test cannot resolve below ~sqrt(eps)).
TAU = {torch.float64: 1e-7, torch.float32: 3e-3}
# Blocks without a prefix (the Gram's diagonal is the reference): round 1
# rejects a column whose Cholesky pivot is below PIVOT_NOISE x its squared norm
# -- the pivot carries ~p eps of that norm in rounding, more for an
# ill-conditioned leading block, so a smaller one is noise, not a residual, and
# goes to round 2's explicit test (raw power blocks of rank-deficient inputs: a
# dependent column accepted on a garbage pivot left Q orthonormal only to 5e-6).
PIVOT_NOISE = {torch.float64: 1e-12, torch.float32: 0.0}
REF_RTOL = 1e-12  # factor.py:41 (_DEFICIENCY_RTOL)
# Second-round threshold per work precision: the reference's own 1e-12 in
# FP64; in FP32 the explicit residuals are resolved only down to ~1e-7, and a
# kept noisy direction perturbs Ritz values only quadratically while a
# dropped one perturbs them to first order, so keep down to the noise floor.
REF_RTOL_BY = {torch.float64: REF_RTOL, torch.float32: 1e-7}


class LocalComm:
    """Single device: reductions are complete already."""

    world = 1
    rank = 0

    def allreduce(self, t):
        return t

    def row_range(self, n):
        return 0, n


class TorchComm:
    """Row-sharded ranks over torch.distributed (NCCL on GPUs, gloo in the
    CPU tests). Sum-allreduce in place on the launching stream."""

    def __init__(self, group=None, n_total=None, row_offset=0):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n_total = n_total
        self.row_offset = row_offset
        # gloo with CUDA tensors (the CPU tests; bench.py's RSVD_DIST_BACKEND=gloo
        # check of the N > 1 path on one GPU): stage through host memory
        self.host_staged = dist.get_backend(group) == "gloo"

    def allreduce(self, t):
        if self.host_staged and t.is_cuda:
            tmp = t.cpu()
            self.dist.all_reduce(tmp, group=self.group)
            t.copy_(tmp)
        elif t.is_contiguous():
            self.dist.all_reduce(t, group=self.group)
        else:  # padded row buffers (krylov.rows_buffer)
            tmp = t.contiguous()
            self.dist.all_reduce(tmp, group=self.group)
            t.copy_(tmp)
        return t

    def all_gather(self, t):
        if self.host_staged and t.is_cuda:
            src = t.cpu()
            out = [torch.empty_like(src) for _ in range(self.world)]
            self.dist.all_gather(out, src, group=self.group)
            return [o.to(t.device) for o in out]
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return out


class HandleComm:
    """The C ABI's own communicator (include/rsvd_b200.h section 8): a per-device
    rsvd_handle carrying an injected / library-built NCCL communicator;
    allreduce is rsvd_handle_allreduce_sum on the current stream. all_gather
    (the sharded sign choice) is a sum-allreduce of zero-padded rank slots.
    ``unique_id`` (128 bytes, from ``nccl_unique_id()`` on one rank and
    distributed by the caller) builds the communicator; ``from_torch`` does
    that over an existing torch.distributed group."""

    def __init__(self, device, world=1, rank=0, unique_id=None, n_total=None, row_offset=0):
        import ctypes

        from . import _lib

        self._L = _lib.load()
        self._ct = ctypes
        h = ctypes.c_void_p()
        _lib.check(self._L.rsvd_handle_create(int(torch.device(device).index or 0), ctypes.byref(h)), "handle_create")
        self.h = h
        if unique_id is not None:
            buf = ctypes.create_string_buffer(bytes(unique_id), 128)
            _lib.check(self._L.rsvd_handle_init_comm(h, buf, 128, int(world), int(rank)), "handle_init_comm")
        self.world, self.rank = int(world), int(rank)
        self.n_total, self.row_offset = n_total, row_offset

    @staticmethod
    def nccl_unique_id():
        import ctypes

        from . import _lib

        buf = ctypes.create_string_buffer(128)
        _lib.check(_lib.load().rsvd_nccl_unique_id(buf, 128), "nccl_unique_id")
        return buf.raw

    @classmethod
    def from_torch(cls, device, group=None, n_total=None, row_offset=0):
        import torch.distributed as dist

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        obj = [cls.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(device, world, rank, obj[0], n_total=n_total, row_offset=row_offset)

    def allreduce(self, t):
        from . import _lib
        from .device import dcode

        buf = t if t.is_contiguous() else t.contiguous()
        _lib.check(self._L.rsvd_handle_allreduce_sum(self.h, self._ct.c_void_p(buf.data_ptr()), buf.numel(),
                                                     dcode(buf), self._ct.c_void_p(
                                                         torch.cuda.current_stream(buf.device).cuda_stream)),
                   "handle_allreduce_sum")
        if buf is not t:
            t.copy_(buf)
        return t

    def all_gather(self, t):
        slots = torch.zeros((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        slots[self.rank] = t
        if t.dtype in (torch.float32, torch.float64):
            self.allreduce(slots)
        else:  # indices: exact through FP64 (|i| < 2^53)
            f = slots.double()
            self.allreduce(f)
            slots = f.to(t.dtype)
        return [slots[i] for i in range(self.world)]

    def __del__(self):
        try:
            self._L.rsvd_handle_destroy(self.h)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def shard_rows(n, world, rank):
    """Contiguous row shard [lo, hi) of rank (rows [g n/G, (g+1) n/G))."""
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return lo, hi


class Workspace:
    """Per-call scratch for the orchestration (small FP64 matrices + masks)."""

    def __init__(self, device, p):
        self.device = device
        self.p = p
        f64 = dict(dtype=torch.float64, device=device)
        i32 = dict(dtype=torch.int32, device=device)
        self.G = torch.empty((p, p), **f64)
        self.T = torch.empty((p, p), **f64)
        self.mask = torch.empty(p, **i32)
        self.ndef = torch.zeros(2, **i32)
        self.ndef_r1 = torch.zeros(2, **i32)
        self.ndef_r3 = torch.zeros(2, **i32)
        self.ref_fin = torch.empty(p, **f64)
        self.mask2 = torch.empty(p, **i32)
        self.ndef2 = torch.zeros(2, **i32)
        self.ref2 = torch.empty(p, **f64)
        self.ref_orig = torch.empty(p, **f64)
        self.ndef_total = torch.zeros(1, **i32)
        self.flag_bool = torch.zeros(1, dtype=torch.bool, device=device)


def rows_buffer(n, p, dtype, device):
    """n x p work block whose rows start on 16-byte boundaries (leading
    dimension padded to a multiple of 4 elements): the tensor-core GEMMs
    read their A operand through TMA, which needs 16-byte aligned rows."""
    p4 = (p + 3) // 4 * 4
    return torch.empty((n, p4), dtype=dtype, device=device)[:, :p]


def _cast_small(ops, T64, dtype, out=None, pred=None):
    if dtype == torch.float64:
        return T64
    if out is None:
        out = torch.empty(T64.shape, dtype=dtype, device=T64.device)
    return ops.convert(T64, out, pred=pred)


def project_out(ops, comm, Qp, V, tmp_c, pred=None, basis=None, planes=None):
    """V <- V - Qp (Qp^T V)  (one block classical Gram-Schmidt pass).
    ``basis`` (exact mode): the digit planes of the basis Qp is the prefix of
    (device.OzBasis) -- both products run as FP64-accurate int8 tensor-core
    GEMMs instead of FP64 DMMA."""
    if Qp is None or Qp.shape[1] == 0:
        return V
    if basis is not None:
        jp = Qp.shape[1]
        basis.gemm(1, jp, V, tmp_c, pred=pred)
        comm.allreduce(tmp_c)
        basis.gemm(0, jp, tmp_c, V, alpha=-1.0, beta=1.0, pred=pred)
        return V
    # planes (FP32, unpredicated calls only): the TN product takes V's split planes
    # when they are current, and the NN product leaves the updated V's behind
    ops.gemm_tn(Qp, V, tmp_c, pred=pred, b_planes=planes if pred is None else None)
    comm.allreduce(tmp_c)
    ops.gemm_nn(Qp, tmp_c, V, alpha=-1.0, beta=1.0, pred=pred, emit=planes if pred is None else None)
    return V


# A third CholeskyQR pass for FP32 blocks (off by default: the chain blocks
# are well conditioned after the first pass and Z is re-orthonormalised in
# FP64; RSVD_FP32_THIRD_PASS=1 restores it for comparison).
FP32_THIRD_PASS = os.environ.get("RSVD_FP32_THIRD_PASS", "0") == "1"
# Projection passes against the prefix before the round-1 Gram (see
# proj_passes); RSVD_PROJ_PASSES overrides (A/B measurement).
_PROJ_ENV = os.environ.get("RSVD_PROJ_PASSES")
# Device-decided sections as CUDA-graph conditional nodes (RSVD_GRAPH_COND=0:
# predicated kernels only, for A/B measurement).
GRAPH_COND = os.environ.get("RSVD_GRAPH_COND", "1") != "0"
# Second FP64 CholeskyQR step on the Ritz vectors only when one step leaves
# ||Z^T Z - I||max above this (or a column was refilled).
Z_REORTH_TOL = 1e-13
# Projected block-Krylov basis: first projection's coefficients formed in
# d-space from W = A^T Q (RSVD_DSPACE_PASS1=0: from Q^T V, A/B).
D_SPACE_PASS1 = os.environ.get("RSVD_DSPACE_PASS1", "1") != "0"
# Exact mode: projections against the final prefix on its int8 digit planes
# (RSVD_OZ_PROJ=0: FP64 DMMA, for A/B measurement).
OZ_PROJECTIONS = os.environ.get("RSVD_OZ_PROJ", "1") != "0"
# Reference-faithful basis: the power chain and the final orthonormalization
# on two streams (RSVD_OVERLAP_FINAL=0: one stream, for A/B measurement).
OVERLAP_FINAL = os.environ.get("RSVD_OVERLAP_FINAL", "1") != "0"
# Projections against Qp inside the second deflation round (see orth_block).
ROUND2_QP_PASSES = int(os.environ.get("RSVD_ROUND2_QP_PASSES", "1"))
# FP32 blocks: split planes emitted by the NN epilogues and reused by the
# following TN products. Off by default: at C4 the split passes fall from 23.5
# to 7.6 ms and the chain's A^T Y from 93.7 to 91.9 ms, but the emitting NN
# epilogues (two 4-byte stores per element on top of C's float4 stores) cost
# 25.7 ms more: 349.6 vs 340.1 ms per factorization (gpurun_out/s5_trace_c4_*).
EMIT_PLANES = os.environ.get("RSVD_EMIT_PLANES", "0") != "0"


def proj_passes(dtype):
    """One projection pass before the round-1 Gram in every precision: the
    decisions that matter for parity (residual <= 1e-12 x original norm,
    factor.py:105) are made in round 2 on explicitly re-projected residuals
    (two more passes), and the final pass projects again after the
    CholeskyQR step. Measured at C2 (exact mode): 39.3 -> 37.2 ms, sigma /
    captured variance / replaced columns unchanged; C1 and the reference
    goldens unchanged to 1e-10 (tests)."""
    if _PROJ_ENV:
        return int(_PROJ_ENV)
    return 1


def orth_block(ops, comm, V, tmp, ws, Qp=None, ref2=None, running=None, n_total=None, row_offset=0,
               tau=None, deflation_count=None, two_round=None, pass1_coef=None, basis=None):
    """Orthonormalize the n x p block V in place (span-preserving, column
    order preserving), against the orthonormal columns Qp when given.

    Round 1: BCGS2 projection against Qp, FP64 Gram, column-ordered Cholesky
      with deflation at ``tau`` (the Gram resolves residuals only down to
      ~sqrt(eps)), Q1 = V R^{-1}, cleaned by one CholeskyQR step.
    Round 2 (FP64, ``two_round``): the columns round 1 rejected are re-tested
      on their EXPLICIT residuals (projected against Qp and Q1) at the
      reference's own threshold 1e-12 x original column norm (factor.py:41,
      105); survivors join Q1, the rest are replaced from the fill stream
      (factor.py:106-112).
    Final: one projection + CholeskyQR step.
    """
    if V.data_ptr() % 16 != 0:
        # the tensor-core GEMMs read their A operand through TMA, which needs a
        # 16-byte aligned base: work on an aligned copy of a misaligned block
        # view (e.g. block j of width p = 50 inside the n x w basis)
        Vw = rows_buffer(V.shape[0], V.shape[1], V.dtype, V.device)
        ops.convert(V, Vw)
        orth_block(ops, comm, Vw, tmp, ws, Qp=Qp, ref2=ref2, running=running, n_total=n_total,
                   row_offset=row_offset, tau=tau, deflation_count=deflation_count, two_round=two_round,
                   pass1_coef=pass1_coef, basis=basis)
        return ops.convert(Vw, V)
    dtype = V.dtype
    p = V.shape[1]
    if two_round is None:
        two_round = os.environ.get("RSVD_TWO_ROUND", "1") != "0"  # "0": A/B timing of round 2's launches
    tau = TAU[dtype] if tau is None else tau
    n_total = V.shape[0] if n_total is None else n_total
    has_prev = Qp is not None and Qp.shape[1] > 0
    tmp_c = torch.empty((Qp.shape[1], p), dtype=dtype, device=V.device) if has_prev else None
    # FP32 blocks: every NN product that writes a block also writes its hi / lo
    # split planes from its epilogue (device.SplitPlanes), and the TN product that
    # reads the block next (Gram, projection, the chain's A^T b) takes those instead
    # of a split pass over the block (C4: 23 of 340 ms were k_split_b). Measured
    # slower as a whole (see EMIT_PLANES), so opt-in: RSVD_EMIT_PLANES=1.
    pl = ops.SplitPlanes.get(V.shape[0], p, V.device) if (dtype == torch.float32 and EMIT_PLANES and
                                                           V.is_cuda) else None
    if has_prev:
        npass = proj_passes(dtype)
        if pass1_coef is not None:
            # first pass with coefficients formed in d-space by the caller
            # (bk_basis: Qp^T A C = (A^T Qp)^T C); the remaining passes and
            # the final pass project with Qp^T V itself
            ops.gemm_nn(Qp, pass1_coef, V, alpha=-1.0, beta=1.0, emit=pl)
            npass -= 1
        for _ in range(npass):
            project_out(ops, comm, Qp, V, tmp_c, basis=basis, planes=pl)
    G = ws.G[:p, :p]
    T = ws.T[:p, :p]
    mask = ws.mask[:p]
    ops.gram(V, G, b_planes=pl)
    comm.allreduce(G)
    if two_round and tau > 0.0 and ref2 is None:
        # original column norms^2 = diag(V^T V): taken from the Gram instead of a
        # separate pass over V (only round 2's 1e-12 test reads them)
        ws.ref_orig[:p].copy_(torch.diagonal(G))
    # round-1 threshold: without separate reference norms the Gram's diagonal is
    # the reference and the pivot-noise floor applies (see PIVOT_NOISE)
    tau2_r1 = tau * tau if ref2 is not None else max(tau * tau, PIVOT_NOISE[dtype])
    # device-decided sections become CUDA-graph IF nodes under capture
    # (device.cond_section); they must not allocate, so their buffers are
    # made here. NCCL collectives stay out of conditional bodies (world 1 only).
    use_cond = GRAPH_COND and isinstance(comm, LocalComm)
    T32 = torch.empty((p, p), dtype=dtype, device=V.device) if dtype != torch.float64 else None
    if two_round and tau > 0.0:
        r1 = ws.ndef_r1  # round-1 [count, base]: round 2 runs on the device only if count > 0
        ops.chol_deflate(G, ref2, tau2_r1, T, mask, r1, None)
        Q1 = rows_buffer(tmp.shape[0], p, dtype, tmp.device)
        ops.gemm_nn(V, _cast_small(ops, T, dtype), Q1, emit=pl)  # Q1 (zero columns at rejected slots)
        ws.ndef.zero_()
        c2 = torch.empty((p, p), dtype=dtype, device=V.device)
        with ops.cond_section(r1, use_cond):
            # round 2 needs Q1 orthonormal enough to project residuals against:
            # one CholeskyQR step, only when round 2 will run
            ops.gram(Q1, G, pred=r1)
            comm.allreduce(G)
            ops.chol_deflate(G, None, 0.0, T, ws.mask2[:p], ws.ndef2, None, pred=r1)
            ops.gemm_nn(Q1, _cast_small(ops, T, dtype, out=T32, pred=r1), tmp, pred=r1)
            ops.convert(tmp, Q1, pred=r1)
            ops.mask_cols(V, mask, pred=r1)  # keep only the rejected columns' residuals
            # the residuals were projected against Qp once before round 1: two
            # passes against Q1 around one more against Qp give each of them the
            # reference's two Gram-Schmidt passes (factor.py:93-98) against every
            # earlier column (RSVD_ROUND2_QP_PASSES=2: the previous Qp, Q1, Qp, Q1)
            if ROUND2_QP_PASSES == 1:
                project_out(ops, comm, Q1, V, c2, pred=r1)
                if has_prev:
                    project_out(ops, comm, Qp, V, tmp_c, pred=r1, basis=basis)
                project_out(ops, comm, Q1, V, c2, pred=r1)
            else:
                if has_prev:
                    project_out(ops, comm, Qp, V, tmp_c, pred=r1, basis=basis)
                project_out(ops, comm, Q1, V, c2, pred=r1)
                if has_prev:
                    project_out(ops, comm, Qp, V, tmp_c, pred=r1, basis=basis)
                project_out(ops, comm, Q1, V, c2, pred=r1)
            ops.gram(V, G, pred=r1)
            comm.allreduce(G)
            ref = ref2 if ref2 is not None else ws.ref_orig[:p]
            rt = REF_RTOL_BY[dtype]
            ops.chol_deflate(G, ref, rt * rt, T, ws.mask2[:p], ws.ndef, running, mask, pred=r1)
            # survivors join the kept columns
            ops.gemm_nn(V, _cast_small(ops, T, dtype, out=T32, pred=r1), Q1, beta=1.0, pred=r1)
            ops.insert_fill(Q1, ws.mask2[:p], ws.ndef, QR_FILL_SEED, row_offset, n_total, pred=r1)
        if pl is not None and pl.describes(Q1):
            pl.split(Q1, pred=r1)  # round 2 changed Q1 (only then: device-predicated)
        out = Q1
    else:
        ops.chol_deflate(G, ref2, tau * tau, T, mask, ws.ndef, running)
        Tw = _cast_small(ops, T, dtype)
        ops.gemm_nn(V, Tw, tmp)
        ops.insert_fill(tmp, mask, ws.ndef, QR_FILL_SEED, row_offset, n_total)
        out = tmp
    if deflation_count is not None:
        deflation_count += ws.ndef[:1]
    # Final pass. A replacement column that collapses against the columns
    # before it (residual <= 1e-6 of its norm, factor.py:111) is redrawn from
    # the next vectors of the same fill stream, as the reference's retry loop
    # does (factor.py:106-116); the repair steps run only if that happened.
    # (without a prefix nothing happens between the norms and the Gram: the
    # Gram's own diagonal is the reference, chol_deflate's default)
    ref_f = None
    if has_prev:
        ref_f = ws.ref_fin[:p]
        ops.colreduce(out, True, ref_f)
        comm.allreduce(ref_f)
        project_out(ops, comm, Qp, out, tmp_c, basis=basis, planes=pl)
    ops.gram(out, G, b_planes=pl)
    comm.allreduce(G)
    r3 = ws.ndef_r3
    ops.chol_deflate(G, ref_f, 1e-12, T, ws.mask2[:p], r3, running)
    ops.gemm_nn(out, _cast_small(ops, T, dtype), V, emit=pl)
    # repair (runs only if a column collapsed): next stream vectors into the
    # collapsed slots, re-project, CholeskyQR
    with ops.cond_section(r3, use_cond):
        ops.insert_fill(V, ws.mask2[:p], r3, QR_FILL_SEED, row_offset, n_total, pred=r3)
        if has_prev:
            project_out(ops, comm, Qp, V, tmp_c, pred=r3, basis=basis)
            project_out(ops, comm, Qp, V, tmp_c, pred=r3, basis=basis)
        ops.gram(V, G, pred=r3)
        comm.allreduce(G)
        ops.chol_deflate(G, None, 0.0, T, ws.mask2[:p], ws.ndef2, None, pred=r3)
        ops.gemm_nn(V, _cast_small(ops, T, dtype, out=T32, pred=r3), out, pred=r3)
        ops.convert(out, V, pred=r3)
    if pl is not None and pl.describes(V):
        pl.split(V, pred=r3)  # the repair changed V (only then: device-predicated)
    if dtype != torch.float64 and FP32_THIRD_PASS:
        # FP32 storage: one more CholeskyQR step (CholeskyQR2 cleanup)
        ops.gram(V, G)
        comm.allreduce(G)
        ops.chol_deflate(G, None, 0.0, T, ws.mask2[:p], ws.ndef2, None)
        ops.gemm_nn(V, _cast_small(ops, T, dtype), out)
        V.copy_(out)
    return V


class BasisResult:
    def __init__(self, Q, q_used, deflated, W=None):
        self.Q = Q
        self.q_used = q_used
        self.deflated = deflated  # device int32 tensor: columns replaced in the final orth
        self.W = W  # A^T Q when the construction produced it (projected BK), else None


def sketch_basis(ops, comm, op, Pi, ws, n_total, row_offset):
    """rsvd.py:224-226: b0 = mgs(A Pi)."""
    n = op.local_rows
    p = Pi.shape[1]
    Y = rows_buffer(n, p, op.dtype, op.device)
    tmp = rows_buffer(n, p, op.dtype, op.device)
    op.apply(Pi, Y)
    running = torch.zeros(1, dtype=torch.int32, device=op.device)
    orth_block(ops, comm, Y, tmp, ws, running=running, n_total=n_total, row_offset=row_offset)
    return Y


# Block-Krylov basis construction for the reduced-precision (FP32) path:
# "projected" orthonormalizes each new block A A^T q_{j-1} against all
# previous blocks as it is produced (block Lanczos with full
# re-orthogonalization, BCGS2 + CholeskyQR). It spans the same Krylov
# subspace as the reference's normalized power blocks + final _mgs of their
# hstack, but represents each block's new directions at full relative
# precision: for high powers those directions are a ~1e-5 residual of the
# raw block, below FP32 / 3xTF32 resolution, and the faithful construction
# measured 2.6e-3 relative error on the C2 tail singular values (median
# 1.1e-4) against the FP64 reference. FP64 keeps the reference-faithful
# construction (its deflation pattern, e.g. C1's 39 replaced columns, is
# part of the parity). RSVD_BK_BASIS=faithful|projected overrides.
BK_BASIS = os.environ.get("RSVD_BK_BASIS", "")


def bk_basis(ops, comm, op, Pi, q, ws, n_total, row_offset):
    """rsvd.py:244-260 — block Krylov basis [b0 .. b_q], orthonormalized.

    Blocks are written straight into the n x w basis buffer K. FP64: the
    reference's structure — normalized power blocks, then the final
    orthonormalization (``_mgs(np.hstack(blocks))``) block by block in place
    (BCGS2 against the already orthonormal prefix). FP32: the projected
    construction (see BK_BASIS above)."""
    n = op.local_rows
    d = op.shape[1]
    p = Pi.shape[1]
    cap_blocks = max(1, min(n_total, d) // p)
    n_blocks = min(q + 1, cap_blocks)
    dev, dt = op.device, op.dtype
    K = rows_buffer(n, n_blocks * p, dt, dev)
    tmp = rows_buffer(n, p, dt, dev)
    C = torch.empty((d, p), dtype=dt, device=dev)
    running = torch.zeros(1, dtype=torch.int32, device=dev)
    projected = BK_BASIS == "projected" or (BK_BASIS != "faithful" and dt != torch.float64)
    b0 = K[:, :p]
    op.apply(Pi, b0)
    orth_block(ops, comm, b0, tmp, ws, running=running, n_total=n_total, row_offset=row_offset)
    if n_blocks == 1:
        return BasisResult(K, 0, torch.zeros(1, dtype=torch.int32, device=dev))
    deflated = torch.zeros(1, dtype=torch.int32, device=dev)
    if projected:
        # One fill stream across the blocks, as one _mgs of the hstack. The
        # chain's A^T q_{j-1} are the columns of W = A^T Q that Rayleigh-Ritz
        # needs (q_{j-1} is final when they are formed), so they are written
        # into W and only A^T q_last is added at the end: one width-p pass
        # over A instead of a width-w one.
        W = rows_buffer(d, n_blocks * p, dt, dev)
        coef = torch.empty((n_blocks * p, p), dtype=dt, device=dev)
        for j in range(1, n_blocks):
            prev = K[:, (j - 1) * p: j * p]
            cur = K[:, j * p: (j + 1) * p]
            Cj = W[:, (j - 1) * p: j * p]
            op.apply_t(prev, Cj)
            comm.allreduce(Cj)
            op.apply(Cj, cur)
            ref2 = ws.ref2[:p]
            ops.colreduce(cur, True, ref2)
            comm.allreduce(ref2)
            c1 = None
            if D_SPACE_PASS1:
                # cur = A Cj, so Qp^T cur = (A^T Qp)^T Cj = W[:, :jp]^T Cj: the
                # first projection's coefficients from the d x jp prefix of W
                # (replicated across ranks: no allreduce) instead of a pass
                # over the n x jp basis
                c1 = coef[: j * p]
                ops.gemm_tn(W[:, : j * p], Cj, c1)
            orth_block(ops, comm, cur, tmp, ws, Qp=K[:, : j * p], ref2=ref2, running=running,
                       n_total=n_total, row_offset=row_offset, deflation_count=deflated, pass1_coef=c1)
        last = W[:, (n_blocks - 1) * p:]
        op.apply_t(K[:, (n_blocks - 1) * p:], last)
        comm.allreduce(last)
        return BasisResult(K, n_blocks - 1, deflated, W=W)
    if OVERLAP_FINAL and isinstance(comm, LocalComm) and dev.type == "cuda":
        return _bk_faithful_overlapped(ops, comm, op, K, C, tmp, ws, n_blocks, p, n_total, row_offset, deflated)
    for j in range(1, n_blocks):
        prev = K[:, (j - 1) * p: j * p]
        cur = K[:, j * p: (j + 1) * p]
        op.apply_t(prev, C)
        comm.allreduce(C)
        op.apply(C, cur)
        running.zero_()
        orth_block(ops, comm, cur, tmp, ws, running=running, n_total=n_total, row_offset=row_offset)
    # final orthonormalization of hstack(blocks): one _mgs call -> one fill stream
    running.zero_()
    # exact mode (FP32 A, FP64 blocks): the projections against the final
    # prefix run on its int8 digit planes, each block sliced in once final
    basis = ops.OzBasis(n, n_blocks * p, dev) if (getattr(op, "oz", None) is not None and
                                                  dt == torch.float64 and OZ_PROJECTIONS) else None
    for j in range(n_blocks):
        cur = K[:, j * p: (j + 1) * p]
        ref2 = ws.ref2[:p]
        ops.colreduce(cur, True, ref2)
        comm.allreduce(ref2)
        orth_block(ops, comm, cur, tmp, ws, Qp=K[:, : j * p] if j else None, ref2=ref2, running=running,
                   n_total=n_total, row_offset=row_offset, deflation_count=deflated, basis=basis)
        if basis is not None and j + 1 < n_blocks:
            basis.slice(K, j * p, p)
    return BasisResult(K, n_blocks - 1, deflated)


_SIDE_STREAMS = {}


def _bk_faithful_overlapped(ops, comm, op, K, C, tmp, ws, n_blocks, p, n_total, row_offset, deflated):
    """The reference-faithful block-Krylov basis with its two sequences on
    two streams: the power chain b_j = mgs(A A^T b_{j-1}) on the caller's
    stream, and the final orthonormalization of hstack(blocks) (block j
    against the final prefix, in place) on a side stream. The only
    dependency between them is that block j may be overwritten by its final
    orthonormalization once the chain has read it (A^T b_j), which an event
    orders; everything else is independent, so the final pass's
    latency-bound small kernels (Grams, Cholesky, projections) fill the gaps
    of the chain's tensor-core products. Same arithmetic, same order per
    block, same results (single rank: NCCL collectives on two streams could
    interleave differently on different ranks, so the sharded path stays
    sequential)."""
    dev, dt = op.device, op.dtype
    n = op.local_rows
    main = torch.cuda.current_stream(dev)
    side = _SIDE_STREAMS.get(dev)
    if side is None:
        side = _SIDE_STREAMS[dev] = torch.cuda.Stream(device=dev)
    ws2 = Workspace(dev, p)
    tmp2 = rows_buffer(n, p, dt, dev)
    running_chain = torch.zeros(1, dtype=torch.int32, device=dev)
    running_final = torch.zeros(1, dtype=torch.int32, device=dev)
    basis = ops.OzBasis(n, n_blocks * p, dev) if (getattr(op, "oz", None) is not None and
                                                  dt == torch.float64 and OZ_PROJECTIONS) else None
    ready = torch.cuda.Event()
    ready.record(main)
    side.wait_event(ready)

    def final(j):
        with torch.cuda.stream(side):
            cur = K[:, j * p: (j + 1) * p]
            ref2 = ws2.ref2[:p]
            ops.colreduce(cur, True, ref2)
            comm.allreduce(ref2)
            orth_block(ops, comm, cur, tmp2, ws2, Qp=K[:, : j * p] if j else None, ref2=ref2, running=running_final,
                       n_total=n_total, row_offset=row_offset, deflation_count=deflated, basis=basis)
            if basis is not None and j + 1 < n_blocks:
                basis.slice(K, j * p, p)

    for j in range(1, n_blocks):
        prev = K[:, (j - 1) * p: j * p]
        cur = K[:, j * p: (j + 1) * p]
        op.apply_t(prev, C)
        comm.allreduce(C)
        consumed = torch.cuda.Event()
        consumed.record(main)  # b_{j-1} has been read by the chain
        side.wait_event(consumed)
        final(j - 1)
        op.apply(C, cur)
        running_chain.zero_()
        orth_block(ops, comm, cur, tmp, ws, running=running_chain, n_total=n_total, row_offset=row_offset)
    last = torch.cuda.Event()
    last.record(main)
    side.wait_event(last)
    final(n_blocks - 1)
    done = torch.cuda.Event()
    done.record(side)
    main.wait_event(done)
    return BasisResult(K, n_blocks - 1, deflated)


def si_basis(ops, comm, op, Pi, q, every, ws, n_total, row_offset):
    """rsvd.py:229-241 — simultaneous (power) iteration."""
    if q == 0:
        return sketch_basis(ops, comm, op, Pi, ws, n_total, row_offset)
    n = op.local_rows
    d = op.shape[1]
    p = Pi.shape[1]
    dev, dt = op.device, op.dtype
    b = rows_buffer(n, p, dt, dev)
    tmp = rows_buffer(n, p, dt, dev)
    C = torch.empty((d, p), dtype=dt, device=dev)
    running = torch.zeros(1, dtype=torch.int32, device=dev)
    op.apply(Pi, b)
    orthonormal = False
    if dt == torch.float32:
        # FP32 blocks cannot carry raw powers the way the reference's FP64 blocks
        # do (a block's small directions sink below 2^-24 of its large ones after
        # a step or two: sigma errors of 50 % measured on low-rank inputs with
        # reorthonormalize_every = 0): orthonormalize after every step. The span
        # is the same in exact arithmetic; the exact / fp64 modes keep the
        # reference's schedule.
        every = 1
    for t in range(1, q + 1):
        op.apply_t(b, C)
        comm.allreduce(C)
        op.apply(C, b)
        orthonormal = False
        if every and t % every == 0:
            running.zero_()
            orth_block(ops, comm, b, tmp, ws, running=running, n_total=n_total, row_offset=row_offset)
            orthonormal = True
    if not orthonormal:
        running.zero_()
        orth_block(ops, comm, b, tmp, ws, running=running, n_total=n_total, row_offset=row_offset)
    return b


class RitzResult:
    def __init__(self, Z, sigma, info, off, zerr):
        self.Z = Z  # n_local x k FP64, signs canonicalized
        self.sigma = sigma  # k FP64
        self.info = info  # int32 [converged, sweeps, ...]
        self.off = off  # FP64 [1]
        self.zerr = zerr  # FP64 [1]: max |Z^T Z - I| (rsvd.py:182-185)


def rayleigh_ritz(ops, comm, op, Q, k, n_total, row_offset, sign_fn=None, W=None):
    """rsvd.py:200-221 with M = W^T W, W = A^T Q (one pass over A; none when
    the basis construction already produced W)."""
    dev = op.device
    w = Q.shape[1]
    d = op.shape[1]
    # W = A^T Q carries the precision of the products: FP64 on the FP64 path;
    # FP32-accurate on the FP32 path (3xTF32 / FP32 SpMM), where it is stored in
    # FP32 and M = W^T W runs on the tensor cores with FP64 output (the FP64
    # CUDA-core Gram of an FP64 copy took 38 ms at C3, w = 1600)
    if W is None:
        wdt = torch.float64 if Q.dtype == torch.float64 else Q.dtype
        W = rows_buffer(d, w, wdt, dev)
        if getattr(op, "oz", None) is not None:
            op.apply_t(Q, W, rayleigh_ritz=True)
        else:
            op.apply_t(Q, W)
        comm.allreduce(W)
    M = torch.empty((w, w), dtype=torch.float64, device=dev)
    ops.gram(W, M)
    # top-k eigenpairs only (rsvd.py:217-220 uses eigvecs[:, :k], eigvals[:k])
    evals, Uk, info = ops.syev_topk(M, k)
    off = torch.zeros(1, dtype=torch.float64, device=dev)
    n = Q.shape[0]
    ws = Workspace(dev, k)
    again = ws.ndef2[:1]
    if Q.dtype == torch.float64:
        Z = rows_buffer(n, k, torch.float64, dev)
        ops.gemm_nn(Q, Uk, Z)
        Z0 = rows_buffer(n, k, torch.float64, dev)
        ws.ndef.zero_()
    else:
        Uk32 = torch.empty((w, k), dtype=Q.dtype, device=dev)
        ops.convert(Uk, Uk32)
        Z32 = rows_buffer(n, k, Q.dtype, dev)
        ops.gemm_nn(Q, Uk32, Z32)
        Z0 = rows_buffer(n, k, torch.float64, dev)
        ops.convert(Z32, Z0)
        # FP64 re-orthonormalization of the n x k Z. Z = Q U_k
        # with Q orthonormal to FP32 precision, so cond(Z) ~ 1 and one FP64
        # CholeskyQR step leaves ||Z^T Z - I|| at ~1e-15; the second step runs
        # (device-decided, a graph IF node under capture) only if the check
        # Gram says otherwise (or a column had to be refilled). The check Gram
        # also gives the orthogonality error reported with the result (the
        # sign canonicalization below only negates columns).
        Z = rows_buffer(n, k, torch.float64, dev)
        G = ws.G
        ops.gram(Z0, G)
        comm.allreduce(G)
        ops.chol_deflate(G, None, 0.0, ws.T, ws.mask, ws.ndef)
        ops.gemm_nn(Z0, ws.T, Z)
        ops.insert_fill(Z, ws.mask, ws.ndef, QR_FILL_SEED, row_offset, n_total, pred=ws.ndef)
    # The check Gram gives the orthogonality error reported with the result;
    # one more CholeskyQR step runs (device-decided) only if it says so. FP64:
    # Z = Q U_k is orthonormal to ~1e-15 whenever Q is; a basis the
    # orthonormalization could only bring to ~1e-6 (raw power blocks of a
    # rank-deficient A, reorthonormalize_every = 0) is repaired here instead of
    # failing PartialSvdResult's check.
    G2 = torch.empty((k, k), dtype=torch.float64, device=dev)
    ops.gram(Z, G2)
    comm.allreduce(G2)
    zerr = ops.ortho_error(G2)
    torch.gt(zerr, Z_REORTH_TOL, out=ws.flag_bool)
    again.copy_(ws.flag_bool)
    again.add_(ws.ndef[:1])
    G3 = torch.empty((k, k), dtype=torch.float64, device=dev)
    z2 = torch.empty_like(zerr)
    with ops.cond_section(again, GRAPH_COND and isinstance(comm, LocalComm)):
        ops.chol_deflate(G2, None, 0.0, ws.T, ws.mask2, ws.ndef_r3, pred=again)
        ops.gemm_nn(Z, ws.T, Z0, pred=again)
        ops.convert(Z0, Z, pred=again)
        # the re-check goes through its own buffer: when the section runs as
        # predicated kernels (row-sharded A: collectives stay unconditional) and
        # the predicate is off, the allreduce must not touch the reduced G2
        G3.zero_()
        ops.gram(Z, G3, pred=again)
        comm.allreduce(G3)
        ops.ortho_error(G3, z2)
        torch.gt(again, 0, out=ws.flag_bool)
        torch.where(ws.flag_bool, z2, zerr, out=zerr)
    if sign_fn is None:
        ops.canonicalize_signs(Z)
    else:
        sign_fn(Z)
    sigma = ops.sqrt_clip(evals)
    return RitzResult(Z, sigma, info, off, zerr)
