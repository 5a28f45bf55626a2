"""Kernel-level parity of the CUDA library against the oracle / FP64
references (run on the B200)."""

import os

import numpy as np
import pytest
import torch

import rsvd_oracle as o
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    from paper_1504_05477_b200 import device

    return device


def _t(a, dt=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)


def _rand(shape, seed):
    return o.gaussian(*shape, o.SeededRng(seed))


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (37, 5, 19), (2000, 20, 1000), (513, 64, 200), (300, 200, 65)])
def test_gemm_nn_f64(ops, m, n, k):
    a, b, c0 = _rand((m, k), 1), _rand((k, n), 2), _rand((m, n), 3)
    C = _t(c0)
    ops.gemm_nn(_t(a), _t(b), C, alpha=0.5, beta=-2.0)
    ref = 0.5 * (a @ b) - 2.0 * c0
    assert np.max(np.abs(C.cpu().numpy() - ref)) <= 1e-12 * max(1.0, np.abs(ref).max()) * np.sqrt(k)


@pytest.mark.parametrize("m,n,k", [(1, 3, 2), (5000, 20, 64), (2000, 200, 1000), (100000, 7, 33)])
def test_gemm_tn_f64(ops, m, n, k):
    a, b = _rand((m, k), 4), _rand((m, n), 5)
    C = torch.empty((k, n), dtype=torch.float64, device="cuda")
    ops.gemm_tn(_t(a), _t(b), C)
    ref = a.T @ b
    assert np.max(np.abs(C.cpu().numpy() - ref)) <= 1e-11 * np.sqrt(m)


def test_gemm_tn_centering_epilogue(ops):
    a, b = _rand((3000, 40), 6), _rand((3000, 9), 7)
    mu = a.mean(axis=0)
    C = torch.empty((40, 9), dtype=torch.float64, device="cuda")
    cs = ops.colreduce(_t(b), square=False)
    ops.gemm_tn(_t(a), _t(b), C, mu=_t(mu), colsum_b=cs)
    ref = (a - mu[None, :]).T @ b
    assert np.max(np.abs(C.cpu().numpy() - ref)) < 1e-10


def test_gemm_f32_paths(ops):
    a, b = _rand((4096, 512), 8).astype(np.float32), _rand((512, 48), 9).astype(np.float32)
    C = torch.empty((4096, 48), dtype=torch.float32, device="cuda")
    ops.gemm_nn(_t(a, torch.float32), _t(b, torch.float32), C)
    ref = a.astype(np.float64) @ b.astype(np.float64)
    assert np.max(np.abs(C.cpu().numpy() - ref)) / np.abs(ref).max() < 2e-6
    y = _rand((4096, 48), 10).astype(np.float32)
    W = torch.empty((512, 48), dtype=torch.float64, device="cuda")
    ops.gemm_tn(_t(a, torch.float32), _t(y, torch.float32), W)
    ref = a.astype(np.float64).T @ y.astype(np.float64)
    assert np.max(np.abs(W.cpu().numpy() - ref)) / np.abs(ref).max() < 2e-6


def test_colreduce_and_convert(ops):
    x = _rand((12345, 70), 11)
    s2 = ops.colreduce(_t(x), True).cpu().numpy()
    s1 = ops.colreduce(_t(x), False).cpu().numpy()
    assert np.allclose(s2, (x * x).sum(0), rtol=1e-13)
    assert np.allclose(s1, x.sum(0), rtol=1e-12, atol=1e-11)
    X = _t(x)
    Y = torch.empty(X.shape, dtype=torch.float32, device="cuda")
    ops.convert(X, Y)
    assert torch.equal(Y, X.float())


def test_chol_deflate_full_rank_and_deficient(ops):
    v = _rand((500, 30), 12)
    G = _t(v.T @ v)
    T = torch.empty((30, 30), dtype=torch.float64, device="cuda")
    mask = torch.empty(30, dtype=torch.int32, device="cuda")
    ndef = torch.zeros(2, dtype=torch.int32, device="cuda")
    ops.chol_deflate(G, None, 1e-14, T, mask, ndef)
    q = v @ T.cpu().numpy()
    assert np.max(np.abs(q.T @ q - np.eye(30))) < 1e-12
    assert int(ndef[0]) == 0
    # make columns 4 and 17 linear combinations of earlier ones
    v[:, 4] = v[:, 0] - 2 * v[:, 3]
    v[:, 17] = v[:, 2] + v[:, 9]
    G = _t(v.T @ v)
    running = torch.tensor([5], dtype=torch.int32, device="cuda")
    ops.chol_deflate(G, None, 1e-14, T, mask, ndef, running)
    m = mask.cpu().numpy()
    assert list(np.nonzero(m)[0]) == [4, 17]
    assert ndef.cpu().tolist() == [2, 5] and int(running[0]) == 7
    Tn = T.cpu().numpy()
    assert np.all(Tn[:, 4] == 0) and np.all(Tn[17, :] == 0)
    keep = [j for j in range(30) if not m[j]]
    qk = (v @ Tn)[:, keep]
    assert np.max(np.abs(qk.T @ qk - np.eye(len(keep)))) < 1e-10


@pytest.mark.parametrize("p", [1, 7, 33, 50, 64])
def test_chol_reg64_halves_match_compact(ops, monkeypatch, p):
    """p <= 64: the two-threads-per-column kernel (default) and the compact
    one-thread-per-column rotating-register kernel -- same operations in the
    same order, bitwise equal T, mask and counts (deficient and inactive
    columns included)."""
    v = _rand((4 * p + 8, p), 60 + p)
    if p >= 7:
        v[:, 5] = v[:, 1] - 2.0 * v[:, 3]
    G = _t(v.T @ v)
    active = torch.ones(p, dtype=torch.int32, device="cuda")
    if p >= 33:
        active[p - 3] = 0
    outs = []
    for mode in ("halves", "compact"):
        if mode == "compact":
            monkeypatch.setenv("RSVD_CHOL_REG_ONE", "1")
        T = torch.empty((p, p), dtype=torch.float64, device="cuda")
        mask = torch.empty(p, dtype=torch.int32, device="cuda")
        ndef = torch.zeros(2, dtype=torch.int32, device="cuda")
        running = torch.tensor([2], dtype=torch.int32, device="cuda")
        ops.chol_deflate(G, None, 1e-14, T, mask, ndef, running, active)
        outs.append((T.clone(), mask.clone(), ndef.clone(), running.clone()))
    for other in outs[1:]:
        for a, b in zip(outs[0], other):
            assert torch.equal(a, b)
    if p >= 7:
        assert int(outs[0][1][5]) == 1


@pytest.mark.parametrize("p", [65, 100, 200, 224])
def test_chol_deflate_blocked_wide(ops, monkeypatch, p):
    """Blocked right-looking factorization (p > 64, k_chol_sweep): the same
    deflation decisions, ndef/running bookkeeping and R^-1 (to rounding) as
    the column-by-column sweep, with deficient columns inside and across the
    16-column block rows, and an inactive column."""
    v = _rand((3 * p, p), 40 + p)
    for j, (a, b) in {5: (0, 3), 17: (2, 9), 40: (16, 33), p - 2: (1, p - 3)}.items():
        v[:, j] = v[:, a] - 0.5 * v[:, b]
    G = _t(v.T @ v)
    active = torch.ones(p, dtype=torch.int32, device="cuda")
    active[p // 2] = 0
    out = {}
    for mode in ("blocked", "unblocked"):
        if mode == "unblocked":
            monkeypatch.setenv("RSVD_CHOL_UNBLOCKED", "1")
        T = torch.empty((p, p), dtype=torch.float64, device="cuda")
        mask = torch.empty(p, dtype=torch.int32, device="cuda")
        ndef = torch.zeros(2, dtype=torch.int32, device="cuda")
        running = torch.tensor([3], dtype=torch.int32, device="cuda")
        ops.chol_deflate(G, None, 1e-14, T, mask, ndef, running, active)
        out[mode] = (T.cpu().numpy(), mask.cpu().numpy(), ndef.cpu().tolist(), int(running[0]))
    Tb, mb, nb, rb = out["blocked"]
    Tu, mu, nu, ru = out["unblocked"]
    assert list(np.nonzero(mb)[0]) == [5, 17, 40, p - 2]
    assert np.array_equal(mb, mu) and nb == nu == [4, 3] and rb == ru == 7
    assert np.max(np.abs(Tb - Tu)) <= 1e-9 * np.max(np.abs(Tu))
    keep = [j for j in range(p) if not mb[j] and j != p // 2]
    qk = (v @ Tb)[:, keep]
    assert np.max(np.abs(qk.T @ qk - np.eye(len(keep)))) < 1e-9


@pytest.mark.parametrize("p", [65, 96, 100, 150, 200])
def test_chol_blk_matches_sweep_bitwise(ops, monkeypatch, p):
    """k_chol_blk (diagonal block factored by one warp, block steps of every
    column in registers: 3 barriers per 16 columns) against k_chol_sweep's
    blocked path (2 barriers per column): same operations in the same order,
    so T, mask and the counts are bitwise equal -- deficient columns inside
    and across blocks and an inactive column included."""
    v = _rand((3 * p, p), 140 + p)
    for j, (a, b) in {5: (0, 3), 17: (2, 9), 40: (16, 33), p - 2: (1, p - 3)}.items():
        v[:, j] = v[:, a] - 0.5 * v[:, b]
    G = _t(v.T @ v)
    active = torch.ones(p, dtype=torch.int32, device="cuda")
    active[p // 2] = 0
    outs = []
    for mode in ("blk", "sweep"):
        if mode == "sweep":
            monkeypatch.setenv("RSVD_CHOL_SWEEP_OLD", "1")
        T = torch.empty((p, p), dtype=torch.float64, device="cuda")
        mask = torch.empty(p, dtype=torch.int32, device="cuda")
        ndef = torch.zeros(2, dtype=torch.int32, device="cuda")
        running = torch.tensor([3], dtype=torch.int32, device="cuda")
        ops.chol_deflate(G, None, 1e-14, T, mask, ndef, running, active)
        outs.append((T.clone(), mask.clone(), ndef.clone(), running.clone()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    assert list(np.nonzero(outs[0][1].cpu().numpy())[0]) == [5, 17, 40, p - 2]


@pytest.mark.parametrize("chunk", [32, 64, 256])
@pytest.mark.parametrize("nb", [4, 100, 128])
def test_spmm_nnz_plan_matches_dense_and_row_plan(ops, nb, chunk):
    """Nonzero-balanced FP32 product (k_spmm_nnz_f32): runs of `chunk`
    nonzeros cut rows anywhere -- rows spanning several runs, runs holding
    many short rows, empty rows (first, middle, last), a run boundary exactly
    on a row boundary -- against the dense FP64 product and, to FP32 rounding
    of the split sums, the warp-per-row plan; alpha / beta applied; repeated
    calls bitwise equal."""
    rng = np.random.default_rng(100 * nb + chunk)
    n, d = 700, 900
    lens = rng.integers(0, 40, n)
    lens[0] = 0
    lens[5] = 3 * chunk + 7     # spans 4+ runs
    lens[6] = 0
    lens[7] = chunk             # a full run's worth
    lens[n - 1] = 0
    lens[100:140] = 1           # many rows inside one run
    A = np.zeros((n, d))
    for r in range(n):
        cols = rng.choice(d, size=min(lens[r], d), replace=False)
        A[r, cols] = rng.lognormal(0, 1, cols.size)
    mask = A != 0
    indptr = np.zeros(n + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(mask.sum(1))
    rows, cols = np.nonzero(mask)
    ip = torch.from_numpy(indptr).cuda().to(torch.int32)
    cl = torch.from_numpy(cols).cuda().to(torch.int32)
    vl = torch.from_numpy(A[rows, cols]).cuda().float()
    B = rng.standard_normal((d, nb))
    C0 = rng.standard_normal((n, nb))
    Bt = torch.from_numpy(B).cuda().float()
    plan = ops.SpmmNnzPlan(ip, chunk=chunk)
    assert plan.nsplit >= 1 and plan.empty_rows.numel() >= 3
    assert ops.SpmmNnzPlan.eligible(cl, vl, Bt, torch.empty((n, nb), device="cuda"))
    A32 = A.astype(np.float32).astype(np.float64)
    for alpha, beta in ((1.0, 0.0), (0.5, 2.0)):
        Ct = torch.from_numpy(C0).cuda().float()
        ops.spmm_nnz_plan(plan, cl, vl, Bt, Ct, alpha=alpha, beta=beta)
        ref = alpha * (A32 @ Bt.double().cpu().numpy()) + beta * torch.from_numpy(C0).float().double().numpy()
        got = Ct.double().cpu().numpy()
        assert np.max(np.abs(got - ref)) < 2e-6 * np.abs(ref).max()
        C2 = torch.from_numpy(C0).cuda().float()
        ops.spmm_nnz_plan(plan, cl, vl, Bt, C2, alpha=alpha, beta=beta)
        assert torch.equal(Ct, C2)
        Cr = torch.from_numpy(C0).cuda().float()
        ops.spmm_csr_plan(ops.SpmmPlan(ip), cl, vl, Bt, Cr, alpha=alpha, beta=beta)
        assert np.max(np.abs(got - Cr.double().cpu().numpy())) < 2e-6 * np.abs(ref).max()


@pytest.mark.parametrize("nb", [8, 100, 300])
def test_csr_slab_tier(ops, nb, monkeypatch):
    """Slab tier of the hybrid CSR product (k_spmm_slab): 500 columns of 5 %
    density stay below the dense-panel threshold used here and above the slab
    threshold, so their rows of X are staged in shared memory; A X against the
    dense FP64 product and against the operator without the tier, ragged and
    empty rows included."""
    from paper_1504_05477_b200.operators import CsrDeviceOp

    rng = np.random.default_rng(nb + 11)
    n, d = 3000, 5000
    mask = rng.random((n, d)) < 0.004
    mask[:, 200:700] |= rng.random((n, 500)) < 0.05
    mask[:, 5] = True
    mask[17] = False  # an empty row
    mask[18, :] = False
    mask[18, 300] = True  # a row with a single slab nonzero
    A = np.zeros((n, d))
    A[mask] = rng.lognormal(0, 1, int(mask.sum()))
    indptr = np.zeros(n + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(mask.sum(1))
    rows, cols = np.nonzero(mask)
    ip = torch.from_numpy(indptr).cuda().to(torch.int32)
    cl = torch.from_numpy(cols).cuda().to(torch.int32)
    vl = torch.from_numpy(A[rows, cols]).cuda().float()
    monkeypatch.setattr(CsrDeviceOp, "SLAB_COLS", 2048)
    op = CsrDeviceOp(ip, cl, vl, d, hot_density=0.2)
    assert op.hot is not None and op.hot["H"] == 1
    assert op.slab is not None and op.slab["cols"].numel() == 500
    assert op.slab["nnz"] == int(mask[:, 200:700].sum())
    monkeypatch.setattr(CsrDeviceOp, "SLAB_COLS", 0)
    plain = CsrDeviceOp(ip, cl, vl, d, hot_density=0.2)
    assert plain.slab is None
    Xt = torch.from_numpy(rng.standard_normal((d, nb))).cuda().float()
    A32 = A.astype(np.float32).astype(np.float64)
    ref = A32 @ Xt.double().cpu().numpy()
    outs = []
    for o_ in (op, plain):
        out = torch.full((n, nb), 7.0, device="cuda")
        o_.apply(Xt, out)
        outs.append(out.double().cpu().numpy())
        assert np.max(np.abs(outs[-1] - ref)) < 2e-6 * np.abs(ref).max()
    # deterministic: a second call is bitwise equal
    out2 = torch.empty((n, nb), device="cuda")
    op.apply(Xt, out2)
    assert np.array_equal(out2.double().cpu().numpy(), outs[0])


def test_fill_stream_matches_host_stream(ops):
    n = 1001  # odd: each vector consumes n+1 uniforms (matrix.py:44-47)
    dev = ops.fill_stream(n, 3, o.QR_FILL_SEED, "cuda").cpu().numpy()
    rng = o.SeededRng(o.QR_FILL_SEED)
    host = np.stack([rng.normal_fill(n) for _ in range(3)])
    assert np.max(np.abs(dev - host)) < 1e-13


@pytest.mark.parametrize("n", [1, 2, 3, 12, 57, 64, 65, 130, 200, 601])
def test_jacobi_vs_oracle(ops, n):
    base = _rand((n, n), 13 + n)
    sym = 0.5 * (base + base.T)
    M, V = _t(sym), _t(np.eye(n))
    info, off = ops.jacobi_sweeps(M, V, 1e-14, 50)
    info = info.cpu().numpy()
    assert info[0] == 1
    vals = np.diag(M.cpu().numpy())
    ref_vals = np.sort(np.linalg.eigvalsh(sym))[::-1] if n > 200 else o.symmetric_eig(sym)[0]
    assert np.max(np.abs(np.sort(vals)[::-1] - ref_vals)) < 1e-12 * max(1.0, np.abs(ref_vals).max()) * max(1.0, np.sqrt(n / 64))
    Vh = V.cpu().numpy()
    assert np.max(np.abs(Vh @ np.diag(vals) @ Vh.T - sym)) < 1e-12 * n
    assert np.max(np.abs(Vh.T @ Vh - np.eye(n))) < 1e-12 * n
    evals, evecs = ops.eig_select(M, V, min(5, n))
    assert np.allclose(evals.cpu().numpy(), ref_vals[: min(5, n)], rtol=1e-12, atol=1e-13)


def test_jacobi_psd_rayleigh_ritz_like(ops):
    # M = W^T W with a decaying spectrum (the Rayleigh-Ritz matrix shape)
    rng = np.random.default_rng(3)
    w = 600
    Q, _ = np.linalg.qr(rng.standard_normal((w, w)))
    lam = (np.arange(1, w + 1) ** -1.0) ** 2
    sym = (Q * lam) @ Q.T
    sym = 0.5 * (sym + sym.T)
    M, V = _t(sym), _t(np.eye(w))
    info, off = ops.jacobi_sweeps(M, V, 1e-14, 50)
    assert int(info[0]) == 1
    evals, evecs = ops.eig_select(M, V, 50)
    ref = np.sort(np.linalg.eigvalsh(sym))[::-1][:50]
    assert np.max(np.abs(evals.cpu().numpy() - ref) / ref) < 1e-10
    E = evecs.cpu().numpy()
    assert np.max(np.abs(sym @ E - E * evals.cpu().numpy())) < 1e-13


def test_jacobi_golden_kernel_contract():
    from paper_1504_05477_b200 import backend

    k = np.load(os.path.join(GOLDEN, "kernels.npz"))
    m, v = k["jac_in"].copy(), np.eye(12)
    off, sweeps, conv = backend.jacobi_sweeps(m, v, 1e-14, 50)
    assert conv
    assert np.allclose(np.sort(np.diag(m)), np.sort(k["jac_diag"]), atol=1e-12)
    recon = v @ np.diag(np.diag(m)) @ v.T
    assert np.max(np.abs(recon - k["jac_in"])) < 1e-12


def test_jacobi_nonconvergence_reports():
    from paper_1504_05477_b200 import backend

    base = _rand((40, 40), 99)
    sym = 0.5 * (base + base.T)
    m, v = sym.copy(), np.eye(40)
    off, sweeps, conv = backend.jacobi_sweeps(m, v, 1e-14, 1)
    assert not conv and sweeps == 1 and off > 0


def test_backend_contract_kats():
    from paper_1504_05477_b200 import backend

    k = np.load(os.path.join(GOLDEN, "kernels.npz"))
    assert np.max(np.abs(backend.mm(k["mm_a"], k["mm_b"]) - k["mm_c"])) < 1e-12
    rows, cols = k["sp_shape"]
    nt = backend.spmm_nt(rows, k["sp_indptr"], k["sp_col"], k["sp_val"], k["sp_bx"])
    assert np.max(np.abs(nt - k["sp_nt"])) < 1e-12
    t = backend.spmm_t(rows, cols, k["sp_indptr"], k["sp_col"], k["sp_val"], k["sp_by"])
    assert np.max(np.abs(t - k["sp_t"])) < 1e-12
    out, st = backend.gauss_fill(7, 987654321)
    g = np.load(os.path.join(GOLDEN, "gauss_fill.npz"))
    assert np.array_equal(out, g["fill_7"])


def test_spmm_csr_ragged_and_empty_rows(ops):
    rng = np.random.default_rng(0)
    n, d = 3000, 700
    nnz_row = rng.integers(0, 90, size=n)
    nnz_row[::17] = 0
    nnz_row[5] = 700  # a full row
    indptr = np.concatenate([[0], np.cumsum(nnz_row)])
    cols = np.concatenate([np.sort(rng.choice(d, size=c, replace=False)) for c in nnz_row])
    vals = rng.standard_normal(indptr[-1])
    b = rng.standard_normal((d, 37))
    y = rng.standard_normal((n, 37))
    got = ops.spmm_csr(_t(indptr, torch.int32), _t(cols, torch.int32), _t(vals), d, _t(b),
                       torch.empty((n, 37), dtype=torch.float64, device="cuda")).cpu().numpy()
    assert np.max(np.abs(got - o.spmm_nt(n, indptr, cols, vals, b))) < 1e-12
    tp, tc, tv = ops.csr_transpose(_t(indptr, torch.int32), _t(cols, torch.int32), _t(vals), n, d)
    got_t = ops.spmm_csr(tp, tc, tv, n, _t(y), torch.empty((d, 37), dtype=torch.float64, device="cuda"))
    assert np.max(np.abs(got_t.cpu().numpy() - o.spmm_t(n, d, indptr, cols, vals, y))) < 1e-11


def test_canonicalize_signs_first_max_tie(ops):
    z = np.array([[0.5, -1.0, 0.0], [-0.5, 1.0, -0.0], [0.1, 0.2, 0.0]])
    Z = _t(z)
    ops.canonicalize_signs(Z)
    ref = o.canonicalize_signs(z.copy())
    assert np.array_equal(Z.cpu().numpy(), ref)
    big = _rand((100000, 13), 21)
    Z = _t(big)
    ops.canonicalize_signs(Z)
    assert np.array_equal(Z.cpu().numpy(), o.canonicalize_signs(big.copy()))


@pytest.mark.parametrize("w,k,kind", [(1, 1, "rand"), (2, 2, "rand"), (3, 1, "rand"), (50, 50, "rand"),
                                      (200, 20, "inv2"), (600, 50, "inv"), (601, 600, "rand"),
                                      (300, 40, "cluster"), (400, 30, "repeated"), (1200, 200, "clustered_c4")])
def test_syev_topk(ops, w, k, kind):
    rng = np.random.default_rng(w + k)
    if kind == "rand":
        base = rng.standard_normal((w, w))
        sym = 0.5 * (base + base.T)
    else:
        Q, _ = np.linalg.qr(rng.standard_normal((w, w)))
        i = np.arange(1, w + 1, dtype=float)
        lam = {"inv2": 1.0 / i ** 2, "inv": 1.0 / i,
               "cluster": np.where(i <= 60, 1.0 + 1e-9 * i, 0.5 / i),
               "repeated": np.where(i <= 10, 2.0, 1.0 / i),
               "clustered_c4": np.where(i <= 200, (1 - 0.001 * i) ** 2, (0.5 / i) ** 2)}[kind]
        sym = (Q * lam) @ Q.T
        sym = 0.5 * (sym + sym.T)
    M = _t(sym)
    evals, evecs, info = ops.syev_topk(M, k)
    assert int(info[0]) == 1
    ref = np.sort(np.linalg.eigvalsh(sym))[::-1][:k]
    ev = evals.cpu().numpy()
    scale = np.abs(np.linalg.eigvalsh(sym)).max()
    assert np.max(np.abs(ev - ref)) < 1e-13 * scale * max(1.0, np.sqrt(w / 64))
    E = evecs.cpu().numpy()
    assert np.max(np.abs(E.T @ E - np.eye(k))) < 1e-11
    assert np.max(np.abs(sym @ E - E * ev)) < 1e-12 * scale * max(1.0, np.sqrt(w / 64))
    assert np.allclose(M.cpu().numpy(), sym)  # input untouched


def test_syev_topk_grid_and_cluster_paths_agree(ops, monkeypatch):
    """w = 600 runs the cluster-resident tridiagonalisation; RSVD_TRIDIAG_GRID
    forces the grid-barrier kernel (the path for w > 608). Same results."""
    rng = np.random.default_rng(7)
    Q, _ = np.linalg.qr(rng.standard_normal((600, 600)))
    lam = 1.0 / np.arange(1, 601, dtype=float)
    sym = (Q * lam) @ Q.T
    sym = 0.5 * (sym + sym.T)
    M = _t(sym)
    ev_c, _, info_c = ops.syev_topk(M, 50)
    monkeypatch.setenv("RSVD_TRIDIAG_GRID", "1")
    ev_g, _, info_g = ops.syev_topk(M, 50)
    assert int(info_c[0]) == 1 and int(info_g[0]) == 1
    ref = np.sort(np.linalg.eigvalsh(sym))[::-1][:50]
    assert np.max(np.abs(ev_c.cpu().numpy() - ref)) < 1e-14
    assert np.max(np.abs(ev_g.cpu().numpy() - ref)) < 1e-14


@pytest.mark.parametrize("w,k", [(4, 2), (40, 10), (600, 50), (608, 30)])
def test_tridiag_cluster_one_barrier_matches_two_barrier(ops, monkeypatch, w, k):
    """Cluster-resident tridiagonalisation (w <= 608, C2): the one-barrier
    kernel (k_tridiag_cluster1) against the two-barrier one, bitwise."""
    rng = np.random.default_rng(w + 1)
    Q, _ = np.linalg.qr(rng.standard_normal((w, w)))
    lam = np.arange(1, w + 1, dtype=float) ** -0.5
    sym = (Q * lam) @ Q.T
    M = _t(0.5 * (sym + sym.T))
    ev1, V1, i1 = ops.syev_topk(M, k)
    monkeypatch.setenv("RSVD_TRIDIAG_TWO_BARRIER", "1")
    ev2, V2, i2 = ops.syev_topk(M, k)
    assert int(i1[0]) == 1 and int(i2[0]) == 1
    assert torch.equal(ev1, ev2) and torch.equal(V1, V2)


@pytest.mark.parametrize("w,k", [(4, 2), (5, 5), (37, 8), (700, 40), (1300, 100)])
def test_tridiag_one_barrier_matches_two_barrier(ops, monkeypatch, w, k):
    """The one-barrier-per-column grid tridiagonalisation (k_tridiag1, the
    path for w > 608: C3-C5) performs the same operations in the same order
    as the two-barrier kernel: eigenvalues and vectors bitwise equal. A
    repeated eigenvalue block exercises the zero-tail (skipped reflector)
    path on the small sizes."""
    rng = np.random.default_rng(w)
    Q, _ = np.linalg.qr(rng.standard_normal((w, w)))
    lam = 1.0 / np.arange(1, w + 1, dtype=float)
    lam[w // 2:] = lam[w // 2]
    sym = (Q * lam) @ Q.T
    sym = 0.5 * (sym + sym.T)
    if w == 5:
        sym = np.diag(np.arange(5.0, 0.0, -1.0))  # already tridiagonal: every reflector skipped
    M = _t(sym)
    monkeypatch.setenv("RSVD_TRIDIAG_GRID", "1")
    ev1, V1, i1 = ops.syev_topk(M, k)
    monkeypatch.setenv("RSVD_TRIDIAG_TWO_BARRIER", "1")
    ev2, V2, i2 = ops.syev_topk(M, k)
    assert int(i1[0]) == 1 and int(i2[0]) == 1
    assert torch.equal(ev1, ev2) and torch.equal(V1, V2)
    # blocked back-transformation (k_backtransform_blk) vs one reflector at a time
    monkeypatch.setenv("RSVD_BT_SEQ", "1")
    ev3, V3, _ = ops.syev_topk(M, k)
    assert torch.equal(ev1, ev3)
    assert torch.max(torch.abs(V1 - V3)).item() < 1e-13
    ref = np.sort(np.linalg.eigvalsh(sym))[::-1][:k]
    assert np.max(np.abs(ev1.cpu().numpy() - ref)) < 1e-13 * max(1.0, abs(ref[0]))


@pytest.mark.parametrize("nb,dtype", [(7, torch.float32), (100, torch.float32), (300, torch.float32),
                                      (600, torch.float32), (64, torch.float64), (300, torch.float64)])
def test_spmm_plan_split_rows_and_wide_blocks(ops, nb, dtype):
    """Load-balanced CSR product: rows longer than the chunk (split, partials
    summed in order), empty rows, column panels of 256 for wide blocks,
    alpha / beta; against a dense numpy product."""
    rng = np.random.default_rng(nb)
    n, d = 300, 2000
    lens = rng.integers(0, 40, n)
    lens[[3, 77, 150]] = [1900, 1300, 700]  # split rows (chunk 512)
    lens[[10, 11]] = 0
    rows, cols = [], []
    for i, m in enumerate(lens):
        c = np.sort(rng.choice(d, size=int(m), replace=False))
        rows += [i] * int(m)
        cols += list(c)
    rows, cols = np.array(rows), np.array(cols)
    vals = rng.standard_normal(rows.size)
    A = np.zeros((n, d))
    A[rows, cols] = vals
    indptr = np.zeros(n + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(np.bincount(rows, minlength=n))
    dev = "cuda"
    ip = torch.from_numpy(indptr).to(dev, torch.int32)
    cl = torch.from_numpy(cols).to(dev, torch.int32)
    vl = torch.from_numpy(vals).to(dev, dtype)
    B = rng.standard_normal((d, nb))
    C0 = rng.standard_normal((n, nb))
    Bt = torch.from_numpy(B).to(dev, dtype)
    Ct = torch.from_numpy(C0).to(dev, dtype)
    plan = ops.SpmmPlan(ip)
    assert plan.nsplit == 3
    ops.spmm_csr_plan(plan, cl, vl, Bt, Ct, alpha=0.5, beta=2.0)
    ref = 0.5 * (A @ B) + 2.0 * C0
    tol = 1e-4 if dtype == torch.float32 else 1e-12
    assert np.max(np.abs(Ct.cpu().double().numpy() - ref)) < tol * np.abs(ref).max()


@pytest.mark.parametrize("nb", [8, 100, 300])
def test_csr_hybrid_hot_columns(ops, nb):
    """Hybrid CSR operator: Zipf-head columns (here every 7th of the first
    140 columns is dense-ish, plus a fully dense column and an empty one)
    densified into a tensor-core panel, the rest gathered; A X and A^T Y
    against dense FP64 products and against the pure-CSR operator."""
    from paper_1504_05477_b200.operators import CsrDeviceOp

    rng = np.random.default_rng(nb + 1)
    n, d = 3000, 5000
    A = np.zeros((n, d))
    mask = rng.random((n, d)) < 0.004
    mask[:, 0:140:7] |= rng.random((n, 20)) < 0.3
    mask[:, 5] = True
    mask[:, 6] = False
    A[mask] = rng.lognormal(0, 1, int(mask.sum()))
    indptr = np.zeros(n + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(mask.sum(1))
    rows, cols = np.nonzero(mask)
    ip = torch.from_numpy(indptr).cuda().to(torch.int32)
    cl = torch.from_numpy(cols).cuda().to(torch.int32)
    vl = torch.from_numpy(A[rows, cols]).cuda().float()
    hyb = CsrDeviceOp(ip, cl, vl, d)
    pure = CsrDeviceOp(ip, cl, vl, d, hot_density=0.0)
    assert hyb.hot is not None and hyb.hot["H"] >= 21 and pure.hot is None
    assert hyb.nnz == pure.nnz == int(mask.sum())
    X = rng.standard_normal((d, nb))
    Y = rng.standard_normal((n, nb))
    Xt, Yt = torch.from_numpy(X).cuda().float(), torch.from_numpy(Y).cuda().float()
    A32 = A.astype(np.float32).astype(np.float64)
    for op in (hyb, pure):
        out = torch.empty((n, nb), device="cuda")
        op.apply(Xt, out)
        ref = A32 @ Xt.double().cpu().numpy()
        assert np.max(np.abs(out.double().cpu().numpy() - ref)) < 2e-6 * np.abs(ref).max()
        out_t = torch.empty((d, nb), device="cuda")
        op.apply_t(Yt, out_t)
        ref_t = A32.T @ Yt.double().cpu().numpy()
        assert np.max(np.abs(out_t.double().cpu().numpy() - ref_t)) < 2e-6 * np.abs(ref_t).max()
        # FP64 output from FP32 operands (the chain's mixed-precision call)
        out64 = torch.empty((d, nb), dtype=torch.float64, device="cuda")
        op.apply_t(Yt, out64)
        assert np.max(np.abs(out64.cpu().numpy() - ref_t)) < 2e-6 * np.abs(ref_t).max()
