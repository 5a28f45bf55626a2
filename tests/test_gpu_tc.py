"""The tcgen05 3xTF32 GEMMs (FP32 path) against FP64 references: shapes
covering partial tiles in M, N and K, both operand majors, split-K
reductions, epilogue options."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TC = 2  # RSVD_GEMM_TC_3XTF32


@pytest.fixture(scope="module")
def ops():
    from paper_1504_05477_b200 import device

    return device


def _r(shape, seed, scale=1.0):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(shape, generator=g, dtype=torch.float64) * scale)


def _rel(got, ref):
    return float((got.double() - ref).abs().max() / ref.abs().max())


@pytest.mark.parametrize("m,n,k", [(128, 8, 32), (1000, 50, 1000), (50000, 50, 10000), (4096, 200, 780),
                                   (333, 96, 68), (20000, 128, 600), (777, 600, 600), (130, 1, 40)])
def test_tc_nn(ops, m, n, k):
    A, B = _r((m, k), 1), _r((k, n), 2)
    A32, B32 = A.float().cuda(), B.float().cuda()
    C = torch.empty((m, n), dtype=torch.float32, device="cuda")
    ops.gemm_nn(A32, B32, C, algo=TC)
    ref = A32.double().cpu() @ B32.double().cpu()
    e = _rel(C.cpu(), ref)
    print(f"NN m={m} n={n} k={k} rel={e:.3e}")
    assert e < 5e-6, e


def test_tc_nn_epilogue(ops):
    m, n, k = 3000, 40, 500
    A, B, C0 = _r((m, k), 3), _r((k, n), 4), _r((m, n), 5)
    rs = _r((n,), 6)
    A32, B32 = A.float().cuda(), B.float().cuda()
    C = C0.float().cuda()
    ops.gemm_nn(A32, B32, C, alpha=-0.5, beta=2.0, row_sub=rs.cuda(), algo=TC)
    ref = -0.5 * (A32.double().cpu() @ B32.double().cpu() - rs.view(1, -1)) + 2.0 * C0.float().double()
    assert _rel(C.cpu(), ref) < 2e-6


def test_tc_nn_strided_views(ops):
    # A = a column window of a wider buffer (ld != k), 16B-aligned base
    m, w, k, n = 5000, 600, 200, 64
    Big = _r((m, w), 7).float().cuda()
    A = Big[:, 100:300]
    B = _r((k, n), 8).float().cuda()
    Cbig = torch.zeros((m, 128), dtype=torch.float32, device="cuda")
    C = Cbig[:, 32:96]
    ops.gemm_nn(A, B, C, algo=TC)
    ref = A.double().cpu() @ B.double().cpu()
    assert _rel(C.cpu(), ref) < 2e-6
    assert float(Cbig[:, :32].abs().max()) == 0.0 and float(Cbig[:, 96:].abs().max()) == 0.0


@pytest.mark.parametrize("m,n,k", [(32, 8, 128), (50000, 50, 10000), (10000, 600, 10000), (3000, 200, 4096),
                                   (1000, 7, 1000), (70001, 64, 132)])
@pytest.mark.parametrize("out", [torch.float32, torch.float64])
def test_tc_tn(ops, m, n, k, out):
    A, B = _r((m, k), 9), _r((m, n), 10)
    A32, B32 = A.float().cuda(), B.float().cuda()
    C = torch.empty((k, n), dtype=out, device="cuda")
    ops.gemm_tn(A32, B32, C, algo=TC)
    ref = A32.double().cpu().T @ B32.double().cpu()
    e = _rel(C.cpu(), ref)
    print(f"TN m={m} n={n} k={k} out={out} rel={e:.3e}")
    assert e < 5e-6, e


def test_tc_tn_centering(ops):
    m, k, n = 20000, 300, 24
    A = (_r((m, k), 11) + 3.0).float().cuda()
    B = _r((m, n), 12).float().cuda()
    mu = A.double().mean(0)
    cs = ops.colreduce(B, square=False)
    C = torch.empty((k, n), dtype=torch.float64, device="cuda")
    ops.gemm_tn(A, B, C, mu=mu, colsum_b=cs, algo=TC)
    ref = (A.double() - mu.view(1, -1)).T @ B.double()
    assert float((C - ref).abs().max() / ref.abs().max()) < 1e-5


def test_tc_deterministic(ops):
    A = _r((30000, 2000), 13).float().cuda()
    B = _r((30000, 50), 14).float().cuda()
    C1 = torch.empty((2000, 50), dtype=torch.float32, device="cuda")
    C2 = torch.empty_like(C1)
    ops.gemm_tn(A, B, C1, algo=TC)
    ops.gemm_tn(A, B, C2, algo=TC)
    assert torch.equal(C1, C2)


def test_auto_dispatch_falls_back_on_misaligned(ops):
    # lda % 4 != 0 -> TMA cannot map it; AUTO must route to the CUDA-core kernel
    A = _r((500, 77), 15).float().cuda()
    B = _r((77, 20), 16).float().cuda()
    C = torch.empty((500, 20), dtype=torch.float32, device="cuda")
    ops.gemm_nn(A, B, C)
    assert _rel(C.cpu(), A.double().cpu() @ B.double().cpu()) < 5e-6
    with pytest.raises(ValueError):
        ops.gemm_nn(A, B, C, algo=TC)


@pytest.mark.parametrize("off", [1, 2, 3])
def test_tc_rejects_misaligned_a_and_auto_falls_back(ops, off):
    # TMA needs 16-byte aligned boxes: a column window starting off floats
    # into an aligned buffer must not take the tensor-core path
    n, w, p = 9000, 400, 50
    Big = _r((n, w), 20 + off).float().cuda()
    V = Big[:, off:off + p]
    T = _r((p, p), 30).float().cuda()
    C = torch.empty((n, p), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        ops.gemm_nn(V, T, C, algo=TC)
    ops.gemm_nn(V, T, C)
    assert _rel(C.cpu(), V.double().cpu() @ T.double().cpu()) < 5e-6


@pytest.mark.parametrize("m,n,k,mode", [(1000, 100, 300, "plain"), (4133, 200, 96, "axpby"), (640, 72, 2048, "rowsub"),
                                        (50000, 104, 50, "axpby")])
def test_nn_epilogue_emits_split_planes(m, n, k, mode):
    """rsvd_gemm_nn_f32_emit: the tcgen05 NN product also writes its output's hi /
    lo split planes from the epilogue. They equal (bitwise) the planes
    rsvd_split_planes cuts from the stored C -- ragged last row block and column
    tile included -- and a TN product fed with them equals the one that splits B
    itself; every epilogue variant (plain, alpha / beta, centred row_sub)."""
    from paper_1504_05477_b200 import device as ops

    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    A = torch.randn((m, k), generator=g, device="cuda")
    B = torch.randn((k, n), generator=g, device="cuda")
    C0 = torch.randn((m, n), generator=g, device="cuda")
    kw = {}
    if mode == "axpby":
        kw = dict(alpha=-1.0, beta=1.0)
    if mode == "rowsub":
        kw = dict(row_sub=torch.randn((1, n), generator=g, device="cuda", dtype=torch.float64))
    Cref = C0.clone()
    ops.gemm_nn(A, B, Cref, **kw)
    C = C0.clone()
    pl = ops.SplitPlanes.get(m, n, "cuda")
    pl.invalidate()
    ops.gemm_nn(A, B, C, emit=pl, **kw)
    assert torch.equal(C, Cref)
    if k <= 64:
        # the skinny CUDA-core path took this shape: nothing emitted, and a TN
        # product offered the stale planes splits B itself
        assert not pl.describes(C)
        Q = torch.randn((m, 136), generator=g, device="cuda")
        o1, o2 = torch.empty((136, n), device="cuda"), torch.empty((136, n), device="cuda")
        ops.gemm_tn(Q, C, o1)
        ops.gemm_tn(Q, C, o2, b_planes=pl)
        assert torch.equal(o1, o2)
        return
    assert pl.describes(C)
    nbytes = int(ops.lib().rsvd_split_planes_bytes(m, n))
    emitted = pl.buf[:nbytes].clone()
    ref = ops.SplitPlanes(nbytes, "cuda")
    ref.buf.zero_()
    ref.split(C)
    # compare the written region: plane rows (columns of C) < n of every k-block
    Kp, Np = (m + 31) // 32 * 32, (n + 31) // 32 * 32
    e = emitted.view(torch.float32).view(Kp // 32, 2, Np, 32)[:, :, :n, :]
    r = ref.buf[:nbytes].view(torch.float32).view(Kp // 32, 2, Np, 32)[:, :, :n, :]
    assert torch.equal(e, r)
    # the TN product on the emitted planes
    Q = torch.randn((m, 136), generator=g, device="cuda")
    out1 = torch.empty((136, n), device="cuda")
    out2 = torch.empty((136, n), device="cuda")
    ops.gemm_tn(Q, C, out1)
    ops.gemm_tn(Q, C, out2, b_planes=pl)
    assert torch.equal(out1, out2)
    G1 = torch.empty((n, n), dtype=torch.float64, device="cuda")
    G2 = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ops.gram(C, G1)
    ops.gram(C, G2, b_planes=pl)
    assert torch.equal(G1, G2)
    # planes of another tensor are ignored
    other = C.clone()
    out3 = torch.empty((136, n), device="cuda")
    ops.gemm_tn(Q, other, out3, b_planes=pl)
    assert torch.equal(out1, out3)
