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
