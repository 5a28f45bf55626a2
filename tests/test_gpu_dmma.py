"""FP64 tensor-core (DMMA) products against FP64 numpy and the CUDA-core FP64
kernels (the reference's FP64 `mm`, _kernels.pyx:56-71, is the contract):
ragged shapes, padded leading dimensions, epilogues and the device predicate."""

import numpy as np
import pytest
import torch

import rsvd_oracle as o

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    from paper_1504_05477_b200 import device

    return device


def _g(shape, seed):
    return o.gaussian(*shape, o.SeededRng(seed))


def _padded(a, pad):
    """Device copy of `a` whose rows are `pad` elements longer (lda > cols)."""
    m, k = a.shape
    buf = torch.zeros((m, k + pad), dtype=torch.float64, device="cuda")
    buf[:, :k] = torch.from_numpy(a).cuda()
    return buf[:, :k]


@pytest.mark.parametrize("algo", ["dmma", "simt"])
@pytest.mark.parametrize("m,n,k,pad", [(1, 1, 1, 0), (129, 33, 17, 3), (2000, 20, 1000, 0), (5000, 50, 3001, 1),
                                       (777, 64, 16, 0), (300, 200, 65, 5), (64, 8, 4, 0), (257, 50, 31, 1), (40000, 64, 300, 0)])
def test_gemm_nn_f64_algos(ops, algo, m, n, k, pad):
    from paper_1504_05477_b200._lib import GEMM_DMMA, GEMM_SIMT

    a, b, c0, rs = _g((m, k), 11), _g((k, n), 12), _g((m, n), 13), _g((1, n), 14)[0]
    A = _padded(a, pad)
    C = torch.from_numpy(c0).cuda()
    ops.gemm_nn(A, torch.from_numpy(b).cuda(), C, alpha=0.75, beta=0.5,
                row_sub=torch.from_numpy(rs).cuda(), algo=GEMM_DMMA if algo == "dmma" else GEMM_SIMT)
    ref = 0.75 * (a @ b - rs[None, :]) + 0.5 * c0
    err = np.max(np.abs(C.cpu().numpy() - ref))
    assert err <= 1e-13 * np.sqrt(k) * max(1.0, np.abs(ref).max()), err


@pytest.mark.parametrize("out", [torch.float64, torch.float32])
@pytest.mark.parametrize("m,n,k,pad", [(1, 3, 2, 0), (5000, 20, 64, 2), (2000, 200, 1000, 0), (100000, 7, 33, 0),
                                       (50000, 50, 130, 1), (17, 65, 129, 0), (3001, 50, 31, 1)])
def test_gemm_tn_f64_dmma(ops, m, n, k, pad, out):
    from paper_1504_05477_b200._lib import GEMM_DMMA

    a, b = _g((m, k), 21), _g((m, n), 22)
    mu = a.mean(axis=0)
    B = torch.from_numpy(b).cuda()
    cs = ops.colreduce(B, square=False)
    C = torch.empty((k, n), dtype=out, device="cuda")
    ops.gemm_tn(_padded(a, pad), B, C, mu=torch.from_numpy(mu).cuda(), colsum_b=cs, algo=GEMM_DMMA)
    ref = (a - mu[None, :]).T @ b
    tol = 1e-12 * np.sqrt(m) if out == torch.float64 else 2e-7 * max(1.0, np.abs(ref).max())
    err = np.max(np.abs(C.double().cpu().numpy() - ref))
    assert err <= tol, err


def test_dmma_matches_simt_closely(ops):
    """Same FP64 arithmetic, different summation order: agreement at 1e-14
    relative on a well-conditioned product (both are FP64-exact FMAs)."""
    from paper_1504_05477_b200._lib import GEMM_DMMA, GEMM_SIMT

    a, b = _g((3000, 800), 31), _g((800, 50), 32)
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    C1 = torch.empty((3000, 50), dtype=torch.float64, device="cuda")
    C2 = torch.empty_like(C1)
    ops.gemm_nn(A, B, C1, algo=GEMM_DMMA)
    ops.gemm_nn(A, B, C2, algo=GEMM_SIMT)
    assert torch.max(torch.abs(C1 - C2)).item() <= 1e-13 * torch.max(torch.abs(C2)).item()
    # TN, deterministic: two runs are bit-identical
    Y = torch.from_numpy(_g((3000, 50), 33)).cuda()
    W1 = torch.empty((800, 50), dtype=torch.float64, device="cuda")
    W2 = torch.empty_like(W1)
    ops.gemm_tn(A, Y, W1, algo=GEMM_DMMA)
    ops.gemm_tn(A, Y, W2, algo=GEMM_DMMA)
    assert torch.equal(W1, W2)


def test_dmma_predicate_skips(ops):
    from paper_1504_05477_b200._lib import GEMM_DMMA

    a, b = _g((256, 64), 41), _g((64, 16), 42)
    C = torch.full((256, 16), 7.0, dtype=torch.float64, device="cuda")
    pred = torch.zeros(1, dtype=torch.int32, device="cuda")
    ops.gemm_nn(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), C, algo=GEMM_DMMA, pred=pred)
    assert torch.all(C == 7.0)
    pred.fill_(1)
    ops.gemm_nn(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), C, algo=GEMM_DMMA, pred=pred)
    assert np.allclose(C.cpu().numpy(), a @ b, rtol=0, atol=1e-12)


def test_dmma_rejects_fp32(ops):
    from paper_1504_05477_b200._lib import GEMM_DMMA

    A = torch.zeros((8, 8), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        ops.gemm_nn(A, A, torch.zeros_like(A), algo=GEMM_DMMA)


@pytest.mark.parametrize("m,n,k,pad", [(1, 1, 1, 0), (50000, 50, 50, 2), (777, 64, 128, 0), (300, 17, 33, 1),
                                       (129, 50, 100, 0), (5000, 64, 3, 3)])
def test_skinny_fp32_products(ops, m, n, k, pad):
    """FP32 CUDA-core products of the orthonormalization (V R^-1, Grams):
    NN with k <= 128 / n <= 64 and TN with k, n <= 64, against FP64 numpy."""
    from paper_1504_05477_b200._lib import GEMM_SKINNY

    a = _g((m, k), 51).astype(np.float32)
    b = _g((k, n), 52).astype(np.float32)
    c0 = _g((m, n), 53).astype(np.float32)
    rs = _g((1, n), 54)[0]
    buf = torch.zeros((m, k + pad), dtype=torch.float32, device="cuda")
    buf[:, :k] = torch.from_numpy(a).cuda()
    A = buf[:, :k]
    C = torch.from_numpy(c0).cuda()
    ops.gemm_nn(A, torch.from_numpy(b).cuda(), C, alpha=-1.0, beta=1.0, row_sub=torch.from_numpy(rs).cuda(),
                algo=GEMM_SKINNY)
    ref = -(a.astype(np.float64) @ b.astype(np.float64) - rs[None, :]) + c0
    scale = np.abs(a).max() * np.abs(b).max() * k + np.abs(c0).max()
    assert np.max(np.abs(C.cpu().numpy() - ref)) <= 4e-7 * scale
    if k <= 64:
        y = _g((m, n), 55).astype(np.float32)
        G = torch.empty((k, n), dtype=torch.float64, device="cuda")
        ops.gemm_tn(A, torch.from_numpy(y).cuda(), G, algo=GEMM_SKINNY)
        ref = a.astype(np.float64).T @ y.astype(np.float64)
        assert np.max(np.abs(G.cpu().numpy() - ref)) <= 1e-6 * max(1.0, np.abs(ref).max())
