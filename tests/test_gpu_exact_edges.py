"""Exact mode (FP32 A, FP64-accurate int8 digit-plane products, the
reference's faithful basis) on the edge shapes the reference's own suite
exercises (test_rsvd.py: tiny and ragged matrices, k = min(n, d), width
capped by min(n, d) // p, rank-deficient and all-zero inputs, q = 0 sketch),
each against the oracle run on the same float32 A upcast to float64."""

import numpy as np
import pytest

import rsvd_oracle as o

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rk():
    import paper_1504_05477_b200 as rk

    return rk


def _check(rk, A32, k, variant, q, p=None, seed=0, tol=1e-9):
    A64 = A32.astype(np.float64)
    ref = o.factorize(o.DenseOp(A64), k, variant, q=q, p=p, seed=seed)
    cfg = rk.RsvdConfig(k=k, variant=variant, q=q, p=p, seed=seed)
    r = rk.factorize(A32, cfg)  # float32 input: exact mode by default
    assert r.q_used == ref.q_used
    s, sr = r.approx_singular_values, ref.sigma
    scale = max(sr.max(), 1e-300)
    assert np.max(np.abs(s - sr)) <= tol * scale, (s, sr)
    z = r.Z.data
    assert np.max(np.abs(z.T @ z - np.eye(z.shape[1]))) <= 1e-10
    return r, ref


@pytest.mark.parametrize("n,d,k,q", [(5, 3, 1, 2), (7, 7, 7, 0), (130, 33, 4, 3), (257, 129, 9, 5),
                                     (1000, 17, 5, 2), (33, 1000, 6, 4)])
def test_exact_ragged_and_tiny(rk, n, d, k, q):
    rng = np.random.default_rng(n * 31 + d)
    A = (rng.standard_normal((n, d)) * np.exp(rng.standard_normal((1, d)))).astype(np.float32)
    _check(rk, A, k, "bk", q)


def test_exact_width_capped_and_rank_deficient(rk):
    rng = np.random.default_rng(3)
    U = rng.standard_normal((400, 6))
    V = rng.standard_normal((6, 90))
    A = (U @ V).astype(np.float32)  # rank 6, cap min(n, d) // p = 4 blocks at p = 20
    r, ref = _check(rk, A, 20, "bk", 9, tol=1e-8)
    assert r.q_used == 3


def test_exact_all_zero_and_zero_rows(rk):
    A = np.zeros((300, 80), dtype=np.float32)
    r, _ = _check(rk, A, 5, "bk", 3)
    assert np.all(r.approx_singular_values == 0.0)
    rng = np.random.default_rng(9)
    B = rng.standard_normal((300, 80)).astype(np.float32)
    B[::7] = 0.0
    B[:, 11] = 0.0
    _check(rk, B, 8, "bk", 4)


def test_exact_wide_dynamic_range(rk):
    """Rows spanning 1e-30 .. 1e30 (per-row digit exponents) and FP32
    subnormal entries."""
    rng = np.random.default_rng(4)
    A = rng.standard_normal((500, 120)) * np.logspace(-30, 30, 500)[:, None]
    A[3, :5] = 1e-42  # FP32 subnormals
    _check(rk, A.astype(np.float32), 6, "bk", 3, tol=1e-8)


@pytest.mark.parametrize("variant,q", [("si", 4), ("sketch", 0)])
def test_exact_si_and_sketch(rk, variant, q):
    rng = np.random.default_rng(5)
    A = (rng.standard_normal((700, 300)) * (np.arange(1, 301) ** -0.7)).astype(np.float32)
    _check(rk, A, 10, variant, q, tol=1e-8)


def test_exact_host_inputs_pipelined_upload(rk, monkeypatch):
    """Public API, exact mode: a pinned host tensor and a pageable numpy array
    go through the panel-pipelined upload (digit planes cut per row panel as it
    lands, rsvd_oz_prepare_rows; panels forced small here, with a ragged last
    panel), a CUDA tensor through the one-shot path: identical digit planes, so
    the three results are bitwise equal. Non-finite input raises the
    reference's ValueError on every path (matrix.py:80-85)."""
    import torch

    from paper_1504_05477_b200 import rsvd

    monkeypatch.setattr(rsvd, "_PANEL_BYTES", 1 << 20)  # 1 MB panels: 7 panels + a ragged tail
    rng = np.random.default_rng(77)
    n, d = 6011, 300
    A = (rng.standard_normal((n, 40)) @ rng.standard_normal((40, d)) / 6.0
         + 1e-3 * rng.standard_normal((n, d))).astype(np.float32)
    cfg = rk.RsvdConfig(k=8, variant="bk", q=4, seed=0)
    outs = []
    for src in (A, torch.from_numpy(A).pin_memory(), torch.from_numpy(A).cuda()):
        for _ in range(2):  # second call of a shape replays the captured graph
            r = rk.factorize(src, cfg)
        outs.append((r.approx_singular_values.copy(), np.array(r.Z.data)))
    for s, z in outs[1:]:
        assert np.array_equal(s, outs[0][0]) and np.array_equal(z, outs[0][1])
    ref = o.factorize(o.DenseOp(A.astype(np.float64)), 8, "bk", q=4, seed=0)
    assert np.max(np.abs(outs[0][0] - ref.sigma)) <= 1e-9 * ref.sigma.max()
    bad = A.copy()
    bad[n - 3, 17] = np.nan
    for src in (bad, torch.from_numpy(bad).pin_memory(), torch.from_numpy(bad).cuda()):
        with pytest.raises(ValueError):
            rk.factorize(src, cfg)
    # and the cached graph still works afterwards
    r = rk.factorize(A, cfg)
    assert np.array_equal(r.approx_singular_values, outs[0][0])


@pytest.mark.parametrize("seed", [91, 104, 355, 385, 391])
def test_raw_power_blocks_of_rank_deficient_input(rk, seed):
    """simultaneous iteration without re-orthonormalization
    (reorthonormalize_every = 0, test_rsvd.py:123-128) on inputs of rank below
    k: the raw power block has exactly dependent columns whose Gram pivots are
    rounding noise. The result is a valid factorization (these cases raised
    'Z must have orthonormal columns' before the pivot-noise floor of round 1
    and the conditional re-orthonormalization of Z) and the singular values
    above the rank match the oracle."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(20, 60))
    d = int(rng.integers(10, 40))
    k = int(min(n, d, rng.integers(5, 30)))
    r = int(rng.integers(1, max(2, min(n, d) // 2 + 1)))
    A = rng.standard_normal((n, r)) @ rng.standard_normal((r, d))
    q = int(rng.integers(1, 6))
    res = rk.factorize(A, rk.RsvdConfig(k=k, variant="si", q=q, seed=seed, reorthonormalize_every=0))
    z = res.Z.data
    assert np.max(np.abs(z.T @ z - np.eye(k))) < 1e-10
    ref = o.factorize(o.DenseOp(A), k, "si", q=q, seed=seed, every=0)
    m = min(r, k)
    assert np.max(np.abs(res.approx_singular_values[:m] - ref.sigma[:m]) / ref.sigma[0]) < 1e-7
    assert np.all(res.approx_singular_values[m:] < 1e-6 * ref.sigma[0])


def test_fp32_mode_si_without_reorthonormalization(rk):
    """precision='fp32' with reorthonormalize_every = 0: FP32 blocks cannot carry
    raw powers (50 % sigma errors measured), so the mode orthonormalizes after
    every step; same span, singular values within the fp32 tolerance."""
    rng = np.random.default_rng(12)
    A = (rng.standard_normal((1196, 60)) @ rng.standard_normal((60, 501))).astype(np.float32)
    ref = o.factorize(o.DenseOp(A.astype(np.float64)), 38, "si", q=3, seed=5, every=0)
    res = rk.factorize(A, rk.RsvdConfig(k=38, variant="si", q=3, seed=5, reorthonormalize_every=0), precision="fp32")
    assert np.max(np.abs(res.approx_singular_values - ref.sigma) / ref.sigma[0]) < 1e-4
