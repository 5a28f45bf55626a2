"""The reference's metric and oracle-SVD suites (pkg/tests/test_metrics.py:38-158,
197-233; test_factor.py:101-143) against the drop-in: the same calls with the
oracle object the reference passes (dense_svd_reference's SvdResult), the same
inputs and tolerances. Everything here computes on the GPU."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rk():
    import paper_1504_05477_b200 as rk

    return rk


@pytest.fixture(scope="module")
def diag_case(rk):
    a = np.diag([3.0, 2.0, 1.0])
    return a, rk.dense_svd_reference(a)


@pytest.fixture(scope="module")
def random_case(rk):
    a = rk.synth_matrix(rk.SyntheticSpec(n=30, d=20, spectrum=np.linspace(4.0, 0.8, 18), seed=70))
    return a, rk.dense_svd_reference(a)


E2 = np.array([[0.0], [1.0], [0.0]])


def _rand_basis(rk, cols, rng):
    return rk.qr_orthonormalize(rk.gaussian(30, cols, rng)).data


# ---- dense_svd_reference (test_factor.py:101-143) ----------------------------


def test_oracle_svd_diagonal_and_rank_one(rk):
    res = rk.dense_svd_reference(np.diag([3.0, 2.0, 1.0]))
    assert np.allclose(res.singular_values, [3.0, 2.0, 1.0], atol=1e-12)
    assert np.allclose(np.abs(res.U.data), np.eye(3), atol=1e-10)
    assert np.allclose(np.abs(res.V.data), np.eye(3), atol=1e-10)
    res = rk.dense_svd_reference(np.array([[2.0], [0.0]]) @ np.array([[0.0], [3.0]]).T)
    assert res.rank == 1 and abs(res.singular_values[0] - 6.0) < 1e-12
    assert rk.dense_svd_reference(np.zeros((4, 3))).rank == 0


@pytest.mark.parametrize("n,d,seed", [(40, 25, 21), (15, 40, 22)])
def test_oracle_svd_reconstruction(rk, n, d, seed):
    a = rk.gaussian(n, d, rk.SeededRng(seed)).data
    res = rk.dense_svd_reference(a)
    recon = res.U.data @ np.diag(res.singular_values) @ res.V.data.T
    assert np.linalg.norm(recon - a) < 1e-8 * np.linalg.norm(a)
    assert np.all(np.diff(res.singular_values) <= 0)


def test_oracle_svd_matches_lapack_and_guard(rk):
    a = rk.gaussian(30, 18, rk.SeededRng(23)).data
    want = np.linalg.svd(a, compute_uv=False)
    assert np.max(np.abs(rk.dense_svd_reference(a).singular_values - want)) < 1e-10 * want[0]
    with pytest.raises(ValueError, match="guard"):
        rk.dense_svd_reference(rk.gaussian(12, 12, rk.SeededRng(24)).data, dim_limit=10)


# ---- Frobenius ratio (test_metrics.py:38-65) ---------------------------------


def test_frob_ratio(rk, diag_case, random_case):
    a, oracle = random_case
    assert abs(rk.frob_error_ratio(a, oracle.U.data[:, :5], oracle) - 1.0) < 1e-10
    rng = rk.SeededRng(71)
    for _ in range(10):
        assert rk.frob_error_ratio(a, _rand_basis(rk, 4, rng), oracle) >= 1 - 1e-10
    d, od = diag_case
    assert abs(rk.frob_error_ratio(d, E2, od) - math.sqrt(2.0)) < 1e-12
    with pytest.raises(ValueError):
        rk.frob_error_ratio(d, np.ones((3, 1)) * 0.9, od)
    one = np.diag([1.0, 0.0, 0.0])
    assert rk.frob_error_ratio(one, np.array([[1.0], [0.0], [0.0]]), rk.dense_svd_reference(one)) == 1.0


# ---- spectral ratio (test_metrics.py:68-90) ----------------------------------


def test_spectral_ratio(rk, diag_case, random_case):
    a, oracle = random_case
    assert abs(rk.spectral_error_ratio(a, oracle.U.data[:, :5], oracle) - 1.0) < 1e-6
    rng = rk.SeededRng(72)
    for _ in range(5):
        assert rk.spectral_error_ratio(a, _rand_basis(rk, 4, rng), oracle) >= 1 - 1e-6
    d, od = diag_case
    assert abs(rk.spectral_error_ratio(d, E2, od) - 1.5) < 1e-6
    one = np.diag([1.0, 0.0, 0.0])
    assert rk.spectral_error_ratio(one, np.array([[1.0], [0.0], [0.0]]), rk.dense_svd_reference(one)) == 1.0


# ---- per-vector errors (test_metrics.py:93-121) ------------------------------


def test_per_vector(rk, diag_case, random_case):
    a, oracle = random_case
    assert np.max(rk.per_vector_errors(a, oracle.U.data[:, :5], oracle)) < 1e-10
    d, od = diag_case
    assert abs(rk.per_vector_errors(d, E2, od)[0] - 1.25) < 1e-12
    z = _rand_basis(rk, 4, rk.SeededRng(73))
    flipped = z * np.array([1.0, -1.0, 1.0, -1.0])[None, :]
    assert np.array_equal(rk.per_vector_errors(a, z, oracle), rk.per_vector_errors(a, flipped, oracle))
    two = np.diag([2.0, 0.0, 0.0])
    o2 = rk.dense_svd_reference(two)
    assert rk.per_vector_errors(two, E2, o2)[0] == 4.0  # absolute, undivided
    rep = rk.compute_error_report(two, E2, o2)
    assert rep.absolute_per_vector and rep.exact_rank


# ---- error function (test_metrics.py:124-158) --------------------------------


def test_error_function(rk, diag_case, random_case):
    a, oracle = random_case
    assert abs(rk.error_function(a, oracle.U.data[:, :3], 3, oracle)) < 1e-9
    d, od = diag_case
    assert abs(rk.error_function(d, E2, 1, od) - 5.0) < 1e-12
    rng = rk.SeededRng(74)
    for _ in range(10):
        z = _rand_basis(rk, 5, rng)
        for l in (1, 3, 5):
            assert rk.error_function(a, z, l, oracle) >= -1e-9
    with pytest.raises(ValueError):
        rk.error_function(a, _rand_basis(rk, 3, rk.SeededRng(75)), 4, oracle)
    # telescoping: E_l - E_{l-1} = sigma_l^2 - ||A^T z_l||^2
    z = _rand_basis(rk, 5, rk.SeededRng(76))
    op = rk.as_operator(a)
    sv = oracle.singular_values
    for l in range(1, 6):
        delta = rk.error_function(a, z, l, oracle) - rk.error_function(a, z, l - 1, oracle)
        direct = float(sv[l - 1] ** 2) - float(np.sum(op.apply_transpose(z[:, l - 1: l]) ** 2))
        assert abs(delta - direct) < 1e-9 * sv[0] ** 2


# ---- error report (test_metrics.py:197-233) ----------------------------------


def test_error_report(rk, random_case):
    a, oracle = random_case
    r = rk.sketch_and_solve(a, rk.RsvdConfig(k=4, variant="sketch", seed=13))
    rep = rk.compute_error_report(a, r.Z, oracle, q=0, variant="sketch", seed=13)
    assert rep.k == 4 and rep.q == 0 and rep.seed == 13 and rep.variant == "sketch"
    assert rep.per_vector_max == float(np.max(rep.per_vector)) and not rep.exact_rank
    with pytest.raises(ValueError):
        rk.ErrorReport(frob_ratio=1.0, spectral_ratio=1.0, per_vector=np.array([0.5, 0.2]), per_vector_max=0.2,
                       exact_rank=False, absolute_per_vector=False, k=2)
    # rotation invariance
    z = _rand_basis(rk, 4, rk.SeededRng(78))
    w = rk.qr_orthonormalize(rk.gaussian(30, 30, rk.SeededRng(79))).data
    dense = rk.as_operator(a).densify().data
    r1 = rk.compute_error_report(a, z, oracle)
    r2 = rk.compute_error_report(w @ dense, w @ z, oracle)
    assert abs(r1.frob_ratio - r2.frob_ratio) < 1e-9
    assert abs(r1.spectral_ratio - r2.spectral_ratio) < 1e-9
    assert abs(r1.per_vector_max - r2.per_vector_max) < 1e-9


# ---- spectral_norm_est (test_factor.py:145-172) -------------------------------


def test_spectral_norm_est(rk):
    est = rk.spectral_norm_est(rk.as_operator(np.diag([3.0, 2.0, 1.0])), tol=1e-10, rng=rk.SeededRng(3))
    assert abs(est - 3.0) < 1e-8
    assert rk.spectral_norm_est(rk.as_operator(np.zeros((3, 3))), tol=1e-9, rng=rk.SeededRng(4)) == 0.0
    a = rk.gaussian(30, 20, rk.SeededRng(25))
    sigma1 = rk.dense_svd_reference(a).singular_values[0]
    assert abs(rk.spectral_norm_max_restarts(rk.as_operator(a), tol=1e-10) - sigma1) / sigma1 < 1e-6
    for seed in range(5):
        b = rk.gaussian(25, 15, rk.SeededRng(40 + seed))
        s1 = rk.dense_svd_reference(b).singular_values[0]
        assert rk.spectral_norm_max_restarts(rk.as_operator(b), tol=1e-9) <= s1 * (1 + 1e-8)
    with pytest.raises(ValueError):
        rk.spectral_norm_est(rk.as_operator(np.eye(2)), tol=0.0)
    # the same estimate as the reference algorithm run on the host (oracle restatement)
    import rsvd_oracle as o

    A = rk.gaussian(40, 30, rk.SeededRng(26)).data
    want = o.spectral_norm_est(lambda x: A @ x, lambda y: A.T @ y, 30, tol=1e-9, max_iters=10000, seed=101)
    got = rk.spectral_norm_est(A, tol=1e-9, rng=rk.SeededRng(101))
    assert abs(got - want) / want < 1e-12


# ---- additive spectral transfer (test_metrics.py:161-194) ---------------------


def test_additive_spectral_check(rk, random_case):
    a, oracle = random_case
    k = 4
    b = oracle.U.data[:, :k] @ np.diag(oracle.singular_values[:k]) @ oracle.V.data[:, :k].T
    res = rk.additive_spectral_check(a, b, k, oracle)
    assert res.passed and abs(res.eta) < 1e-9
    assert abs(res.spectral_sq - oracle.singular_values[k] ** 2) < 1e-9
    dense = rk.as_operator(a).densify().data
    r = rk.sketch_and_solve(a, rk.RsvdConfig(k=4, variant="sketch", seed=12))
    assert rk.additive_spectral_check(a, r.Z.data @ (r.Z.data.T @ dense), 4, oracle).passed
    rng = rk.SeededRng(77)
    for _ in range(20):
        y = _rand_basis(rk, 4, rng)
        assert rk.additive_spectral_check(a, y @ (y.T @ dense), 4, oracle).passed
    with pytest.raises(ValueError):
        rk.additive_spectral_check(a, dense, 4, oracle)
