"""The reference's own entry-point behaviour suite (pkg/tests/test_rsvd.py:88-262:
simultaneous iteration, block Krylov, sketch-and-solve, post_process, result
invariants) run against the drop-in on the GPU: same inputs (the pinned
SeededRng / gaussian / synth_matrix streams), same calls, same tolerances.
The reference's host-side helpers the cases lean on (dense_svd_reference,
qr_orthonormalize, frob_error_ratio) are numpy here: they are checkers, not the
path under test. float64 inputs -> the FP64 (DMMA) path; the tiny shapes
(3 x 3, 20 x 20, 30 x 20 ...) are the edge cases of every tile size."""

import numpy as np
import pytest

import rsvd_oracle as o

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rk():
    import paper_1504_05477_b200 as rk

    return rk


def _g(rk, rows, cols, seed):
    return rk.gaussian(rows, cols, rk.SeededRng(seed)).data


def _orth_err(z):
    return np.max(np.abs(z.T @ z - np.eye(z.shape[1])))


def _qr(x):
    q, _ = np.linalg.qr(x)
    return q


# ---- simultaneous iteration (test_rsvd.py:88-130) ---------------------------


@pytest.mark.parametrize("seed", [0, 3, 4, 6, 7])
def test_si_dominant_direction_on_diagonal(rk, seed):
    a = np.diag([3.0, 2.0, 1.0])
    r = rk.simultaneous_iteration(a, rk.RsvdConfig(k=1, variant="si", q=11, seed=seed))
    assert 3.0 - 1e-6 <= r.approx_singular_values[0] <= 3.0 + 1e-12
    assert abs(r.Z.data[0, 0]) > 1 - 1e-6


def test_si_orthonormal_output(rk):
    a = _g(rk, 60, 40, 50)
    r = rk.simultaneous_iteration(a, rk.RsvdConfig(k=6, variant="si", q=4, seed=1))
    assert _orth_err(r.Z.data) < 1e-10
    ref = o.factorize(o.DenseOp(a), 6, "si", q=4, seed=1)
    assert np.max(np.abs(r.approx_singular_values - ref.sigma) / ref.sigma) < 1e-10


def test_si_bitwise_deterministic(rk):
    a = _g(rk, 30, 20, 51)
    cfg = rk.RsvdConfig(k=3, variant="si", q=5, seed=9)
    assert np.array_equal(rk.simultaneous_iteration(a, cfg).Z.data, rk.simultaneous_iteration(a, cfg).Z.data)


def test_si_rejections(rk):
    with pytest.raises(ValueError):
        rk.simultaneous_iteration(np.ones((3, 2)), rk.RsvdConfig(k=3, variant="si", q=1))
    with pytest.raises(ValueError):
        rk.simultaneous_iteration(np.eye(3), rk.RsvdConfig(k=1, variant="bk", q=1))


@pytest.mark.parametrize("every", [0, 1, 3])
def test_si_reorthonormalization_interval(rk, every):
    a = _g(rk, 25, 18, 52)
    cfg = rk.RsvdConfig(k=3, variant="si", q=6, seed=2, reorthonormalize_every=every)
    r = rk.simultaneous_iteration(a, cfg)
    assert _orth_err(r.Z.data) < 1e-10
    ref = o.factorize(o.DenseOp(a), 3, "si", q=6, seed=2, every=every)
    assert np.max(np.abs(r.approx_singular_values - ref.sigma) / ref.sigma) < 1e-9


# ---- block Krylov (test_rsvd.py:131-162) ------------------------------------


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_bk_diagonal_padded(rk, seed):
    a = np.zeros((20, 20))
    a[0, 0], a[1, 1], a[2, 2] = 3.0, 2.0, 1.0
    r = rk.block_krylov(a, rk.RsvdConfig(k=1, variant="bk", q=3, seed=seed))
    assert abs(r.approx_singular_values[0] - 3.0) < 1e-8


def test_bk_width_matches_blocks_and_saturation_cap(rk):
    # _bk_basis(op, 4, 3) -> 4 blocks, q_used 3; (20 x 12, p = 4, q = 50) -> 12 // 4 = 3 blocks, q_used 2
    a = _g(rk, 40, 30, 53)
    r = rk.block_krylov(a, rk.RsvdConfig(k=4, variant="bk", q=3, seed=7))
    assert r.q_used == 3 and _orth_err(r.Z.data) < 1e-10
    b = _g(rk, 20, 12, 54)
    r = rk.block_krylov(b, rk.RsvdConfig(k=4, variant="bk", q=50, seed=8))
    assert r.q_used == 2 and r.Z.data.shape == (20, 4)
    ref = o.factorize(o.DenseOp(b), 4, "bk", q=50, seed=8)
    assert ref.q_used == 2
    assert np.max(np.abs(r.approx_singular_values - ref.sigma) / ref.sigma) < 1e-9


def test_bk_block_width_beyond_rows_rejected(rk):
    a = _g(rk, 5, 30, 55)
    with pytest.raises(ValueError):
        rk.block_krylov(a, rk.RsvdConfig(k=5, variant="bk", q=1, p=6))


def test_bk_bitwise_deterministic(rk):
    a = _g(rk, 30, 20, 56)
    cfg = rk.RsvdConfig(k=3, variant="bk", q=3, seed=11)
    assert np.array_equal(rk.block_krylov(a, cfg).Z.data, rk.block_krylov(a, cfg).Z.data)


# ---- sketch-and-solve (test_rsvd.py:163-186) --------------------------------


def test_sketch_rank_one_forcing(rk):
    a = np.diag([1.0, 0.0, 0.0])
    r = rk.sketch_and_solve(a, rk.RsvdConfig(k=1, variant="sketch", seed=5))
    assert abs(abs(r.Z.data[0, 0]) - 1.0) < 1e-12
    assert abs(r.approx_singular_values[0] - 1.0) < 1e-12


def test_sketch_frobenius_ratio_at_least_one(rk):
    a = _g(rk, 50, 30, 57)
    s = np.linalg.svd(a, compute_uv=False)
    best = np.sqrt(np.sum(s[5:] ** 2))  # ||A - A_5||_F
    for seed in range(5):
        z = rk.sketch_and_solve(a, rk.RsvdConfig(k=5, variant="sketch", seed=seed)).Z.data
        assert np.linalg.norm(a - z @ (z.T @ a)) / best >= 1 - 1e-10


def test_q_zero_equivalence_across_variants(rk):
    a = _g(rk, 30, 22, 58)
    outs = [rk.factorize(a, rk.RsvdConfig(k=4, variant=v, q=0, seed=21)).Z.data for v in ("si", "bk", "sketch")]
    assert np.array_equal(outs[0], outs[2])
    assert np.array_equal(outs[1], outs[2])


# ---- post_process (test_rsvd.py:187-238) ------------------------------------


def _synth(rk, n, d, spectrum, seed):
    return rk.as_dense_array(rk.synth_matrix(rk.SyntheticSpec(n=n, d=d, spectrum=spectrum, seed=seed)))


def test_post_process_true_singular_basis_is_fixed_point(rk):
    a = _synth(rk, 20, 12, np.linspace(4.0, 1.0, 10), 60)
    u, s, _ = np.linalg.svd(a, full_matrices=False)
    z, sigma = rk.post_process(a, u[:, :5].copy(), 5)
    assert np.max(np.abs(sigma - s[:5])) < 1e-10
    for i in range(5):
        assert abs(abs(z.data[:, i] @ u[:, i]) - 1.0) < 1e-8


def test_post_process_full_identity_basis_recovers_svd(rk):
    a = _synth(rk, 25, 15, np.linspace(3.0, 0.9, 15), 61)
    u, s, _ = np.linalg.svd(a, full_matrices=False)
    z, sigma = rk.post_process(a, np.eye(25), 5)
    assert np.max(np.abs(sigma - s[:5]) / s[:5]) < 1e-8
    for i in range(5):
        assert abs(z.data[:, i] @ u[:, i]) > 1 - 1e-6


def test_post_process_prefix_beats_random_bases_in_span(rk):
    a = _g(rk, 25, 16, 62)
    q = _qr(_g(rk, 25, 8, 63))
    z, _ = rk.post_process(a, q, 6)
    rng = rk.SeededRng(64)
    for l in (1, 3, 6):
        zl = z.data[:, :l]
        err_z = np.linalg.norm(a - zl @ (zl.T @ a))
        for _ in range(50):
            y = _qr(q @ rk.gaussian(8, l, rng).data)
            assert err_z <= np.linalg.norm(a - y @ (y.T @ a)) + 1e-9


def test_post_process_rejections(rk):
    with pytest.raises(ValueError):
        rk.post_process(np.eye(4), np.eye(4)[:, :2].copy(), 3)
    with pytest.raises(ValueError):
        rk.post_process(np.eye(4), np.ones((4, 2)), 2)


def test_post_process_sign_canonicalization(rk):
    a = _g(rk, 20, 14, 65)
    z, _ = rk.post_process(a, _qr(_g(rk, 20, 5, 66)), 5)
    for j in range(5):
        col = z.data[:, j]
        assert col[np.argmax(np.abs(col))] > 0


# ---- result invariants (test_rsvd.py:239-265) -------------------------------


@pytest.mark.parametrize("variant", ["si", "bk", "sketch"])
def test_values_descending_and_bounded(rk, variant):
    a = _synth(rk, 30, 20, np.linspace(5.0, 0.5, 18), 67)
    r = rk.factorize(a, rk.RsvdConfig(k=6, variant=variant, q=3, seed=3))
    sv = r.approx_singular_values
    assert np.all(np.diff(sv) <= 0)
    assert np.all(sv <= 5.0 * (1 + 1e-8))
    assert np.all(sv >= 0)


def test_k_above_rank_still_returns_basis(rk):
    a = _g(rk, 20, 2, 68) @ _g(rk, 8, 2, 69).T  # rank 2, k = 4
    r = rk.factorize(a, rk.RsvdConfig(k=4, variant="si", q=3, seed=4))
    assert _orth_err(r.Z.data) < 1e-10
    assert r.approx_singular_values[3] < 1e-6 * r.approx_singular_values[0]


def test_wall_time_recorded(rk):
    r = rk.factorize(_g(rk, 30, 20, 70), rk.RsvdConfig(k=3, variant="bk", q=1, seed=0))
    assert r.wall_time_ms > 0.0


# ---- qr_orthonormalize (test_factor.py:19-53) -------------------------------


def test_qr_identity_unchanged(rk):
    assert np.array_equal(rk.qr_orthonormalize(np.eye(3)).data, np.eye(3))


def test_qr_rank_deficient_hand_case(rk):
    q = rk.qr_orthonormalize(np.array([[3.0, 0.0], [4.0, 0.0]])).data
    assert np.allclose(q[:, 0], [0.6, 0.8], atol=1e-15)
    assert abs(np.linalg.norm(q[:, 1]) - 1.0) < 1e-12  # replacement column
    assert abs(q[:, 0] @ q[:, 1]) < 1e-12


def test_qr_random_block_contract(rk):
    m = _g(rk, 50, 8, 4)
    q = rk.qr_orthonormalize(m).data
    assert _orth_err(q) < 1e-12
    assert np.linalg.norm(q @ (q.T @ m) - m) < 1e-10 * np.linalg.norm(m)
    # same basis as the reference's column-by-column _mgs (positive diagonal R: no sign freedom)
    assert np.max(np.abs(q - o.mgs(m))) < 1e-12


def test_qr_always_full_width_even_for_duplicates(rk):
    base = _g(rk, 30, 3, 5)
    q = rk.qr_orthonormalize(np.hstack([base, base, base])).data
    assert q.shape == (30, 9)
    assert _orth_err(q) < 1e-12
    ref = o.mgs(np.hstack([base, base, base]))
    assert np.max(np.abs(q[:, :3] - ref[:, :3])) < 1e-12
    # the six replaced columns come from the same seeded fill stream
    assert np.max(np.abs(q - ref)) < 1e-9


def test_qr_rows_less_than_cols_rejected(rk):
    with pytest.raises(ValueError):
        rk.qr_orthonormalize(np.ones((2, 3)))


def test_qr_deterministic_including_replacement(rk):
    m = np.array([[3.0, 0.0], [4.0, 0.0], [0.0, 0.0]])
    assert np.array_equal(rk.qr_orthonormalize(m).data, rk.qr_orthonormalize(m).data)


def test_qr_wider_than_one_block(rk):
    m = _g(rk, 700, 150, 6).copy()  # three blocks of QR_BLOCK columns, the last ragged
    m[:, 100] = m[:, 3] - 2.0 * m[:, 77]  # a dependent column in the second block
    q = rk.qr_orthonormalize(m).data
    assert _orth_err(q) < 1e-12
    ref = o.mgs(m)
    assert list(o.mgs.last_replaced) == [100]
    assert np.max(np.abs(q - ref)) < 1e-9


# ---- symmetric_eig (test_factor.py:55-100) ----------------------------------


def test_eig_diagonal(rk):
    res = rk.symmetric_eig(np.diag([2.0, 1.0]))
    assert res.eigenvalues.tolist() == [2.0, 1.0]
    assert np.array_equal(res.eigenvectors.data, np.eye(2))


def test_eig_exchange_matrix(rk):
    res = rk.symmetric_eig(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert np.allclose(res.eigenvalues, [1.0, -1.0], atol=1e-12)
    v = res.eigenvectors.data
    s = 1.0 / np.sqrt(2.0)
    assert np.allclose(np.abs(v), [[s, s], [s, s]], atol=1e-12)
    assert np.allclose(v.T @ v, np.eye(2), atol=1e-12)


@pytest.mark.parametrize("n,seed", [(6, 17), (9, 18), (40, 23)])
def test_eig_reconstruction_and_orthonormal_vectors(rk, n, seed):
    base = _g(rk, n, n, seed)
    m = 0.5 * (base + base.T)
    res = rk.symmetric_eig(m)
    v = res.eigenvectors.data
    assert np.max(np.abs(v @ np.diag(res.eigenvalues) @ v.T - m)) < 1e-10
    assert _orth_err(v) < 1e-10
    assert np.max(np.abs(res.eigenvalues - np.linalg.eigvalsh(m)[::-1])) < 1e-10


def test_eig_rejections(rk):
    with pytest.raises(ValueError):
        rk.symmetric_eig(np.ones((2, 3)))
    with pytest.raises(ValueError):
        rk.symmetric_eig(np.array([[0.0, 1.0], [0.0, 0.0]]))


def test_eig_nonconvergence_carries_residual(rk):
    base = _g(rk, 8, 8, 19)
    with pytest.raises(rk.ConvergenceError) as err:
        rk.symmetric_eig(0.5 * (base + base.T), tol=0.0, max_sweeps=1)
    assert err.value.residual is not None and err.value.residual > 0
