"""The reference's container / operator suite (pkg/tests/test_matrix.py:22-183,
288-306) against the drop-in's matrix.py: the seeded stream, gaussian,
DenseMatrix and SparseMatrixCSR invariants run on the host (no GPU needed: the
stream is the C ABI's host function); matmul / spmm / MatrixOperator /
frobenius_norm_sq run on the GPU (-m gpu)."""

import numpy as np
import pytest

import rsvd_oracle as o


@pytest.fixture(scope="module")
def rk():
    import paper_1504_05477_b200 as rk

    return rk


def _random_csr(rk, n, d, seed, density=0.1):
    rng = rk.SeededRng(seed)
    vals = rng.normal_fill(n * d)
    gate = rng.normal_fill(n * d)
    idx = np.nonzero(gate < np.quantile(gate, density))[0]
    return rk.SparseMatrixCSR.from_coo(n, d, idx // d, idx % d, vals[idx])


# ---- host side: SeededRng, gaussian, DenseMatrix (test_matrix.py:22-92) ------


def test_rng_seed_range_validated(rk):
    for bad in (-1, 1 << 64):
        with pytest.raises(ValueError):
            rk.SeededRng(bad)


def test_rng_streams(rk):
    assert np.array_equal(rk.SeededRng(42).normal_fill(1001), rk.SeededRng(42).normal_fill(1001))
    assert not np.array_equal(rk.SeededRng(1).normal_fill(64), rk.SeededRng(2).normal_fill(64))
    assert np.array_equal(rk.SeededRng(42).normal_fill(1001), o.SeededRng(42).normal_fill(1001))
    rng = rk.SeededRng(9)
    split = np.concatenate([rng.normal_fill(4), rng.normal_fill(2)])
    whole = rk.SeededRng(9).normal_fill(6)
    assert np.array_equal(split, whole)
    # 3 samples consume two full pairs; the next fill starts at pair 3
    rng = rk.SeededRng(9)
    rng.normal_fill(3)
    assert np.array_equal(rng.normal_fill(2), whole[4:6])


def test_gaussian_contract(rk):
    g = rk.gaussian(3, 2, rk.SeededRng(7))
    assert g.shape == (3, 2) and np.all(np.isfinite(g.data))
    x = rk.gaussian(1000, 1, rk.SeededRng(1)).data
    assert -0.15 < x.mean() < 0.15 and 0.8 < x.var() < 1.2
    assert np.array_equal(rk.gaussian(10, 4, rk.SeededRng(3)).data, rk.gaussian(10, 4, rk.SeededRng(3)).data)
    for rows, cols in [(0, 3), (3, 0), (0, 0)]:
        with pytest.raises(ValueError):
            rk.gaussian(rows, cols, rk.SeededRng(0))


def test_dense_matrix_contract(rk):
    with pytest.raises(ValueError):
        rk.DenseMatrix(np.array([[1.0, np.nan]]))
    with pytest.raises(ValueError):
        rk.DenseMatrix(np.array([[np.inf, 0.0]]))
    m = rk.DenseMatrix(np.ones((2, 2)))
    with pytest.raises(ValueError):
        m.data[0, 0] = 5.0
    src = np.ones((2, 2))
    rk.DenseMatrix(src)
    src[0, 0] = 3.0  # the caller's array stays writable


def test_sparse_invariants_enforced(rk):
    S = rk.SparseMatrixCSR
    with pytest.raises(ValueError):  # decreasing row_ptr
        S(2, 2, [0, 2, 1], [0, 1], [1.0, 1.0])
    with pytest.raises(ValueError):  # unsorted columns within a row
        S(1, 3, [0, 2], [2, 0], [1.0, 1.0])
    with pytest.raises(ValueError):  # explicit zero value
        S(1, 2, [0, 1], [0], [0.0])
    with pytest.raises(ValueError):  # column out of bounds
        S(1, 2, [0, 1], [2], [1.0])
    sp = S.from_coo(2, 2, [0, 0, 1, 1], [0, 0, 1, 1], [1.5, 2.0, 1.0, -1.0])
    assert sp.nnz == 1
    assert sp.toarray().tolist() == [[3.5, 0.0], [0.0, 0.0]]


def test_product_shape_checks_need_no_device(rk):
    with pytest.raises(ValueError):
        rk.matmul(np.ones((2, 3)), np.ones((2, 2)))
    sp = _random_csr(rk, 5, 4, 25)
    with pytest.raises(ValueError):
        rk.spmm(sp, np.ones((5, 2)))
    with pytest.raises(ValueError):
        rk.spmm(sp, np.ones((4, 2)), transpose_A=True)
    with pytest.raises(TypeError):
        rk.spmm(np.ones((4, 4)), np.ones((4, 2)))
    op = rk.as_operator(np.ones((3, 2)))
    assert rk.as_operator(op) is op and op.shape == (3, 2) and not op.is_sparse and op.nnz == 6


# ---- device side: matmul, spmm, MatrixOperator, Frobenius (:94-183, :288-306) -


@pytest.mark.gpu
def test_matmul_cases(rk):
    b = rk.gaussian(3, 4, rk.SeededRng(5))
    assert np.array_equal(rk.matmul(np.eye(3), b).data, b.data)
    assert rk.matmul(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[0.0], [1.0]])).data.tolist() == [[2.0], [4.0]]
    a = rk.gaussian(17, 9, rk.SeededRng(11)).data
    c = rk.gaussian(9, 5, rk.SeededRng(12)).data
    assert np.max(np.abs(rk.matmul(a, c).data - o.mm_naive(a, c))) < 1e-12  # the reference's fixed-order triple loop
    a = rk.gaussian(20, 30, rk.SeededRng(13)).data
    c = rk.gaussian(30, 8, rk.SeededRng(14)).data
    assert np.array_equal(rk.matmul(a, c).data, rk.matmul(a, c).data)


@pytest.mark.gpu
def test_spmm_cases(rk):
    eye = rk.SparseMatrixCSR.from_coo(3, 3, [0, 1, 2], [0, 1, 2], [1.0, 1.0, 1.0])
    b = rk.gaussian(3, 5, rk.SeededRng(2))
    assert np.array_equal(rk.spmm(eye, b).data, b.data)
    a = rk.SparseMatrixCSR.from_coo(2, 2, [0], [1], [2.0])
    assert rk.spmm(a, np.array([[1.0], [1.0]])).data.tolist() == [[2.0], [0.0]]
    sp = _random_csr(rk, 30, 20, 21)
    b = rk.gaussian(20, 6, rk.SeededRng(22)).data
    assert np.max(np.abs(rk.spmm(sp, b).data - sp.toarray() @ b)) < 1e-12
    sp = _random_csr(rk, 30, 20, 23)
    b = rk.gaussian(30, 4, rk.SeededRng(24)).data
    assert np.max(np.abs(rk.spmm(sp, b, transpose_A=True).data - sp.toarray().T @ b)) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("sparse", [False, True])
def test_matrix_operator_apply_and_transpose(rk, sparse):
    if sparse:
        m = _random_csr(rk, 40, 25, 26, density=0.2)
        dense = m.toarray()
    else:
        m = rk.gaussian(40, 25, rk.SeededRng(27))
        dense = m.data
    op = rk.as_operator(m)
    assert op.is_sparse == sparse and op.shape == (40, 25) and op.nnz == np.count_nonzero(dense)
    x = rk.gaussian(25, 7, rk.SeededRng(28)).data
    y = rk.gaussian(40, 3, rk.SeededRng(29)).data
    assert np.max(np.abs(op.apply(x) - dense @ x)) < 1e-12
    assert np.max(np.abs(op.apply_transpose(y) - dense.T @ y)) < 1e-12
    assert op.apply(x[:, 0]).shape == (40, 1)  # a vector is a one-column block
    with pytest.raises(ValueError):
        op.apply(y)
    with pytest.raises(ValueError):
        op.apply_transpose(x)
    assert np.array_equal(op.densify().data, dense)
    # the operator handle is accepted wherever a matrix is
    r1 = rk.block_krylov(op, rk.RsvdConfig(k=3, variant="bk", q=2, seed=1))
    r2 = rk.block_krylov(m, rk.RsvdConfig(k=3, variant="bk", q=2, seed=1))
    assert np.array_equal(r1.Z.data, r2.Z.data)


@pytest.mark.gpu
def test_frobenius(rk):
    assert rk.frobenius_norm_sq(np.diag([3.0, 2.0, 1.0])) == 14.0
    assert rk.frobenius_norm_sq(np.zeros((4, 3))) == 0.0
    a = rk.gaussian(20, 12, rk.SeededRng(31))
    want = float(np.sum(np.linalg.svd(a.data, compute_uv=False) ** 2))
    assert abs(rk.frobenius_norm_sq(a) - want) / want < 1e-10
    sp = _random_csr(rk, 12, 9, 33)
    assert abs(rk.frobenius_norm_sq(rk.MatrixOperator(sp)) - float(np.sum(sp.toarray() ** 2))) < 1e-12


# ---- synthetic inputs (test_synth.py) ----------------------------------------


def test_synthetic_spec_contract(rk):
    spec = rk.SyntheticSpec(n=8, d=6, spectrum=np.array([2.0, 1.0]), seed=3)
    again = rk.SyntheticSpec.from_dict(spec.to_dict())
    assert (again.n, again.d, again.seed) == (spec.n, spec.d, spec.seed)
    assert np.array_equal(again.spectrum, spec.spectrum)
    for bad in (np.array([1.0, 2.0]), np.array([1.0, -0.5]), np.array([])):  # ascending, negative, empty
        with pytest.raises(ValueError):
            rk.SyntheticSpec(n=4, d=4, spectrum=bad)
    with pytest.raises(ValueError):  # longer than min(n, d)
        rk.SyntheticSpec(n=3, d=5, spectrum=np.array([3.0, 2.0, 1.0, 0.5]))


@pytest.mark.gpu
def test_synth_matrix_cases(rk):
    a = rk.synth_matrix(rk.SyntheticSpec(n=3, d=3, spectrum=np.array([3.0, 2.0, 1.0]), seed=1))
    assert np.max(np.abs(rk.dense_svd_reference(a).singular_values - [3.0, 2.0, 1.0])) < 1e-10 * 3.0
    z = rk.synth_matrix(rk.SyntheticSpec(n=4, d=3, spectrum=np.zeros(3), seed=2))
    assert np.all(z.data == 0.0)
    spec = rk.SyntheticSpec(n=10, d=8, spectrum=np.linspace(2.0, 0.5, 6), seed=5)
    assert np.array_equal(rk.synth_matrix(spec).data, rk.synth_matrix(spec).data)
    want = o.synth_matrix(10, 8, np.linspace(2.0, 0.5, 6), seed=5)  # the reference's fixed-order triple loop
    assert np.max(np.abs(rk.synth_matrix(spec).data - want)) < 1e-14


@pytest.mark.gpu
def test_synth_adversarial_flat_top_spectral_floor(rk):
    # six equal top values at sqrt(10), tail of ones: every rank-5 projector
    # leaves spectral residual exactly sqrt(10) (exact oracle on the residual)
    spectrum = np.concatenate([np.full(6, np.sqrt(10.0)), np.ones(100)])
    a = rk.synth_matrix(rk.SyntheticSpec(n=106, d=106, spectrum=spectrum, seed=7))
    oracle = rk.dense_svd_reference(a)
    assert abs(oracle.singular_values[5] ** 2 - 10.0) < 1e-8
    rng = rk.SeededRng(8)
    for _ in range(5):
        z = rk.qr_orthonormalize(rk.gaussian(106, 5, rng)).data
        resid = a.data - z @ (z.T @ a.data)
        top = rk.dense_svd_reference(resid).singular_values[0]
        assert abs(top / oracle.singular_values[5] - 1.0) < 1e-6
