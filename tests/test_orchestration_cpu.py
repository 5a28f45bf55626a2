"""CPU tests of the device orchestration (krylov.py) through a torch-CPU
test double of the op interface, and of the row-sharded path with
torch.distributed gloo at world size 2."""

import os

import numpy as np
import pytest
import torch

import cpu_ops
import rsvd_oracle as o
from paper_1504_05477_b200 import krylov


def _run(A, k, variant, q, seed=0, comm=None, n_total=None, row_offset=0, mu=None, every=1):
    op = cpu_ops.CpuDenseOp(torch.from_numpy(A), n_total=n_total, row_offset=row_offset, mu=mu)
    c = comm if comm is not None else krylov.LocalComm()
    p = k
    pi = torch.from_numpy(o.gaussian(A.shape[1], p, o.SeededRng(seed)))
    ws = krylov.Workspace("cpu", p)
    nt = op.n_total
    if variant == "bk":
        qe = o.resolve_q("bk", q)
        br = krylov.bk_basis(cpu_ops, c, op, pi, qe, ws, nt, row_offset)
        Q = br.Q
    elif variant == "si":
        Q = krylov.si_basis(cpu_ops, c, op, pi, q, every, ws, nt, row_offset)
    else:
        Q = krylov.sketch_basis(cpu_ops, c, op, pi, ws, nt, row_offset)
    sign_fn = None
    if comm is not None and comm.world > 1:
        from paper_1504_05477_b200.dist import sharded_canonicalize_signs

        sign_fn = lambda Z: sharded_canonicalize_signs(Z, comm, ops=cpu_ops)  # noqa: E731
    rr = krylov.rayleigh_ritz(cpu_ops, c, op, Q, k, nt, row_offset, sign_fn=sign_fn)
    return rr, Q


@pytest.mark.parametrize("variant,q", [("bk", 4), ("si", 5), ("sketch", 0)])
def test_orchestration_matches_oracle_fp64(variant, q):
    A = o.synth_matrix(300, 120, 1.0 / np.arange(1, 121), seed=2, mm=o.mm_blas)
    rr, Q = _run(A, 8, variant, q)
    ref = o.factorize(o.DenseOp(A), 8, variant, q=q, seed=0)
    assert np.max(np.abs(rr.sigma.numpy() - ref.sigma) / ref.sigma) < 1e-10
    Qn = Q.numpy()
    assert np.max(np.abs(Qn.T @ Qn - np.eye(Qn.shape[1]))) < 1e-12
    assert np.max(np.abs(rr.Z.numpy() - ref.Z)) < 1e-8
    assert float(rr.zerr[0]) < 1e-12


def test_deficient_krylov_basis_replacement():
    # rank-deficient chain (C1-like): the final orthonormalization must
    # deflate and refill, keeping an orthonormal n x w basis
    A = o.synth_matrix(400, 200, 1.0 / np.arange(1, 201), seed=0, mm=o.mm_blas)
    rr, Q = _run(A, 10, "bk", 9)
    ref = o.factorize(o.DenseOp(A), 10, "bk", q=9, seed=0)
    assert len(ref.replaced) > 0
    Qn = Q.numpy()
    assert Qn.shape == (400, 100)
    assert np.max(np.abs(Qn.T @ Qn - np.eye(100))) < 1e-12
    assert np.max(np.abs(rr.sigma.numpy() - ref.sigma) / ref.sigma) < 1e-10


def test_centering_double_matches_explicit():
    rng = np.random.default_rng(1)
    X = rng.uniform(-5, 5, 60) + rng.standard_normal((500, 60)) * np.exp(-np.arange(60) / 10.0)
    mu = torch.from_numpy(X.mean(0))
    rr, _ = _run(X, 6, "bk", 3, mu=mu)
    ref = o.factorize(o.DenseOp(X - X.mean(0)), 6, "bk", q=3, seed=0)
    assert np.max(np.abs(rr.sigma.numpy() - ref.sigma) / ref.sigma) < 1e-10


def _worker(rank, world, port, A, k, variant, q, out_path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = A.shape[0]
    lo, hi = krylov.shard_rows(n, world, rank)
    comm = krylov.TorchComm(n_total=n, row_offset=lo)
    rr, _ = _run(np.ascontiguousarray(A[lo:hi]), k, variant, q, comm=comm, n_total=n, row_offset=lo)
    from paper_1504_05477_b200.dist import gather_rows

    Z = gather_rows(rr.Z, comm)
    if rank == 0:
        np.savez(out_path, Z=Z.numpy(), sigma=rr.sigma.numpy(), zerr=rr.zerr.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("variant,q", [("bk", 5), ("si", 3)])
def test_row_sharded_gloo_world2_matches_unsharded(tmp_path, variant, q):
    import torch.multiprocessing as mp

    A = o.synth_matrix(401, 90, 1.0 / np.sqrt(np.arange(1, 91)), seed=4, mm=o.mm_blas)
    out = str(tmp_path / "r.npz")
    port = 29500 + (os.getpid() % 1000)
    mp.spawn(_worker, args=(2, port, A, 6, variant, q, out), nprocs=2, join=True)
    got = np.load(out)
    ref, _ = _run(A, 6, variant, q)
    assert np.max(np.abs(got["sigma"] - ref.sigma.numpy()) / ref.sigma.numpy()) < 1e-10
    assert np.max(np.abs(got["Z"] - ref.Z.numpy())) < 1e-8
    assert float(got["zerr"][0]) < 1e-12


def test_shard_rows_partition():
    for n in (1, 7, 1000003):
        for w in (1, 2, 3, 8):
            spans = [krylov.shard_rows(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
