"""The C ABI's per-device handle with a library-built NCCL communicator
(include/rsvd_b200.h section 8): one rank on the box's GPU (every gpurun box
has one), through the same factorization code the row-sharded path runs."""

import numpy as np
import pytest
import torch

import rsvd_oracle as o

pytestmark = pytest.mark.gpu


def test_handle_nccl_world1_allreduce_and_factorization():
    import paper_1504_05477_b200 as rk
    from paper_1504_05477_b200 import krylov, rsvd
    from paper_1504_05477_b200.operators import DenseDeviceOp

    uid = krylov.HandleComm.nccl_unique_id()
    assert len(uid) == 128
    comm = krylov.HandleComm("cuda:0", world=1, rank=0, unique_id=uid)
    for dt in (torch.float32, torch.float64):
        t = torch.randn((37, 5), device="cuda", dtype=dt)
        ref = t.clone()
        comm.allreduce(t)
        torch.cuda.synchronize()
        assert torch.equal(t, ref)  # one rank: the sum is the partial
    g = comm.all_gather(torch.arange(6, device="cuda", dtype=torch.int64))
    assert len(g) == 1 and torch.equal(g[0].cpu(), torch.arange(6))
    A = torch.from_numpy(o.synth_matrix(900, 300, 1.0 / np.arange(1, 301), seed=5, mm=o.mm_blas)).cuda()
    cfg = rk.RsvdConfig(k=10, variant="bk", q=6, seed=0)
    comm.n_total, comm.row_offset = 900, 0
    d1 = rsvd.run_device(DenseDeviceOp(A, n_total=900, comm=comm), cfg, comm=comm)
    d0 = rsvd.run_device(DenseDeviceOp(A), cfg)
    assert np.max(np.abs(d1.sigma.cpu().numpy() - d0.sigma.cpu().numpy()) / d0.sigma.cpu().numpy()) < 1e-12
