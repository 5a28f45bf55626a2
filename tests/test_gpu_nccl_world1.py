"""torch.distributed NCCL with one rank on the box's GPU: the bench's N > 1
code path (krylov.TorchComm allreduces on the launching stream, the
factorization captured as a CUDA graph WITH its NCCL collectives inside, the
eager fallback agreement) as far as a one-GPU box can take it. Runs in a
subprocess so that the process group does not leak into the other tests."""

import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent("""
    import os, sys
    sys.path.insert(0, %r)
    sys.path.insert(0, os.path.join(%r, "oracle"))
    import numpy as np, torch, torch.distributed as dist
    import rsvd_oracle as o
    import paper_1504_05477_b200 as rk
    from paper_1504_05477_b200 import krylov, rsvd
    from paper_1504_05477_b200.operators import DenseDeviceOp
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29600 + os.getpid() %% 300), RANK="0", WORLD_SIZE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    A64 = o.synth_matrix(1500, 300, 1.0 / np.arange(1, 301), seed=5, mm=o.mm_blas)
    for exact, variant, q in ((False, "bk", 6), (True, "bk", 4), (False, "si", 3)):
        A = torch.from_numpy(A64).cuda()
        if exact:
            A = A.float()
        cfg = rk.RsvdConfig(k=10, variant=variant, q=q, seed=0)
        comm = krylov.TorchComm(n_total=1500, row_offset=0)
        op = DenseDeviceOp(A, n_total=1500, comm=comm, exact=exact)
        base = rsvd.run_device(DenseDeviceOp(A, exact=exact), cfg)
        eager = rsvd.run_device(op, cfg, comm=comm)
        g = rsvd.GraphedFactorization(op, cfg, comm=comm)   # NCCL allreduces inside the capture
        for _ in range(3):
            df = g.run()
        torch.cuda.synchronize()
        s0, s1, s2 = (x.sigma.cpu().numpy() for x in (base, eager, df))
        assert np.max(np.abs(s1 - s0) / s0) < 1e-12, (variant, exact, "eager")
        assert np.max(np.abs(s2 - s0) / s0) < 1e-12, (variant, exact, "graph")
        assert float(df.zerr.cpu()[0]) < 1e-12
    dist.destroy_process_group()
    print("NCCL_WORLD1_OK")
""") % (ROOT, ROOT)


def test_torchcomm_nccl_one_rank_eager_and_graph_capture():
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, timeout=600)
    assert "NCCL_WORLD1_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
