"""Exercise bench.cpu_baseline_sparse on a small C3-like CSR (seconds), so a
crash in the parity block shows up before the full C3 reference run."""
import os
import sys
import types

import json

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1504_05477_b200 as rk  # noqa: E402
from paper_1504_05477_b200 import rsvd  # noqa: E402
from paper_1504_05477_b200.operators import CsrDeviceOp  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    cfgd = dict(n=6000, d=3000, k=20, q=3, sparse=True, variant="bk", mode="fp32")
    indptr, colv, valv = bench.make_csr(cfgd, dev)
    cfg = rk.RsvdConfig(k=20, variant="bk", q=3, seed=0)
    op = CsrDeviceOp(indptr, colv, valv, cfgd["d"])
    g = rsvd.GraphedFactorization(op, cfg)
    Pi = rk.gaussian(cfgd["d"], cfg.p, rk.SeededRng(0)).data
    df = g.run(Pi)
    torch.cuda.synchronize()
    args = types.SimpleNamespace(cpu_budget_sparse=120.0, no_spectral=False, spectral_iters=2000, no_fp64=False)
    res = bench.cpu_baseline_sparse(indptr, colv, valv, cfgd, cfg, Pi, args, df)
    print(json.dumps(res, indent=1))
    assert res["parity"]["pass"], res


if __name__ == "__main__":
    main()
