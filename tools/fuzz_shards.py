"""Randomized sweep of the row-sharded factorization as virtual shards on one
GPU (tests/test_gpu_shards.py's in-process communicator): random shapes, shard
counts 2..5 (ragged and single-row shards included), variants and modes,
against the unsharded run on the same device. GPU only.

    python tools/fuzz_shards.py [cases] [seed]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import paper_1504_05477_b200 as rk
import test_gpu_shards as ts

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
fails = 0
for it in range(cases):
    world = int(rng.integers(2, 6))
    n = int(rng.choice([rng.integers(world, 40), rng.integers(40, 600), rng.integers(600, 4000)]))
    d = int(rng.choice([rng.integers(2, 40), rng.integers(40, 600)]))
    k = int(rng.integers(1, min(n, d, 40) + 1))
    variant = str(rng.choice(["bk", "si", "sketch"]))
    q = int(rng.integers(0, 5))
    mode = str(rng.choice(["fp64", "exact", "fp32"]))
    kind = str(rng.choice(["gauss", "lowrank", "scaled"]))
    if kind == "lowrank":
        r = int(rng.integers(1, max(2, min(n, d) // 2 + 1)))
        A = rng.standard_normal((n, r)) @ rng.standard_normal((r, d))
    else:
        A = rng.standard_normal((n, d)) * (np.exp(rng.standard_normal((1, d))) if kind == "scaled" else 1.0)
    At = torch.from_numpy(A).cuda()
    if mode != "fp64":
        At = At.float()
    exact = mode == "exact"
    desc = f"case {it}: {n}x{d} world={world} k={k} {variant} q={q} {kind} mode={mode}"
    try:
        cfg = rk.RsvdConfig(k=k, variant=variant, q=q, seed=it)
        Z1, s1, d1, _ = ts._single(rk, At, cfg, exact)
        scale = max(float(s1.max()), 1e-300)
        tol = {"fp64": 1e-9, "exact": 1e-8, "fp32": 2e-4}[mode]
        if kind == "lowrank":
            tol = max(tol, 5e-8)
        for rank, (Z, s, dd, zerr) in enumerate(ts._sharded(rk, At, cfg, world, exact)):
            bad = []
            err = float(np.max(np.abs(s - s1))) / scale
            if not err <= tol:
                bad.append(f"sigma {err:.2e} > {tol}")
            if not zerr <= 1e-10:
                bad.append(f"zerr {zerr:.2e}")
            if not np.max(np.abs(Z.T @ Z - np.eye(k))) <= 1e-10:
                bad.append("Z^T Z")
            if dd != d1 and mode == "fp64":
                bad.append(f"replaced {dd} != {d1}")
            if bad:
                fails += 1
                print("FAIL", desc, f"rank {rank}:", "; ".join(bad), flush=True)
                break
    except Exception as exc:  # noqa: BLE001
        fails += 1
        print("EXC ", desc, repr(exc)[:300], flush=True)
print(f"{cases} cases, {fails} failures")
sys.exit(1 if fails else 0)
