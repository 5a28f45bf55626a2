import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
import numpy as np
import paper_1504_05477_b200 as rk
import rsvd_oracle as o
bad = 0
for seed in range(400):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(20, 60)); d = int(rng.integers(10, 40)); k = int(min(n, d, rng.integers(5, 30)))
    r = int(rng.integers(1, max(2, min(n, d) // 2 + 1)))
    A = rng.standard_normal((n, r)) @ rng.standard_normal((r, d))
    q = int(rng.integers(1, 6))
    for variant, every in (("si", 0), ("si", 1), ("bk", 1)):
        if variant == "bk" and k > n:
            continue
        try:
            res = rk.factorize(A, rk.RsvdConfig(k=k, variant=variant, q=q, seed=seed, reorthonormalize_every=every))
        except Exception as exc:
            bad += 1
            print(f"EXC seed={seed} {n}x{d} r={r} k={k} q={q} {variant} every={every}: {exc!r}"[:250], flush=True)
print("done", bad)
