"""Phase timing of the public-API call factorize(A_host_pinned) at a bench
config (argv[1], default c2) in its bench precision mode. GPU only."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import bench
import paper_1504_05477_b200 as rk
from paper_1504_05477_b200 import rsvd
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfgd = bench.CONFIGS[name]
A = bench.make_matrix(cfgd, "cuda")
Ah = A.cpu().pin_memory(); del A
cfg = rk.RsvdConfig(k=cfgd["k"], variant=cfgd["variant"], q=cfgd["q"], seed=0)
kw = dict(center=bool(cfgd.get("pca")), precision=cfgd["mode"])
call = lambda X: rk.factorize(X, cfg, **kw)  # noqa: E731
for _ in range(3):
    call(Ah)
torch.cuda.synchronize()
key = list(rsvd._GRAPH_CACHE.keys())[0]
buf, op, graphed, pi, _ = rsvd._GRAPH_CACHE[key]
def tm(f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize(); return r, (time.perf_counter() - t0) * 1e3
_, t_up = tm(lambda: buf.copy_(Ah, non_blocking=True))
_, t_fin = tm(lambda: rsvd._upload_into(buf, Ah))
df, t_g = tm(lambda: graphed.run(pi))
_, t_finish = tm(lambda: rsvd._finish(df, cfg, time.perf_counter()))
_, t_total = tm(lambda: call(Ah))
gb = Ah.numel() * Ah.element_size() / 1e9
print(f"{name}: upload {t_up:.1f} ms ({gb/t_up*1e3:.1f} GB/s), upload+validate {t_fin:.1f}, graph {t_g:.1f}, finish {t_finish:.1f}, total call {t_total:.1f} ms")
# timers around the real call path
T = {}
def wrap(mod, name):
    f = getattr(mod, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(*a, **k); torch.cuda.synchronize()
        T[name] = T.get(name, 0) + (time.perf_counter() - t0) * 1e3
        return r
    setattr(mod, name, g)
for nm in ("_graph_cache_key", "_upload_into", "_finish"):
    wrap(rsvd, nm)
GR = rsvd.GraphedFactorization.run
def grun(self, *a, **k):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = GR(self, *a, **k); torch.cuda.synchronize()
    T["graph.run"] = T.get("graph.run", 0) + (time.perf_counter() - t0) * 1e3
    return r
rsvd.GraphedFactorization.run = grun
An = Ah.numpy().copy()  # pageable
for label, X in (("pinned", Ah), ("numpy", An), ("numpy", An)):
    T.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    call(X)
    torch.cuda.synchronize()
    print(label, "call", round((time.perf_counter() - t0) * 1e3, 1), {k: round(v, 1) for k, v in T.items()}, flush=True)
