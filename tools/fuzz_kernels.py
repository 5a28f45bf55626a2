"""Randomized sweep of the product kernels behind the C ABI against FP64 torch
references: rsvd_gemm_nn / rsvd_gemm_tn (FP32 3xTF32 and FP64 DMMA; strided
views, alpha / beta, centering epilogues), rsvd_oz_gemm (digit-plane products),
the CSR operator (A X and A^T Y, FP32 and FP64, hybrid hot panel) and
rsvd_syev_topk. GPU only; exits 1 on any failure.

    python tools/fuzz_kernels.py [cases] [seed]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1504_05477_b200 import device as ops
from paper_1504_05477_b200.operators import CsrDeviceOp

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
dev = torch.device("cuda", 0)
fails = 0


def dim(big):
    return int(rng.choice([rng.integers(1, 10), rng.integers(10, 130), rng.integers(130, big)]))


def rnd(shape, dt, pad=0):
    """Random matrix as a column window of a wider buffer (row pitch != columns)."""
    m, n = shape
    off = int(rng.choice([0, 4, 8])) if pad else 0
    buf = torch.from_numpy(rng.standard_normal((m, n + pad + off))).to(device=dev, dtype=dt)
    return buf[:, off: off + n]


def rel(got, ref):
    return float((got.double() - ref).abs().max() / max(float(ref.abs().max()), 1e-300))


def report(name, desc, err, tol):
    global fails
    if not err <= tol:
        fails += 1
        print(f"FAIL {name} {desc}: {err:.3e} > {tol}", flush=True)


for it in range(cases):
    kind = str(rng.choice(["nn", "tn", "oz", "csr", "syev"]))
    try:
        if kind in ("nn", "tn"):
            dt = torch.float32 if rng.random() < 0.6 else torch.float64
            tol = 5e-6 if dt == torch.float32 else 1e-13
            m, n, k = dim(30000), dim(260), dim(3000)
            pad = int(rng.choice([0, 4, 12]))
            alpha, beta = (1.0, 0.0) if rng.random() < 0.5 else (float(rng.normal()), float(rng.normal()))
            if kind == "nn":
                A, B, C = rnd((m, k), dt, pad), rnd((k, n), dt, pad), rnd((m, n), dt, pad)
                rs = torch.from_numpy(rng.standard_normal((1, n))).to(dev) if rng.random() < 0.3 else None
                ref = alpha * (A.double() @ B.double() - (rs if rs is not None else 0.0)) + beta * C.double()
                ops.gemm_nn(A, B, C, alpha=alpha, beta=beta, row_sub=rs)
                scale = (A.double().abs() @ B.double().abs()).max()
            else:
                A, B = rnd((m, k), dt, pad), rnd((m, n), dt, pad)
                odt = torch.float64 if rng.random() < 0.5 else dt
                C = rnd((k, n), odt, pad)
                mu = cs = None
                if rng.random() < 0.3:
                    mu = torch.from_numpy(rng.standard_normal((k, 1))).to(dev)
                    cs = B.double().sum(dim=0).view(1, -1).contiguous()
                ref = alpha * (A.double().T @ B.double() - (mu @ cs if mu is not None else 0.0)) + beta * C.double()
                ops.gemm_tn(A, B, C, alpha=alpha, beta=beta, mu=None if mu is None else mu.view(-1),
                            colsum_b=None if cs is None else cs.view(-1))
                scale = (A.double().abs().T @ B.double().abs()).max()
            err = float((C.double() - ref).abs().max() / max(float(scale), 1e-300))
            report(kind, f"{dt} m={m} n={n} k={k} pad={pad} a={alpha:.2f} b={beta:.2f}", err, tol)
        elif kind == "oz":
            n, d, p = dim(20000), dim(3000), dim(200)
            A = rnd((n, d), torch.float32).contiguous() * torch.exp(torch.randn((n, 1), device=dev)).float()
            P = ops.OzPlanes(A)
            for trans in (0, 1):
                B = rnd((n if trans else d, p), torch.float64, 4)
                C = rnd((d if trans else n, p), torch.float64, 4)
                beta = float(rng.choice([0.0, 1.0, -0.7]))
                Ad = A.double()
                ref = 1.3 * ((Ad.T if trans else Ad) @ B) + beta * C
                scale = ((Ad.abs().T if trans else Ad.abs()) @ B.abs()).max()
                ops.oz_gemm(P, B, C, trans=trans, alpha=1.3, beta=beta)
                err = float((C - ref).abs().max() / float(scale))
                # A^T Y folds A's row exponents into Y before it is cut into 48-bit
                # digits: with e^+-3 row spreads the sum keeps ~1e-12 of |A|^T |Y|
                report("oz", f"n={n} d={d} p={p} trans={trans} beta={beta}", err, 5e-12 if trans else 5e-13)
        elif kind == "csr":
            n, d, nb = dim(20000), dim(5000), dim(260)
            dt = torch.float32 if rng.random() < 0.5 else torch.float64
            dens = float(rng.choice([0.002, 0.02, 0.2]))
            M = rng.standard_normal((n, d)) * (rng.random((n, d)) < dens)
            if rng.random() < 0.5 and d > 4:  # a few dense (hot) columns
                hot = rng.choice(d, size=max(1, d // 50), replace=False)
                M[:, hot] = rng.standard_normal((n, hot.size))
            if rng.random() < 0.3:
                M[rng.random(n) < 0.3] = 0.0  # empty rows
            r, c = np.nonzero(M)
            indptr = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=n))])
            it32 = torch.int32
            op = CsrDeviceOp(torch.from_numpy(indptr).to(dev, it32), torch.from_numpy(c).to(dev, it32),
                             torch.from_numpy(M[r, c]).to(dev, dt), d)
            Md = torch.from_numpy(M).to(dev)
            X = rnd((d, nb), dt)
            Y = rnd((n, nb), dt)
            o1 = torch.empty((n, nb), dtype=dt, device=dev)
            o2 = torch.empty((d, nb), dtype=dt, device=dev)
            op.apply(X.contiguous(), o1)
            op.apply_t(Y.contiguous(), o2)
            tol = 5e-6 if dt == torch.float32 else 1e-13
            s1 = float((Md.abs() @ X.double().abs()).max()) or 1.0
            s2 = float((Md.abs().T @ Y.double().abs()).max()) or 1.0
            report("csr A X", f"{dt} n={n} d={d} nb={nb} dens={dens}", float((o1.double() - Md @ X.double()).abs().max()) / s1, tol)
            report("csr A^T Y", f"{dt} n={n} d={d} nb={nb} dens={dens}", float((o2.double() - Md.T @ Y.double()).abs().max()) / s2, tol)
        else:
            w = int(rng.choice([rng.integers(1, 40), rng.integers(40, 650), rng.integers(650, 1300)]))
            k = int(rng.integers(1, min(w, 200) + 1))
            B = rng.standard_normal((w, max(1, int(w * rng.choice([0.3, 1.0, 2.0])))))
            Mh = B @ B.T
            M = torch.from_numpy(Mh).to(dev)
            ev, U, info = ops.syev_topk(M, k)
            lam = np.linalg.eigvalsh(Mh)[::-1][:k]
            evh, Uh = ev.cpu().numpy(), U.cpu().numpy()
            report("syev values", f"w={w} k={k}", float(np.max(np.abs(evh - lam)) / lam[0]), 1e-12)
            report("syev orth", f"w={w} k={k}", float(np.max(np.abs(Uh.T @ Uh - np.eye(k)))), 1e-11)
            report("syev resid", f"w={w} k={k}", float(np.max(np.abs(Mh @ Uh - Uh * evh)) / lam[0]), 1e-11)
    except Exception as exc:  # noqa: BLE001
        fails += 1
        print(f"EXC {kind} case {it}: {exc!r}"[:300], flush=True)
print(f"{cases} cases, {fails} failures")
sys.exit(1 if fails else 0)
