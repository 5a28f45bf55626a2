"""Generate golden vectors by importing the REFERENCE package (rsvdkit 0.1.0).

Run in the build container only (the reference does not exist on the GPU
box):

    cp -r /root/reference/pkg /tmp/refbuild/ && (cd /tmp/refbuild/pkg &&
        python setup.py build_ext --inplace)
    RSVDKIT_SRC=/tmp/refbuild/pkg/src python tests/golden/make_golden.py

Writes small .npz fixtures next to this script. Everything here is the
reference's own output (compiled backend) on seeded inputs; the tests pin
both the oracle restatement and the CUDA path against these files.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

SRC = os.environ.get("RSVDKIT_SRC", "/tmp/refbuild/pkg/src")
sys.path.insert(0, SRC)
import rsvdkit as rk  # noqa: E402
from rsvdkit import backend  # noqa: E402
from rsvdkit.factor import _mgs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def save(name, **arrs):
    np.savez_compressed(os.path.join(OUT, name), **arrs)
    print("wrote", name, {k: getattr(v, "shape", v) for k, v in arrs.items()})


def main():
    assert rk.active_backend() == "compiled", "build the reference extension first"
    meta = {"reference": "rsvdkit " + rk.__version__, "backend": rk.active_backend()}

    # 1. Gaussian stream KATs (test_backends.py:21-34 shapes), Pi for C1.
    g = {}
    for count in (1, 2, 7, 100, 1001):
        out, st = backend.gauss_fill(count, 987654321)
        g[f"fill_{count}"] = out
        g[f"state_{count}"] = np.array([st], dtype=np.uint64)
    pi = rk.gaussian(1000, 20, rk.SeededRng(0)).data
    g["pi_c1_head"] = pi.ravel()[:64].copy()
    g["pi_c1_sum"] = np.array([pi.sum(), (pi * pi).sum()])
    meta["pi_c1_sha256"] = sha(pi)
    fill = rk.SeededRng(0x5EED_F111_0C0F_FEE5).normal_fill(4096)
    g["qr_fill_head"] = fill
    save("gauss_fill.npz", **g)

    # 2. Kernel KATs: mm, spmm, Jacobi.
    rng = rk.SeededRng(1234)
    a = rk.gaussian(23, 17, rng).data
    b = rk.gaussian(17, 9, rng).data
    dense = rk.gaussian(15, 11, rng).data
    dense = np.where(np.abs(dense) > 1.0, dense, 0.0)
    ri, ci = np.nonzero(dense)
    sp = rk.SparseMatrixCSR.from_coo(15, 11, ri, ci, dense[ri, ci])
    bx = rk.gaussian(11, 6, rng).data
    by = rk.gaussian(15, 4, rng).data
    base = rk.gaussian(12, 12, rng).data
    sym = 0.5 * (base + base.T)
    m1, v1 = sym.copy(), np.eye(12)
    off, sweeps, conv = backend.jacobi_sweeps(m1, v1, 1e-14, 50)
    eig = rk.symmetric_eig(sym)
    save(
        "kernels.npz",
        mm_a=a, mm_b=b, mm_c=backend.mm(a, b),
        sp_indptr=sp.row_ptr, sp_col=sp.col_idx, sp_val=sp.values, sp_shape=np.array(sp.shape),
        sp_bx=bx, sp_nt=backend.spmm_nt(sp.rows, sp.row_ptr, sp.col_idx, sp.values, bx),
        sp_by=by, sp_t=backend.spmm_t(sp.rows, sp.cols, sp.row_ptr, sp.col_idx, sp.values, by),
        jac_in=sym, jac_diag=np.diag(m1).copy(), jac_v=v1, jac_sweeps=np.array([sweeps]),
        eig_vals=eig.eigenvalues, eig_vecs=eig.eigenvectors.data,
    )

    # 3. Small end-to-end cases through the public API (shapes from
    #    test_rsvd.py / test_acceptance.py), all three variants.
    cases = {}

    def run(name, A, cfg):
        r = rk.factorize(A, cfg)
        d = A if isinstance(A, np.ndarray) else None
        cases[name] = dict(
            sigma=r.approx_singular_values.copy(), Z=r.Z.data.copy(), q_used=r.q_used,
            cfg=dict(k=cfg.k, variant=cfg.variant.value, p=cfg.p, q=cfg.q, seed=cfg.seed,
                     every=cfg.reorthonormalize_every),
        )
        if d is not None:
            cases[name]["A"] = d
        return r

    g1 = rk.gaussian(40, 30, rk.SeededRng(53)).data
    run("bk_40x30_k4_q3", g1, rk.RsvdConfig(k=4, variant="bk", q=3, seed=7))
    g2 = rk.gaussian(60, 40, rk.SeededRng(50)).data
    run("si_60x40_k6_q4", g2, rk.RsvdConfig(k=6, variant="si", q=4, seed=1))
    g3 = rk.gaussian(25, 18, rk.SeededRng(52)).data
    for every in (0, 1, 3):
        run(f"si_25x18_k3_q6_every{every}", g3,
            rk.RsvdConfig(k=3, variant="si", q=6, seed=2, reorthonormalize_every=every))
    diag = np.zeros((20, 20))
    diag[0, 0], diag[1, 1], diag[2, 2] = 3.0, 2.0, 1.0
    run("bk_diag_padded", diag, rk.RsvdConfig(k=1, variant="bk", q=3, seed=0))
    u = rk.gaussian(20, 2, rk.SeededRng(68)).data
    v = rk.gaussian(8, 2, rk.SeededRng(69)).data
    run("si_rank2_k4", u @ v.T, rk.RsvdConfig(k=4, variant="si", q=3, seed=4))
    g4 = rk.gaussian(30, 22, rk.SeededRng(58)).data
    for variant in ("si", "bk", "sketch"):
        run(f"q0_{variant}", g4, rk.RsvdConfig(k=4, variant=variant, q=0, seed=21))
    spec = rk.SyntheticSpec(n=120, d=80, spectrum=1.0 / np.arange(1, 81), seed=5)
    a5 = rk.synth_matrix(spec).data
    run("bk_synth_120x80_k5_q4", a5, rk.RsvdConfig(k=5, variant="bk", q=4, seed=0))
    run("bk_synth_120x80_k8_q8_p10", a5, rk.RsvdConfig(k=8, variant="bk", q=8, p=10, seed=3))
    # a clustered small-gap spectrum (C4-like), deficient Krylov basis
    clus = np.concatenate([1 - 0.001 * np.arange(1, 31), 0.5 / np.arange(31, 101)])
    spec = rk.SyntheticSpec(n=300, d=100, spectrum=np.sort(clus)[::-1], seed=9)
    a6 = rk.synth_matrix(spec, check=False).data
    run("bk_clustered_300x100_k10_q7", a6, rk.RsvdConfig(k=10, variant="bk", q=7, seed=0))
    # sparse CSR case through spmm / spmm_t
    rng = rk.SeededRng(77)
    dense = rk.gaussian(90, 70, rng).data
    dense = np.where(np.abs(dense) > 1.3, dense, 0.0)
    ri, ci = np.nonzero(dense)
    sp = rk.SparseMatrixCSR.from_coo(90, 70, ri, ci, dense[ri, ci])
    r = rk.block_krylov(sp, rk.RsvdConfig(k=6, variant="bk", q=4, seed=2))
    cases["bk_csr_90x70_k6_q4"] = dict(
        sigma=r.approx_singular_values.copy(), Z=r.Z.data.copy(), q_used=r.q_used,
        cfg=dict(k=6, variant="bk", p=6, q=4, seed=2, every=1),
        csr_indptr=sp.row_ptr, csr_col=sp.col_idx, csr_val=sp.values, csr_shape=np.array(sp.shape),
    )
    flat = {}
    for name, c in cases.items():
        for key, val in c.items():
            if key == "cfg":
                flat[f"{name}__cfg"] = np.array(json.dumps(val))
            else:
                flat[f"{name}__{key}"] = np.asarray(val)
    save("cases.npz", **flat)

    # 4. C1 (BASELINE configs[0]): reference construction, reference run.
    t0 = time.time()
    spec = rk.SyntheticSpec(n=2000, d=1000, spectrum=1.0 / np.arange(1, 1001), seed=0)
    A = rk.synth_matrix(spec, check=False).data
    t1 = time.time()
    cfg = rk.RsvdConfig(k=20, variant="bk", q=8, seed=0)
    r = rk.block_krylov(A, cfg)
    from rsvdkit import rsvd as rsvd_mod

    op = rk.as_operator(A)
    basis, q_used = rsvd_mod._bk_basis(op, 20, cfg.resolve_q(1000), rk.SeededRng(0))
    z = r.Z.data
    captured = np.sum((A.T @ z) ** 2, axis=0)
    resid = A - z @ (z.T @ A)
    exact = float(np.linalg.norm(resid, 2))
    oracle_sv = np.zeros(21)
    oracle_sv[:] = 1.0 / np.arange(1, 22)

    class _O:
        singular_values = oracle_sv

    est = rk.spectral_error_ratio(A, r.Z, _O) * oracle_sv[20]
    save(
        "c1.npz",
        sigma=r.approx_singular_values, Z=z, captured=captured, q_used=np.array([r.q_used]),
        spectral_exact=np.array([exact]), spectral_est=np.array([est]),
        A_head=A.ravel()[:256].copy(), A_sums=np.array([A.sum(), (A * A).sum(), np.abs(A).sum()]),
        basis_width=np.array([basis.shape[1]]), wall_time_ms=np.array([r.wall_time_ms]),
    )
    meta["c1"] = dict(A_sha256=sha(A), synth_s=t1 - t0, wall_time_ms=r.wall_time_ms,
                      q_used=r.q_used, basis_width=int(basis.shape[1]))
    with open(os.path.join(OUT, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
