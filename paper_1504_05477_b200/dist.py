"""Row-sharded multi-GPU helpers: A is split by rows across
ranks; A X is local, every reduction over rows is an allreduce (krylov.py),
and these helpers handle the two steps that need more than a sum.

  * sign canonicalization (rsvd.py:192-197) needs the GLOBAL first
    largest-magnitude entry per column: each rank reports (signed value,
    global row) for its rows, the ranks all-gather them and every rank picks
    the same winner (largest |value|, then smallest row), then flips locally.
  * the result Z is returned on every rank (all-gather of the row blocks).
"""

from __future__ import annotations

import torch

from . import device as ops


def sharded_canonicalize_signs(Z, comm, ops=ops):
    val, idx = ops.col_absargmax(Z, comm.row_offset)
    vals = comm.all_gather(val)
    idxs = comm.all_gather(idx)
    V = torch.stack(vals)  # world x k
    I = torch.stack(idxs)
    absv = V.abs()
    best = absv.max(dim=0).values
    cand = torch.where(absv == best, I, torch.full_like(I, torch.iinfo(torch.int64).max))
    win = cand.argmin(dim=0)
    sign_val = V.gather(0, win.view(1, -1)).view(-1).contiguous()
    ops.flip_by_sign(Z, sign_val)
    return Z


def gather_rows(Z, comm):
    """All-gather the row blocks of Z (uneven shards padded)."""
    n_local = torch.tensor([Z.shape[0]], dtype=torch.int64, device=Z.device)
    sizes = [int(t.item()) for t in comm.all_gather(n_local)]
    mx = max(sizes)
    pad = torch.zeros((mx, Z.shape[1]), dtype=Z.dtype, device=Z.device)
    pad[: Z.shape[0]] = Z
    parts = comm.all_gather(pad)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0)
