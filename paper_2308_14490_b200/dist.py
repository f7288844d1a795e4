"""Multi-GPU AZ solve: probe columns and right-hand sides sharded over ranks.

One process per GPU; torch.distributed (NCCL on GPUs) is the plumbing, every arithmetic step runs
in libaz through the `Ops` adapter (GpuOps).  Steps (Alg. 1):

  1. rank g computes b' = (I - A Z*) b for its share of the right-hand-side columns and the sketch
     S = (A - A Z* A) Omega for its share of the probe columns (Philox keyed by the GLOBAL column, so
     the probes are the single-GPU ones): no communication (a1-a6 of SURVEY.md §8(a));
  2. all-to-all re-block: the column-sharded [S | b'] becomes G row blocks (the exchange step);
  3. local TSQR of each row block -> [R_g | c_g] (k1 x k, az_qr_r_partial), all-gather of these
     small factors, and a second TSQR of the stacked factors on every rank -> [R_S | Q^T b'];
  4. truncated SVD solve y = V_k Sigma_k^-1 U_k^T (Q^T b') on every rank (identical inputs, so
     identical results; no broadcast needed);
  5. x2 = Omega y and the step-2 correction x = x2 + Z*(b - A x2) for the rank's right-hand-side
     columns, then all-gather of x (b and x are replicated on every rank).

The orchestration is backend-agnostic (duck-typed `ops`), so the host logic (shard ranges, the
re-blocking, the factor merge) is tested on CPU with the gloo backend at world size 2.
"""
from __future__ import annotations

from typing import List, Optional, Tuple

import torch
import torch.distributed as dist


def split(n: int, parts: int) -> List[int]:
    """Balanced contiguous partition of range(n): boundaries b[0] = 0 <= ... <= b[parts] = n."""
    return [(n * g) // parts for g in range(parts + 1)]


def colmajor_empty(rows: int, cols: int, like: torch.Tensor) -> torch.Tensor:
    return torch.empty((cols, rows), dtype=torch.float64, device=like.device).t()


def reblock(local: torch.Tensor, col_owner: List[Tuple[int, int, int]], k: int, row_splits: List[int],
            group=None) -> torch.Tensor:
    """Column-sharded -> row-blocked.

    local: (rows x c_me) column-major, this rank's columns in the order listed for it in col_owner.
    col_owner: for every rank g, a list of (global column, ...) is given as runs (g, c0, c1): rank g's
               local columns j = 0.. map to global columns c0..c1-1 of its runs, runs concatenated
               in list order.
    Returns this rank's row block (rows_me x k) column-major, columns in global order.
    """
    G = dist.get_world_size(group)
    me = dist.get_rank(group)
    rows = local.shape[0]
    assert rows == row_splits[-1]
    ncols = [0] * G
    for g, c0, c1 in col_owner:
        ncols[g] += c1 - c0
    assert local.shape[1] == ncols[me]
    rb = [row_splits[h + 1] - row_splits[h] for h in range(G)]
    # send buffer: for every destination h, my columns restricted to h's rows, as (c_me x rb[h]) row-major
    lt = local.t()                                   # c_me x rows, row-major view of the column-major block
    send = torch.cat([lt[:, row_splits[h]:row_splits[h + 1]].contiguous().reshape(-1) for h in range(G)]) \
        if ncols[me] > 0 else torch.empty(0, dtype=local.dtype, device=local.device)
    recv = torch.empty(sum(ncols[g] * rb[me] for g in range(G)), dtype=local.dtype, device=local.device)
    dist.all_to_all_single(recv, send, output_split_sizes=[ncols[g] * rb[me] for g in range(G)],
                           input_split_sizes=[ncols[me] * rb[h] for h in range(G)], group=group)
    out = colmajor_empty(rb[me], k, local)
    off = 0
    pos = [0] * G     # running offset into each source's local column list
    chunks = []
    for g in range(G):
        chunks.append(recv[off:off + ncols[g] * rb[me]].view(ncols[g], rb[me]))
        off += ncols[g] * rb[me]
    for g, c0, c1 in col_owner:
        blk = chunks[g][pos[g]:pos[g] + (c1 - c0)]   # (c1 - c0) x rows_me
        out[:, c0:c1] = blk.t()
        pos[g] += c1 - c0
    return out


def solve_sharded(ops, b: torch.Tensor, theta: float, R: int, max_blocks: int = 1, p_over: int = 10,
                  group=None) -> Tuple[torch.Tensor, dict]:
    """Distributed AZ solve; b: rows x nrhs column-major, replicated on every rank.  Returns x
    (N x nrhs, replicated) and a report {rank, probes, saturated}.  Collective over `group`."""
    G = dist.get_world_size(group)
    me = dist.get_rank(group)
    rows, N = ops.rows, ops.N
    nrhs = b.shape[1]
    qs = split(nrhs, G)
    q0, q1 = qs[me], qs[me + 1]
    bp = ops.resid(b[:, q0:q1]) if q1 > q0 else None       # my b' columns
    row_splits = split(rows, G)
    rank_k, kp, y = 0, 0, None
    saturated = False
    for nb in range(1, max_blocks + 1):
        kp = nb * R
        k = kp + nrhs
        ps = split(kp, G)
        p0, p1 = ps[me], ps[me + 1]
        parts = []
        if p1 > p0:
            parts.append(ops.sketch(p0, p1 - p0))
        if bp is not None:
            parts.append(bp)
        if parts:
            local = parts[0] if len(parts) == 1 else torch.cat([t.t() for t in parts]).t()
        else:
            local = colmajor_empty(rows, 0, b)
        owner = []
        for g in range(G):
            if ps[g + 1] > ps[g]:
                owner.append((g, ps[g], ps[g + 1]))
            if qs[g + 1] > qs[g]:
                owner.append((g, kp + qs[g], kp + qs[g + 1]))
        A = reblock(local, owner, k, row_splits, group)
        Rg = ops.qr_partial(A, kp)                               # kp x k
        Rg = Rg.t().contiguous()                                 # k x kp row-major == Rg column-major, packed
        gathered = [torch.empty_like(Rg) for _ in range(G)]
        dist.all_gather(gathered, Rg, group=group)
        # stack the G factors by rows: (G kp) x k column-major
        stacked = colmajor_empty(G * kp, k, b)
        for g in range(G):
            stacked[g * kp:(g + 1) * kp, :] = gathered[g].t()
        Rf = ops.qr_partial(stacked, kp)                        # [R_S | Q^T b'] (kp x k)
        y, _, rank_k = ops.tsvd(Rf, kp, nrhs, theta)
        saturated = rank_k > kp - p_over
        if not saturated:
            break
    # x2 = Omega y and step 2 for my right-hand sides
    xs = None
    if q1 > q0:
        x2 = ops.omega_apply(0, y[:, q0:q1])
        r = ops.apply_A(x2)
        r = b[:, q0:q1] - r
        xs = x2 + ops.apply_Zstar(ops.contig(r))
    # all-gather the x columns (pad to the largest share)
    qmax = max(qs[g + 1] - qs[g] for g in range(G))
    buf = torch.zeros((qmax, N), dtype=torch.float64, device=b.device)
    if xs is not None:
        buf[:q1 - q0] = xs.t()
    allx = [torch.empty_like(buf) for _ in range(G)]
    dist.all_gather(allx, buf, group=group)
    x = colmajor_empty(N, nrhs, b)
    for g in range(G):
        c = qs[g + 1] - qs[g]
        if c:
            x[:, qs[g]:qs[g + 1]] = allx[g][:c].t()
    return x, {"rank": int(rank_k), "probes": int(kp), "saturated": bool(saturated)}


class GpuOps:
    """libaz entry points behind the solve_sharded interface (CUDA tensors, column-major)."""

    def __init__(self, plan):
        self.plan = plan
        self.rows, self.N = plan.rows, plan.N

    @staticmethod
    def contig(t):
        from .api import colmajor
        return colmajor(t)

    def resid(self, b):
        return self.plan.apply_resid(self.contig(b))

    def sketch(self, col0, ncols):
        return self.plan.sketch(col0, ncols)

    def qr_partial(self, A, k1):
        from .api import qr_r, qr_r_partial
        A = self.contig(A)
        if A.shape[1] <= 128:
            return qr_r_partial(A, k1)
        if A.shape[0] < A.shape[1]:     # the blocked path needs m >= k: zero rows leave R unchanged
            Z = colmajor_empty(A.shape[1], A.shape[1], A)
            Z.zero_()
            Z[:A.shape[0]] = A
            A = Z
        return qr_r(A)[:k1]

    def tsvd(self, Rf, r, nrhs, theta):
        from .api import tsvd_solve
        return tsvd_solve(self.contig(Rf), r, nrhs, theta)

    def omega_apply(self, col0, y):
        return self.plan.omega_apply(col0, self.contig(y))

    def apply_A(self, x):
        return self.plan.apply_A(self.contig(x))

    def apply_Zstar(self, y):
        return self.plan.apply_Zstar(self.contig(y))
