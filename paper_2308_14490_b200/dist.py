"""Multi-GPU AZ solve: probe columns and right-hand sides sharded over ranks.

One process per GPU; torch.distributed (NCCL on GPUs) moves the data, every arithmetic step runs
in libaz through the `Ops` adapter (GpuOps).  Steps (Alg. 1):

  1. rank g computes b' = (I - A Z*) b for its share of the right-hand-side columns and the sketch
     S = (A - A Z* A) Omega for its share of each new probe block (Philox keyed by the GLOBAL
     column, so the probes are the single-GPU ones): no communication (a1-a6 of SURVEY.md §8(a));
  2. all-to-all re-block of the NEW columns only: the column-sharded block becomes row blocks
     appended to the rank's rows of the earlier blocks (the exchange step);
  3. TSQR over a FIXED tree: the rows are cut into NLEAF leaves whatever the world size (rank g owns
     NLEAF/G consecutive leaves), each leaf gives [R_l | c_l] (k1 x k, az_qr_r_partial), and a binary
     tree of pairwise merges (left over right, by the owner of the left child; a factor crosses to
     another rank only where the two children live on different ranks, one factor per rank and
     level) ends in [R_S | Q^T b'] on rank 0;
  4. truncated SVD solve y = V_k Sigma_k^-1 U_k^T (Q^T b') on rank 0; y (probes x nrhs) and the rank
     are broadcast;
  5. x2 = Omega y and the step-2 correction x = x2 + Z*(b - A x2) (az_omega_apply, az_step2) for the
     rank's right-hand-side columns, then all-gather of x (b and x are replicated).

Shards of probe and right-hand-side columns are aligned to column PAIRS: libaz packs two real
columns into one complex FFT vector, so a column's rounding depends on its partner; pair-aligned
shards give every column the same partner at every world size.  With the fixed leaf tree, every
operation then sees the same operands at G = 1, 2, 4, 8 and x is bitwise identical across G
(SURVEY.md §4 "bitwise-identical across G"; H6).

The orchestration is backend-agnostic (duck-typed `ops`), so the host logic (shard ranges, the
re-blocking, the fixed tree, the determinism across G) is tested on CPU with the gloo backend at
world sizes 1, 2 and 4 (tests/test_dist.py).
"""
from __future__ import annotations

from typing import List, Tuple

import torch
import torch.distributed as dist

NLEAF = 8     # leaves of the TSQR tree, independent of the world size (G must divide it)


def split(n: int, parts: int) -> List[int]:
    """Balanced contiguous partition of range(n): boundaries b[0] = 0 <= ... <= b[parts] = n."""
    return [(n * g) // parts for g in range(parts + 1)]


def split_pairs(n: int, parts: int) -> List[int]:
    """Partition of range(n) into `parts` contiguous runs whose boundaries fall on even columns
    (a column and its complex-packing partner 2p, 2p + 1 stay on one rank)."""
    npairs = (n + 1) // 2
    return [min(n, 2 * b) for b in split(npairs, parts)]


def colmajor_empty(rows: int, cols: int, like: torch.Tensor) -> torch.Tensor:
    return torch.empty((cols, rows), dtype=torch.float64, device=like.device).t()


def reblock(local: torch.Tensor, col_owner: List[Tuple[int, int, int]], k: int, row_splits: List[int],
            group=None) -> torch.Tensor:
    """Column-sharded -> row-blocked.

    local: (rows x c_me) column-major, this rank's columns in the order listed for it in col_owner.
    col_owner: runs (g, c0, c1): rank g's local columns j = 0.. map to columns c0..c1-1 of the
               result (0 <= c < k), runs concatenated in list order.
    Returns this rank's row block (rows_me x k) column-major.
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


def tree_merge(ops, facs: dict, nleaf: int, lpr: int, k1: int, k: int, like: torch.Tensor, group=None):
    """Binary reduction of the nleaf leaf factors [R_l | c_l] (k1 x k each) over a FIXED tree: node i of
    level l (covering leaves i 2^l .. (i + 1) 2^l - 1) is the TSQR of its two children stacked (left
    over right), computed by the owner of its first leaf; a child on another rank is sent there.  The
    same merges in the same order at every world size; the root ends on rank 0 (returned there,
    None elsewhere).  Each rank sends at most one factor per level (log2 nleaf levels)."""
    me = dist.get_rank(group)
    cur = dict(facs)                 # node index -> factor, for the nodes this rank holds
    width = 1                        # leaves per node at the current level
    while width < nleaf:
        nxt = {}
        ops_ = []
        for i in range(0, nleaf // width, 2):
            left, right = i * width, (i + 1) * width          # first leaves of the two children
            ol, orr = left // lpr, right // lpr                # their owners
            if orr != ol:
                if me == orr:
                    ops_.append(dist.P2POp(dist.isend, cur.pop(i + 1).t().contiguous(), ol, group=group))
                elif me == ol:
                    buf = torch.empty((k, k1), dtype=torch.float64, device=like.device)
                    ops_.append(dist.P2POp(dist.irecv, buf, orr, group=group))
                    cur[("in", i + 1)] = buf
        if ops_:
            for req in dist.batch_isend_irecv(ops_):
                req.wait()
        for i in range(0, nleaf // width, 2):
            left = i * width
            if left // lpr != me:
                continue
            rt = cur.pop(i + 1) if (i + 1) in cur else cur.pop(("in", i + 1)).t()
            lt = cur.pop(i)
            st = colmajor_empty(2 * k1, k, like)
            st[:k1] = lt
            st[k1:] = rt
            nxt[i // 2] = ops.qr_partial(st, k1)
        cur = nxt
        width *= 2
    return cur.get(0)


def solve_sharded(ops, b: torch.Tensor, theta: float, R: int, max_blocks: int = 1, p_over: int = 10,
                  group=None, nleaf: int = NLEAF) -> Tuple[torch.Tensor, dict]:
    """Distributed AZ solve; b: rows x nrhs column-major, replicated on every rank.  Returns x
    (N x nrhs, replicated) and a report {rank, probes, saturated}.  Collective over `group`."""
    G = dist.get_world_size(group)
    me = dist.get_rank(group)
    if nleaf % G:
        raise ValueError(f"world size {G} must divide the {nleaf} leaves of the TSQR tree")
    rows, N = ops.rows, ops.N
    nrhs = b.shape[1]
    qs = split_pairs(nrhs, G)
    q0, q1 = qs[me], qs[me + 1]
    bp = ops.resid(b[:, q0:q1]) if q1 > q0 else colmajor_empty(rows, 0, b)   # my b' columns
    leaves = split(rows, nleaf)
    lpr = nleaf // G                                          # leaves per rank
    row_splits = [leaves[g * lpr] for g in range(G + 1)]
    r_lo = row_splits[me]
    # right-hand sides re-blocked once: my rows of b'
    owner_b = [(g, qs[g], qs[g + 1]) for g in range(G) if qs[g + 1] > qs[g]]
    Bme = reblock(bp, owner_b, nrhs, row_splits, group)      # rows_me x nrhs
    Sme = colmajor_empty(row_splits[me + 1] - r_lo, 0, b)    # my rows of the probe columns so far
    rank_k, kp, y = 0, 0, None
    saturated = False
    for nb in range(1, max_blocks + 1):
        c0 = (nb - 1) * R                                    # the new block's global probe columns
        kp = nb * R
        k = kp + nrhs
        ps = split_pairs(R, G)
        p0, p1 = ps[me], ps[me + 1]
        new = ops.sketch(c0 + p0, p1 - p0) if p1 > p0 else colmajor_empty(rows, 0, b)
        owner = [(g, ps[g], ps[g + 1]) for g in range(G) if ps[g + 1] > ps[g]]
        Snew = reblock(new, owner, R, row_splits, group)     # rows_me x R
        # my rows of [S | b'] (rows_me x k): earlier blocks, the new block, b'
        Sme = torch.cat([Sme.t(), Snew.t()]).t() if Sme.shape[1] else Snew
        Ame = torch.cat([Sme.t(), Bme.t()]).t()
        facs = {}
        for leaf in range(me * lpr, (me + 1) * lpr):
            a0, a1 = leaves[leaf] - r_lo, leaves[leaf + 1] - r_lo
            facs[leaf] = ops.qr_partial(Ame[a0:a1].clone(), kp)   # kp x k; az_qr_r_partial overwrites its input
        Rf = tree_merge(ops, facs, nleaf, lpr, kp, k, b, group)    # [R_S | Q^T b'] on rank 0, None elsewhere
        # the truncated SVD on rank 0; y (kp x nrhs) and the rank are broadcast
        info = torch.zeros(1, dtype=torch.float64, device=b.device)
        if me == 0:
            y, _, rank_k = ops.tsvd(Rf, kp, nrhs, theta)
            y = ops.contig(y)
            info[0] = rank_k
        else:
            y = colmajor_empty(kp, nrhs, b)
        ybuf = y.t().contiguous()                             # nrhs x kp row-major == y column-major
        dist.broadcast(ybuf, 0, group=group)
        dist.broadcast(info, 0, group=group)
        y = ybuf.t()
        rank_k = int(info[0].item())
        saturated = rank_k > kp - p_over
        if not saturated:
            break
    # x2 = Omega y and steps 2-3 (az_step2) for my right-hand sides, all in libaz
    qmax = max(qs[g + 1] - qs[g] for g in range(G))
    buf = torch.zeros((qmax, N), dtype=torch.float64, device=b.device)
    if q1 > q0:
        x2 = ops.omega_apply(0, y[:, q0:q1])
        xs = ops.step2(x2, b[:, q0:q1])
        buf[:q1 - q0] = xs.t()
    # all-gather the x columns (padded to the largest share)
    allx = torch.empty((G * qmax, N), dtype=torch.float64, device=b.device)
    dist.all_gather_into_tensor(allx, buf, group=group)
    x = colmajor_empty(N, nrhs, b)
    for g in range(G):
        c = qs[g + 1] - qs[g]
        if c:
            x[:, qs[g]:qs[g + 1]] = allx[g * qmax:g * qmax + c].t()
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
        if A.shape[0] < A.shape[1]:     # fewer rows than columns (a small leaf): zero rows leave R unchanged
            Z = colmajor_empty(A.shape[1], A.shape[1], A)
            Z.zero_()
            Z[:A.shape[0]] = A
            A = Z
        if A.shape[1] <= 128:
            return qr_r_partial(A, k1)
        return qr_r(A)[:k1]

    def tsvd(self, Rf, r, nrhs, theta):
        from .api import tsvd_solve
        return tsvd_solve(self.contig(Rf), r, nrhs, theta)

    def omega_apply(self, col0, y):
        return self.plan.omega_apply(col0, self.contig(y))

    def step2(self, x2, b):
        return self.plan.step2(self.contig(x2), self.contig(b))
