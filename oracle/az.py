"""AZ algorithm (Alg. 1), truncated-SVD least squares and evaluation.

Test infrastructure only (see oracle/__init__.py).

O1  `tsvd_lsq`        dense truncated-SVD least squares of A x = b (the judge's reference,
                      SURVEY.md §8(c-1); "computed using a truncated SVD").
O2  `az_solve`        Alg. 1 step by step with the randomized low-rank
                      solver of PAPER.md:269 for step 1, over operator callables so the same
                      code runs with dense matrices (small cases) or the FFT operators of
                      `circulant.PeriodicOperators` (large cases).
    `Problem`         A, Z* (with zero columns over boundary rows)
                      as callables, built from `dense` / `circulant`.
    `evaluate`        the approximant sum_j x_j phi_j(t) on a test grid.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Optional

import numpy as np

from paper_2308_14490_b200 import inputs as I
from . import circulant as C
from . import dense as D
from .kernel import periodized
from .philox import probe_matrix


# --------------------------------------------------------------------------------------
# O1: dense truncated SVD least squares
# --------------------------------------------------------------------------------------

def tsvd_lsq(A: np.ndarray, b: np.ndarray, tol: float):
    """Minimum-norm LSQ over singular directions with sigma_k > tol * sigma_1."""
    U, s, Vt = np.linalg.svd(A, full_matrices=False)
    k = int((s > tol * s[0]).sum()) if s.size and s[0] > 0 else 0
    coef = (U[:, :k].T @ b) / s[:k, None] if b.ndim == 2 else (U[:, :k].T @ b) / s[:k]
    return Vt[:k].T @ coef, k, s


def tsvd_lsq_multi(A: np.ndarray, b: np.ndarray, tols):
    """`tsvd_lsq` at several truncation levels from one SVD of A (the oracle's determinacy
    delta_det compares the solutions at tol and tol/100).
    Returns [(x, k) per tol], s."""
    U, s, Vt = np.linalg.svd(A, full_matrices=False)
    out = []
    for tol in tols:
        k = int((s > tol * s[0]).sum()) if s.size and s[0] > 0 else 0
        out.append((Vt[:k].T @ ((U[:, :k].T @ b) / s[:k, None]), k))
    return out, s


# --------------------------------------------------------------------------------------
# the problem: A and Z* as operators
# --------------------------------------------------------------------------------------

@dataclasses.dataclass
class Problem:
    cfg: I.Config
    M: int                      # interior rows
    Mb: int                     # boundary rows
    N: int
    apply_A: Callable           # (N, k) -> (M + Mb, k)
    apply_Zstar: Callable       # (M + Mb, k) -> (N, k); ignores the boundary rows
    zstar_norm: float
    n_dropped: int


def make_problem(cfg: I.Config, backend: str = "fft", dense_A: Optional[np.ndarray] = None) -> Problem:
    """Build A = [R A^c ; beta A^b] and Z* = [F B^dag P E, 0].

    backend "dense": A is the entrywise dense matrix (dense.assemble_A) and Z* uses the
                     extended-precision DFT matrices ("ld") -- O2 of SURVEY.md §8(c-2).
    backend "fft":   A = R A^c applied through the paper's factorisation with numpy.fft,
                     boundary rows as dense rows; Z* with numpy.fft (binary64).
    """
    msk = I.mask(cfg).astype(bool).reshape(-1)
    M = int(msk.sum())
    Mb = cfg.n_boundary
    N = cfg.N
    sym = C.Symbol(cfg.dim, cfg.n, cfg.s, cfg.eps, cfg.T, cfg.row_op, alpha=cfg.row_scale, k0sq=cfg.k0sq,
                   backend="ld" if backend == "dense" else "fft", n_y=cfg.ny, T_y=cfg.Ty)
    ops = C.PeriodicOperators(sym, cfg.tol)
    Ab = None
    if Mb:
        Ab = D.boundary_matrix(cfg)

    def zstar(y):
        y = np.asarray(y)
        y2 = y.reshape(y.shape[0], -1)
        out = np.empty((N, y2.shape[1]), dtype=np.float64)
        for c in range(y2.shape[1]):
            g = np.zeros(msk.shape[0], dtype=C.LD if backend == "dense" else np.float64)
            g[msk] = y2[:M, c]                                    # E (zero padding); boundary rows ignored
            out[:, c] = np.real(ops.apply_Zstar_grid(g)).astype(np.float64)
        return out.reshape((N,) + y.shape[1:])

    if backend == "dense":
        Ad = D.assemble_A(cfg) if dense_A is None else dense_A

        def apply_A(x):
            return Ad @ x
    else:
        def apply_A(x):
            x = np.asarray(x)
            x2 = x.reshape(N, -1)
            out = np.empty((M + Mb, x2.shape[1]), dtype=np.float64)
            for c in range(x2.shape[1]):
                out[:M, c] = np.real(ops.apply_Ac(x2[:, c]))[msk]    # R A^c x
                if Mb:
                    out[M:, c] = Ab @ x2[:, c]
            return out.reshape((M + Mb,) + x.shape[1:])

    return Problem(cfg, M, Mb, N, apply_A, zstar, ops.zstar_norm(), ops.n_dropped)


# --------------------------------------------------------------------------------------
# O2: Alg. 1 with the randomized step-1 solver
# --------------------------------------------------------------------------------------

@dataclasses.dataclass
class AZResult:
    x: np.ndarray
    x_step1: np.ndarray
    rank: int
    probes_used: int
    saturated: bool
    sketch_sigma: np.ndarray
    b_prime: np.ndarray
    S: Optional[np.ndarray] = None


def step1_apply(prob: Problem, v: np.ndarray) -> np.ndarray:
    """(A - A Z* A) v."""
    Av = prob.apply_A(v)
    return Av - prob.apply_A(prob.apply_Zstar(Av))


def resid_apply(prob: Problem, b: np.ndarray) -> np.ndarray:
    """(I - A Z*) b  (right-hand side of Alg. 1 line 1)."""
    return b - prob.apply_A(prob.apply_Zstar(b))


def az_solve(prob: Problem, b: np.ndarray, theta: float, R: int, seed: int,
             p: int = 10, max_blocks: int = 1, keep_S: bool = False,
             omega_fn: Optional[Callable] = None) -> AZResult:
    """Alg. 1.

    Step 1: solve (I - A Z*) A x2 = (I - A Z*) b with the randomized low-rank solver
            (PAPER.md:257, 269): S = (A - A Z* A) Omega, truncated SVD of S
            (sigma > theta * sigma_1), y = V_k Sigma_k^-1 U_k^T b', x2 = Omega y.
            Probes are drawn in blocks of R until the sketch is unsaturated
            (rank <= probes - p), at most `max_blocks` blocks (reading F1).
    Step 2: x1 = Z* (b - A x2).
    Step 3: x = x1 + x2.
    """
    b2 = b.reshape(b.shape[0], -1)
    N = prob.N
    omega = omega_fn or (lambda cols: probe_matrix(prob.cfg, cols, seed))
    bp = resid_apply(prob, b2)                                   # b' = (I - A Z*) b
    cols = []
    blocks = []
    while True:
        j0 = len(cols)
        cj = list(range(j0, j0 + R))
        cols += cj
        blocks.append(step1_apply(prob, omega(cj)))              # S = (A - A Z* A) Omega
        S = np.hstack(blocks)
        U, sig, Vt = np.linalg.svd(S, full_matrices=False)       # "SVD of an (r+p)-by-M matrix"
        k = int((sig > theta * sig[0]).sum()) if sig[0] > 0 else 0
        if k <= len(cols) - p or len(blocks) >= max_blocks:
            break
    y = Vt[:k].T @ ((U[:, :k].T @ bp) / sig[:k, None])
    x2 = omega(cols) @ y                                          # x2 = Omega y
    x1 = prob.apply_Zstar(b2 - prob.apply_A(x2))                 # step 2
    x = x1 + x2                                                   # step 3
    return AZResult(x.reshape((N,) + b.shape[1:]), x2, k, len(cols), k > len(cols) - p,
                    sig, bp, S if keep_S else None)


# --------------------------------------------------------------------------------------
# evaluation of the approximant (verification only)
# --------------------------------------------------------------------------------------

def evaluate(cfg: I.Config, x: np.ndarray, grid: I.TestGrid) -> np.ndarray:
    """sum_j x_j phi_j(t) at the test-grid points inside Omega: (n_inside, nrhs)."""
    c = I.center_axis(cfg)
    X = x.reshape(cfg.N, -1)
    if cfg.dim == 1:
        t = grid.axes[0]
        if cfg.n <= 4096:
            Phi = periodized(t[:, None] - c[None, :], cfg.eps, cfg.T, 0)
            return (Phi @ X)[grid.inside]
        # large n: the sum over centres within +-W of each point (phi^per < 1e-170 beyond W = 40
        # centres at eps h = 0.5); the omitted terms are below binary64 resolution of the sum
        W = 40
        j0 = np.rint((t + cfg.T) / cfg.h).astype(np.int64)
        js = (j0[:, None] + np.arange(-W, W + 1)[None, :]) % cfg.n
        Phi = periodized(t[:, None] - c[js], cfg.eps, cfg.T, 0)
        return np.einsum("pw,pwr->pr", Phi, X[js])[grid.inside]
    Px = periodized(grid.axes[0][:, None] - c[None, :], cfg.eps, cfg.T, 0)
    Py = periodized(grid.axes[1][:, None] - I.center_axis(cfg, 1)[None, :], cfg.eps, cfg.Ty, 0)
    out = []
    for r in range(X.shape[1]):
        F = Px @ X[:, r].reshape(cfg.n, cfg.ny) @ Py.T
        out.append(F[grid.inside])
    return np.stack(out, axis=1)


def relative_residual(prob: Problem, x: np.ndarray, b: np.ndarray) -> np.ndarray:
    b2 = b.reshape(b.shape[0], -1)
    r = prob.apply_A(x.reshape(prob.N, -1)) - b2
    return np.linalg.norm(r, axis=0) / np.linalg.norm(b2, axis=0)
