"""Dense collocation matrices, assembled entry by entry (Sec. 2.2-2.3, 5.1-5.2, 6.2.1).

Test infrastructure only (see oracle/__init__.py).

Row order: interior collocation rows in natural row-major grid order (x outer),
then boundary rows in the caller's order.  The paper orders rows like Pi X~
(PAPER.md:142); the least-squares problem is invariant under a row permutation
(reading R19 in DESIGN.md), and natural order is what the C ABI exposes.
Column order: j = j_x n + j_y.
"""
from __future__ import annotations

import numpy as np

from paper_2308_14490_b200 import inputs as I
from .kernel import periodized


def _Phi(points: np.ndarray, centers: np.ndarray, eps: float, T: float, order: int) -> np.ndarray:
    """Phi[i, j] = phi^per_order(points[i] - centers[j])."""
    return periodized(points[:, None] - centers[None, :], eps, T, order)


def assemble_rows(cfg: I.Config, pts: np.ndarray, kind: str) -> np.ndarray:
    """Rows of A at `pts` (1-D: (m,), 2-D: (m, 2)).

    kind "value":     phi_j(x)
    kind "laplacian": alpha (phi_jx'' phi_jy + phi_jx phi_jy'' + k0^2 phi_jx phi_jy)
                      1-D: alpha (phi_j'' + k0^2 phi_j)
    """
    c = I.center_axis(cfg)
    eps, T = cfg.eps, cfg.T
    cy, Ty = I.center_axis(cfg, 1), cfg.Ty          # 2-D: the y axis has its own centres and period
    if cfg.dim == 1:
        pts = np.asarray(pts, dtype=np.float64)
        if pts.ndim == 2:          # (m, 1) boundary points
            pts = pts[:, 0]
        if kind == "value":
            return _Phi(pts, c, eps, T, 0)
        return cfg.row_scale * (_Phi(pts, c, eps, T, 2) + cfg.k0sq * _Phi(pts, c, eps, T, 0))
    X0 = _Phi(pts[:, 0], c, eps, T, 0)
    Y0 = _Phi(pts[:, 1], cy, eps, Ty, 0)
    if kind == "value":
        # entry (i, jx*n_y + jy) = phi(x_i - c_jx) phi(y_i - c_jy)
        return (X0[:, :, None] * Y0[:, None, :]).reshape(pts.shape[0], -1)
    X2 = _Phi(pts[:, 0], c, eps, T, 2)
    Y2 = _Phi(pts[:, 1], cy, eps, Ty, 2)
    L = X2[:, :, None] * Y0[:, None, :] + X0[:, :, None] * Y2[:, None, :]
    if cfg.k0sq:
        L = L + cfg.k0sq * (X0[:, :, None] * Y0[:, None, :])
    return cfg.row_scale * L.reshape(pts.shape[0], -1)


def boundary_matrix(cfg: I.Config, pts=None, coefs=None) -> np.ndarray:
    """beta A^b: Dirichlet rows beta phi_j(x_b), or, where the plan gives Robin
    coefficients [a, b, n_x, n_y] (the flower of PAPER.md:839-846), beta (a phi_j + b n . grad phi_j)(x_b)
    with grad phi_j = (phi'(x - c_jx) phi(y - c_jy), phi(x - c_jx) phi'(y - c_jy))."""
    pts = I.boundary_points(cfg) if pts is None else np.asarray(pts, dtype=np.float64)
    coefs = I.boundary_coefs(cfg) if coefs is None else coefs
    if coefs is None or cfg.dim == 1:
        return cfg.boundary_weight * assemble_rows(cfg, pts, "value")
    c, cy = I.center_axis(cfg), I.center_axis(cfg, 1)
    X0 = _Phi(pts[:, 0], c, cfg.eps, cfg.T, 0)
    Y0 = _Phi(pts[:, 1], cy, cfg.eps, cfg.Ty, 0)
    X1 = _Phi(pts[:, 0], c, cfg.eps, cfg.T, 1)
    Y1 = _Phi(pts[:, 1], cy, cfg.eps, cfg.Ty, 1)
    a, b, nx, ny = (coefs[:, i][:, None, None] for i in range(4))
    rows = a * X0[:, :, None] * Y0[:, None, :] + b * (nx * X1[:, :, None] * Y0[:, None, :]
                                                     + ny * X0[:, :, None] * Y1[:, None, :])
    return cfg.boundary_weight * rows.reshape(pts.shape[0], -1)


def assemble_A(cfg: I.Config) -> np.ndarray:
    """A = [A^i ; beta A^b], shape (M + M_b, N)."""
    kind = "laplacian" if cfg.row_op == I.ROW_LAPLACIAN else "value"
    Ai = assemble_rows(cfg, I.collocation_points(cfg), kind)
    if cfg.n_boundary == 0:
        return Ai
    return np.vstack([Ai, boundary_matrix(cfg)])


def assemble_Ac(cfg: I.Config) -> np.ndarray:
    """Full periodic matrix A^c on the whole oversampled grid, natural order."""
    g = I.grid_axis(cfg)
    kind = "laplacian" if cfg.row_op == I.ROW_LAPLACIAN else "value"
    if cfg.dim == 1:
        return assemble_rows(cfg, g, kind)
    X, Y = np.meshgrid(g, I.grid_axis(cfg, 1), indexing="ij")
    return assemble_rows(cfg, np.stack([X.ravel(), Y.ravel()], axis=1), kind)


def boundary_row(cfg: I.Config, pt, window: int | None = None, coef=None) -> np.ndarray:
    """One boundary row (used for sampled parity at full size)."""
    pt = np.asarray(pt, dtype=np.float64)[None, :]
    return boundary_matrix(cfg, pt, None if coef is None else np.asarray(coef, dtype=np.float64)[None, :])[0]


def A_row_entries(cfg: I.Config, i_grid, half_width: int = 40):
    """Nonzero window of interior row for grid index i_grid (1-D int, 2-D (qx, qy)).

    Returns (column indices, values) for the columns within +-half_width centers per
    axis; outside that window phi^per < 1e-170 for eps h = 0.5 (exp(-(0.5*40)^2) ~ 1e-174),
    far below binary64 resolution of the row sum.  Used for sampled full-size parity.
    Pinned against the entrywise dense row (tests/test_oracle_pins.py).
    """
    n, s = cfg.n, cfg.s
    g = I.grid_axis(cfg)
    c = I.center_axis(cfg)
    kind = 2 if cfg.row_op == I.ROW_LAPLACIAN else 0
    if cfg.dim == 1:
        q = int(i_grid)
        j0 = q // s
        js = (np.arange(j0 - half_width, j0 + half_width + 1)) % n
        js = np.unique(js)
        vals = periodized(g[q] - c[js], cfg.eps, cfg.T, kind)
        if kind:
            vals = cfg.row_scale * (vals + cfg.k0sq * periodized(g[q] - c[js], cfg.eps, cfg.T, 0))
        return js, vals
    qx, qy = i_grid
    ny, gy, cy, Ty = cfg.ny, I.grid_axis(cfg, 1), I.center_axis(cfg, 1), cfg.Ty
    jx = np.unique(np.arange(qx // s - half_width, qx // s + half_width + 1) % n)
    jy = np.unique(np.arange(qy // s - half_width, qy // s + half_width + 1) % ny)
    x0 = periodized(g[qx] - c[jx], cfg.eps, cfg.T, 0)
    y0 = periodized(gy[qy] - cy[jy], cfg.eps, Ty, 0)
    if kind:
        x2 = periodized(g[qx] - c[jx], cfg.eps, cfg.T, 2)
        y2 = periodized(gy[qy] - cy[jy], cfg.eps, Ty, 2)
        V = cfg.row_scale * (x2[:, None] * y0[None, :] + x0[:, None] * y2[None, :]
                             + cfg.k0sq * x0[:, None] * y0[None, :])
    else:
        V = x0[:, None] * y0[None, :]
    cols = (jx[:, None] * ny + jy[None, :]).ravel()
    return cols, V.ravel()
