"""Seeded, synthetic workload inputs shared by the oracle and the CUDA path.

This module holds NONE of the AZ method's arithmetic (no kernel sums, no
symbols, no transforms, no least squares).  It only produces the data that
both sides consume as inputs:

* the configuration table (BASELINE.json configs[0..4] plus reduced members of
  the same families, SURVEY.md §8 table / §8(d) inputs table);
* the collocation mask on the oversampled grid (PAPER.md:120-123 Eq. set_X,
  PAPER.md:586-589 Eq. set_X_2d; closed membership);
* the boundary points of config 4 ("M^b points along the
  boundary");
* the right-hand-side samples and the manufactured exact solutions;
* the evaluation (test) grids.

The probe matrix Omega is NOT generated here: each side implements the same
counter-based Philox4x32-10 generator itself (oracle/philox.py and
csrc/az_common.cuh (probe_pair)), per the task rules.

Grid conventions (PAPER.md:76-83 Eqs. set_centers / set_Xtilde with T=1):
  centers  c_j = -1 + j*h,          h = 2/n,      j = 0..n-1
  grid     x_q = -1 + q*(2/(s*n)),                q = 0..s*n-1
Every coordinate is exact in binary64 for the power-of-two sizes used.
2-D arrays are row-major with x the OUTER (slow) index, y the inner one
("j = (m-1)N^y + n").
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, List, Optional, Tuple

import numpy as np

# --------------------------------------------------------------------------------------
# configuration table
# --------------------------------------------------------------------------------------

ROW_VALUE = 0       # interior rows are plain kernel values (function approximation)
ROW_LAPLACIAN = 1   # interior rows are alpha * Laplacian of the kernel (Poisson, config 4)


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    dim: int              # 1 or 2
    n: int                # centers per axis (paper N, N^x = N^y)
    s: int                # oversampling factor per axis (paper s; BASELINE "L")
    domain: str           # "interval" | "disk" | "star" | "box"
    row_op: int           # ROW_VALUE | ROW_LAPLACIAN
    nrhs: int
    R: int                # probe block size (BASELINE "R")
    seed: int
    tol: float
    boundary_weight: float = 0.0   # beta (config 4: 10)
    n_boundary: int = 0            # M_b
    T: float = 1.0
    k0sq: float = 0.0              # Helmholtz term of the LAPLACIAN rows (0 = Poisson)
    eps_h: float = 0.5             # eps * h: 0.5 in every BASELINE config; the paper's regime is eps_h_paper(tau0)
    n_y: int = 0                   # 2-D anisotropic boxes: centers along y (0 = n)
    T_y: float = 0.0               # half-period along y (0 = T); the box is [-T, T) x [-T_y, T_y)
    rhs_kind: str = ""             # "" = the family's default data; "mms" = manufactured solution (flower)

    @property
    def ny(self) -> int:
        return self.n_y or self.n

    @property
    def Ty(self) -> float:
        return self.T_y or self.T

    @property
    def h(self) -> float:
        return 2.0 * self.T / self.n

    @property
    def hy(self) -> float:
        return 2.0 * self.Ty / self.ny

    @property
    def eps(self) -> float:
        # BASELINE: eps = 0.5 / h  (SURVEY.md §0 naming trap 3); eps_h overrides for the paper's regime
        return self.eps_h / self.h

    @property
    def grid_n(self) -> int:
        return self.s * self.n

    @property
    def N(self) -> int:
        return self.n if self.dim == 1 else self.n * self.ny

    @property
    def spectral_probes(self) -> bool:
        # the probe definition of the plan (reading R35): 1-D boxes whose fine grid is longer
        # than 2048 points (the GPU's four-step layout) draw each probe column pair in the frequency
        # domain; every other plan draws Omega entrywise.  Data only: each side generates its own.
        return self.dim == 1 and self.s * self.n > 2048

    @property
    def row_scale(self) -> float:
        # alpha: 1 for value rows; -1/(2 eps^2) for Laplacian rows (PAPER.md:704,
        # "we normalize A^i with the factor -2 eps^2")
        if self.row_op == ROW_LAPLACIAN:
            return -1.0 / (2.0 * self.eps * self.eps)
        return 1.0


def _disk_R(n: int, s: int) -> int:
    # BASELINE configs[2]: "R sized 1.5x the boundary point count (~1.5*pi*0.8*512)"
    return int(round(1.5 * math.pi * 0.8 * s * n))


def eps_h_paper(tau0: float) -> float:
    """The paper's shape-parameter regime eps = c N with c from Eq. (4),
    c = pi / (2 T sqrt(2 log(1 + tau0^-2))), h = 2T/N:  eps h = pi / sqrt(2 log(1 + tau0^-2)).
    (the paper uses tau0 = 1e-10 in 1-D and 1e-5 in 2-D.)"""
    return math.pi / math.sqrt(2.0 * math.log1p(tau0 ** -2))


def make_config(family: str, n: int, *, nrhs: int = 1, R: Optional[int] = None,
                seed: int = 0, s: int = 2, name: Optional[str] = None, eps_h: Optional[float] = None) -> Config:
    """Members of the BASELINE families at any size (reduced members for parity); eps_h overrides
    eps * h (default 0.5)."""
    return _with_eps(_make_config(family, n, nrhs=nrhs, R=R, seed=seed, s=s, name=name), eps_h)


def _make_config(family: str, n: int, *, nrhs: int = 1, R: Optional[int] = None,
                 seed: int = 0, s: int = 2, name: Optional[str] = None) -> Config:
    if family.endswith("_paper"):
        # the same family in the paper's own eps regime (tau0 = 1e-10 in 1-D, 1e-5 in 2-D)
        base = family[:-len("_paper")]
        c = make_config(base, n, nrhs=nrhs, R=R, seed=seed, s=s, name=name or f"{base}_paper_n{n}")
        return dataclasses.replace(c, eps_h=eps_h_paper(1e-10 if c.dim == 1 else 1e-5))
    if family == "interval":
        return Config(name or f"interval_n{n}", 1, n, s, "interval", ROW_VALUE, nrhs,
                      R if R is not None else 40, seed, 1e-12)
    if family == "box1d":      # Omega = whole periodic box (periodic special case)
        return Config(name or f"box1d_n{n}", 1, n, s, "box", ROW_VALUE, nrhs,
                      R if R is not None else 16, seed, 1e-12)
    if family == "disk":
        return Config(name or f"disk_n{n}", 2, n, s, "disk", ROW_VALUE, nrhs,
                      R if R is not None else _disk_R(n, s), seed, 1e-10)
    if family == "box2d":
        return Config(name or f"box2d_n{n}", 2, n, s, "box", ROW_VALUE, nrhs,
                      R if R is not None else 16, seed, 1e-10)
    if family == "star":
        return Config(name or f"star_n{n}", 2, n, s, "star", ROW_LAPLACIAN, nrhs,
                      R if R is not None else 8 * n, seed, 1e-10,
                      boundary_weight=10.0, n_boundary=4 * n)
    if family == "ode":
        # SURVEY.md §8(f) f2, PAPER.md Example 6.1 (:694-705, Fig. 8 :823-830): u'' + k^2 u = 0 on [-1, 1],
        # u(+-1) = sin(+-n/5), k = n/5, box T = 1.5, s = 2; Dirichlet rows at the two endpoints (beta = 1)
        return Config(name or f"ode_n{n}", 1, n, s, "ode", ROW_LAPLACIAN, nrhs,
                      R if R is not None else 40, seed, 1e-10,
                      boundary_weight=1.0, n_boundary=2, T=1.5, k0sq=(n / 5.0) ** 2)
    if family == "helm":
        # 2-D Helmholtz Delta u + k0^2 u = f on the star domain,
        # the c4 geometry and weights with k0^2 = 25 (k0 = 5: k0^2 is not an eigenvalue of the
        # manufactured u = sin3x cos2y, whose -Delta eigenvalue is 13)
        return Config(name or f"helm_n{n}", 2, n, s, "star", ROW_LAPLACIAN, nrhs,
                      R if R is not None else 8 * n, seed, 1e-10,
                      boundary_weight=10.0, n_boundary=4 * n, k0sq=25.0)
    if family == "ellipse":
        # SURVEY.md §8(f) f3, PAPER.md:644-647 (Fig. 7): the ellipse x^2 + 4 y^2 <= 1 in the anisotropic
        # box T^x = 1.4, T^y = 0.7 with N^x = 2 N^y (the paper's N^x = 100, N^y = 50 give h^x = h^y;
        # power-of-two N here), f = sin(N^x x / 10 + N^y y / 10), value rows.  R: 1.5 x the collocation
        # points along the boundary (the disk rule of BASELINE configs[2] applied to the ellipse's
        # perimeter, Ramanujan's approximation)
        per = math.pi * (3 * 1.5 - math.sqrt((3 + 0.5) * (1 + 1.5)))
        return Config(name or f"ellipse_n{n}", 2, n, s, "ellipse", ROW_VALUE, nrhs,
                      R if R is not None else int(round(1.5 * per * s * n / 2.8)), seed, 1e-10,
                      T=1.4, n_y=n // 2, T_y=0.7)
    if family == "ellipse_t":
        # the same ellipse with the long axis along y (4 x^2 + y^2 <= 1, T^x = 0.7, T^y = 1.4, N^y = 2 N^x):
        # exercises the other orientation of the anisotropic passes
        per = math.pi * (3 * 1.5 - math.sqrt((3 + 0.5) * (1 + 1.5)))
        return Config(name or f"ellipse_t_n{n}", 2, n, s, "ellipse_t", ROW_VALUE, nrhs,
                      R if R is not None else int(round(1.5 * per * s * 2 * n / 2.8)), seed, 1e-10,
                      T=0.7, n_y=2 * n, T_y=1.4)
    if family == "ellipse_bvp":
        # Poisson on the ellipse in the anisotropic box (c4's row operator, Dirichlet rows beta = 10 at
        # 4 N^x boundary points): the boundary windows differ per axis
        c = _make_config("ellipse", n, nrhs=nrhs, R=R, seed=seed, s=s, name=name or f"ellipse_bvp_n{n}")
        return dataclasses.replace(c, row_op=ROW_LAPLACIAN, boundary_weight=10.0, n_boundary=4 * n)
    if family in ("flower", "flower_mms"):
        # Delta u + 4 u = f on a smooth flower with a circular hole
        # of diameter 0.2 cut out; homogeneous Neumann rows on the outer boundary (2 N points), Dirichlet
        # rows on the inner one (N points), box [-1, 1]^2 (the paper: N = 100, 200 + 100 points).  The
        # flower curve is not given: r = 0.7 + 0.1 cos 5 theta, hole centred at the origin (reading R29).
        # "flower" is the paper's data (f = exp(-4((x + 0.3)^2 + y^2)^2), zero boundary data); "flower_mms"
        # the same operator with the manufactured u = sin(2x + 3y) (inhomogeneous Neumann / Dirichlet data)
        return Config(name or f"{family}_n{n}", 2, n, s, "flower", ROW_LAPLACIAN, nrhs,
                      R if R is not None else 8 * n, seed, 1e-10,
                      boundary_weight=10.0, n_boundary=3 * n, k0sq=4.0,
                      rhs_kind="mms" if family == "flower_mms" else "")
    raise ValueError(f"unknown family {family!r}")


def _with_eps(c: Config, eps_h: Optional[float]) -> Config:
    return c if eps_h is None else dataclasses.replace(c, eps_h=eps_h)


# BASELINE.json configs[0..4]
CONFIGS = {
    "c1": make_config("interval", 256, nrhs=1, R=40, seed=0, name="c1"),
    "c2": make_config("interval", 1 << 20, nrhs=64, R=64, seed=1, name="c2"),
    "c3": make_config("disk", 256, nrhs=1, R=1930, seed=2, name="c3"),
    "c4": make_config("star", 128, nrhs=1, R=1024, seed=3, name="c4"),
    "c5": make_config("disk", 512, nrhs=8, R=3072, seed=4, name="c5"),
}


def get_config(name: str) -> Config:
    return CONFIGS[name]


# --------------------------------------------------------------------------------------
# geometry data (inputs, not method)
# --------------------------------------------------------------------------------------

def grid_axis(cfg: Config, axis: int = 0) -> np.ndarray:
    """Oversampled grid coordinates along one axis, x_q = -T + q*2T/(s n) (axis 1: T_y, n_y)."""
    T, n = (cfg.T, cfg.n) if axis == 0 else (cfg.Ty, cfg.ny)
    L = cfg.s * n
    return -T + np.arange(L, dtype=np.float64) * (2.0 * T / L)


def center_axis(cfg: Config, axis: int = 0) -> np.ndarray:
    T, n = (cfg.T, cfg.n) if axis == 0 else (cfg.Ty, cfg.ny)
    return -T + np.arange(n, dtype=np.float64) * (2.0 * T / n)


def _in_domain(domain: str, x: np.ndarray, y: Optional[np.ndarray] = None) -> np.ndarray:
    # Closed membership, computed in binary64 exactly as SURVEY.md §8(c-4) #13 states.
    if domain == "interval":
        return (-0.5 <= x) & (x <= 0.5)
    if domain == "ode":
        return (-1.0 <= x) & (x <= 1.0)
    if domain == "box":
        return np.ones(np.broadcast(x, x if y is None else y).shape, dtype=bool)
    if domain == "disk":
        return x * x + y * y <= 0.64
    if domain == "star":
        return np.hypot(x, y) <= 0.6 + 0.15 * np.cos(5.0 * np.arctan2(y, x))
    if domain == "ellipse":
        return x * x + 4.0 * y * y <= 1.0
    if domain == "flower":
        rr = np.hypot(x, y)
        return (rr <= flower_radius(np.arctan2(y, x))) & (rr >= FLOWER_HOLE)
    if domain == "ellipse_t":
        return 4.0 * x * x + y * y <= 1.0
    raise ValueError(domain)


def mask(cfg: Config) -> np.ndarray:
    """uint8 collocation mask on the full oversampled grid, natural row-major order.

    1-D: shape (s n,).  2-D: shape (s n, s n_y), x outer.
    """
    g = grid_axis(cfg)
    if cfg.dim == 1:
        return _in_domain(cfg.domain, g).astype(np.uint8)
    X, Y = np.meshgrid(g, grid_axis(cfg, 1), indexing="ij")
    return _in_domain(cfg.domain, X, Y).astype(np.uint8)


def collocation_points(cfg: Config) -> np.ndarray:
    """Interior collocation points in natural order: (M,) in 1-D, (M, 2) in 2-D."""
    g = grid_axis(cfg)
    m = mask(cfg).astype(bool)
    if cfg.dim == 1:
        return g[m]
    X, Y = np.meshgrid(g, grid_axis(cfg, 1), indexing="ij")
    return np.stack([X[m], Y[m]], axis=1)


def star_radius(theta: np.ndarray) -> np.ndarray:
    return 0.6 + 0.15 * np.cos(5.0 * theta)


FLOWER_HOLE = 0.1      # radius of the cut-out circle (diameter 0.2)


def flower_radius(theta: np.ndarray) -> np.ndarray:
    return 0.7 + 0.1 * np.cos(5.0 * theta)


def _flower_outer(m: int):
    """m points on the flower curve, theta_k = 2 pi k / m, and the outward unit normals."""
    th = 2.0 * np.pi * np.arange(m, dtype=np.float64) / m
    r = flower_radius(th)
    dr = -0.5 * np.sin(5.0 * th)
    tx, ty = dr * np.cos(th) - r * np.sin(th), dr * np.sin(th) + r * np.cos(th)
    nrm = np.hypot(tx, ty)
    return np.stack([r * np.cos(th), r * np.sin(th)], axis=1), np.stack([ty / nrm, -tx / nrm], axis=1)


def _flower_inner(m: int):
    """m points on the hole's circle and the normals pointing out of the domain (into the hole)."""
    th = 2.0 * np.pi * np.arange(m, dtype=np.float64) / m
    c, s_ = np.cos(th), np.sin(th)
    return np.stack([FLOWER_HOLE * c, FLOWER_HOLE * s_], axis=1), np.stack([-c, -s_], axis=1)


def boundary_coefs(cfg: "Config") -> Optional[np.ndarray]:
    """(M_b, 4) rows [a, b, n_x, n_y]: boundary row b is beta (a phi_j + b n . grad phi_j)(x_b)
    (Robin form; Dirichlet a = 1, b = 0; Neumann a = 0, b = 1/eps -- reading R29 scales the normal
    derivative by 1/eps so both row kinds are O(1)).  None: every boundary row is Dirichlet."""
    if cfg.domain != "flower" or cfg.n_boundary == 0:
        return None
    no, ni = 2 * cfg.n, cfg.n
    _, nout = _flower_outer(no)
    _, nin = _flower_inner(ni)
    co = np.concatenate([np.zeros((no, 1)), np.full((no, 1), 1.0 / cfg.eps), nout], axis=1)
    ci = np.concatenate([np.ones((ni, 1)), np.zeros((ni, 1)), nin], axis=1)
    return np.ascontiguousarray(np.vstack([co, ci]))


def boundary_points(cfg: Config) -> np.ndarray:
    """(M_b, 2) boundary points, theta_k = 2 pi k / M_b."""
    if cfg.n_boundary == 0:
        return np.zeros((0, max(cfg.dim, 1)), dtype=np.float64)
    if cfg.domain == "ode":
        return np.array([[-1.0], [1.0]])
    if cfg.domain == "flower":
        return np.vstack([_flower_outer(2 * cfg.n)[0], _flower_inner(cfg.n)[0]])
    th = 2.0 * np.pi * np.arange(cfg.n_boundary, dtype=np.float64) / cfg.n_boundary
    if cfg.domain == "ellipse":
        return np.stack([np.cos(th), 0.5 * np.sin(th)], axis=1)
    if cfg.domain != "star":
        raise ValueError("boundary points are defined for the star and ellipse domains only")
    r = star_radius(th)
    return np.stack([r * np.cos(th), r * np.sin(th)], axis=1)


# --------------------------------------------------------------------------------------
# right-hand sides and exact solutions (manufactured data)
# --------------------------------------------------------------------------------------

def exact_functions(cfg: Config) -> List[Callable]:
    """The functions the approximant should reproduce, one per RHS column.

    For the Poisson config this is the manufactured solution u (the approximant is
    u's expansion); for approximation configs it is f itself.
    """
    if cfg.row_op == ROW_LAPLACIAN and cfg.dim == 1:
        kk = cfg.n / 5.0
        return [lambda x: np.sin(kk * x)]
    if cfg.domain == "flower":
        # the paper's flower problem has no closed-form solution: only the manufactured variant does
        return [lambda x, y: np.sin(2 * x + 3 * y)] if cfg.rhs_kind == "mms" else []
    if cfg.row_op == ROW_LAPLACIAN:
        return [lambda x, y: np.sin(3 * x) * np.cos(2 * y)]
    if cfg.dim == 1:
        if cfg.nrhs == 1:
            return [lambda x: np.exp(x) * np.cos(8 * x)]
        return [(lambda k: (lambda x: np.cos(k * x) * np.exp(-x * x)))(k)
                for k in range(1, cfg.nrhs + 1)]
    if cfg.domain in ("ellipse", "ellipse_t"):
        # PAPER.md:644 f(x, y) = sin(N^x x / 10 + N^y y / 10); extra columns shift the phase
        kx, ky = cfg.n / 10.0, cfg.ny / 10.0
        return [(lambda k: (lambda x, y: np.sin(kx * x + ky * y + k)))(k) for k in range(cfg.nrhs)]
    if cfg.nrhs == 1:
        return [lambda x, y: np.exp(x + y) * np.sin(3 * x) * np.cos(2 * y)]
    return [(lambda k: (lambda x, y: np.cos(k * x + y) * np.exp(-(x * x + y * y))))(k)
            for k in range(1, cfg.nrhs + 1)]


def _laplacian_of_u(x, y, k0sq=0.0):
    # u = sin(3x) cos(2y)  =>  Delta u + k0^2 u = (k0^2 - 13) u  (BASELINE configs[3] "f=Delta u": k0 = 0)
    return (k0sq - 13.0) * np.sin(3 * x) * np.cos(2 * y)


def rhs(cfg: Config) -> np.ndarray:
    """b, shape (M + M_b, nrhs), float64, column-major-friendly (Fortran order).

    Interior rows: alpha * f(x_i) (alpha = row_scale; f = Delta u for Poisson).
    Boundary rows: beta * u(x_b)  (SURVEY.md §8(c-4) #11 "multiply rows and data by beta").
    """
    pts = collocation_points(cfg)
    fns = exact_functions(cfg)
    M = pts.shape[0]
    Mb = cfg.n_boundary
    b = np.zeros((M + Mb, cfg.nrhs), dtype=np.float64, order="F")
    if cfg.row_op == ROW_LAPLACIAN and cfg.dim == 1:
        # u'' + k^2 u = 0 for u = sin(k x): interior data 0, boundary data beta u(+-1)
        b[:M, 0] = 0.0
        b[M:, 0] = cfg.boundary_weight * fns[0](boundary_points(cfg)[:, 0])
        return b
    if cfg.domain == "flower":
        bp, bc = boundary_points(cfg), boundary_coefs(cfg)
        if cfg.rhs_kind == "mms":
            # u = sin(2x + 3y): Delta u + k0^2 u = (k0^2 - 13) u; n . grad u = (2 n_x + 3 n_y) cos(2x + 3y)
            b[:M, 0] = cfg.row_scale * (cfg.k0sq - 13.0) * np.sin(2 * pts[:, 0] + 3 * pts[:, 1])
            u = np.sin(2 * bp[:, 0] + 3 * bp[:, 1])
            dn = (2 * bc[:, 2] + 3 * bc[:, 3]) * np.cos(2 * bp[:, 0] + 3 * bp[:, 1])
            b[M:, 0] = cfg.boundary_weight * (bc[:, 0] * u + bc[:, 1] * dn)
        else:
            # f = exp(-4((x + 0.3)^2 + y^2)^2), homogeneous boundary data
            b[:M, 0] = cfg.row_scale * np.exp(-4.0 * ((pts[:, 0] + 0.3) ** 2 + pts[:, 1] ** 2) ** 2)
        return b
    if cfg.row_op == ROW_LAPLACIAN:
        b[:M, 0] = cfg.row_scale * _laplacian_of_u(pts[:, 0], pts[:, 1], cfg.k0sq)
        bp = boundary_points(cfg)
        b[M:, 0] = cfg.boundary_weight * fns[0](bp[:, 0], bp[:, 1])
        return b
    for k, f in enumerate(fns):
        b[:M, k] = f(pts) if cfg.dim == 1 else f(pts[:, 0], pts[:, 1])
    return b


# --------------------------------------------------------------------------------------
# evaluation grids (verification only, never timed)
# --------------------------------------------------------------------------------------

@dataclasses.dataclass
class TestGrid:
    axes: Tuple[np.ndarray, ...]      # tensor axes
    inside: np.ndarray                # bool, shape = tensor shape
    exact: np.ndarray                 # (n_points_inside, nrhs) exact values


def test_grid(cfg: Config, points_1d: Optional[int] = None) -> TestGrid:
    fns = exact_functions(cfg)
    if cfg.dim == 1:
        m = points_1d or (2001 if cfg.n <= 4096 else 65537)
        t = (np.linspace(-0.5, 0.5, m) if cfg.domain == "interval" else
             np.linspace(-1, 1, m) if cfg.domain == "ode" else np.linspace(-1, 1, m, endpoint=False))
        inside = np.ones(m, dtype=bool)
        ex = np.stack([f(t) for f in fns], axis=1)
        return TestGrid((t,), inside, ex)
    m = points_1d or 401
    if cfg.domain == "flower":
        t = u = np.linspace(-0.9, 0.9, m)
    elif cfg.domain == "ellipse":
        t, u = np.linspace(-1.0, 1.0, m), np.linspace(-0.5, 0.5, (m + 1) // 2)
    elif cfg.domain == "ellipse_t":
        t, u = np.linspace(-0.5, 0.5, (m + 1) // 2), np.linspace(-1.0, 1.0, m)
    else:
        lim = {"disk": 0.8, "star": 0.75, "box": 1.0}[cfg.domain]
        t = np.linspace(-lim, lim, m) if cfg.domain != "box" else np.linspace(-1, 1, m, endpoint=False)
        u = t
    X, Y = np.meshgrid(t, u, indexing="ij")
    inside = _in_domain(cfg.domain, X, Y)
    ex = (np.stack([f(X[inside], Y[inside]) for f in fns], axis=1) if fns else
          np.zeros((int(inside.sum()), 0)))
    return TestGrid((t, u), inside, ex)


def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """Seeded N(0,1) test vectors for operator parity tests (not the AZ probes)."""
    rng = np.random.default_rng(seed)
    return np.asfortranarray(rng.standard_normal((rows, cols)))
