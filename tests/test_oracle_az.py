"""Pins for oracle/az.py: dense TSVD LSQ, Alg. 1, evaluation (CPU only)."""
import numpy as np
import pytest

from oracle import az
from oracle import dense as D
from oracle import kernel as K
from paper_2308_14490_b200 import inputs as I


# ---------------------------------------------------------------- O1: tsvd_lsq

def test_tsvd_identity_and_rank1():
    b = np.arange(5.0)
    x, k, _ = az.tsvd_lsq(np.eye(5), b, 1e-12)
    assert k == 5 and np.allclose(x, b, rtol=0, atol=1e-15)
    u = np.array([3.0, 4.0, 0.0]) / 5
    v = np.array([1.0, 2.0, 2.0]) / 3
    x, k, _ = az.tsvd_lsq(np.outer(u, v), u, 1e-12)
    assert k == 1 and np.allclose(x, v, atol=1e-15)


def test_tsvd_matches_qr_lstsq_when_well_conditioned():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((20, 12))
    b = rng.standard_normal(20)
    x, k, _ = az.tsvd_lsq(A, b, 1e-14)
    Q, R = np.linalg.qr(A)
    xr = np.linalg.solve(R, Q.T @ b)                       # independent QR-based solve
    assert k == 12 and np.linalg.norm(x - xr) < 1e-12 * np.linalg.norm(xr)


# ---------------------------------------------------------------- Alg. 1 identities

def _toy_problem(A, Z):
    cfg = I.Config("toy", 1, A.shape[1], 1, "box", 0, 1, 4, 0, 1e-12)
    return az.Problem(cfg, A.shape[0], 0, A.shape[1], lambda x: A @ x, lambda y: Z @ y, 1.0, 0)


def test_az_with_identity():
    A = np.eye(6)
    b = np.linspace(-1, 1, 6)[:, None]
    r = az.az_solve(_toy_problem(A, A), b, 1e-12, R=4, seed=0,
                    omega_fn=lambda cols: np.random.default_rng(0).standard_normal((6, 4))[:, cols])
    assert r.rank == 0 and np.allclose(r.x, b, atol=1e-15) and np.allclose(r.x_step1, 0)


def test_az_with_exact_inverse():
    rng = np.random.default_rng(1)
    A = rng.standard_normal((8, 8)) + 8 * np.eye(8)
    b = rng.standard_normal((8, 1))
    Om = rng.standard_normal((8, 4))
    r = az.az_solve(_toy_problem(A, np.linalg.inv(A)), b, 1e-12, R=4, seed=0, keep_S=True,
                    omega_fn=lambda cols: Om[:, cols])
    # step-1 matrix is numerically zero (relative to ||A||); whatever step 1 returns,
    # step 2 restores x = Z* b exactly since Z* A = I
    assert np.linalg.norm(r.S) < 1e-13 * np.linalg.norm(A) * 4
    assert np.allclose(r.x, np.linalg.solve(A, b), rtol=1e-12)


def test_az_low_rank_perturbation_exact():
    """A = A0 + rank 3, Z* = A0^-1 (square, invertible): A - A Z* A has rank 3, step 1
    captures it and AZ solves A x = b to roundoff (Sherman-Morrison-Woodbury in AZ form)."""
    rng = np.random.default_rng(2)
    A0 = rng.standard_normal((20, 20)) + 6 * np.eye(20)
    A = A0 + rng.standard_normal((20, 3)) @ rng.standard_normal((3, 20))
    b = rng.standard_normal((20, 1))
    Om = rng.standard_normal((20, 13))
    r = az.az_solve(_toy_problem(A, np.linalg.inv(A0)), b, 1e-12, R=13, seed=0,
                    omega_fn=lambda cols: Om[:, cols])
    assert r.rank == 3
    assert np.linalg.norm(A @ r.x - b) < 1e-11 * np.linalg.norm(b)


# ---------------------------------------------------------------- the paper's problems

@pytest.fixture(scope="module")
def c1():
    cfg = I.get_config("c1")
    A = D.assemble_A(cfg)
    b = I.rhs(cfg)
    x, k, s = az.tsvd_lsq(A, b, cfg.tol)
    return cfg, A, b, x


def test_c1_oracle_manufactured_error(c1):
    cfg, A, b, x = c1
    g = I.test_grid(cfg)
    f = az.evaluate(cfg, x, g)
    assert np.max(np.abs(f - g.exact)) / np.max(np.abs(g.exact)) < 1e-9


@pytest.mark.parametrize("backend", ["dense", "fft"])
def test_c1_az_matches_tsvd(c1, backend):
    """Alg. 1 with probes reaches the O1 approximant (<= 1e-9 ||f||) and residual bar (F3)."""
    cfg, A, b, x = c1
    prob = az.make_problem(cfg, backend, dense_A=A)
    r = az.az_solve(prob, b, 1e-12, cfg.R, cfg.seed, max_blocks=4)
    g = I.test_grid(cfg)
    fo, fa = az.evaluate(cfg, x, g), az.evaluate(cfg, r.x, g)
    assert np.max(np.abs(fa - fo)) / np.max(np.abs(fo)) < 1e-9
    ro = np.linalg.norm(A @ x - b) / np.linalg.norm(b)
    ra = np.linalg.norm(A @ r.x - b) / np.linalg.norm(b)
    assert ra <= max(2 * ro, 1e-12)
    # Theorem 7: rank <= 4W, with tau0 from eps h = 0.5 and delta = theta
    W = K.theorem7_W(1e-12, K.tau0_from_eps_h(0.5))
    assert 5 <= r.rank <= 4 * W
    assert not r.saturated
    # moderate coefficient norm ("||a||/sqrt(N)" stays O(1); SPEC.md:369 bound 10)
    assert np.linalg.norm(r.x) / np.sqrt(cfg.N) < 10


def test_1d_rank_constant_in_n():
    """Fig. 3 / Theorem 7: the step-1 rank does not grow with N."""
    ranks = []
    for n in (64, 128, 256, 512):
        cfg = I.make_config("interval", n, R=40)
        prob = az.make_problem(cfg, "fft")
        r = az.az_solve(prob, I.rhs(cfg), 1e-12, 40, 0)
        ranks.append(r.rank)
    assert max(ranks) - min(ranks) <= 2, ranks


def test_periodic_box_step1_vanishes():
    """Omega = bounding box: A = A^c, Z* is its pseudo-inverse, step 1 is (numerically) zero
    and AZ returns the periodic least-squares solution."""
    cfg = I.make_config("box1d", 64)
    prob = az.make_problem(cfg, "dense")
    rng = np.random.default_rng(0)
    v = rng.standard_normal((cfg.N, 3))
    Kv = az.step1_apply(prob, v)
    assert np.linalg.norm(Kv) < 1e-12 * np.linalg.norm(prob.apply_A(v))
    # a function that is exactly one basis function -> unit coefficient vector
    j = 17
    b = D.assemble_A(cfg)[:, j:j + 1]
    r = az.az_solve(prob, b, 1e-12, 8, 0)
    e = np.zeros((cfg.N, 1))
    e[j] = 1
    assert np.linalg.norm(r.x - e) < 1e-10


def test_fft_and_dense_backends_agree_on_operators():
    cfg = I.make_config("star", 12)
    pd = az.make_problem(cfg, "dense")
    pf = az.make_problem(cfg, "fft")
    rng = np.random.default_rng(4)
    v = rng.standard_normal((cfg.N, 2))
    y = rng.standard_normal((pd.M + pd.Mb, 2))
    assert np.linalg.norm(pd.apply_A(v) - pf.apply_A(v)) < 1e-14 * np.linalg.norm(pd.apply_A(v))
    zd, zf = pd.apply_Zstar(y), pf.apply_Zstar(y)
    assert np.linalg.norm(zd - zf) < 1e-13 * pd.zstar_norm * np.linalg.norm(y)


def test_evaluate_unit_coefficients():
    cfg = I.make_config("disk", 8)
    g = I.test_grid(cfg, 21)
    j = 3 * 8 + 5
    x = np.zeros(cfg.N)
    x[j] = 1
    f = az.evaluate(cfg, x, g)[:, 0]
    X, Y = np.meshgrid(*g.axes, indexing="ij")
    c = I.center_axis(cfg)
    ref = K.periodized(X - c[3], cfg.eps, 1.0) * K.periodized(Y - c[5], cfg.eps, 1.0)
    assert np.allclose(f, ref[g.inside], rtol=1e-14, atol=1e-300)


def test_ellipse_orientations_agree():
    """the ellipse problem posed with the long axis along x (ellipse, N^x = 2 N^y)
    and along y (ellipse_t, N^y = 2 N^x) is the same problem with x and y exchanged: the dense O1
    solutions agree after transposing the coefficient array, which pins the per-axis bookkeeping
    (centres, periods, column order j = jx N^y + jy) of the anisotropic assembly."""
    ca, cb = I.make_config("ellipse", 32), I.make_config("ellipse_t", 16)
    xa, ka, _ = az.tsvd_lsq(D.assemble_A(ca), I.rhs(ca), ca.tol)
    xb, kb, _ = az.tsvd_lsq(D.assemble_A(cb), I.rhs(cb), cb.tol)
    assert ka == kb
    Xa = xa.reshape(32, 16)
    Xb = xb.reshape(16, 32)
    assert np.linalg.norm(Xa - Xb.T) <= 1e-4 * np.linalg.norm(Xa)   # coefficients: rounding-level non-uniqueness
    ga, gb = I.test_grid(ca, 101), I.test_grid(cb, 101)
    fa, fb = az.evaluate(ca, xa, ga), az.evaluate(cb, xb, gb)
    Fa = np.zeros(ga.inside.shape)
    Fa[ga.inside] = fa[:, 0]
    Fb = np.zeros(gb.inside.shape)
    Fb[gb.inside] = fb[:, 0]
    assert np.max(np.abs(Fa - Fb.T)) <= 1e-6 * np.max(np.abs(Fa))   # O1 determinacy at tol = 1e-10 (F4)
