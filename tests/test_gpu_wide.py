"""GPU parity of the wide dense path used by the 2-D configs (SURVEY.md §8(a) a7-a8 with
k > 128 columns): blocked Householder QR (az_qrw.cu) and block one-sided Jacobi SVD
(az_svdw.cu), then whole 2-D solves against the oracle (O1 dense TSVD, O2 Alg. 1 step by step)
on reduced members of the c3/c5 (disk) and c4 (star, Laplacian + Dirichlet rows) families."""
import numpy as np
import pytest

from paper_2308_14490_b200 import inputs as I
from oracle import az as OA
from oracle import dense as OD

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.asfortranarray(a)).cuda()


def _host(t):
    return t.cpu().numpy()


def _graded(m, k, seed, lo=-14):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, k)))
    V, _ = np.linalg.qr(rng.standard_normal((k, k)))
    sig = np.logspace(0, lo, k)
    return (U * sig) @ V.T, sig


@pytest.mark.parametrize("m,k", [(600, 129), (3000, 200), (4099, 517), (20000, 256), (1500, 1500)])
def test_qr_r_wide(m, k):
    from paper_2308_14490_b200.api import qr_r
    A, sig = _graded(m, k, m + k)
    R = _host(qr_r(_dev(A)))
    assert np.allclose(np.tril(R, -1), 0)
    # backward stability: R^T R = A^T A up to O(u ||A||^2)
    assert np.linalg.norm(R.T @ R - A.T @ A) <= 1e-13 * np.linalg.norm(A) ** 2
    sR = np.linalg.svd(R, compute_uv=False)
    assert np.max(np.abs(sR - sig)) <= 1e-13 * sig[0]
    # R agrees with LAPACK's Householder R up to row signs
    Rl = np.linalg.qr(A, mode="r")
    D = np.sign(np.diag(R)) * np.sign(np.diag(Rl))
    assert np.linalg.norm(D[:, None] * R - Rl) <= 1e-12 * np.linalg.norm(Rl)


def test_qr_r_wide_bitwise_reproducible():
    from paper_2308_14490_b200.api import qr_r
    A, _ = _graded(5000, 300, 7)
    R1 = _host(qr_r(_dev(A)))
    R2 = _host(qr_r(_dev(A)))
    assert np.array_equal(R1, R2)


@pytest.mark.parametrize("r,nrhs", [(129, 1), (200, 8), (517, 3), (1024, 64)])
def test_tsvd_solve_wide(r, nrhs):
    from paper_2308_14490_b200.api import tsvd_solve
    rng = np.random.default_rng(r)
    U, _ = np.linalg.qr(rng.standard_normal((r, r)))
    V, _ = np.linalg.qr(rng.standard_normal((r, r)))
    sig = np.concatenate([np.logspace(0, -9, r // 2), np.logspace(-14, -16, r - r // 2)])   # clear gap
    RS = np.triu(np.linalg.qr((U * sig) @ V.T, mode="r"))   # upper triangular, same singular values
    c = rng.standard_normal((r, nrhs))
    Rf = np.hstack([RS, c])
    y, s, k = tsvd_solve(_dev(Rf), r, nrhs, 1e-12)
    y, s = _host(y), _host(s)
    assert k == r // 2
    Uf, sf, Vt = np.linalg.svd(RS)
    assert np.max(np.abs(s - sf)) <= 1e-13 * sf[0]
    ref = Vt[:k].T @ ((Uf[:, :k].T @ c) / sf[:k, None])
    assert np.linalg.norm(y - ref) <= 100 * 1.1e-16 * (sf[0] / sf[k - 1]) * np.linalg.norm(ref)


def _approx_err(cfg, x, ref_x, grid):
    f = OA.evaluate(cfg, x, grid)
    fr = OA.evaluate(cfg, ref_x, grid)
    return np.max(np.abs(f - fr), axis=0) / np.max(np.abs(fr), axis=0)


# reduced members of the 2-D families; R = the family's block rule, adaptive blocks (reading R5)
WIDE_CASES = [("disk_n32", I.make_config("disk", 32), 8),
              ("star_n32", I.make_config("star", 32), 8),
              ("helm_n32", I.make_config("helm", 32), 8),      # SURVEY.md §8(f) f2 (2-D Helmholtz)
              ("disk_n32_nrhs3", I.make_config("disk", 32, nrhs=3, R=128), 12),
              # anisotropic boxes
              ("ellipse_n32", I.make_config("ellipse", 32), 8),
              ("ellipse_t_n16", I.make_config("ellipse_t", 16), 8),
              ("ellipse_bvp_n32", I.make_config("ellipse_bvp", 32), 8),
              ("ellipse_n64", I.make_config("ellipse", 64), 8),
              # the flower (Neumann + Dirichlet rows), the paper's data and the
              # manufactured variant
              ("flower_n32", I.make_config("flower", 32), 8),
              ("flower_mms_n32", I.make_config("flower_mms", 32), 8)]


@pytest.mark.parametrize("name,cfg,max_blocks", WIDE_CASES, ids=[c[0] for c in WIDE_CASES])
def test_solve_2d_matches_oracle(name, cfg, max_blocks):
    from paper_2308_14490_b200.api import Plan
    plan = Plan.from_config(cfg)
    b = I.rhs(cfg)
    theta = max(cfg.tol * 1e-2, 1e-12)
    x, rep = plan.solve(_dev(b), theta, cfg.R, max_blocks)
    x = _host(x)
    assert not rep["saturated"], rep
    grid = I.test_grid(cfg)
    A = OD.assemble_A(cfg)
    # O1: dense truncated SVD (the plain definition)
    xo, _, _ = OA.tsvd_lsq(A, b, cfg.tol)
    res = np.linalg.norm(A @ x - b, axis=0) / np.linalg.norm(b, axis=0)
    ro = np.linalg.norm(A @ xo - b, axis=0) / np.linalg.norm(b, axis=0)
    # F3 reading: within 2x of the oracle's; the absolute 1e-8 bar applies where the oracle meets it
    # (a reduced n = 32 disk is itself only resolved to ~2e-7)
    assert np.all(res <= np.maximum(2 * ro, 1e-12)), (res, ro)
    assert np.all((res <= 1e-8) | (ro > 0.5e-8)), (res, ro)
    # O1 determinacy: the oracle's own spread between tol and tol / 100
    xo2, _, _ = OA.tsvd_lsq(A, b, cfg.tol / 100)
    det = _approx_err(cfg, xo2, xo, grid)
    err = _approx_err(cfg, x, xo, grid)
    assert np.all(err <= np.maximum(1e-9, 2 * det)), (err, det)
    # O2: same algorithm step by step (same Philox probes, same block rule).  In 2-D the sketch
    # singular values below ~1e-10 sigma_1 are rounding noise of K (||Z*|| ~ 5e6),
    # so the count above theta = 1e-12 (and hence the probe count) is not a determined quantity
    # (several correct results): only the approximant is compared.
    prob = OA.make_problem(cfg, "fft")
    r2 = OA.az_solve(prob, b, theta, cfg.R, cfg.seed, max_blocks=max_blocks)
    err2 = _approx_err(cfg, x, r2.x.reshape(cfg.N, -1), grid)
    assert np.all(err2 <= np.maximum(1e-9, 2 * det)), (err2, det)


GOLDEN = __import__("os").path.join(__import__("os").path.dirname(__file__), "golden")


@pytest.mark.parametrize("name", ["c4", "c3", "c5"])
def test_solve_2d_full_size(name, parity_record):
    """BASELINE configs 3, 4 and 5 at full size on the 401^2 test grids (reading R22).

    c4: against the dense O1 golden (tests/golden/c4_o1.npz, written by make_o1_golden.py, which
    calls only oracle/: LAPACK's SVD of the 19,632 x 16,384 entrywise A), with the
    bar max(1e-9, 2 delta_det), delta_det the oracle's own spread between tol and tol/100
    (SURVEY.md §8(c) F4), and the residual within max(2 rho_O1, 1e-12) and <= 1e-8 (F3).
    c3 / c5: parity unpinned by a dense oracle (69 GB / 1.1 TB dense A): the
    manufactured solution on the 401^2 grid and the residual through the oracle's independent
    FFT operator, both <= 1e-8 (F5 reading (b)).  The sketch must be unsaturated (reading R5)."""
    import os
    from paper_2308_14490_b200.api import Plan
    cfg = I.get_config(name)
    plan = Plan.from_config(cfg)
    b = I.rhs(cfg)
    x, rep = plan.solve(_dev(b), max(cfg.tol * 1e-2, 1e-12), cfg.R, 16 if cfg.n < 512 else 6)
    x = _host(x)
    assert not rep["saturated"] and rep["rank"] <= rep["probes"] - 10
    grid = I.test_grid(cfg)
    assert grid.axes[0].size == 401
    f = OA.evaluate(cfg, x, grid)
    scale = np.max(np.abs(grid.exact), axis=0)
    err = np.max(np.abs(f - grid.exact), axis=0) / scale
    prob = OA.make_problem(cfg, "fft")
    res = OA.relative_residual(prob, x, b)
    rec = dict(case=name, probes=int(rep["probes"]), rank=int(rep["rank"]), err_vs_exact=float(err.max()),
               resid=float(res.max()))
    if name == "c4":
        g = np.load(os.path.join(GOLDEN, "c4_o1.npz"))
        fo = OA.evaluate(cfg, g["x_tol"], grid)
        fo2 = OA.evaluate(cfg, g["x_tol100"], grid)
        so = np.max(np.abs(fo), axis=0)
        det = np.max(np.abs(fo2 - fo), axis=0) / so
        e1 = np.max(np.abs(f - fo), axis=0) / so
        ro = g["res_tol"]
        rec.update(approx_vs_o1=float(e1.max()), delta_det=float(det.max()), resid_o1=float(ro.max()),
                   bar=float(np.maximum(1e-9, 2 * det).max()))
        parity_record(**rec)
        assert np.all(e1 <= np.maximum(1e-9, 2 * det)), (e1, det)
        assert np.all(res <= np.maximum(2 * ro, 1e-12)) and np.all(res <= 1e-8), (res, ro)
    else:
        parity_record(**rec, note="parity unpinned by a dense oracle (SURVEY.md §8(c) F5)")
    assert np.all(err <= 1e-8), err
    assert np.all(res <= 1e-8), res


FACTOR_CASES = [("c1", I.get_config("c1"), 4), ("interval_n4096_4step", I.make_config("interval", 4096, nrhs=6, R=40), 4),
                # one probe block of <= 64 on the four-step layout: the factor keeps A Omega (step 2 as a GEMM)
                ("interval_n8192_4step_mb1", I.make_config("interval", 8192, nrhs=6, R=48), 1),
                ("disk_n32", I.make_config("disk", 32), 8), ("star_n32", I.make_config("star", 32), 8)]


@pytest.mark.parametrize("name,cfg,max_blocks", FACTOR_CASES, ids=[c[0] for c in FACTOR_CASES])
def test_factorize_and_solve_factored_matches_solve(name, cfg, max_blocks):
    """Factorisation reuse: one az_factorize, then az_solve_factored for the
    config's right-hand sides and for a second, different set -- each against a full az_solve /
    the oracle (approximant parity; coefficients are not unique)."""
    from paper_2308_14490_b200.api import Factor, Plan
    plan = Plan.from_config(cfg)
    theta = max(cfg.tol * 1e-2, 1e-12)
    fac = Factor(plan, theta, cfg.R, max_blocks)
    assert not fac.report["saturated"]
    grid = I.test_grid(cfg)
    b = I.rhs(cfg)
    xf, _ = fac.solve(_dev(b))
    xs, rep = plan.solve(_dev(b), theta, cfg.R, max_blocks)
    assert fac.report["probes"] == rep["probes"] or cfg.dim == 2   # 2-D: noise-determined (reading R24)
    err = _approx_err(cfg, _host(xf), _host(xs), grid)
    assert np.all(err <= 1e-9), err
    # a second right-hand side on the same factor: a different smooth function, vs the oracle O1
    if cfg.N <= 1024:
        rng = np.random.default_rng(1)
        A = OD.assemble_A(cfg)
        coef = rng.standard_normal((cfg.N, 2)) * np.exp(-0.05 * np.arange(cfg.N))[:, None]
        b2 = A @ coef                                   # exactly representable data
        x2, _ = fac.solve(_dev(b2))
        res = np.linalg.norm(A @ _host(x2) - b2, axis=0) / np.linalg.norm(b2, axis=0)
        xo, _, _ = OA.tsvd_lsq(A, b2, cfg.tol)
        ro = np.linalg.norm(A @ xo - b2, axis=0) / np.linalg.norm(b2, axis=0)
        assert np.all(res <= np.maximum(2 * ro, 1e-10)), (res, ro)


@pytest.mark.parametrize("nrhs", [1, 3, 11, 30, 48])
def test_factored_explicit_matches_compact(nrhs, monkeypatch):
    """The explicit factored form (Q1 = Q[:, :kp] and Omega materialised; memory-bound tsgemv passes
    for few right-hand sides, tiled GEMMs above) against the compact form (Householder panels
    re-applied, probes regenerated): the same factorisation, so the approximants agree to rounding,
    for right-hand-side counts on both sides of the tsgemv/GEMM switch and with ragged 8-groups."""
    from paper_2308_14490_b200.api import Factor, Plan
    cfg = I.make_config("disk", 32)
    plan = Plan.from_config(cfg)
    theta = max(cfg.tol * 1e-2, 1e-12)
    rng = np.random.default_rng(nrhs)
    A = OD.assemble_A(cfg)
    coef = rng.standard_normal((cfg.N, nrhs)) * np.exp(-0.05 * np.arange(cfg.N))[:, None]
    b = A @ coef                                        # exactly representable data
    monkeypatch.setenv("AZ_FACTOR_EXPLICIT", "1")
    fe = Factor(plan, theta, cfg.R, 8)
    monkeypatch.setenv("AZ_FACTOR_EXPLICIT", "0")
    fc = Factor(plan, theta, cfg.R, 8)
    assert fe.report["probes"] == fc.report["probes"] and fe.report["rank"] == fc.report["rank"]
    xe, _ = fe.solve(_dev(b))
    xc, _ = fc.solve(_dev(b))
    grid = I.test_grid(cfg)
    err = _approx_err(cfg, _host(xe), _host(xc), grid)
    assert np.all(err <= 1e-9), err
    re = np.linalg.norm(A @ _host(xe) - b, axis=0)
    rc = np.linalg.norm(A @ _host(xc) - b, axis=0)
    assert np.all(np.abs(re - rc) <= 1e-8 * np.linalg.norm(b, axis=0)), (re, rc)


def test_factored_four_step_m_path_compact_and_explicit(monkeypatch):
    """Four-step factors with one probe block keep M = Omega - Z* A Omega and solve x = Z* b + M y;
    with the compact Householder form (AZ_FACTOR_EXPLICIT=0) and the explicit Q1 the approximants
    agree with a full az_solve."""
    from paper_2308_14490_b200.api import Factor, Plan
    cfg = I.make_config("interval", 8192, nrhs=6, R=48)
    plan = Plan.from_config(cfg)
    theta = max(cfg.tol * 1e-2, 1e-12)
    b = I.rhs(cfg)
    xs, _ = plan.solve(_dev(b), theta, cfg.R, 1)
    grid = I.test_grid(cfg)
    for mode in ("1", "0"):
        monkeypatch.setenv("AZ_FACTOR_EXPLICIT", mode)
        fac = Factor(plan, theta, cfg.R, 1)
        xf, _ = fac.solve(_dev(b))
        err = _approx_err(cfg, _host(xf), _host(xs), grid)
        assert np.all(err <= 1e-9), (mode, err)


PAPER_EPS_CASES = [("interval_paper_n256", I.make_config("interval_paper", 256), 4),
                   ("interval_paper_n1024", I.make_config("interval_paper", 1024), 8),
                   ("disk_paper_n32", I.make_config("disk_paper", 32), 12),
                   ("star_paper_n32", I.make_config("star_paper", 32), 12)]


@pytest.mark.parametrize("name,cfg,max_blocks", PAPER_EPS_CASES, ids=[c[0] for c in PAPER_EPS_CASES])
def test_paper_eps_regime(name, cfg, max_blocks):
    """the paper's own shape parameter eps = cN with c from Eq. (4) (tau0 = 1e-10 in
    1-D, 1e-5 in 2-D), where ||Z*|| reaches 1e8-1e9.  Judged against O1 (the
    dense truncated SVD) with its own determinacy as the bar (F4), the residual against O1's (F3), and
    in 1-D the step-1 rank against Theorem 7's bound 4W."""
    from paper_2308_14490_b200.api import Plan
    from oracle import kernel as K
    plan = Plan.from_config(cfg)
    b = I.rhs(cfg)
    theta = max(cfg.tol * 1e-2, 1e-12)
    x, rep = plan.solve(_dev(b), theta, cfg.R, max_blocks)
    x = _host(x)
    assert not rep["saturated"]
    A = OD.assemble_A(cfg)
    grid = I.test_grid(cfg)
    xo, _, _ = OA.tsvd_lsq(A, b, cfg.tol)
    xo2, _, _ = OA.tsvd_lsq(A, b, cfg.tol / 100)
    det = _approx_err(cfg, xo2, xo, grid)
    err = _approx_err(cfg, x, xo, grid)
    assert np.all(err <= np.maximum(1e-9, 2 * det)), (err, det)
    res = np.linalg.norm(A @ x - b, axis=0) / np.linalg.norm(b, axis=0)
    ro = np.linalg.norm(A @ xo - b, axis=0) / np.linalg.norm(b, axis=0)
    assert np.all(res <= np.maximum(2 * ro, 1e-12)), (res, ro)
    if cfg.dim == 1:
        assert rep["rank"] <= 4 * K.theorem7_W(theta, 1e-10)
