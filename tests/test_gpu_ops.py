"""GPU parity of the operator entry points (az_apply_*, az_sketch) against the CPU oracle.

Tolerances:
  A, A^T:          ||y - y_ref|| <= 1e-12 ||y_ref||                 (dense entrywise reference)
  Z*:              ||x - x_ref|| <= 1e-12 ||Z*||_2 ||y||             (extended-precision closed form, O2)
  A - A Z* A:      ||y - y_ref|| <= 1e-12 ||A||_2^2 ||Z*||_2 ||v||
  I - A Z*:        ||y - y_ref|| <= 1e-12 ||A||_2 ||Z*||_2 ||b||
Each bound is the forward-error scale of the composite in binary64 (the reference itself is
computed with 64-bit-mantissa DFTs).

On top of those scale-derived bounds every operator test also holds the ACHIEVED error, normwise
relative to the reference (||y - y_ref|| / ||y_ref||), to 10x the error a binary64 FFT
implementation reaches (measured with numpy's FFT against the same references):
A, A^T 2e-14 (measured <= 1.8e-15); Z* 2e-10 (<= 1.8e-11); A - A Z* A and I - A Z* 1e-10 in 1-D
(<= 1.2e-11) and 1e-9 in 2-D (~1e-10).  The paper-regime family (eps from Eq. 4, ||Z*|| ~ 1e8,
PAPER.md:437) is outside those measurements: its achieved errors are recorded, not held to them.
Achieved errors go to the parity log (tests/conftest.py PARITY_LOG).
"""
import numpy as np
import pytest

from paper_2308_14490_b200 import inputs as I
from oracle import az as OA
from oracle import dense as OD
from oracle import philox as OP

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASES = [
    ("c1", I.get_config("c1")),
    ("interval_n64", I.make_config("interval", 64)),
    ("interval_n1024", I.make_config("interval", 1024)),
    ("interval_n256_s4", I.make_config("interval", 256, s=4)),
    ("box1d_n128", I.make_config("box1d", 128)),
    ("interval_n2048_4step", I.make_config("interval", 2048)),
    ("interval_n8192_4step", I.make_config("interval", 8192)),
    ("box1d_n4096_4step", I.make_config("box1d", 4096)),
    ("disk_n8", I.make_config("disk", 8)),
    ("disk_n32", I.make_config("disk", 32)),
    ("star_n16", I.make_config("star", 16)),
    ("star_n32", I.make_config("star", 32)),
    ("helm_n16", I.make_config("helm", 16)),      # Helmholtz rows, k0^2 = 25
    ("ode_n64", I.make_config("ode", 64)),        # f2: 1-D ODE, two Dirichlet rows, box T = 1.5
    ("ode_n256", I.make_config("ode", 256)),
    ("box2d_n16", I.make_config("box2d", 16)),
    # anisotropic boxes (T^x != T^y, N^x != N^y), both orientations, and the
    # Poisson + Dirichlet-row variant whose boundary windows differ per axis
    ("ellipse_n32", I.make_config("ellipse", 32)),
    ("ellipse_t_n16", I.make_config("ellipse_t", 16)),
    ("ellipse_bvp_n32", I.make_config("ellipse_bvp", 32)),
    ("ellipse_paper_n16", I.make_config("ellipse", 16, eps_h=I.eps_h_paper(1e-5))),
    # Helmholtz on the flower with a hole, Neumann (outer) + Dirichlet (inner) rows
    ("flower_n16", I.make_config("flower", 16)),
    ("flower_mms_n32", I.make_config("flower_mms", 32)),
]


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def setup(request):
    from paper_2308_14490_b200.api import Plan
    name, cfg = request.param
    plan = Plan.from_config(cfg)
    prob = OA.make_problem(cfg, "dense" if cfg.N <= 2048 else "fft")
    A = OD.assemble_A(cfg)
    return cfg, plan, prob, A


def _dev(a):
    return torch.from_numpy(np.asfortranarray(a)).cuda()


def _host(t):
    return t.cpu().numpy()


def _rel(y, ref):
    return np.linalg.norm(y - ref) / np.linalg.norm(ref)


TIGHT = {"A": 2e-14, "Zstar": 2e-10, "K1": 1e-10, "K2": 1e-9}


def _achieved(record, cfg, kind, y, ref):
    """Normwise relative error per column; recorded, and held to the TIGHT bar of its kind."""
    y, ref = y.reshape(y.shape[0], -1), ref.reshape(ref.shape[0], -1)
    err = max(_rel(y[:, c], ref[:, c]) for c in range(y.shape[1]))
    key = kind if kind in ("A", "Zstar") else f"K{cfg.dim}"
    bar = TIGHT[key]
    record(case=cfg.name, op=kind, achieved=float(err), bar=bar)
    # the whole periodic box makes A - A Z* A and I - A Z* vanish (their output is rounding noise, a
    # relative error is meaningless there: test_box_step1_operator_vanishes holds those cases)
    degenerate = cfg.domain == "box" and kind not in ("A", "Zstar")
    if cfg.eps_h == 0.5 and not degenerate:
        assert err <= bar, (kind, err, bar)
    return err


def test_plan_info(setup):
    cfg, plan, prob, A = setup
    assert plan.M == int(I.mask(cfg).sum()) and plan.N == cfg.N and plan.Mb == cfg.n_boundary
    sv = np.sqrt(prob_sigma2(cfg))
    assert plan.sigma_max == pytest.approx(sv.max(), rel=1e-12)
    assert plan.zstar_norm == pytest.approx(prob.zstar_norm, rel=1e-9)


def prob_sigma2(cfg):
    from oracle import circulant as C
    sym = C.Symbol(cfg.dim, cfg.n, cfg.s, cfg.eps, cfg.T, cfg.row_op, alpha=cfg.row_scale, k0sq=cfg.k0sq,
                   n_y=cfg.ny, T_y=cfg.Ty)
    return sym.sigma2


@pytest.mark.parametrize("nvec", [1, 2, 5])
def test_apply_A_and_At(setup, nvec, parity_record):
    cfg, plan, prob, A = setup
    x = I.gaussian_matrix(cfg.N, nvec, 10 + nvec)
    y = _host(plan.apply_A(_dev(x)))
    ref = A @ x
    for c in range(nvec):
        assert _rel(y[:, c], ref[:, c]) <= 1e-12
    _achieved(parity_record, cfg, "A", y, ref)
    yy = I.gaussian_matrix(A.shape[0], nvec, 20 + nvec)
    xt = _host(plan.apply_At(_dev(yy)))
    reft = A.T @ yy
    for c in range(nvec):
        assert _rel(xt[:, c], reft[:, c]) <= 1e-12
    _achieved(parity_record, cfg, "A", xt, reft)


def test_adjoint_identity(setup):
    cfg, plan, prob, A = setup
    u = I.gaussian_matrix(cfg.N, 3, 1)
    v = I.gaussian_matrix(A.shape[0], 3, 2)
    Au = _host(plan.apply_A(_dev(u)))
    Atv = _host(plan.apply_At(_dev(v)))
    lhs, rhs = np.sum(Au * v, 0), np.sum(u * Atv, 0)
    assert np.all(np.abs(lhs - rhs) <= 1e-12 * np.linalg.norm(Au, axis=0) * np.linalg.norm(v, axis=0))


@pytest.mark.parametrize("nvec", [1, 3])
def test_apply_Zstar(setup, nvec, parity_record):
    cfg, plan, prob, A = setup
    y = I.gaussian_matrix(A.shape[0], nvec, 30 + nvec)
    x = _host(plan.apply_Zstar(_dev(y)))
    ref = prob.apply_Zstar(y)
    for c in range(nvec):
        assert np.linalg.norm(x[:, c] - ref[:, c]) <= 1e-12 * plan.zstar_norm * np.linalg.norm(y[:, c])
    _achieved(parity_record, cfg, "Zstar", x, ref)


@pytest.mark.parametrize("nvec", [2, 3])
def test_apply_step1_and_resid(setup, nvec, parity_record):
    cfg, plan, prob, A = setup
    nA = plan.sigma_max
    v = I.gaussian_matrix(cfg.N, nvec, 40 + nvec)
    y = _host(plan.apply_step1(_dev(v)))
    ref = OA.step1_apply(prob, v)
    for c in range(nvec):
        assert np.linalg.norm(y[:, c] - ref[:, c]) <= 1e-12 * nA * nA * plan.zstar_norm * np.linalg.norm(v[:, c])
    _achieved(parity_record, cfg, "step1", y, ref)
    b = I.gaussian_matrix(A.shape[0], nvec, 50 + nvec)
    r = _host(plan.apply_resid(_dev(b)))
    refr = OA.resid_apply(prob, b)
    for c in range(nvec):
        assert np.linalg.norm(r[:, c] - refr[:, c]) <= 1e-12 * nA * plan.zstar_norm * np.linalg.norm(b[:, c])
    _achieved(parity_record, cfg, "resid", r, refr)
    # on the interior block I - A Z* is a projector complement: ||b'_i|| <= ||b_i|| (Lemma 5
    # proof); boundary rows are outside that statement
    M = plan.M
    assert np.all(np.linalg.norm(r[:M], axis=0) <= np.linalg.norm(b[:M], axis=0) * (1 + 1e-12))


def test_sketch_matches_oracle_probes(setup, parity_record):
    cfg, plan, prob, A = setup
    col0, ncols = 5, 7      # ragged: odd count, non-zero global offset
    S = _host(plan.sketch(col0, ncols))
    Om = OP.probe_matrix(cfg, list(range(col0, col0 + ncols)), cfg.seed)
    ref = OA.step1_apply(prob, Om)
    nA = plan.sigma_max
    for c in range(ncols):
        assert np.linalg.norm(S[:, c] - ref[:, c]) <= 1e-12 * nA * nA * plan.zstar_norm * np.linalg.norm(Om[:, c])
    _achieved(parity_record, cfg, "sketch", S, ref)


def test_leading_dimension_and_empty(setup):
    cfg, plan, prob, A = setup
    x = I.gaussian_matrix(cfg.N, 3, 7)
    big = torch.zeros((3, cfg.N + 5), dtype=torch.float64, device="cuda").t()[: cfg.N]   # ld = N + 5
    big.copy_(_dev(x))
    y = _host(plan.apply_A(big))
    assert _rel(y, A @ x) <= 1e-12
    e = torch.empty((0, cfg.N), dtype=torch.float64, device="cuda").t()
    out = plan.apply_A(e)
    assert out.shape == (A.shape[0], 0)


def test_probe_generator_bitwise_reproducible(setup):
    cfg, plan, prob, A = setup
    s1 = plan.sketch(0, 4)
    s2 = plan.sketch(0, 4)
    assert torch.equal(s1, s2)
    s3 = plan.sketch(2, 2)       # same global columns -> same values
    assert torch.equal(s1[:, 2:4], s3)


FULL_CASES = [(n, I.get_config(n)) for n in ("c2", "c3", "c4", "c5")] + [
    # the largest sizes the plan accepts: 1-D n = 2^21 (four-step 2048 x 1024), 2-D n = 1024 (2048^2 grid)
    ("interval_n2^21", I.make_config("interval", 1 << 21, nrhs=3)),
    ("disk_n1024", I.make_config("disk", 1024, nrhs=1)),
]


@pytest.mark.parametrize("name,cfg", FULL_CASES, ids=[c[0] for c in FULL_CASES])
def test_full_size_sampled_and_normwise(name, cfg, parity_record):
    """BASELINE full sizes (c2: n = 2^20, fine grid 2^21; c3/c4/c5: 256^2 / 128^2 / 512^2 centres)
    in the bench's launch configuration: sampled rows of A x against the windowed exact row sums
    (interior and, for c4, boundary rows), and the composite operators against the FFT oracle
    normwise (reading R9)."""
    from paper_2308_14490_b200.api import Plan
    plan = Plan.from_config(cfg)
    prob = OA.make_problem(cfg, "fft")
    rng = np.random.default_rng(0)
    x = I.gaussian_matrix(cfg.N, 2, 3)
    y = _host(plan.apply_A(_dev(x)))
    rows = np.argwhere(I.mask(cfg).reshape(-1)).ravel()
    gn = cfg.grid_n
    for r in rng.choice(plan.M, 64, replace=False):
        g = rows[r] if cfg.dim == 1 else (rows[r] // gn, rows[r] % gn)
        cols, vals = OD.A_row_entries(cfg, g, half_width=40 if cfg.dim == 1 else 16)
        ref = vals @ x[cols]
        assert np.all(np.abs(y[r] - ref) <= 1e-12 * np.abs(vals) @ np.abs(x[cols]))
    if cfg.n_boundary:
        bpts = I.boundary_points(cfg)
        for i in rng.choice(cfg.n_boundary, 8, replace=False):
            rowv = OD.boundary_row(cfg, bpts[i])
            ref = rowv @ x
            assert np.all(np.abs(y[plan.M + i] - ref) <= 1e-12 * np.abs(rowv) @ np.abs(x))
    ref = prob.apply_A(x)
    assert _rel(y, ref) <= 1e-12
    _achieved(parity_record, cfg, "A", y, ref)
    nA = plan.sigma_max
    S = _host(plan.sketch(0, 4))
    Om = OP.probe_matrix(cfg, [0, 1, 2, 3], cfg.seed)
    refS = OA.step1_apply(prob, Om)
    for c in range(4):
        assert np.linalg.norm(S[:, c] - refS[:, c]) <= 1e-12 * nA * nA * plan.zstar_norm * np.linalg.norm(Om[:, c])
    # the full-size references are the binary64 FFT oracle (numpy.fft), not the extended-precision
    # closed form: the achieved error is the sum of both implementations' rounding (recorded; held
    # to 10x the reduced-size bars)
    errS = max(_rel(S[:, c], refS[:, c]) for c in range(4))
    parity_record(case=name, op="sketch_full", achieved=float(errS), bar=10 * TIGHT[f"K{cfg.dim}"])
    assert errS <= 10 * TIGHT[f"K{cfg.dim}"]
    b = I.rhs(cfg)[:, :3]
    z = _host(plan.apply_Zstar(_dev(b)))
    refz = prob.apply_Zstar(b)
    for c in range(b.shape[1]):
        assert np.linalg.norm(z[:, c] - refz[:, c]) <= 1e-12 * plan.zstar_norm * np.linalg.norm(b[:, c])
    errZ = max(_rel(z[:, c], refz[:, c]) for c in range(b.shape[1]))
    parity_record(case=name, op="Zstar_full", achieved=float(errZ), bar=10 * TIGHT["Zstar"])
    assert errZ <= 10 * TIGHT["Zstar"]


def _plan_kwargs(cfg, **over):
    kw = dict(dim=cfg.dim, n=cfg.n, L=cfg.s, T=cfg.T, eps=cfg.eps, op=cfg.row_op, row_scale=cfg.row_scale,
              mask=I.mask(cfg).reshape(-1), boundary_xy=I.boundary_points(cfg) if cfg.n_boundary else None,
              boundary_weight=cfg.boundary_weight, zstar_rcond=cfg.tol, seed=cfg.seed)
    kw.update(over)
    return kw


@pytest.mark.parametrize("case", ["n_not_pow2", "n_too_large_1d", "n_too_large_2d", "L_3_in_2d", "ny_ratio_4",
                                  "no_oversampling", "rcond_1", "robin_in_1d"])
def test_plan_create_rejects_unsupported(case):
    """Argument and size errors come back as status codes before any launch (az.h conventions)."""
    from paper_2308_14490_b200._lib import AZError
    from paper_2308_14490_b200.api import Plan
    c1, d = I.make_config("interval", 64), I.make_config("disk", 16)
    bad = {
        "n_not_pow2": lambda: Plan(**_plan_kwargs(c1, n=48, mask=np.ones(96, np.uint8))),
        "n_too_large_1d": lambda: Plan(**_plan_kwargs(c1, n=1 << 22, mask=np.ones(1 << 23, np.uint8))),
        "n_too_large_2d": lambda: Plan(**_plan_kwargs(d, n=2048, mask=np.ones(4096 * 4096, np.uint8))),
        "L_3_in_2d": lambda: Plan(**_plan_kwargs(d, L=3, mask=np.ones(48 * 48, np.uint8))),
        "ny_ratio_4": lambda: Plan(**_plan_kwargs(d, n_y=64, mask=np.ones(32 * 128, np.uint8))),
        "no_oversampling": lambda: Plan(**_plan_kwargs(c1, L=1, mask=np.ones(64, np.uint8))),
        "rcond_1": lambda: Plan(**_plan_kwargs(c1, zstar_rcond=1.0)),
        "robin_in_1d": lambda: Plan(**_plan_kwargs(I.make_config("ode", 64), boundary_xy=np.array([[-1.0], [1.0]]),
                                                   boundary_coef=np.zeros((2, 4)))),
    }[case]
    with pytest.raises(AZError):
        bad()


def test_box_step1_operator_vanishes():
    """Degenerate case of the method: Omega = the whole periodic box (E = R = I), where A Z* A = A
    (Z* is the pseudo-inverse of A^c), so the step-1 operator and the step-1
    right-hand side of data in the range of A vanish to rounding and the sketch has rank 0."""
    from paper_2308_14490_b200.api import Plan
    for cfg in (I.make_config("box1d", 4096), I.make_config("box2d", 32)):
        plan = Plan.from_config(cfg)
        v = I.gaussian_matrix(cfg.N, 3, 1)
        y = _host(plan.apply_step1(_dev(v)))
        Av = _host(plan.apply_A(_dev(v)))
        assert np.linalg.norm(y) <= 1e-11 * plan.zstar_norm * plan.sigma_max * np.linalg.norm(Av)
        # data in the range of A (the periodic box has no boundary, so f must be representable)
        b = Av + 0.0
        r = _host(plan.apply_resid(_dev(b)))
        assert np.linalg.norm(r) <= 1e-11 * plan.zstar_norm * plan.sigma_max * np.linalg.norm(b)


@pytest.mark.parametrize("name,cfg", [("c1", I.get_config("c1")), ("interval_n8192_4step", I.make_config("interval", 8192)),
                                      ("star_n16", I.make_config("star", 16)), ("disk_n32", I.make_config("disk", 32))],
                         ids=["c1", "interval_n8192_4step", "star_n16", "disk_n32"])
def test_step2_entry_matches_oracle(name, cfg, parity_record):
    """az_step2 (steps 2-3 of Alg. 1 for a given step-1 solution): x = x2 + Z*(b - A x2)
    against the oracle's operators on random x2 and b, for an odd column count (the complex packing's
    unpaired last column) and a padded leading dimension."""
    from paper_2308_14490_b200.api import Plan
    plan = Plan.from_config(cfg)
    prob = OA.make_problem(cfg, "dense" if cfg.N <= 2048 else "fft")
    x2 = I.gaussian_matrix(cfg.N, 3, 71)
    b = I.gaussian_matrix(plan.rows, 3, 72)
    big = torch.zeros((3, cfg.N + 3), dtype=torch.float64, device="cuda").t()[: cfg.N]   # ld = N + 3
    big.copy_(_dev(x2))
    x = _host(plan.step2(big, _dev(b)))
    ref = x2 + prob.apply_Zstar(b - prob.apply_A(x2))
    # forward error of x2 + Z*(b - A x2) in binary64: ||Z*|| (||b|| + ||A|| ||x2||) u-scale
    for c in range(3):
        scale = plan.zstar_norm * (np.linalg.norm(b[:, c]) + plan.sigma_max * np.linalg.norm(x2[:, c]))
        assert np.linalg.norm(x[:, c] - ref[:, c]) <= 1e-12 * scale
    parity_record(case=cfg.name, op="step2", achieved=float(max(_rel(x[:, c], ref[:, c]) for c in range(3))))
