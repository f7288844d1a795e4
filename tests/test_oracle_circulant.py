"""Pins for oracle/circulant.py and oracle/dense.py (CPU only).

The symbols are checked against the definition B = P Pi A^c F computed densely,
against the Poisson-summation closed form of Lemma 4's proof, and against LAPACK
singular values of the entrywise A^c (Lemma 3).  The operators are checked
against entrywise dense matrices and numpy's pseudo-inverse.
"""
import numpy as np
import pytest

from oracle import circulant as C
from oracle import dense as D
from oracle import kernel as K
from paper_2308_14490_b200 import inputs as I


def _cfg(dim, n, s=2, domain="box", row_op=0, eps_h=0.5, k0sq=0.0):
    c = I.Config("t", dim, n, s, domain, row_op, 1, 8, 0, 1e-10, k0sq=k0sq)
    return c


@pytest.mark.parametrize("n,s", [(16, 2), (16, 3), (32, 2)])
def test_block_diagonalisation_definition(n, s):
    """B = P Pi A^c F is block-column diagonal with diagonals = Lemma 3's DFT (sqrt(N) reading)."""
    cfg = _cfg(1, n, s)
    Ac = D.assemble_Ac(cfg).astype(C.LD)
    perm = C.polyphase_index(n, s)
    F = C.dft_F(n)
    P = np.zeros((s * n, s * n), dtype=C.CLD)
    for i in range(s):
        P[i * n:(i + 1) * n, i * n:(i + 1) * n] = F.conj().T
    B = P @ Ac[perm, :].astype(C.CLD) @ F
    v = C.kernel_samples(cfg.eps, cfg.T, n, s, 0, C.LD)
    d = C.diagonals(v, "ld")
    for i in range(s):
        Di = B[i * n:(i + 1) * n]
        off = Di - np.diag(np.diag(Di))
        assert np.max(np.abs(off)) < 1e-15 * np.max(np.abs(Di))
        assert np.max(np.abs(np.diag(Di) - d[i])) < 1e-15 * np.max(np.abs(d))
    # diagonals_dense computes diag(F* A^c_i F) directly
    assert np.max(np.abs(C.diagonals_dense(v) - d)) < 1e-15 * np.max(np.abs(d))


@pytest.mark.parametrize("n,s,eps_h", [(16, 2, 0.5), (256, 2, 0.5), (64, 3, 0.5), (128, 2, 0.9)])
def test_symbol_poisson_closed_form(n, s, eps_h):
    """Lemma 4 proof: DFT of kernel samples = periodic sum of the Gaussian FT."""
    eps = eps_h / (2.0 / n)
    v = C.kernel_samples(eps, 1.0, n, s, 0)
    d = C.diagonals(v, "fft")
    cf = C.poisson_closed_form(eps, 1.0, n, s)
    assert np.max(np.abs(d - cf)) < 5e-14 * np.max(np.abs(cf))
    # and the extended-precision DFT of the same samples agrees with numpy's FFT
    dl = C.diagonals(C.kernel_samples(eps, 1.0, n, s, 0, C.LD), "ld") if n <= 64 else d
    assert np.max(np.abs(dl.astype(np.complex128) - d)) < 1e-14 * np.max(np.abs(d))


def test_min_of_d1_at_half():
    """Lemma 4: d_1 is real, positive, minimal at k = N/2 (0-based)."""
    n = 128
    eps = 0.5 / (2.0 / n)
    d = C.diagonals(C.kernel_samples(eps, 1.0, n, 2, 0), "fft")
    assert np.max(np.abs(d[0].imag)) < 1e-13 * np.max(np.abs(d[0]))
    assert np.all(d[0].real > 0)
    assert int(np.argmin(d[0].real)) == n // 2


@pytest.mark.parametrize("dim,n,row_op,k0sq", [(1, 32, 0, 0.0), (1, 64, 0, 0.0), (2, 8, 0, 0.0), (2, 8, 1, 0.0),
                                               (1, 32, 1, 25.0), (2, 8, 1, 25.0), (2, 16, 1, 7.0)])
def test_lemma3_singular_values(dim, n, row_op, k0sq):
    """Singular values of the entrywise A^c (LAPACK) = sqrt(sum_i |d_i(k)|^2); with k0^2 > 0 this pins
    the Helmholtz rows alpha (Delta + k0^2) phi of the dense assembly and of the symbol together."""
    cfg = _cfg(dim, n, row_op=row_op, k0sq=k0sq)
    Ac = D.assemble_Ac(cfg)
    sv = np.linalg.svd(Ac, compute_uv=False)
    sym = C.Symbol(dim, n, 2, cfg.eps, cfg.T, row_op, alpha=cfg.row_scale, k0sq=k0sq)
    ours = np.sort(np.sqrt(sym.sigma2))[::-1]
    assert np.max(np.abs(sv - ours)) < 1e-13 * sv[0]


def test_laplacian_symbol_k0sq_degenerate():
    """with the order-0 symbol substituted for order 2, k0^2=0 gives 2x the value symbol."""
    n, s = 8, 2
    cfg = _cfg(2, n)
    d0 = C.diagonals(C.kernel_samples(cfg.eps, 1.0, n, s, 0), "fft")
    sv = C.Symbol(2, n, s, cfg.eps, 1.0, 0)
    sl = C.Symbol(2, n, s, cfg.eps, 1.0, 1, alpha=1.0, diag_fn=lambda order: d0)
    assert np.max(np.abs(sl.d - 2 * sv.d)) < 1e-15 * np.max(np.abs(sl.d))


@pytest.mark.parametrize("s", [2, 3])
def test_pinv_moore_penrose_and_s2_closed_form(s):
    n = 8
    rng = np.random.default_rng(3)
    d = rng.standard_normal((s, n)) + 1j * rng.standard_normal((s, n))
    sym = C.Symbol.__new__(C.Symbol)
    sym.d = d
    sym.sigma2 = (np.abs(d) ** 2).sum(0)
    dt, nd = sym.pinv(1e-12)
    assert nd == 0
    if s == 2:
        den = np.abs(d[0]) ** 2 + np.abs(d[1]) ** 2
        assert np.allclose(dt[0], np.conj(d[0]) / den, rtol=1e-15)
        assert np.allclose(dt[1], np.conj(d[1]) / den, rtol=1e-15)
    B = np.vstack([np.diag(d[i]) for i in range(s)])
    Bd = np.hstack([np.diag(dt[i]) for i in range(s)])
    assert np.allclose(B @ Bd @ B, B, atol=1e-13)
    assert np.allclose(Bd @ B @ Bd, Bd, atol=1e-13)
    assert np.allclose((B @ Bd).conj().T, B @ Bd, atol=1e-13)
    assert np.allclose(Bd @ B, np.eye(n), atol=1e-13)
    assert np.allclose(Bd, np.linalg.pinv(B), atol=1e-12)


@pytest.mark.parametrize("dim,n,row_op,backend",
                         [(1, 64, 0, "fft"), (1, 32, 0, "ld"), (2, 16, 0, "fft"), (2, 8, 0, "ld"),
                          (2, 16, 1, "fft"), (2, 8, 1, "ld")])
def test_apply_Ac_matches_entrywise(dim, n, row_op, backend):
    """A^c = Pi^T P* B F* equals the entrywise matrix."""
    cfg = _cfg(dim, n, row_op=row_op)
    Ac = D.assemble_Ac(cfg)
    sym = C.Symbol(dim, n, 2, cfg.eps, cfg.T, row_op, alpha=cfg.row_scale, backend=backend)
    ops = C.PeriodicOperators(sym, 0.0)
    rng = np.random.default_rng(0)
    a = rng.standard_normal(n ** dim)
    y = np.real(ops.apply_Ac(a)).astype(np.float64)
    ref = Ac @ a
    assert np.linalg.norm(y - ref) <= 1e-14 * np.linalg.norm(ref) * (10 if backend == "fft" else 1)


@pytest.mark.parametrize("dim,n,eps_h", [(1, 32, 1.0), (2, 8, 1.0), (1, 32, 0.5)])
def test_zstar_full_box_is_pseudo_inverse(dim, n, eps_h):
    """With Omega = box (E = I), Z* = F B^dag P Pi is the pseudo-inverse of A^c."""
    cfg = _cfg(dim, n)
    eps = eps_h / cfg.h
    Ac = _Ac_eps(cfg, eps)
    sym = C.Symbol(dim, n, 2, eps, cfg.T, 0, backend="ld")
    ops = C.PeriodicOperators(sym, 0.0)
    L = Ac.shape[0]
    Z = np.stack([np.real(ops.apply_Zstar_grid(np.eye(L, dtype=C.LD)[:, i])).astype(np.float64)
                  for i in range(L)], axis=1)
    cond = np.linalg.cond(Ac)
    ref = np.linalg.pinv(Ac, rcond=1e-15)
    assert np.linalg.norm(Z - ref) <= 1e-15 * cond * cond * np.linalg.norm(ref) + 1e-12
    # Moore-Penrose identities
    nrm = np.linalg.norm(Ac)
    assert np.linalg.norm(Ac @ Z @ Ac - Ac) <= 1e-15 * cond * nrm * 10
    assert np.linalg.norm((Ac @ Z).T - Ac @ Z) <= 1e-15 * cond * 10
    # Lemma 5: ||I - A^c Z*|| <= 2
    assert np.linalg.norm(np.eye(L) - Ac @ Z, 2) <= 2 + 1e-8


def _grid_pts(cfg):
    g = I.grid_axis(cfg)
    if cfg.dim == 1:
        return g
    X, Y = np.meshgrid(g, g, indexing="ij")
    return np.stack([X.ravel(), Y.ravel()], axis=1)


def _Ac_eps(cfg, eps):
    g = I.grid_axis(cfg)
    c = I.center_axis(cfg)
    P1 = K.periodized(g[:, None] - c[None, :], eps, 1.0)
    if cfg.dim == 1:
        return P1
    return np.einsum("ak,bl->abkl", P1, P1).reshape(len(g) ** 2, cfg.n ** 2)


def test_lemma5_and_zero_columns_on_star():
    """Lemma 5 on a BVP instance, and Z*'s zero columns over boundary rows."""
    from oracle import az
    cfg = I.make_config("star", 12)
    prob = az.make_problem(cfg, "dense")
    A = D.assemble_A(cfg)
    Mt = prob.M + prob.Mb
    Z = prob.apply_Zstar(np.eye(Mt))
    # ||I - A Z*|| restricted to the interior block (I - A^i Z^i is the paper's Lemma 5 object)
    Ai = A[:prob.M]
    assert np.linalg.norm(np.eye(prob.M) - Ai @ Z[:, :prob.M], 2) <= 2 + 1e-8
    # zero columns: perturbing boundary entries leaves Z* y bitwise unchanged
    rng = np.random.default_rng(0)
    y = rng.standard_normal(Mt)
    y2 = y.copy()
    y2[prob.M:] += rng.standard_normal(prob.Mb)
    assert np.array_equal(prob.apply_Zstar(y), prob.apply_Zstar(y2))
    assert np.all(Z[:, prob.M:] == 0)


def test_laplacian_threshold_drops_only_the_mean_mode():
    """The periodic Laplacian symbol vanishes at k = 0 (integral of phi'' over a period is 0)."""
    cfg = I.make_config("star", 32)
    sym = C.Symbol(2, 32, 2, cfg.eps, 1.0, 1, alpha=cfg.row_scale)
    dt, nd = sym.pinv(cfg.tol)
    assert nd == 1
    assert np.all(dt[:, 0] == 0) and np.all(np.abs(dt[:, 1:]).sum(0) > 0)


def test_dense_A_rows_match_window_entries():
    cfg = I.make_config("star", 16)
    A = D.assemble_A(cfg)
    msk = I.mask(cfg)
    q = np.argwhere(msk)[5]
    cols, vals = D.A_row_entries(cfg, tuple(q), half_width=8)
    row = np.zeros(cfg.N)
    row[cols] = vals
    assert np.allclose(row, A[5], rtol=1e-14, atol=1e-300)


@pytest.mark.parametrize("k0sq", [0.0, 25.0])
def test_helmholtz_rows_are_the_operator_applied_to_the_expansion(k0sq):
    """PAPER.md:741-752 (and :698 in 1-D): a LAPLACIAN row at x applied to coefficients c equals
    alpha (Delta u + k0^2 u)(x) for u = sum_j c_j phi_j -- checked against a 4th-order finite
    difference Laplacian of the value rows (independent of the order-2 kernel formula)."""
    n = 16
    cfg = _cfg(2, n, row_op=1, k0sq=k0sq)
    rng = np.random.default_rng(3)
    c = rng.standard_normal(cfg.N)
    x = np.array([[0.13, -0.27], [-0.41, 0.05]])
    hd = 1e-3

    def u(p):
        return D.assemble_rows(cfg, p, "value") @ c

    lap = np.zeros(len(x))
    for ax in range(2):
        e = np.zeros(2)
        e[ax] = hd
        lap += (-u(x + 2 * e) + 16 * u(x + e) - 30 * u(x) + 16 * u(x - e) - u(x - 2 * e)) / (12 * hd * hd)
    rows = D.assemble_rows(cfg, x, "laplacian") @ c
    ref = cfg.row_scale * (lap + k0sq * u(x))
    assert np.allclose(rows, ref, rtol=1e-6, atol=1e-6 * np.abs(cfg.row_scale) * np.max(np.abs(lap)))


# ---- anisotropic boxes (T^x != T^y, N^x != N^y) ----

def _acfg(n, ny, T, Ty, row_op=0, eps_h=0.5):
    import dataclasses
    base = I.make_config("box2d", n, eps_h=eps_h)
    return dataclasses.replace(base, n_y=ny, T=T, T_y=Ty, row_op=row_op)


@pytest.mark.parametrize("n,ny,T,Ty,row_op,backend", [(16, 8, 1.4, 0.7, 0, "fft"), (8, 16, 0.7, 1.4, 0, "fft"),
                                                     (16, 8, 1.4, 0.7, 1, "fft"), (8, 4, 1.4, 0.9, 1, "ld"),
                                                     (16, 4, 1.0, 1.3, 0, "ld")])
def test_aniso_apply_Ac_matches_entrywise(n, ny, T, Ty, row_op, backend):
    """A^c = Pi^T P* B F* with B = B^x (x) B^y from each axis' own (N, T) equals the entrywise
    matrix of the per-axis periodised kernels."""
    cfg = _acfg(n, ny, T, Ty, row_op)
    Ac = D.assemble_Ac(cfg)
    assert Ac.shape == (4 * n * ny, n * ny)
    sym = C.Symbol(2, n, 2, cfg.eps, T, row_op, alpha=cfg.row_scale, backend=backend, n_y=ny, T_y=Ty)
    ops = C.PeriodicOperators(sym, 0.0)
    a = np.random.default_rng(n + ny).standard_normal(n * ny)
    y = np.real(ops.apply_Ac(a)).astype(np.float64)
    ref = Ac @ a
    assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)


@pytest.mark.parametrize("row_op", [0, 1])
def test_aniso_axis_swap_invariance(row_op):
    """Swapping the roles of x and y (N^x <-> N^y, T^x <-> T^y) transposes every grid and
    coefficient array: the FFT-built operators of the two configurations agree after the
    index permutation.  Catches an axis mixed up anywhere in the 2-D factorisation."""
    a_cfg, b_cfg = _acfg(16, 8, 1.4, 0.7, row_op), _acfg(8, 16, 0.7, 1.4, row_op)
    b_cfg = __import__("dataclasses").replace(b_cfg, eps_h=a_cfg.eps * b_cfg.h)   # same eps in both
    assert abs(a_cfg.eps - b_cfg.eps) < 1e-12 * a_cfg.eps
    ops = []
    for c in (a_cfg, b_cfg):
        sym = C.Symbol(2, c.n, 2, c.eps, c.T, row_op, alpha=c.row_scale, n_y=c.ny, T_y=c.Ty)
        ops.append(C.PeriodicOperators(sym, 1e-10))
    a = np.random.default_rng(5).standard_normal((16, 8))
    ya = np.real(ops[0].apply_Ac(a.reshape(-1))).reshape(32, 16)
    yb = np.real(ops[1].apply_Ac(a.T.reshape(-1))).reshape(16, 32)
    assert np.linalg.norm(ya - yb.T) <= 1e-13 * np.linalg.norm(ya)
    g = np.random.default_rng(6).standard_normal((32, 16))
    za = np.real(ops[0].apply_Zstar_grid(g.reshape(-1))).reshape(16, 8)
    zb = np.real(ops[1].apply_Zstar_grid(g.T.reshape(-1))).reshape(8, 16)
    assert np.linalg.norm(za - zb.T) <= 1e-12 * np.linalg.norm(za)


@pytest.mark.parametrize("row_op", [0, 1])
def test_aniso_lemma3_singular_values(row_op):
    """Singular values of the entrywise anisotropic A^c (LAPACK) = sqrt(sum_i |d_i(k)|^2)."""
    cfg = _acfg(16, 8, 1.4, 0.7, row_op)
    sv = np.linalg.svd(D.assemble_Ac(cfg), compute_uv=False)
    sym = C.Symbol(2, 16, 2, cfg.eps, 1.4, row_op, alpha=cfg.row_scale, n_y=8, T_y=0.7)
    ours = np.sort(np.sqrt(sym.sigma2))[::-1]
    assert np.max(np.abs(sv - ours)) < 1e-13 * sv[0]


def test_aniso_zstar_full_box_is_pseudo_inverse():
    """Omega = the anisotropic box (E = I): Z* = F B^dag P Pi is the pseudo-inverse of A^c."""
    cfg = _acfg(8, 4, 1.4, 0.7, 0, eps_h=1.0)
    Ac = D.assemble_Ac(cfg)
    sym = C.Symbol(2, 8, 2, cfg.eps, 1.4, 0, backend="ld", n_y=4, T_y=0.7)
    ops = C.PeriodicOperators(sym, 0.0)
    L = Ac.shape[0]
    Z = np.stack([np.real(ops.apply_Zstar_grid(np.eye(L, dtype=C.LD)[:, i])).astype(np.float64)
                  for i in range(L)], axis=1)
    cond = np.linalg.cond(Ac)
    ref = np.linalg.pinv(Ac, rcond=1e-15)
    assert np.linalg.norm(Z - ref) <= 1e-15 * cond * cond * np.linalg.norm(ref) + 1e-12
    assert np.linalg.norm(Ac @ Z @ Ac - Ac) <= 1e-14 * cond * np.linalg.norm(Ac)
