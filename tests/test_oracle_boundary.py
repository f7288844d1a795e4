"""Pins for the Robin / Neumann boundary rows of the flower example (SURVEY.md §8(f) f4,
PAPER.md:839-850; CPU only).

The oracle's boundary rows beta (a phi_j + b n . grad phi_j)(x_b) are built from the order-1
periodised kernel; here they are checked against central differences of the VALUE rows along the
normal (which use only the order-0 kernel), and the flower geometry against its definition."""
import numpy as np
import pytest

from oracle import az as OA
from oracle import dense as D
from paper_2308_14490_b200 import inputs as I


@pytest.mark.parametrize("n", [16, 32])
def test_neumann_rows_are_normal_derivatives_of_value_rows(n):
    cfg = I.make_config("flower", n)
    pts, coef = I.boundary_points(cfg), I.boundary_coefs(cfg)
    B = D.boundary_matrix(cfg)
    delta = 1e-4 * cfg.h
    nrm = coef[:, 2:]
    Vp = D.assemble_rows(cfg, pts + delta * nrm, "value")
    Vm = D.assemble_rows(cfg, pts - delta * nrm, "value")
    V0 = D.assemble_rows(cfg, pts, "value")
    ref = cfg.boundary_weight * (coef[:, :1] * V0 + coef[:, 1:2] * (Vp - Vm) / (2 * delta))
    scale = cfg.boundary_weight * np.abs(V0).max()
    assert np.max(np.abs(B - ref)) <= 1e-6 * scale
    # Dirichlet rows (the hole) are exactly the value rows
    inner = coef[:, 1] == 0
    assert inner.sum() == n and np.array_equal(B[inner], cfg.boundary_weight * V0[inner])


def test_flower_geometry():
    cfg = I.make_config("flower", 32)
    pts, coef = I.boundary_points(cfg), I.boundary_coefs(cfg)
    assert pts.shape == (96, 2) and coef.shape == (96, 4)
    outer, inner = pts[:64], pts[64:]
    th = np.arctan2(outer[:, 1], outer[:, 0])
    assert np.allclose(np.hypot(outer[:, 0], outer[:, 1]), I.flower_radius(th), atol=1e-14)
    assert np.allclose(np.hypot(inner[:, 0], inner[:, 1]), I.FLOWER_HOLE, atol=1e-15)
    # unit normals, perpendicular to the curve (central-difference tangent), pointing out of Omega
    assert np.allclose(np.hypot(coef[:, 2], coef[:, 3]), 1.0, atol=1e-14)
    fine, fnrm = I._flower_outer(8192)
    tan = np.roll(fine, -1, 0) - np.roll(fine, 1, 0)
    assert np.max(np.abs((tan * fnrm).sum(1))) <= 1e-5 * np.max(np.hypot(tan[:, 0], tan[:, 1]))   # O(dtheta^2)
    step = 1e-3
    assert not np.any(I._in_domain("flower", *(outer + step * coef[:64, 2:]).T))
    assert np.all(I._in_domain("flower", *(outer - step * coef[:64, 2:]).T))
    assert not np.any(I._in_domain("flower", *(inner + step * coef[64:, 2:]).T))
    assert np.all(I._in_domain("flower", *(inner - step * coef[64:, 2:]).T))


def test_flower_manufactured_solution_converges():
    """O1 on the manufactured flower problem (u = sin(2x + 3y) with its Neumann / Dirichlet data):
    the error against u falls with n (the paper's flower has no closed-form solution)."""
    errs = []
    for n in (16, 32):
        cfg = I.make_config("flower_mms", n)
        A, b = D.assemble_A(cfg), I.rhs(cfg)
        x, _, _ = OA.tsvd_lsq(A, b, cfg.tol)
        g = I.test_grid(cfg, 81)
        f = OA.evaluate(cfg, x, g)
        errs.append(np.max(np.abs(f - g.exact)) / np.max(np.abs(g.exact)))
    assert errs[1] < 0.2 * errs[0] and errs[1] < 2e-2, errs
