"""Host-side input generation (no method arithmetic): sizes, masks, boundary points."""
import numpy as np
import pytest

from paper_2308_14490_b200 import inputs as I


@pytest.mark.parametrize("name,M,Mb,N", [("c1", 257, 0, 256), ("c3", 131753, 0, 65536),
                                         ("c4", 19120, 512, 16384)])
def test_config_row_counts(name, M, Mb, N):
    # M interior rows (closed membership on the collocation grid)
    cfg = I.get_config(name)
    assert int(I.mask(cfg).sum()) == M
    assert cfg.n_boundary == Mb and cfg.N == N


def test_c2_c5_sizes_cheaply():
    c2 = I.get_config("c2")
    g = I.grid_axis(c2)
    assert int(((g >= -0.5) & (g <= 0.5)).sum()) == 1048577
    assert I.get_config("c5").R == 3072 and I.get_config("c3").R == 1930


def test_grid_exact_and_eps():
    cfg = I.get_config("c1")
    g = I.grid_axis(cfg)
    assert g[0] == -1.0 and np.all(np.diff(g) == 2.0 / 512)
    assert cfg.eps * cfg.h == 0.5 and cfg.eps == 64.0


def test_boundary_points_on_star():
    cfg = I.get_config("c4")
    bp = I.boundary_points(cfg)
    r = np.hypot(bp[:, 0], bp[:, 1])
    th = np.arctan2(bp[:, 1], bp[:, 0])
    assert bp.shape == (512, 2)
    assert np.max(np.abs(r - I.star_radius(th))) < 1e-12


def test_rhs_layout():
    cfg = I.get_config("c4")
    b = I.rhs(cfg)
    assert b.shape == (19632, 1) and b.flags.f_contiguous
    assert cfg.row_scale == -1.0 / 2048   # eps = n/4 = 32 (SURVEY.md §8(d) prints -1/512 in error)
    pts = I.collocation_points(cfg)
    assert np.allclose(b[:5, 0], cfg.row_scale * -13 * np.sin(3 * pts[:5, 0]) * np.cos(2 * pts[:5, 1]))
