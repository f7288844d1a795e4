"""Pins for oracle/kernel.py and oracle/philox.py (CPU only).

Each test checks the oracle against something other than itself: values quoted
by SPEC.md/PAPER.md (tests/golden/), finite differences, symmetry, published
known-answer vectors, distribution moments.
"""
import math
import os

import numpy as np
import pytest

from oracle import kernel as K
from oracle import philox as P

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden_rows():
    rows = []
    with open(os.path.join(GOLD, "spec_kernel_values.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            name, args, val, tol, *_ = line.split()
            kv = dict(a.split("=") for a in args.split(","))
            rows.append((name, {k: float(v) for k, v in kv.items()}, float(val), float(tol)))
    return rows


@pytest.mark.parametrize("name,args,val,tol", _golden_rows())
def test_golden_kernel_values(name, args, val, tol):
    if name == "periodized_eval":
        got = float(K.periodized(args["x"], args["eps"], args["T"], int(args["order"])))
    elif name == "shape_constant":
        got = K.shape_constant(args["T"], args["tau0"])
    elif name == "kernel_eval":
        f = K.phi if int(args["order"]) == 0 else K.phi2
        got = float(f(args["r"], args["eps"]))
    elif name == "theorem7_W":
        got = K.theorem7_W(args["delta"], args["tau0"])
    else:
        raise AssertionError(name)
    if tol == 0:
        assert got == val
    else:
        assert abs(got - val) <= tol * abs(val) + 5e-7 * (name == "periodized_eval"), (name, got, val)


@pytest.mark.parametrize("eps", [1.0, 3.0, 64.0])
def test_phi2_matches_finite_difference(eps):
    # central differences of phi^per agree with the order-2 periodisation
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, 100)
    h = 1e-5 / max(1.0, eps / 4)
    fd = (K.periodized(x + h, eps, 1.0) - 2 * K.periodized(x, eps, 1.0) + K.periodized(x - h, eps, 1.0)) / (h * h)
    ex = K.periodized(x, eps, 1.0, 2)
    scale = 2 * eps * eps
    assert np.max(np.abs(fd - ex)) / scale < 1e-4


@pytest.mark.parametrize("eps", [1.0, 3.0, 64.0])
def test_phi1_matches_finite_difference_and_is_odd(eps):
    """The order-1 periodisation (Neumann rows) is the derivative of phi^per:
    4th-order central differences of order 0 agree, it is odd and 2T-periodic, and its sum over a
    full period of samples vanishes (the derivative of a periodic function has zero mean)."""
    rng = np.random.default_rng(2)
    x = rng.uniform(-1, 1, 100)
    h = 1e-3 / max(1.0, eps / 4)
    f = lambda t: K.periodized(t, eps, 1.0)
    fd = (-f(x + 2 * h) + 8 * f(x + h) - 8 * f(x - h) + f(x - 2 * h)) / (12 * h)
    ex = K.periodized(x, eps, 1.0, 1)
    assert np.max(np.abs(fd - ex)) / eps < 1e-7
    assert np.allclose(K.periodized(-x, eps, 1.0, 1), -ex, rtol=1e-13, atol=1e-13 * eps)
    assert np.allclose(K.periodized(x + 2.0, eps, 1.0, 1), ex, rtol=1e-12, atol=1e-12 * eps)
    g = np.arange(-512, 512) / 512.0
    assert abs(K.periodized(g, min(eps, 8.0), 1.0, 1).sum()) < 1e-10 * min(eps, 8.0)


@pytest.mark.parametrize("order", [0, 2])
def test_periodicity_and_evenness(order):
    x = np.linspace(-3, 3, 77)
    for eps in (0.7, 5.0, 64.0):
        a = K.periodized(x, eps, 1.0, order)
        assert np.allclose(a, K.periodized(x + 2.0, eps, 1.0, order), rtol=1e-13, atol=1e-13 * (2 * eps * eps if order else 1.0))
        assert np.allclose(a, K.periodized(-x, eps, 1.0, order), rtol=1e-13, atol=1e-13 * (2 * eps * eps if order else 1.0))


def test_periodized_tail_negligible():
    # first omitted translate below unit roundoff of the retained sum
    eps, T = 1.0, 1.0
    mm = K._m_max(eps, T)
    x = 0.9
    tail = K.phi(x - 2 * (mm + 1) * T, eps) + K.phi(x + 2 * (mm + 1) * T, eps)
    assert tail < 1e-16 * K.periodized(x, eps, T)


def test_shape_constant_monotone_and_inverse():
    # SPEC.md:70 monotonicity; and eps h = 2 T c round-trips through tau0_from_eps_h
    assert K.shape_constant(2.0, 1e-10) == pytest.approx(K.shape_constant(1.0, 1e-10) / 2, rel=1e-15)
    assert K.shape_constant(1.0, 1e-8) > K.shape_constant(1.0, 1e-10)
    t0 = K.tau0_from_eps_h(0.5)
    assert 2.0 * 1.0 * K.shape_constant(1.0, t0) == pytest.approx(0.5, rel=1e-12)


def test_philox_known_answers():
    with open(os.path.join(GOLD, "philox4x32_10_kat.txt")) as f:
        rows = [l.split() for l in f if l.strip() and not l.startswith("#")]
    for r in rows:
        v = [int(t, 16) for t in r]
        out = P.philox4x32_10(*[np.uint64(t) for t in v[:6]])
        assert [int(o) for o in out] == v[6:], r


def test_probe_moments_and_layout():
    N = 20001
    Om = P.probes(N, [0, 1, 7, 123456789], seed=5)
    assert Om.shape == (N, 4) and Om.flags.f_contiguous
    assert abs(Om.mean()) < 0.02
    assert abs(Om.var() - 1.0) < 0.03
    # independence between columns and between the cos/sin members of a pair
    c = np.corrcoef(Om.T)
    assert np.max(np.abs(c - np.eye(4))) < 0.05
    assert abs(np.corrcoef(Om[0::2][:10000, 0], Om[1::2][:10000, 0])[0, 1]) < 0.05
    # counter-based: a column does not depend on which other columns are requested
    assert np.array_equal(P.probes(N, [7], seed=5)[:, 0], Om[:, 2])
    # different seeds differ
    assert not np.array_equal(P.probes(N, [7], seed=6)[:, 0], Om[:, 2])
    # normal quantiles (Kolmogorov-Smirnov against the standard normal CDF)
    from scipy import stats
    assert stats.kstest(Om.ravel(), "norm").pvalue > 1e-3


def test_spectral_probes_definition_by_brute_force_dft():
    """Reading R35: column pair P is Re / Im of u_P[j] = (1/n) sum_k v_P[k] e^{+2 pi i j k / n},
    v_P[k] = sqrt(n) (z0 + i z1) from Philox counter (k, P + 2^63) -- checked against an O(n^2)
    explicit inverse DFT (catches a sign, scale or index error of the numpy route)."""
    n, seed = 64, 3
    for P_ in (0, 5):
        Om = P.spectral_probes(n, [2 * P_, 2 * P_ + 1], seed)
        z0, z1 = P.normal_pairs(np.arange(n, dtype=np.uint64), np.uint64(P_ | (1 << 63)), seed)
        v = np.sqrt(n) * (z0 + 1j * z1)
        jj, kk = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        u = (np.exp(2j * np.pi * jj * kk / n) @ v) / n
        assert np.max(np.abs(Om[:, 0] - u.real)) <= 1e-13
        assert np.max(np.abs(Om[:, 1] - u.imag)) <= 1e-13
    # a column does not depend on which others are requested (odd column alone, out of order)
    Om = P.spectral_probes(n, [7, 4, 5], seed)
    assert np.array_equal(Om[:, 2], P.spectral_probes(n, [4, 5], seed)[:, 1])
    assert np.array_equal(Om[:, 0], P.spectral_probes(n, [6, 7], seed)[:, 1])


def test_spectral_probes_are_iid_standard_normal():
    """The distribution claim of reading R35: entries N(0,1), columns (also the two of a pair and
    the entries of one column) uncorrelated, and a different stream from the entrywise probes."""
    n = 1 << 14
    Om = P.spectral_probes(n, list(range(8)), seed=1)
    assert Om.shape == (n, 8) and Om.flags.f_contiguous
    assert abs(Om.mean()) < 0.02
    assert abs(Om.var() - 1.0) < 0.03
    c = np.corrcoef(Om.T)
    assert np.max(np.abs(c - np.eye(8))) < 0.05
    assert abs(np.corrcoef(Om[:-1, 0], Om[1:, 0])[0, 1]) < 0.05     # neighbouring entries
    from scipy import stats
    assert stats.kstest(Om.ravel(), "norm").pvalue > 1e-3
    E = P.probes(n, list(range(8)), seed=1)
    assert np.max(np.abs(np.corrcoef(np.hstack([Om, E]).T)[:8, 8:])) < 0.05
    # the plan rule: 1-D boxes with more than 2048 fine-grid points (the four-step layout)
    from paper_2308_14490_b200 import inputs as I
    assert I.make_config("interval", 2048).spectral_probes and not I.make_config("interval", 1024).spectral_probes
    assert not I.get_config("c1").spectral_probes and I.get_config("c2").spectral_probes
    assert not I.get_config("c3").spectral_probes
    cfg = I.make_config("interval", 2048)
    assert np.array_equal(P.probe_matrix(cfg, [3], cfg.seed), P.spectral_probes(cfg.N, [3], cfg.seed))
