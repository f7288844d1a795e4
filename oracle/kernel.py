"""Gaussian RBF, derivatives and periodisation (Sec. 2.1).

Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import math

import numpy as np


def phi(r, eps):
    """Gaussian RBF, PAPER.md:54 Eq. (rbf): phi(r) = exp(-eps^2 r^2)."""
    r = np.asarray(r)
    return np.exp(-(eps * eps) * r * r)


def phi1(r, eps):
    """First derivative of Eq. (rbf): phi'(r) = -2 eps^2 r exp(-eps^2 r^2) -- the
    Neumann rows n . grad phi_j of the flower example."""
    r = np.asarray(r)
    e2 = eps * eps
    return -2.0 * e2 * r * np.exp(-e2 * r * r)


def phi2(r, eps):
    """Second derivative: phi''(r) = -2 eps^2 exp(-eps^2 r^2) (1 - 2 eps^2 r^2)."""
    r = np.asarray(r)
    e2 = eps * eps
    return -2.0 * e2 * np.exp(-e2 * r * r) * (1.0 - 2.0 * e2 * r * r)


def _m_max(eps: float, T: float) -> int:
    # Keep every translate that does not underflow in binary64 for |x - 2mT| measured
    # from the nearest period: exp(-745) is below the smallest subnormal.
    return 1 + int(math.ceil(math.sqrt(745.0) / (2.0 * T * eps)))


def periodized(x, eps, T, order: int = 0):
    """phi^per(x) = sum_m phi(x - 2 m T), PAPER.md:58-59 Eq. (periodic_rbf).

    order 0 -> phi, 1 -> phi', 2 -> phi'' (the periodisation of the
    derivative is the derivative of the periodisation, term by term).
    All non-underflowing translates are summed.
    """
    x = np.asarray(x)
    if x.dtype != np.longdouble:
        x = x.astype(np.float64)
    if order not in (0, 1, 2):
        raise ValueError("order must be 0, 1 or 2")
    f = (phi, phi1, phi2)[order]
    center = np.round(x / (2.0 * T))
    mm = _m_max(eps, T)
    out = np.zeros_like(x)
    for d in range(-mm, mm + 1):
        out = out + f(x - 2.0 * (center + d) * T, eps)
    return out


def shape_constant(T: float, tau0: float) -> float:
    """PAPER.md:65-67 Eq. (4): c = pi / (2 T sqrt(2 log(1 + tau0^-2))), natural log."""
    if not (T > 0 and 0 < tau0 < 1):
        raise ValueError("need T > 0 and 0 < tau0 < 1")
    return math.pi / (2.0 * T * math.sqrt(2.0 * math.log1p(tau0 ** -2)))


def theorem7_W(delta: float, tau0: float) -> float:
    """PAPER.md:453-455 (Theorem 7): W = (1/pi) sqrt(-2 log(delta) log(1 + tau0^-2))."""
    return math.sqrt(-2.0 * math.log(delta) * math.log1p(tau0 ** -2)) / math.pi


def tau0_from_eps_h(eps_h: float) -> float:
    """Invert Eq. (4) with eps = c N, h = 2T/N:  eps h = 2 T c = pi / sqrt(2 log(1+tau0^-2)).

    Used to express BASELINE's eps*h = 0.5 in the paper's tau0 (SURVEY.md §0 trap 3).
    """
    L = (math.pi / eps_h) ** 2 / 2.0        # = log(1 + tau0^-2)
    return 1.0 / math.sqrt(math.expm1(L))
