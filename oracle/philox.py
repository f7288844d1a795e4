"""Philox4x32-10 counter-based generator + Box-Muller, the probe matrix Omega.

Test infrastructure only (see oracle/__init__.py).  This is an independent
implementation of the same generator the CUDA path uses (csrc/az_common.cuh (probe_pair));
the two share no code (task rules: "each side implements the same
counter-based generator").

Probes: PAPER.md:269 ("r+p matrix vector products" with a random matrix) and
SPEC.md:272 (i.i.d. standard normal Omega).  Specification ("Probe
generator"):
  key     = (seed mod 2^32, seed >> 32)
  counter = (m mod 2^32, m >> 32, j mod 2^32, j >> 32),   m = i >> 1 (row pair), j = global column
  x0..x3  = Philox4x32-10(counter, key)
  u1 = (((x1 << 32) | x0) >> 11) + 1) * 2^-53      in (0, 1]
  u2 = (((x3 << 32) | x2) >> 11)      * 2^-53      in [0, 1)
  Omega[2m, j]   = sqrt(-2 ln u1) cos(2 pi u2)
  Omega[2m+1, j] = sqrt(-2 ln u1) sin(2 pi u2)
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint64(0x9E3779B9)
W1 = np.uint64(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)
S32 = np.uint64(32)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32 with 10 rounds (Salmon et al., SC'11).  Inputs are uint64 arrays holding 32-bit values."""
    c0, c1, c2, c3 = (np.asarray(v, dtype=np.uint64) & MASK32 for v in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint64) & MASK32
    k1 = np.asarray(k1, dtype=np.uint64) & MASK32
    for _ in range(10):
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> S32, p0 & MASK32
        hi1, lo1 = p1 >> S32, p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & MASK32, lo1, (hi0 ^ c3 ^ k1) & MASK32, lo0
        k0 = (k0 + W0) & MASK32
        k1 = (k1 + W1) & MASK32
    return c0, c1, c2, c3


def probes(N: int, cols, seed: int) -> np.ndarray:
    """Omega[:, cols] as an (N, len(cols)) float64 Fortran array."""
    cols = np.asarray(cols, dtype=np.uint64)
    npair = (N + 1) // 2
    m = np.arange(npair, dtype=np.uint64)[:, None]
    j = cols[None, :]
    seed = np.uint64(seed)
    x0, x1, x2, x3 = philox4x32_10(m & MASK32, m >> S32, j & MASK32, j >> S32,
                                   seed & MASK32, seed >> S32)
    a = ((x1 << S32) | x0) >> np.uint64(11)
    b = ((x3 << S32) | x2) >> np.uint64(11)
    u1 = (a + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = b.astype(np.float64) * 2.0 ** -53
    r = np.sqrt(-2.0 * np.log(u1))
    out = np.empty((2 * npair, cols.shape[0]), dtype=np.float64)
    out[0::2] = r * np.cos(2.0 * np.pi * u2)
    out[1::2] = r * np.sin(2.0 * np.pi * u2)
    return np.asfortranarray(out[:N])
