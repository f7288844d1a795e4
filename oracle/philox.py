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
1-D plans with more than 2048 fine-grid points draw their probes in the frequency domain
instead (`spectral_probes`, reading R35); `probe_matrix` picks the definition.
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


def normal_pairs(m, j, seed: int):
    """The two standard normals (z0, z1) of counter (m, j): Box-Muller of one Philox4x32-10 block."""
    m = np.asarray(m, dtype=np.uint64)
    j = np.asarray(j, dtype=np.uint64)
    seed = np.uint64(seed)
    x0, x1, x2, x3 = philox4x32_10(m & MASK32, m >> S32, j & MASK32, j >> S32,
                                   seed & MASK32, seed >> S32)
    a = ((x1 << S32) | x0) >> np.uint64(11)
    b = ((x3 << S32) | x2) >> np.uint64(11)
    u1 = (a + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = b.astype(np.float64) * 2.0 ** -53
    r = np.sqrt(-2.0 * np.log(u1))
    return r * np.cos(2.0 * np.pi * u2), r * np.sin(2.0 * np.pi * u2)


def probes(N: int, cols, seed: int) -> np.ndarray:
    """Omega[:, cols] as an (N, len(cols)) float64 Fortran array."""
    cols = np.asarray(cols, dtype=np.uint64)
    npair = (N + 1) // 2
    m = np.arange(npair, dtype=np.uint64)[:, None]
    z0, z1 = normal_pairs(m, cols[None, :], seed)
    out = np.empty((2 * npair, cols.shape[0]), dtype=np.float64)
    out[0::2] = z0
    out[1::2] = z1
    return np.asfortranarray(out[:N])


SPECTRAL_TAG = 1 << 63


def spectral_probes(n: int, cols, seed: int) -> np.ndarray:
    """Omega[:, cols] of the spectral probe definition (reading R35), (n, len(cols)) Fortran.

    Column pair P (columns 2P, 2P+1) is the real / imaginary part of u_P = IFFT_n(v_P) with the
    unnormalised spectrum v_P[k] = sqrt(n) (z0 + i z1), (z0, z1) = normal_pairs(k, P + 2^63), i.e.
        u_P[j] = (1/n) sum_k v_P[k] exp(+2 pi i j k / n).
    (The DFT of a vector of i.i.d. N(0,1) + i N(0,1) entries is sqrt(n) x a unitary map of it, so
    v_P has i.i.d. circular entries of variance 2n and Omega's columns are i.i.d. N(0,1) -- pinned by
    tests/test_oracle_kernel.py.)  A plain length-n inverse DFT in numpy."""
    cols = [int(c) for c in cols]
    out = np.empty((n, len(cols)), dtype=np.float64, order="F")
    k = np.arange(n, dtype=np.uint64)
    cache = {}
    for idx, c in enumerate(cols):
        P = c // 2
        if P not in cache:
            z0, z1 = normal_pairs(k, np.uint64(P | SPECTRAL_TAG), seed)
            v = np.sqrt(float(n)) * (z0 + 1j * z1)
            cache[P] = np.fft.ifft(v)
        out[:, idx] = cache[P].real if c % 2 == 0 else cache[P].imag
    return out


def probe_matrix(cfg, cols, seed: int) -> np.ndarray:
    """Omega[:, cols] of the plan `cfg` (inputs.Config): spectral probes where cfg.spectral_probes
    (1-D boxes with more than 2048 fine-grid points), entrywise Philox otherwise."""
    if cfg.spectral_probes:
        return spectral_probes(cfg.N, cols, seed)
    return probes(cfg.N, cols, seed)
