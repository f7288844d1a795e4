"""Block-column circulant structure of the periodic problem (Sec. 3.1, 5.1, 6.2.2).

Test infrastructure only (see oracle/__init__.py).

Notation follows the paper:
  F      unitary DFT, F_kl = exp(+2 pi i (k-1)(l-1)/N) / sqrt(N)
  Pi     permutation grouping the L = sN grid points into s shifted grids
  P      block diagonal matrix with F* on the diagonal                     PAPER.md:167-173 Eq. (P)
  B      = P Pi A^c F, block-column diagonal, diagonals d_i
  B^dag  blocks D~_i = (sum_j D_j* D_j)^-1 D_i*                           PAPER.md:190-209 Eq. (B_pinv)
  Z*     = F B^dag P E
  2-D:   B = B^x (x) B^y; Laplacian rows B = B2^x(x)B0^y + B0^x(x)B2^y + k0^2 B0^x(x)B0^y
                                                                           PAPER.md:577, 796-806

Two transform backends are offered for the same formulas:
  "ld"  explicit DFT matrices in extended precision (numpy longdouble, 64-bit
        mantissa) -- the Z* reference of SURVEY.md §8(c-2) O2;
  "fft" numpy.fft in binary64 (a library primitive serving as the step F / F*),
        for the large configurations.

Readings (listed in DESIGN.md):
  * Lemma 3 writes d_i = F* v_i; with the unitary F of PAPER.md:163
    the diagonal of F* C F for a circulant C with first column v is sqrt(N) F* v,
    i.e. the plain (unnormalised, e^{-i}) DFT of v.  We define the diagonals as
    diag(F* A^c_i F), which is what B = P Pi A^c F states; `diagonals_dense`
    computes exactly that and the tests pin it to the sqrt(N) F* v form and to
    the Poisson-summation closed form of Lemma 4's proof.
  * explicit_d has e^{+i...}; for the unshifted grid (i=1) the
    sign is immaterial (v_1 is even); for i >= 2 it is the complex conjugate of
    diag(F* A^c_i F).  We follow the definition of B.
  * Thresholding ("eigenvalue-thresholded", BASELINE north star): with
    sigma(k)^2 = sum_i |d_i(k)|^2 (the squared singular values of B, hence of A^c),
    D~_i(k) = conj(d_i(k)) / sigma(k)^2 if sigma(k) > rcond * max sigma, else 0.
"""
from __future__ import annotations

import functools

import numpy as np

from .kernel import periodized

LD = np.longdouble
CLD = np.clongdouble
PI_LD = LD("3.14159265358979323846264338327950288419716939937510")


# --------------------------------------------------------------------------------------
# DFT matrices and the permutation Pi
# --------------------------------------------------------------------------------------

@functools.lru_cache(maxsize=16)
def dft_F(N: int) -> np.ndarray:
    """Paper's unitary F, extended precision."""
    k = np.arange(N)
    kl = np.outer(k, k) % N                   # exact integer phase index
    ang = (2 * PI_LD / N) * kl.astype(LD)
    return (np.cos(ang) + 1j * np.sin(ang)).astype(CLD) / np.sqrt(LD(N))


def polyphase_index(n: int, s: int) -> np.ndarray:
    """Pi as an index map: (Pi g)[i*n + k] = g[k*s + i]  (rows k + (j-1)s)."""
    i = np.arange(s)[:, None]
    k = np.arange(n)[None, :]
    return (k * s + i).reshape(-1)


# --------------------------------------------------------------------------------------
# per-axis diagonals d_i (Lemma 3) and closed forms
# --------------------------------------------------------------------------------------

def kernel_samples(eps: float, T: float, n: int, s: int, order: int = 0, dtype=np.float64):
    """v_i[k] = phi_1(x~_{i,k}) with phi_1(x) = phi^per(x - c_1), c_1 = -T (Lemma 3).

    x~_{i,k} - c_1 = i h_L + k h_N (0-based i, k).  Returns shape (s, n).
    """
    hN = 2.0 * T / n
    hL = 2.0 * T / (s * n)
    i = np.arange(s, dtype=dtype)[:, None]
    k = np.arange(n, dtype=dtype)[None, :]
    x = i * dtype(hL) + k * dtype(hN)
    return periodized(x, eps, T, order)


def circulant(v: np.ndarray) -> np.ndarray:
    """Dense circulant block with first column v: C[k, j] = v[(k - j) mod n]."""
    n = v.shape[0]
    idx = (np.arange(n)[:, None] - np.arange(n)[None, :]) % n
    return v[idx]


def diagonals_dense(v: np.ndarray) -> np.ndarray:
    """d_i = diag(F* A^c_i F) by dense products in extended precision (B = P Pi A^c F)."""
    s, n = v.shape
    F = dft_F(n)
    out = np.empty((s, n), dtype=CLD)
    for i in range(s):
        C = circulant(v[i].astype(LD)).astype(CLD)
        out[i] = np.diag(F.conj().T @ C @ F)
    return out


def diagonals(v: np.ndarray, backend: str = "fft") -> np.ndarray:
    """d_i = sqrt(N) F* v_i  (Lemma 3 with the sqrt(N) reading): the e^{-i} DFT of v_i."""
    s, n = v.shape
    if backend == "fft":
        return np.fft.fft(v.astype(np.float64), axis=1)
    F = dft_F(n)
    return np.sqrt(LD(n)) * (v.astype(LD).astype(CLD) @ F.conj())   # rows: (F* v_i)^T = v_i^T conj(F)


def poisson_closed_form(eps: float, T: float, n: int, s: int, q_max: int = 8) -> np.ndarray:
    """Lemma 4 proof, Poisson summation of the kernel samples:

    sum_m exp(-eps^2 (m h + delta)^2) e^{-2 pi i k m / n}
        = (sqrt(pi)/(eps h)) sum_q exp(-pi^2 (k/n - q)^2 / (eps h)^2) e^{+2 pi i (k/n - q) delta / h}
    with delta = i h/s the shift of grid i.  Returns (s, n) complex (binary64).
    """
    h = 2.0 * T / n
    eh = eps * h
    k = np.arange(n)[None, :, None] / n
    q = np.arange(-q_max, q_max + 1)[None, None, :]
    delta = (np.arange(s)[:, None, None] * h / s)
    nu = k - q
    terms = np.exp(-(np.pi ** 2) * nu * nu / (eh * eh)) * np.exp(2j * np.pi * nu * delta / h)
    return (np.sqrt(np.pi) / eh) * terms.sum(axis=2)


# --------------------------------------------------------------------------------------
# 1-D / 2-D symbols and the pseudo-inverse
# --------------------------------------------------------------------------------------

class Symbol:
    """Diagonals of B for a dim-d problem, shape (P, N) with P = s^d phases, N = n (1-D) or
    N^x N^y (2-D; the y axis may have its own N^y and T^y, "N = N^x N^y").

    Phase p enumerates (p_x, p_y) row-major; frequency index (k_x, k_y) row-major.
    """

    def __init__(self, dim: int, n: int, s: int, eps: float, T: float, row_op: int,
                 alpha: float = 1.0, k0sq: float = 0.0, backend: str = "fft",
                 diag_fn=None, n_y: int = 0, T_y: float = 0.0):
        self.dim, self.n, self.s, self.eps, self.T = dim, n, s, eps, T
        self.ny, self.Ty = (n_y or n), (T_y or T)
        self.backend = backend
        dt = LD if backend == "ld" else np.float64

        def axis_d(order, nn, TT, axis):
            if diag_fn is not None:
                return diag_fn(order) if axis == 0 or (nn, TT) == (n, T) else diag_fn(order, axis)
            return diagonals(kernel_samples(eps, TT, nn, s, order, dt), backend)

        d0 = axis_d(0, n, T, 0)
        if dim == 1:
            if row_op != 0:
                d2 = axis_d(2, n, T, 0)
                self.d = alpha * (d2 + k0sq * d0)          # 1-D ODE rows, normalised
            else:
                self.d = d0
        else:
            ny = self.ny
            d0y = axis_d(0, ny, self.Ty, 1)                # B^y: the y axis' own samples (N^y, T^y)
            if row_op == 0:
                # B = B^x (x) B^y
                self.d = np.einsum("ak,bl->abkl", d0, d0y).reshape(s * s, n * ny)
            else:
                d2 = axis_d(2, n, T, 0)
                d2y = axis_d(2, ny, self.Ty, 1)
                # B = B2^x (x) B0^y + B0^x (x) B2^y + k0^2 B0^x (x) B0^y
                t = (np.einsum("ak,bl->abkl", d2, d0y) + np.einsum("ak,bl->abkl", d0, d2y)
                     + k0sq * np.einsum("ak,bl->abkl", d0, d0y))
                self.d = alpha * t.reshape(s * s, n * ny)
        self.sigma2 = (np.abs(self.d) ** 2).sum(axis=0)   # diag of B*B

    def pinv(self, rcond: float):
        """Diagonals of B^dag, thresholded (PAPER.md:190-209 + threshold reading)."""
        smax2 = self.sigma2.max()
        keep = self.sigma2 > (rcond * rcond) * smax2
        dt = np.where(keep[None, :], np.conj(self.d) / np.where(keep, self.sigma2, 1.0)[None, :], 0.0)
        return dt, int((~keep).sum())


# --------------------------------------------------------------------------------------
# transforms along axes (the steps F, F*, P, P*)
# --------------------------------------------------------------------------------------

def _F_axis(x: np.ndarray, axis: int, backend: str, inverse: bool) -> np.ndarray:
    """Apply F (inverse=False) or F* (inverse=True) along `axis` (unitary)."""
    n = x.shape[axis]
    if backend == "fft":
        # F a = sqrt(n) * ifft(a);  F* a = fft(a) / sqrt(n)
        if inverse:
            return np.fft.fft(x, axis=axis) / np.sqrt(n)
        return np.fft.ifft(x, axis=axis) * np.sqrt(n)
    M = dft_F(n)
    if inverse:
        M = M.conj().T
    xm = np.moveaxis(x.astype(CLD), axis, -1)
    return np.moveaxis(xm @ M.T, -1, axis)


def _to_phases(g: np.ndarray, dim: int, n: int, s: int, ny: int = 0) -> np.ndarray:
    """Pi (per axis) on a natural-order grid vector: returns (P, N) phase blocks."""
    if dim == 1:
        return g.reshape(n, s).T.copy()
    ny = ny or n
    G = g.reshape(n, s, ny, s)              # [k_x, p_x, k_y, p_y]
    return G.transpose(1, 3, 0, 2).reshape(s * s, n * ny).copy()


def _from_phases(c: np.ndarray, dim: int, n: int, s: int, ny: int = 0) -> np.ndarray:
    """Pi^T: (P, N) phase blocks back to the natural-order grid vector."""
    if dim == 1:
        return c.T.reshape(-1).copy()
    ny = ny or n
    G = c.reshape(s, s, n, ny).transpose(2, 0, 3, 1)
    return G.reshape(-1).copy()


def _F_coeff(a: np.ndarray, dim: int, n: int, backend: str, inverse: bool, ny: int = 0) -> np.ndarray:
    if dim == 1:
        return _F_axis(a, 0, backend, inverse)
    A = a.reshape(n, ny or n)
    A = _F_axis(A, 0, backend, inverse)
    A = _F_axis(A, 1, backend, inverse)
    return A.reshape(-1)


def _P_blocks(c: np.ndarray, dim: int, n: int, backend: str, inverse: bool, ny: int = 0) -> np.ndarray:
    """P = blockdiag(F*) (inverse=True) or P* = blockdiag(F) (inverse=False), per phase block."""
    if dim == 1:
        return _F_axis(c, 1, backend, inverse)
    C = c.reshape(c.shape[0], n, ny or n)
    C = _F_axis(C, 1, backend, inverse)
    C = _F_axis(C, 2, backend, inverse)
    return C.reshape(c.shape[0], -1)


class PeriodicOperators:
    """A^c, Z* and friends built from the paper's factorisation (Sec. 3.2.2, 5.2)."""

    def __init__(self, sym: Symbol, rcond: float):
        self.sym = sym
        self.dt, self.n_dropped = sym.pinv(rcond)
        self.dim, self.n, self.s, self.backend = sym.dim, sym.n, sym.s, sym.backend
        self.ny = sym.ny

    def apply_Ac(self, a: np.ndarray) -> np.ndarray:
        """A^c a = Pi^T P* B F* a  (natural-order full grid output)."""
        y = _F_coeff(a, self.dim, self.n, self.backend, inverse=True, ny=self.ny)        # F* a
        c = self.sym.d * y[None, :]                                                     # B
        c = _P_blocks(c, self.dim, self.n, self.backend, inverse=False, ny=self.ny)      # P*
        return _from_phases(c, self.dim, self.n, self.s, ny=self.ny)                    # Pi^T

    def apply_Zstar_grid(self, g: np.ndarray) -> np.ndarray:
        """Z* restricted to a grid vector already extended by zeros (E applied): F B^dag P Pi g."""
        c = _to_phases(g, self.dim, self.n, self.s, ny=self.ny)                         # Pi
        c = _P_blocks(c, self.dim, self.n, self.backend, inverse=True, ny=self.ny)       # P
        y = (self.dt * c).sum(axis=0)                                                   # B^dag
        return _F_coeff(y, self.dim, self.n, self.backend, inverse=False, ny=self.ny)   # F

    def zstar_norm(self) -> float:
        """||Z*||_2 = 1 / (smallest kept singular value of A^c) (unitary F, P)."""
        s2 = self.sym.sigma2
        keep = np.abs(self.dt).sum(axis=0) > 0
        # singular values of A^c: sigma(k) = sqrt(sum_i |d_i(k)|^2) with the sqrt(N) reading
        # of Lemma 3 divided back out: A^c = Pi^T P* B F* has the singular values of B.
        return float(1.0 / np.sqrt(s2[keep].min()))
