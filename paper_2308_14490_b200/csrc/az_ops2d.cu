// 2-D operators: A, A^T, Z*, A - A Z* A, I - A Z* on the tensor-product problem (Sec. 5,
// Sec. 6.2) as a small number of HBM passes over row-major [x][y] arrays (y contiguous).
//
// Fine-grid formulation per axis (see az_ops1d.cu and DESIGN.md): for value rows
//   A^c a = IFFT2_L( W(kx) W(ky) . a^(kx mod n, ky mod n) ) / L^2,
// for Laplacian rows (k0^2 = 0) the symbol is alpha (W2(kx) W0(ky) + W0(kx) W2(ky)).
// Z* = F B^dag P E becomes: FFT2_L of the zero-padded data, fold the s^2 aliases with conj(W),
// multiply by zinv = 1/sigma^2 (thresholded), IFFT2_n.
//
// Pass structure (each pass = one kernel over a batch of vector pairs, complex packing of two
// real vectors per pair):
//   K1  rows  (y, n):  coefficient input (vector or Philox probes) -> FFT_n
//   K2  cols  (x):     FFT_n -> [store v^] -> expand to the s x s aliases x W / L^2 -> IFFT_L
//   K3  rows  (y, L):  IFFT_L -> E R (mask) -> FFT_L
//   K4  cols  (x):     FFT_L of the s fine columns -> fold conj(W) -> x zinv -> (r^ = v^ - w^)
//                      -> expand x W / L^2 -> IFFT_L      (or IFFT_n for Z*, A^T)
//   K5  rows  (y, L):  IFFT_L -> R (gather the collocation rows)  [-> b - . for I - A Z*]
//   Z1  rows  (y, L):  E (scatter the rows onto the grid) -> FFT_L
//   Z3  rows  (y, n):  IFFT_n -> coefficient output
//   KB  boundary rows beta phi_j(x_b) as separable windowed sums, KBT its adjoint.
#include <algorithm>
#include <cmath>

#include "az_fft.cuh"
#include "az_internal.h"

struct P2 {
  const cplx* W0;
  const cplx* W2;
  const cplx* W0y;   // the y axis' symbols (== W0 / W2 for square boxes)
  const cplx* W2y;
  const double* zinv;
  const int32_t* pos;
  const uint8_t* mask;
  const cplx* tw;
  const double* bw;
  const int32_t* bj;
  int lap;
  double k0sq;
  double alpha, beta, eps, T, h;
  int n, s, L;      // x axis (the column passes)
  int ny, Ly;       // y axis (the row passes, contiguous)
  int64_t M, Mb, N, GG;
  uint64_t seed;
  cplx* C1;
  cplx* G;
  const double* in;
  int64_t ldin;
  double* out;
  int64_t ldout;
  int64_t nvec;
  int64_t col0;
  int64_t pair0;
  int win, win_y;   // boundary windows (centres along x / y)
};

// alpha (W2x W0y + W0x W2y + k0^2 W0x W0y) for LAPLACIAN / Helmholtz rows
AZ_D cplx sym2(const P2& a, int kx, int ky) {
  if (!a.lap) return cmul(a.W0[kx], a.W0y[ky]);
  const cplx w00 = cmul(a.W0[kx], a.W0y[ky]);
  return cscale(cadd(cadd(cmul(a.W2[kx], a.W0y[ky]), cmul(a.W0[kx], a.W2y[ky])), cscale(w00, a.k0sq)), a.alpha);
}

struct Cols {
  int64_t cre, cim;
  bool has_im;
};
AZ_D Cols pair_cols(const P2& a, int b) {
  Cols c;
  c.cre = 2 * (a.pair0 + b);
  c.cim = c.cre + 1;
  c.has_im = c.cim < a.nvec;
  return c;
}

// ------------------------------------------------------------------------------------------
// row passes
// ------------------------------------------------------------------------------------------
enum { RK_IN_COEF = 0, RK_FINE_MASK = 1, RK_OUT_GATHER = 2, RK_OUT_RESID = 3, RK_IN_ROWS = 4,
       RK_OUT_COEF = 5, RK_COEF_W = 6 };

template <int LEN, int KIND, int SRC>
__global__ void __launch_bounds__(256) k2_rows(P2 a, int nrows, double cout) {
  extern __shared__ cplx sm[];
  constexpr int TPF = LEN / 8;
  constexpr int RPC = 256 / TPF > 0 ? 256 / TPF : 1;
  const int f = threadIdx.x / TPF, j = threadIdx.x % TPF;
  const int row = blockIdx.x * RPC + f;
  const bool live = row < nrows;
  const int b = blockIdx.y;
  const Cols cc = pair_cols(a, b);
  cplx* buf = sm + f * spad_len(LEN);
  cplx* C1b = a.C1 + (int64_t)b * a.N;
  cplx* Gb = a.G + (int64_t)b * a.GG;

  // ---- load ----
  if constexpr (KIND == RK_IN_COEF) {
    if constexpr (SRC == SRC_PROBE) {
      for (int e = j; e < LEN / 2; e += TPF) {
        cpair pr = {czero(), czero()};
        if (live) {
          const int64_t i = (int64_t)row * a.ny + 2 * e;
          pr = probe_cplx_pair((uint64_t)(i >> 1), (uint64_t)(a.col0 + cc.cre), (uint64_t)(a.col0 + cc.cim),
                               cc.has_im, a.seed);
        }
        buf[spad(2 * e)] = pr.a;
        buf[spad(2 * e + 1)] = pr.b;
      }
    } else {
      for (int e = j; e < LEN; e += TPF) {
        cplx v = czero();
        if (live) {
          const int64_t i = (int64_t)row * a.ny + e;
          v.x = a.in[i + cc.cre * a.ldin];
          v.y = cc.has_im ? a.in[i + cc.cim * a.ldin] : 0.0;
        }
        buf[spad(e)] = v;
      }
    }
  } else if constexpr (KIND == RK_IN_ROWS) {
    for (int e = j; e < LEN; e += TPF) {
      cplx v = czero();
      if (live) {
        const int r = a.pos[(int64_t)row * a.Ly + e];
        if (r >= 0) {
          v.x = a.in[r + cc.cre * a.ldin];
          v.y = cc.has_im ? a.in[r + cc.cim * a.ldin] : 0.0;
        }
      }
      buf[spad(e)] = v;
    }
  } else if constexpr (KIND == RK_OUT_COEF || KIND == RK_COEF_W) {
    for (int e = j; e < LEN; e += TPF) buf[spad(e)] = live ? C1b[(int64_t)row * a.ny + e] : czero();
  } else {   // fine rows
    for (int e = j; e < LEN; e += TPF) buf[spad(e)] = live ? Gb[(int64_t)row * a.Ly + e] : czero();
  }
  __syncthreads();

  // ---- transform(s) ----
  if constexpr (KIND == RK_IN_COEF || KIND == RK_IN_ROWS) {
    fft_smem<LEN, -1>(buf, j, a.tw, TWN);
  } else if constexpr (KIND == RK_FINE_MASK) {
    fft_smem<LEN, 1>(buf, j, a.tw, TWN);
    for (int e = j; e < LEN; e += TPF)
      if (!live || !a.mask[(int64_t)row * a.Ly + e]) buf[spad(e)] = czero();
    __syncthreads();
    fft_smem<LEN, -1>(buf, j, a.tw, TWN);
  } else {
    fft_smem<LEN, 1>(buf, j, a.tw, TWN);
  }

  if (!live) return;
  // ---- store ----
  if constexpr (KIND == RK_IN_COEF) {
    for (int e = j; e < LEN; e += TPF) C1b[(int64_t)row * a.ny + e] = buf[spad(e)];
  } else if constexpr (KIND == RK_IN_ROWS || KIND == RK_FINE_MASK) {
    for (int e = j; e < LEN; e += TPF) Gb[(int64_t)row * a.Ly + e] = buf[spad(e)];
  } else if constexpr (KIND == RK_OUT_GATHER || KIND == RK_OUT_RESID) {
    for (int e = j; e < LEN; e += TPF) {
      const int r = a.pos[(int64_t)row * a.Ly + e];
      if (r >= 0) {
        const cplx v = buf[spad(e)];
        if constexpr (KIND == RK_OUT_RESID) {
          a.out[r + cc.cre * a.ldout] = a.in[r + cc.cre * a.ldin] - v.x;
          if (cc.has_im) a.out[r + cc.cim * a.ldout] = a.in[r + cc.cim * a.ldin] - v.y;
        } else {
          a.out[r + cc.cre * a.ldout] = v.x;
          if (cc.has_im) a.out[r + cc.cim * a.ldout] = v.y;
        }
      }
    }
  } else if constexpr (KIND == RK_OUT_COEF) {
    for (int e = j; e < LEN; e += TPF) {
      const int64_t i = (int64_t)row * a.ny + e;
      const cplx v = buf[spad(e)];
      a.out[i + cc.cre * a.ldout] = v.x * cout;
      if (cc.has_im) a.out[i + cc.cim * a.ldout] = v.y * cout;
    }
  } else {   // RK_COEF_W: spatial coefficients of the pair, kept in C1 for the boundary rows
    for (int e = j; e < LEN; e += TPF) C1b[(int64_t)row * a.ny + e] = cscale(buf[spad(e)], cout);
  }
}

// ------------------------------------------------------------------------------------------
// column passes (x direction); a CTA owns TC adjacent coefficient columns ky and their s fine
// columns ky + my n.  Threads: TC * NN/8; the length-L FFTs use L/(NN/8) values per thread.
// ------------------------------------------------------------------------------------------
enum { CK_EXPAND = 0, CK_EXPAND_KEEP = 1, CK_STEP1 = 2, CK_RESID = 3, CK_ZSTAR = 4, CK_AT = 5 };

template <int NN, int LL, int TC, int KIND, int WANT_W>
__global__ void __launch_bounds__(TC * NN / 8) k2_cols(P2 a) {
  extern __shared__ cplx sm[];
  constexpr int TPF = NN / 8;
  constexpr int PLN = spad_len(NN), PLL = spad_len(LL);
  constexpr int NT = TC * TPF;
  const int tid = threadIdx.x;
  const int f = tid / TPF, j = tid % TPF;
  const int b = blockIdx.y;
  const int c0 = blockIdx.x * TC;
  const int n = NN, s = LL / NN;        // x axis
  const int ny = a.ny, Ly = a.Ly;       // y axis: row strides of the coefficient / fine arrays
  cplx* bufN = sm;
  cplx* bufL = sm + TC * PLN;
  cplx* C1b = a.C1 + (int64_t)b * a.N;
  cplx* Gb = a.G + (int64_t)b * a.GG;
  const double cA = 1.0 / ((double)LL * (double)Ly);

  if constexpr (KIND == CK_EXPAND || KIND == CK_EXPAND_KEEP) {
    for (int e = tid; e < NN * TC; e += NT) {
      const int row = e / TC, c = e % TC;
      bufN[c * PLN + spad(row)] = C1b[(int64_t)row * ny + c0 + c];
    }
    __syncthreads();
    fft_smem<NN, -1>(bufN + f * PLN, j, a.tw, TWN);
    if constexpr (KIND == CK_EXPAND_KEEP) {
      for (int e = tid; e < NN * TC; e += NT) {
        const int row = e / TC, c = e % TC;
        C1b[(int64_t)row * ny + c0 + c] = bufN[c * PLN + spad(row)];
      }
    }
  } else {
    // fold the s^2 aliases: acc(kx, ky) = sum_{mx,my} conj(W) U
    for (int e = tid; e < NN * TC; e += NT) bufN[(e % TC) * PLN + spad(e / TC)] = czero();
    for (int my = 0; my < s; ++my) {
      for (int e = tid; e < LL * TC; e += NT) {
        const int row = e / TC, c = e % TC;
        bufL[c * PLL + spad(row)] = Gb[(int64_t)row * Ly + c0 + c + my * ny];
      }
      __syncthreads();
      fft_smem<LL, -1, TPF>(bufL + f * PLL, j, a.tw, TWN);
      for (int e = tid; e < NN * TC; e += NT) {
        const int kx = e / TC, c = e % TC;
        const int kyf = c0 + c + my * ny;
        cplx acc = bufN[c * PLN + spad(kx)];
        for (int mx = 0; mx < s; ++mx) {
          const int kxf = kx + mx * n;
          acc = cadd(acc, cmulc(bufL[c * PLL + spad(kxf)], sym2(a, kxf, kyf)));
        }
        bufN[c * PLN + spad(kx)] = acc;
      }
      __syncthreads();
    }
    for (int e = tid; e < NN * TC; e += NT) {
      const int kx = e / TC, c = e % TC;
      const int64_t k = (int64_t)kx * ny + c0 + c;
      cplx v = bufN[c * PLN + spad(kx)];
      if constexpr (KIND != CK_AT) v = cscale(v, a.zinv[k]);
      if constexpr (KIND == CK_STEP1) v = csub(C1b[k], v);       // r^ = v^ - w^
      bufN[c * PLN + spad(kx)] = v;
    }
    __syncthreads();
  }

  // ---- expand to the fine grid and inverse transform along x ----
  if constexpr (KIND == CK_EXPAND || KIND == CK_EXPAND_KEEP || KIND == CK_STEP1 || KIND == CK_RESID) {
    for (int my = 0; my < s; ++my) {
      for (int e = tid; e < LL * TC; e += NT) {
        const int kxf = e / TC, c = e % TC;
        const int kyf = c0 + c + my * ny;
        bufL[c * PLL + spad(kxf)] = cscale(cmul(bufN[c * PLN + spad(kxf & (n - 1))], sym2(a, kxf, kyf)), cA);
      }
      __syncthreads();
      fft_smem<LL, 1, TPF>(bufL + f * PLL, j, a.tw, TWN);
      for (int e = tid; e < LL * TC; e += NT) {
        const int row = e / TC, c = e % TC;
        Gb[(int64_t)row * Ly + c0 + c + my * ny] = bufL[c * PLL + spad(row)];
      }
      __syncthreads();
    }
  }
  if constexpr (KIND == CK_ZSTAR || KIND == CK_AT || WANT_W) {
    fft_smem<NN, 1>(bufN + f * PLN, j, a.tw, TWN);
    for (int e = tid; e < NN * TC; e += NT) {
      const int row = e / TC, c = e % TC;
      C1b[(int64_t)row * ny + c0 + c] = bufN[c * PLN + spad(row)];
    }
  }
}

// ------------------------------------------------------------------------------------------
// boundary rows: beta * sum_{jx,jy} phi^per(xb - c_jx) phi^per(yb - c_jy) w[jx][jy]
// one warp per (boundary point, pair); w from C1 (spatial, complex pair) or from the input
// coefficient columns.
// ------------------------------------------------------------------------------------------
template <int FROM_INPUT, int RESID>
__global__ void k2_boundary_rows(P2 a) {
  const int bp = blockIdx.x, b = blockIdx.y, lane = threadIdx.x;
  const Cols cc = pair_cols(a, b);
  const cplx* C1b = a.C1 + (int64_t)b * a.N;
  const int n = a.n, ny = a.ny, W = a.win, Wy = a.win_y;
  // Robin form (k_stencil2): weight of centre (t, l) = P[t] Y0[l] + Q[t] Y1[l]
  const double* wP = a.bw + (4 * bp + 0) * 64;
  const double* wY0 = a.bw + (4 * bp + 1) * 64;
  const double* wQ = a.bw + (4 * bp + 2) * 64;
  const double* wY1 = a.bw + (4 * bp + 3) * 64;
  const int jx0 = a.bj[2 * bp], jy0 = a.bj[2 * bp + 1];
  cplx acc = czero();
  for (int l = lane; l < Wy; l += 32) {
    const int jy = ((jy0 + l) % ny + ny) % ny;
    const double y0 = wY0[l], y1 = wY1[l];
    for (int t = 0; t < W; ++t) {
      const int jx = ((jx0 + t) % n + n) % n;
      const int64_t i = (int64_t)jx * ny + jy;
      cplx w;
      if (FROM_INPUT) {
        w.x = a.in[i + cc.cre * a.ldin];
        w.y = cc.has_im ? a.in[i + cc.cim * a.ldin] : 0.0;
      } else {
        w = C1b[i];
      }
      acc = cadd(acc, cscale(w, fma(wP[t], y0, wQ[t] * y1)));
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  if (lane == 0) {
    const int64_t r = a.M + bp;
    acc = cscale(acc, a.beta);
    if (RESID) {
      a.out[r + cc.cre * a.ldout] = a.in[r + cc.cre * a.ldin] - acc.x;
      if (cc.has_im) a.out[r + cc.cim * a.ldout] = a.in[r + cc.cim * a.ldin] - acc.y;
    } else {
      a.out[r + cc.cre * a.ldout] = acc.x;
      if (cc.has_im) a.out[r + cc.cim * a.ldout] = acc.y;
    }
  }
}

// A^T boundary part: x[jx][jy] += beta phi phi y_b  (scatter-add, after the interior part)
__global__ void k2_boundary_adjoint(P2 a) {
  const int bp = blockIdx.x, b = blockIdx.y, lane = threadIdx.x;
  const Cols cc = pair_cols(a, b);
  const int n = a.n, ny = a.ny, W = a.win, Wy = a.win_y;
  const double* wP = a.bw + (4 * bp + 0) * 64;
  const double* wY0 = a.bw + (4 * bp + 1) * 64;
  const double* wQ = a.bw + (4 * bp + 2) * 64;
  const double* wY1 = a.bw + (4 * bp + 3) * 64;
  const int jx0 = a.bj[2 * bp], jy0 = a.bj[2 * bp + 1];
  const int64_t r = a.M + bp;
  const double vre = a.beta * a.in[r + cc.cre * a.ldin];
  const double vim = cc.has_im ? a.beta * a.in[r + cc.cim * a.ldin] : 0.0;
  for (int l = lane; l < Wy; l += 32) {
    const int jy = ((jy0 + l) % ny + ny) % ny;
    const double y0 = wY0[l], y1 = wY1[l];
    for (int t = 0; t < W; ++t) {
      const int jx = ((jx0 + t) % n + n) % n;
      const double w = fma(wP[t], y0, wQ[t] * y1);
      const int64_t i = (int64_t)jx * ny + jy;
      atomicAdd(&a.out[i + cc.cre * a.ldout], vre * w);
      if (cc.has_im) atomicAdd(&a.out[i + cc.cim * a.ldout], vim * w);
    }
  }
}

// ------------------------------------------------------------------------------------------
// host orchestration
// ------------------------------------------------------------------------------------------
template <int LEN, int KIND, int SRC>
static az_status_t rows(const P2& a, int nrows, int nb, double cout, cudaStream_t st) {
  constexpr int TPF = LEN / 8;
  constexpr int RPC = 256 / TPF > 0 ? 256 / TPF : 1;
  const size_t sm = (size_t)RPC * spad_len(LEN) * sizeof(cplx);
  auto kern = k2_rows<LEN, KIND, SRC>;
  AZ_CUDA_CHECK(az_smem_attr(kern, sm));
  static const char* names[] = {"2d_rows_in_coef", "2d_rows_fine_mask", "2d_rows_out_gather", "2d_rows_out_resid",
                                "2d_rows_in_rows", "2d_rows_out_coef", "2d_rows_coef_w"};
  AzTrace tr(names[KIND], st, nb);
  kern<<<dim3(az_div_up(nrows, RPC), nb), RPC * TPF, sm, st>>>(a, nrows, cout);
  AZ_LAUNCH_CHECK();
  return AZ_OK;
}

template <int NN, int NY, int KIND, int WANT_W>
static az_status_t cols(const P2& a, int nb, cudaStream_t st) {
  constexpr int LL = 2 * NN;
  constexpr int TC0 = 2048 / NN;
  constexpr int TC1 = TC0 < 2 ? 2 : (TC0 > NN ? NN : TC0);
  constexpr int TC = TC1 > NY ? NY : TC1;   // adjacent y columns per CTA
  const size_t sm = (size_t)TC * (spad_len(NN) + spad_len(LL)) * sizeof(cplx);
  auto kern = k2_cols<NN, LL, TC, KIND, WANT_W>;
  AZ_CUDA_CHECK(az_smem_attr(kern, sm));
  static const char* names[] = {"2d_cols_expand", "2d_cols_expand_keep", "2d_cols_step1", "2d_cols_resid",
                                "2d_cols_zstar", "2d_cols_at"};
  AzTrace tr(names[KIND], st, nb);
  kern<<<dim3(az_div_up(NY, TC), nb), TC * NN / 8, sm, st>>>(a);
  AZ_LAUNCH_CHECK();
  return AZ_OK;
}

template <int NN, int NY>
static az_status_t run2d(const P2& a0, int op, int src, int64_t npairs, int64_t Bmax, cudaStream_t st) {
  constexpr int LL = 2 * NN, LY = 2 * NY;   // x: column passes; y: row passes
  const double n2 = (double)NN * NY;
  for (int64_t p0 = 0; p0 < npairs; p0 += Bmax) {
    P2 a = a0;
    a.pair0 = p0;
    const int nb = (int)std::min<int64_t>(Bmax, npairs - p0);
    const bool bnd = a.Mb > 0;
    switch (op) {
      case OP_A:
        AZ_TRY(rows<NY, RK_IN_COEF, SRC_VEC>(a, NN, nb, 1.0, st));
        AZ_TRY((cols<NN, NY, CK_EXPAND, 0>(a, nb, st)));
        AZ_TRY(rows<LY, RK_OUT_GATHER, SRC_VEC>(a, LL, nb, 1.0, st));
        if (bnd) {
          AzTrace tr("2d_boundary", st, nb);
          k2_boundary_rows<1, 0><<<dim3((unsigned)a.Mb, nb), 32, 0, st>>>(a);
          AZ_LAUNCH_CHECK();
        }
        break;
      case OP_STEP1:
        if (src == SRC_PROBE)
          AZ_TRY(rows<NY, RK_IN_COEF, SRC_PROBE>(a, NN, nb, 1.0, st));
        else
          AZ_TRY(rows<NY, RK_IN_COEF, SRC_VEC>(a, NN, nb, 1.0, st));
        AZ_TRY((cols<NN, NY, CK_EXPAND_KEEP, 0>(a, nb, st)));
        AZ_TRY(rows<LY, RK_FINE_MASK, SRC_VEC>(a, LL, nb, 1.0, st));
        if (bnd)
          AZ_TRY((cols<NN, NY, CK_STEP1, 1>(a, nb, st)));
        else
          AZ_TRY((cols<NN, NY, CK_STEP1, 0>(a, nb, st)));
        AZ_TRY(rows<LY, RK_OUT_GATHER, SRC_VEC>(a, LL, nb, 1.0, st));
        if (bnd) {
          AZ_TRY(rows<NY, RK_COEF_W, SRC_VEC>(a, NN, nb, 1.0 / n2, st));
          AzTrace tr("2d_boundary", st, nb);
          k2_boundary_rows<0, 0><<<dim3((unsigned)a.Mb, nb), 32, 0, st>>>(a);
          AZ_LAUNCH_CHECK();
        }
        break;
      case OP_RESID:
        AZ_TRY(rows<LY, RK_IN_ROWS, SRC_VEC>(a, LL, nb, 1.0, st));
        if (bnd)
          AZ_TRY((cols<NN, NY, CK_RESID, 1>(a, nb, st)));
        else
          AZ_TRY((cols<NN, NY, CK_RESID, 0>(a, nb, st)));
        AZ_TRY(rows<LY, RK_OUT_RESID, SRC_VEC>(a, LL, nb, 1.0, st));
        if (bnd) {
          AZ_TRY(rows<NY, RK_COEF_W, SRC_VEC>(a, NN, nb, 1.0 / n2, st));
          AzTrace tr("2d_boundary", st, nb);
          k2_boundary_rows<0, 1><<<dim3((unsigned)a.Mb, nb), 32, 0, st>>>(a);
          AZ_LAUNCH_CHECK();
        }
        break;
      case OP_ZSTAR:
        AZ_TRY(rows<LY, RK_IN_ROWS, SRC_VEC>(a, LL, nb, 1.0, st));
        AZ_TRY((cols<NN, NY, CK_ZSTAR, 0>(a, nb, st)));
        AZ_TRY(rows<NY, RK_OUT_COEF, SRC_VEC>(a, NN, nb, 1.0 / n2, st));
        break;
      case OP_AT:
        AZ_TRY(rows<LY, RK_IN_ROWS, SRC_VEC>(a, LL, nb, 1.0, st));
        AZ_TRY((cols<NN, NY, CK_AT, 0>(a, nb, st)));
        AZ_TRY(rows<NY, RK_OUT_COEF, SRC_VEC>(a, NN, nb, 1.0 / ((double)LL * LY), st));
        if (bnd) {
          AzTrace tr("2d_boundary", st, nb);
          k2_boundary_adjoint<<<dim3((unsigned)a.Mb, nb), 32, 0, st>>>(a);
          AZ_LAUNCH_CHECK();
        }
        break;
    }
  }
  return AZ_OK;
}

az_status_t az2_apply(az_plan_s* p, int op, int src, const double* in, int64_t ldin, double* out,
                      int64_t ldout, int64_t nvec, int64_t col0, cudaStream_t st) {
  P2 a;
  a.W0 = p->d_W0;
  a.W2 = p->d_W2;
  a.W0y = p->d_W0y;
  a.W2y = p->d_W2y;
  a.zinv = p->d_zinv;
  a.pos = p->d_pos;
  a.mask = p->d_mask;
  a.tw = p->d_tw;
  a.bw = p->d_bw;
  a.bj = p->d_bj;
  a.lap = p->op == AZ_ROW_LAPLACIAN;
  a.k0sq = p->k0sq;
  a.alpha = p->alpha;
  a.beta = p->beta;
  a.eps = p->eps;
  a.T = p->T;
  a.h = 2.0 * p->T / (double)p->n;
  a.n = (int)p->n;
  a.s = (int)p->s;
  a.L = (int)p->L;
  a.ny = (int)p->ny;
  a.Ly = (int)p->Ly;
  a.M = p->M;
  a.Mb = p->Mb;
  a.N = p->N;
  a.GG = p->G;
  a.seed = p->seed;
  a.C1 = p->d_C1;
  a.G = p->d_G;
  a.in = in;
  a.ldin = ldin;
  a.out = out;
  a.ldout = ldout;
  a.nvec = nvec;
  a.col0 = col0;
  a.pair0 = 0;
  a.win = p->win;
  a.win_y = p->win_y;
  const int64_t npairs = (nvec + 1) / 2;
  if (p->s != 2) {
    az_set_error("2-D layout supports L = 2 only");
    return AZ_ERR_NOT_SUPPORTED;
  }
  // square boxes, and anisotropic ones with n_y = n / 2 or 2 n
#define AZ_RUN2D(NX, NY) \
  if (p->n == NX && p->ny == NY) return run2d<NX, NY>(a, op, src, npairs, p->Bmax, st);
  AZ_RUN2D(8, 8) AZ_RUN2D(16, 16) AZ_RUN2D(32, 32) AZ_RUN2D(64, 64) AZ_RUN2D(128, 128) AZ_RUN2D(256, 256)
  AZ_RUN2D(512, 512) AZ_RUN2D(1024, 1024)
  AZ_RUN2D(16, 8) AZ_RUN2D(32, 16) AZ_RUN2D(64, 32) AZ_RUN2D(128, 64) AZ_RUN2D(256, 128) AZ_RUN2D(512, 256)
  AZ_RUN2D(1024, 512)
  AZ_RUN2D(8, 16) AZ_RUN2D(16, 32) AZ_RUN2D(32, 64) AZ_RUN2D(64, 128) AZ_RUN2D(128, 256) AZ_RUN2D(256, 512)
  AZ_RUN2D(512, 1024)
#undef AZ_RUN2D
  az_set_error("2-D: unsupported n");
  return AZ_ERR_NOT_SUPPORTED;
}
