// Blocked Householder QR for the wide sketches of the 2-D configs (SURVEY.md §8(a) a7:
// "tall-skinny QR of [S | b']", k = probes + nrhs up to ~12k columns; "SVD of an
// (r+p)-by-M matrix ... O(r^2 M)").  Only R (and Q^T b') is needed; Q stays implicit as
// compact-WY panels  H_p = I - V_p T_p V_p^T  (Schreiber & Van Loan), V_p stored below the diagonal
// of the factored columns (LAPACK dgeqrf layout, unit diagonal implicit), T_p in a side buffer.
//
// Per panel of QB = 64 columns:
//   k_qr_panel  (cooperative, one CTA per SM): column-by-column Householder (dlarfg convention,
//               beta = -sign(alpha) ||x||) over the panel; each CTA owns a contiguous row range and
//               touches only its rows, so the only cross-CTA traffic is two partial-sum vectors per
//               column (2 grid barriers per column).  The same dot products give T (dlarft, forward
//               columnwise: T[0:j, j] = -tau_j T[0:j, 0:j] V[:, 0:j]^T v_j).
//   trailing update  C <- (I - V T^T V^T) C = C - V (T^T (V^T C)):  split-K DMMA GEMM for V^T C,
//               an ordered reduction fused with T^T, and a DMMA rank-64 update; all reductions run in
//               a fixed order, so R is bitwise reproducible.
// New probe blocks are added incrementally: the previous panels are applied to the new columns
// (az_qrw_apply), then the new columns are factored (az_qrw_factor); the right-hand sides b' get the
// same treatment, so their top rows end up as Q^T b'.
#include <cooperative_groups.h>

#include <algorithm>

#include "az_internal.h"
#include "az_mma.cuh"

namespace cg = cooperative_groups;

constexpr int QB = 64;            // panel width
constexpr int QB0 = 8;            // base panel width of the recursive panel factorisation
static_assert(QB0 <= 16 && QB >= 64, "k_qr_panel packs 2 x 16 partial slots per column parity into QB");
constexpr int PANEL_THREADS = 512;

AZ_D double qr_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct PanelArgs {
  double* A;
  int64_t lda, m;   // rows of A
  int64_t j0;       // first column (and diagonal row) of the panel
  int nb;           // panel columns (<= QB)
  int64_t chunk;    // rows per CTA
  double* T;        // QB x QB out (column-major)
  double* part;     // gridDim.x * (1 + QB) partial sums
};

__global__ void __launch_bounds__(PANEL_THREADS, 1) k_qr_panel(PanelArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[PANEL_THREADS / 32];
  __shared__ double dsum[QB];
  __shared__ double Ts[QB * QB];
  __shared__ double sc[3];
  const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  constexpr int NW = PANEL_THREADS / 32;
  const int64_t rb = a.j0 + (int64_t)c * a.chunk;
  const int64_t re = min(a.m, rb + a.chunk);
  double* R1 = a.part;          // G
  double* R2 = a.part + G;      // G x QB
  for (int e = tid; e < QB * QB; e += PANEL_THREADS) Ts[e] = 0.0;
  for (int j = 0; j < a.nb; ++j) {
    const int64_t jc = a.j0 + j;
    double* col = a.A + jc * a.lda;
    const int64_t rlo = max(rb, jc + 1);
    const bool owner = jc >= rb && jc < re;
    // ---- phase A: ONE reduction per column (one grid barrier instead of two): slot l of the
    // partials is the dot of the UNSCALED column j with column l over rows > jc (slot j: ||x||^2),
    // slot 16 + l is row jc of column l (only its owner contributes, so the sum is exact).  Then
    // d_l = v_j^T A[:, l] (v_j[jc] = 1) = A[jc, l] + scale * dot_l.  The partials are double-buffered
    // by column parity: a CTA one column step ahead writes the other buffer ----
    double* P2 = R2 + (j & 1) * 32;
    for (int l = w; l < a.nb; l += NW) {
      const double* cl = a.A + (a.j0 + l) * a.lda;
      double d = 0.0;
      for (int64_t r = rlo + lane; r < re; r += 32) d = fma(col[r], cl[r], d);
      d = qr_warp_sum(d);
      if (lane == 0) {
        P2[(int64_t)c * QB + l] = d;
        P2[(int64_t)c * QB + 16 + l] = owner ? cl[jc] : 0.0;
      }
    }
    grid.sync();
    // ---- phase B: fixed-order cross-CTA sums (every CTA the same numbers in the same order) ----
    for (int l = w; l < 2 * a.nb; l += NW) {   // one warp per slot, lanes over the CTAs' partials
      const int sl = l < a.nb ? l : 16 + (l - a.nb);
      double t = 0.0;
      for (int i = lane; i < G; i += 32) t += P2[(int64_t)i * QB + sl];
      t = qr_warp_sum(t);
      if (lane == 0) dsum[sl] = t;   // (dsum has QB slots)
    }
    __syncthreads();
    if (tid == 0) {
      const double sig = dsum[j];
      const double alpha = dsum[16 + j];
      double beta = alpha, tau = 0.0, scale = 0.0;
      if (sig > 0.0) {
        const double nrm = sqrt(fma(alpha, alpha, sig));
        beta = alpha >= 0.0 ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      sc[0] = beta;
      sc[1] = tau;
      sc[2] = scale;
    }
    __syncthreads();
    const double scale = sc[2], tau = sc[1];
    if (tid < a.nb && tid != j) dsum[tid] = fma(scale, dsum[tid], dsum[16 + tid]);   // d_l
    __syncthreads();
    for (int64_t r = rlo + tid; r < re; r += PANEL_THREADS) col[r] *= scale;
    // ---- phase D: apply H_j to the remaining panel columns; extend T ----
    if (tau != 0.0) {
      const int64_t nr = re - rlo;
      const int ncl = a.nb - j - 1;
      if (nr > 0)
        for (int l = j + 1; l < j + 1 + ncl; ++l) {     // columns outer, rows across threads (no div/mod)
          double* cl = a.A + (a.j0 + l) * a.lda;
          const double wl = -tau * dsum[l];
          for (int64_t r = rlo + tid; r < re; r += PANEL_THREADS) cl[r] = fma(wl, col[r], cl[r]);
        }
      if (owner)
        for (int l = j + 1 + tid; l < a.nb; l += PANEL_THREADS) a.A[(a.j0 + l) * a.lda + jc] -= tau * dsum[l];
    }
    if (owner && tid == 0) col[jc] = sc[0];
    // T[0:j, j] = -tau T[0:j, 0:j] d[0:j];  T[j][j] = tau
    if (c == 0) {
      for (int i = tid; i < j; i += PANEL_THREADS) {
        double t = 0.0;
        for (int q = i; q < j; ++q) t = fma(Ts[q * QB + i], dsum[q], t);
        Ts[j * QB + i] = -tau * t;
      }
      if (tid == 0) Ts[j * QB + j] = tau;
    }
    __syncthreads();
  }
  if (c == 0)
    for (int e = tid; e < QB * QB; e += PANEL_THREADS) a.T[e] = Ts[e];
}

// ------------------------------------------------------------------------------------------
// V element (row r, panel column l) with the implicit unit diagonal / zero upper part.
// ------------------------------------------------------------------------------------------
AZ_D double v_elem(const double* A, int64_t lda, int64_t j0, int nb, int64_t r, int l) {
  if (l >= nb) return 0.0;
  const int64_t d = r - j0;
  if (d < QB) {
    if (d == l) return 1.0;
    if (d < l) return 0.0;
  }
  return A[(j0 + l) * lda + r];
}

struct UpdArgs {
  const double* V;   // the factored matrix holding the panel (column j0.. of it)
  int64_t ldv;
  int64_t j0;        // panel's first column == first active row
  int nb;
  int64_t m;         // rows
  double* C;         // target columns (rows indexed like V)
  int64_t ldc;
  int64_t nt;        // target column count
  int64_t kchunk;    // rows per split-K chunk
  double* Wpart;     // KC x QB x nt
  double* Wfin;      // QB x nt (column-major, ld QB)
  const double* T;   // QB x QB
  int applyQ;        // 0: C <- Q^T C (W' = T^T W), 1: C <- Q C (W' = T W)
};

// Wpart[kc] = V^T C over rows [j0 + kc kchunk, ...): CTA tile 64 (panel cols) x 64 (target cols).
constexpr int VT_BK = 32, VT_S = 36;
__global__ void __launch_bounds__(256) k_qr_vtc(UpdArgs a) {
  __shared__ double smv[2 * QB * VT_S];
  double* As = smv;                  // IMAJ [m = panel col][k = row]
  double* Bs = smv + QB * VT_S;      // IMAJ [n = target col][k = row]
  static_assert(4 * 32 * 33 <= 2 * QB * VT_S, "reduction scratch must fit in the operand tiles");
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wm = w & 1, wn = (w >> 1) & 1, wk = w >> 2;
  const int64_t n0 = (int64_t)blockIdx.x * 64;
  const int kc = blockIdx.y;
  const int64_t r0 = a.j0 + (int64_t)kc * a.kchunk;
  const int64_t r1 = min(a.m, r0 + a.kchunk);
  double acc[4][4][2];
  acc_zero(acc);
  // per-thread load slots: 64 x 32 tile = 2048 elements = 8 per thread; k fastest
  const int lk = tid & 31, li = tid >> 5;   // element (i = li + 8 t, k = lk)
  double va[8], vb[8];
  auto load = [&](int64_t rr) {
    const int64_t r = rr + lk;
    if (rr >= a.j0 + QB) {   // (uniform) below the panel's unit triangle: V is the stored column
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int i = li + 8 * t;
        va[t] = (r < r1 && i < a.nb) ? a.V[(a.j0 + i) * a.ldv + r] : 0.0;
        vb[t] = (r < r1 && n0 + i < a.nt) ? a.C[(n0 + i) * a.ldc + r] : 0.0;
      }
    } else {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int i = li + 8 * t;
        va[t] = r < r1 ? v_elem(a.V, a.ldv, a.j0, a.nb, r, i) : 0.0;
        vb[t] = (r < r1 && n0 + i < a.nt) ? a.C[(n0 + i) * a.ldc + r] : 0.0;
      }
    }
  };
  load(r0);
  for (int64_t rr = r0; rr < r1; rr += VT_BK) {
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      As[(li + 8 * t) * VT_S + lk] = va[t];
      Bs[(li + 8 * t) * VT_S + lk] = vb[t];
    }
    __syncthreads();
    if (rr + VT_BK < r1) load(rr + VT_BK);   // next tile in flight during the MMAs
    warp_mma<4, 4, IMAJ, IMAJ>(acc, As, VT_S, Bs, VT_S, wm * 32, wn * 32, wk * 16, 16, lane);
  }
  // reduce the two k halves: warps wk = 1 write, wk = 0 add (scratch reuses the operand tiles)
  __syncthreads();
  double* rs = smv + (w & 3) * 32 * 33;
  if (wk == 1) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) rs[acc_row(0, i, lane) * 33 + acc_col(0, j, e, lane)] = acc[i][j][e];
  }
  __syncthreads();
  if (wk == 0) {
    double* W = a.Wpart + (int64_t)kc * QB * a.nt;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int ml = acc_row(0, i, lane), nl = acc_col(0, j, e, lane);
          const int64_t n = n0 + wn * 32 + nl;
          if (n < a.nt) W[n * QB + wm * 32 + ml] = acc[i][j][e] + rs[ml * 33 + nl];
        }
  }
}

// Wfin[:, n] = T^T sum_kc Wpart[kc][:, n]   (ordered sum; 4 target columns per CTA, 64 threads each)
__global__ void __launch_bounds__(256) k_qr_wred(UpdArgs a, int KC) {
  constexpr int TS = QB + 1;   // padded: rows (T^T path) and columns (T path) both conflict-free
  __shared__ double Ts[QB * TS];
  __shared__ double ws[4][QB];
  const int tid = threadIdx.x, l = tid & 63, g = tid >> 6;
  for (int e = tid; e < QB * QB; e += 256) Ts[(e / QB) * TS + (e % QB)] = a.T[e];
  const int64_t n = (int64_t)blockIdx.x * 4 + g;
  double s = 0.0;
  if (n < a.nt)
    for (int kc = 0; kc < KC; ++kc) s += a.Wpart[(int64_t)kc * QB * a.nt + n * QB + l];
  ws[g][l] = s;
  __syncthreads();
  if (n < a.nt) {
    double t = 0.0;
    if (!a.applyQ)
      for (int i = 0; i <= l; ++i) t = fma(Ts[l * TS + i], ws[g][i], t);    // (T^T)[l][i] = T[i][l]
    else
      for (int i = l; i < QB; ++i) t = fma(Ts[i * TS + l], ws[g][i], t);    // T[l][i], i >= l
    a.Wfin[n * QB + l] = t;
  }
}

// C[rows j0.., n] -= V[rows, 0:QB] Wfin[0:QB, n]: a CTA owns 128 rows and sweeps all target
// columns in tiles of 64, so its V tile is read from HBM once.  The accumulators start from C
// (DMMA computes D = A B + C with A = -V), and the next tile's C fragments and W' tile are
// fetched into registers while the current tile's MMAs run.
constexpr int UP_SA = 132, UP_SB = 68;
// PF = 1: the next tile's C fragments are prefetched into registers during the current tile's MMAs
// (with the current tile and W' that is ~80 doubles per thread: 1 CTA per SM without spills);
// PF = 0: C is loaded at the tile's start and only W' is prefetched (2 CTAs per SM)
template <int PF>
__global__ void __launch_bounds__(256, PF ? 1 : 2) k_qr_upd(UpdArgs a) {
  extern __shared__ double sm[];
  double* As = sm;                    // KMAJ [k = panel col][m = row], stride 132 (holds -V)
  double* Bs = sm + QB * UP_SA;       // IMAJ [n = target col][k], stride 68
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wm = w & 3, wn = w >> 2;
  const int64_t rbase = a.j0 + (int64_t)blockIdx.x * 128;
  {
    // the CTA's 128 x QB block of -V: all of a thread's loads in flight before the first store (the
    // rolled loop waited for each group of four loads: ~20 % of the warp samples at nt = 2048)
    constexpr int NV = QB * 128 / 256;
    double vv[NV];
#pragma unroll
    for (int t = 0; t < NV; ++t) {
      const int e = tid + 256 * t, l = e >> 7, ri = e & 127;
      const int64_t r = rbase + ri;
      vv[t] = r < a.m ? v_elem(a.V, a.ldv, a.j0, a.nb, r, l) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < NV; ++t) {
      const int e = tid + 256 * t, l = e >> 7, ri = e & 127;
      As[l * UP_SA + ri] = -vv[t];
    }
  }
  double acc[4][4][2];
  double wv[16];
  auto load_c = [&](int64_t n0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t r = rbase + acc_row(wm * 32, i, lane);
          const int64_t n = n0 + acc_col(wn * 32, j, e, lane);
          acc[i][j][e] = (r < a.m && n < a.nt) ? a.C[n * a.ldc + r] : 0.0;
        }
  };
  auto load_w = [&](int64_t n0) {
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int e = tid + 256 * t, n = e >> 6, l = e & 63;
      wv[t] = (n0 + n < a.nt) ? a.Wfin[(n0 + n) * QB + l] : 0.0;
    }
  };
  if (PF) load_c(0);
  load_w(0);
  for (int64_t n0 = 0; n0 < a.nt; n0 += 64) {
    __syncthreads();                  // previous tile's MMAs are done with Bs
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int e = tid + 256 * t, n = e >> 6, l = e & 63;
      Bs[n * UP_SB + l] = wv[t];
    }
    __syncthreads();
    auto mma_store = [&](double (&cc)[4][4][2]) {
      warp_mma<4, 4, KMAJ, IMAJ>(cc, As, UP_SA, Bs, UP_SB, wm * 32, wn * 32, 0, QB, lane);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t r = rbase + acc_row(wm * 32, i, lane);
            const int64_t n = n0 + acc_col(wn * 32, j, e, lane);
            if (r < a.m && n < a.nt) a.C[n * a.ldc + r] = cc[i][j][e];
          }
    };
    if constexpr (PF != 0) {
      double cur[4][4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          cur[i][j][0] = acc[i][j][0];
          cur[i][j][1] = acc[i][j][1];
        }
      if (n0 + 64 < a.nt) load_c(n0 + 64);   // next C fragments in flight
      if (n0 + 64 < a.nt) load_w(n0 + 64);   // next W' tile in flight
      mma_store(cur);
    } else {
      load_c(n0);
      if (n0 + 64 < a.nt) load_w(n0 + 64);
      mma_store(acc);
    }
  }
}

// AZ_QR_UPD_PF: 1 (register prefetch of the next C tile, one CTA per SM) or 0 (two CTAs per SM)
static int upd_pf() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("AZ_QR_UPD_PF");
    v = e ? atoi(e) : 1;
  }
  return v;
}

// ------------------------------------------------------------------------------------------
// T of a QB-wide panel from its Gram matrix: Gv = V^T V (split-K DMMA partials over row chunks,
// V with the implicit unit diagonal), then the dlarft recurrence
//   T[j][j] = tau_j,  T[0:j, j] = -tau_j T[0:j, 0:j] Gv[0:j, j]
// with tau_j read off the diagonals of the base-panel T factors.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_qr_vtv(UpdArgs a) {
  __shared__ double Xs[QB * VT_S];   // IMAJ [col][k]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wm = w & 1, wn = (w >> 1) & 1, wk = w >> 2;
  const int kc = blockIdx.x;
  const int64_t r0 = a.j0 + (int64_t)kc * a.kchunk;
  const int64_t r1 = min(a.m, r0 + a.kchunk);
  double acc[4][4][2];
  acc_zero(acc);
  const int lk = tid & 31, li = tid >> 5;
  double v[8];
  auto load = [&](int64_t rr) {
    const int64_t r = rr + lk;
#pragma unroll
    for (int t = 0; t < 8; ++t) v[t] = r < r1 ? v_elem(a.V, a.ldv, a.j0, a.nb, r, li + 8 * t) : 0.0;
  };
  load(r0);
  for (int64_t rr = r0; rr < r1; rr += VT_BK) {
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 8; ++t) Xs[(li + 8 * t) * VT_S + lk] = v[t];
    __syncthreads();
    if (rr + VT_BK < r1) load(rr + VT_BK);
    warp_mma<4, 4, IMAJ, IMAJ>(acc, Xs, VT_S, Xs, VT_S, wm * 32, wn * 32, wk * 16, 16, lane);
  }
  double* W = a.Wpart + (int64_t)kc * QB * QB;
  // the two k halves: the first writes the partial, the second adds to it
  if (wk == 0)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) W[acc_col(wn * 32, j, e, lane) * QB + acc_row(wm * 32, i, lane)] = acc[i][j][e];
  __syncthreads();
  if (wk == 1)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) W[acc_col(wn * 32, j, e, lane) * QB + acc_row(wm * 32, i, lane)] += acc[i][j][e];
}

__global__ void __launch_bounds__(256) k_qr_tbuild(const double* Wpart, int KC, const double* Tslots, int nb,
                                                    double* T) {
  extern __shared__ double smt[];
  double* Gv = smt;              // QB x QB
  double* Ts = smt + QB * QB;    // QB x QB
  __shared__ double tau[QB];
  const int tid = threadIdx.x;
  for (int e = tid; e < QB * QB; e += 256) {
    double t = 0.0;
    for (int kc = 0; kc < KC; ++kc) t += Wpart[(int64_t)kc * QB * QB + e];
    Gv[e] = t;
    Ts[e] = 0.0;
  }
  for (int j = tid; j < QB; j += 256) tau[j] = j < nb ? Tslots[(j / QB0) * QB * QB + (j % QB0) * QB + (j % QB0)] : 0.0;
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (tid < j) {
      double t = 0.0;
      for (int q = tid; q < j; ++q) t = fma(Ts[q * QB + tid], Gv[j * QB + q], t);   // (T Gv[:, j])[tid]
      Ts[j * QB + tid] = -tau[j] * t;
    }
    if (tid == 0) Ts[j * QB + j] = tau[j];
    __syncthreads();
  }
  for (int e = tid; e < QB * QB; e += 256) T[e] = Ts[e];
}

// ------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------
static int qrw_sms() {
  static int s = 0;
  if (!s) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    if (s <= 0) s = 148;
  }
  return s;
}

static int64_t qrw_kc(int64_t rows) {   // split-K chunks for V^T C
  return std::max<int64_t>(1, std::min<int64_t>(4 * qrw_sms(), (rows + 255) / 256));
}

// workspace: [panel partials | Wpart (KC x QB x nt) | Wfin (QB x nt)]
static size_t qrw_part_bytes() {
  // panel partial sums + (QB / QB0) base-panel T slots
  return (((size_t)qrw_sms() * (1 + QB) * sizeof(double) + 255) & ~(size_t)255) +
         (size_t)(QB / QB0) * QB * QB * sizeof(double);
}

size_t az_qrw_ws_bytes(int64_t m, int64_t ncols_max) {
  const int64_t KC = qrw_kc(m);
  const int64_t nt = std::max<int64_t>(ncols_max, 64);
  return qrw_part_bytes() + (size_t)(KC + 1) * QB * nt * sizeof(double) + 256;
}

// Apply panels [p0, p1) of the factored matrix V (panel p = columns p QB ..) to the target columns.
// Panel p starts at column pj0[p] (== its first active row) and has pnb[p] columns; its T is at
// Tbuf + p QB^2.
static az_status_t qrw_apply_dir(const double* V, int64_t ldv, int64_t m, const int64_t* pj0, const int* pnb,
                                 const double* Tbuf, int64_t p0, int64_t p1, double* C, int64_t ldc, int64_t nt,
                                 void* ws, size_t ws_bytes, cudaStream_t st, int applyQ);

az_status_t az_qrw_apply(const double* V, int64_t ldv, int64_t m, const int64_t* pj0, const int* pnb,
                         const double* Tbuf, int64_t p0, int64_t p1, double* C, int64_t ldc, int64_t nt, void* ws,
                         size_t ws_bytes, cudaStream_t st) {
  return qrw_apply_dir(V, ldv, m, pj0, pnb, Tbuf, p0, p1, C, ldc, nt, ws, ws_bytes, st, 0);
}

// C <- Q C with Q = H_(p0) ... H_(p1-1): panels in reverse order, W' = T W
az_status_t az_qrw_apply_q(const double* V, int64_t ldv, int64_t m, const int64_t* pj0, const int* pnb,
                           const double* Tbuf, int64_t p0, int64_t p1, double* C, int64_t ldc, int64_t nt, void* ws,
                           size_t ws_bytes, cudaStream_t st) {
  return qrw_apply_dir(V, ldv, m, pj0, pnb, Tbuf, p0, p1, C, ldc, nt, ws, ws_bytes, st, 1);
}

static az_status_t qrw_apply_dir(const double* V, int64_t ldv, int64_t m, const int64_t* pj0, const int* pnb,
                                 const double* Tbuf, int64_t p0, int64_t p1, double* C, int64_t ldc, int64_t nt,
                                 void* ws, size_t ws_bytes, cudaStream_t st, int applyQ) {
  if (nt <= 0) return AZ_OK;
  if (ws_bytes < az_qrw_ws_bytes(m, nt)) {
    az_set_error("az_qrw_apply: workspace too small");
    return AZ_ERR_WORKSPACE;
  }
  const size_t ups = (size_t)(QB * UP_SA + 64 * UP_SB) * sizeof(double);
  AZ_CUDA_CHECK(az_smem_attr(k_qr_upd<1>, ups));
  AZ_CUDA_CHECK(az_smem_attr(k_qr_upd<0>, ups));
  for (int64_t pi = 0; pi < p1 - p0; ++pi) {
    const int64_t p = applyQ ? p1 - 1 - pi : p0 + pi;
    UpdArgs u;
    u.applyQ = applyQ;
    u.V = V;
    u.ldv = ldv;
    u.j0 = pj0[p];
    u.nb = pnb[p];
    u.m = m;
    u.C = C;
    u.ldc = ldc;
    u.nt = nt;
    const int64_t rows = m - u.j0;
    if (rows <= 0) continue;
    const int64_t KC = qrw_kc(rows);
    u.kchunk = (rows + KC - 1) / KC;
    u.Wpart = (double*)((char*)ws + qrw_part_bytes());   // (also the V^T V partials of k_qr_vtv)
    u.Wfin = u.Wpart + (size_t)KC * QB * nt;
    u.T = Tbuf + p * QB * QB;
    {
      AzTrace tr("qrw_vtc", st, 2 * rows * u.nb * nt);
      k_qr_vtc<<<dim3(az_div_up(nt, 64), (unsigned)KC), 256, 0, st>>>(u);
      AZ_LAUNCH_CHECK();
    }
    {
      AzTrace tr("qrw_wred", st);
      k_qr_wred<<<az_div_up(nt, 4), 256, 0, st>>>(u, (int)KC);
      AZ_LAUNCH_CHECK();
    }
    {
      AzTrace tr("qrw_upd", st, 2 * rows * u.nb * nt);
      if (upd_pf())
        k_qr_upd<1><<<az_div_up(rows, 128), 256, ups, st>>>(u);
      else
        k_qr_upd<0><<<az_div_up(rows, 128), 256, ups, st>>>(u);
      AZ_LAUNCH_CHECK();
    }
  }
  return AZ_OK;
}

// Factor columns [c0, c1) of A (columns < c0 already factored and applied to these columns).
// Appends the new panels to (pj0, pnb) starting at index *np (capacity checked by the caller).
az_status_t az_qrw_factor(double* A, int64_t lda, int64_t m, int64_t c0, int64_t c1, double* Tbuf, int64_t* pj0,
                          int* pnb, int64_t* np, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (c1 > m) {
    az_set_error("az_qrw_factor: more columns (%lld) than rows (%lld)", (long long)c1, (long long)m);
    return AZ_ERR_NOT_SUPPORTED;
  }
  if (ws_bytes < az_qrw_ws_bytes(m, c1 - c0)) {
    az_set_error("az_qrw_factor: workspace too small");
    return AZ_ERR_WORKSPACE;
  }
  int maxb = 0;
  AZ_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, k_qr_panel, PANEL_THREADS, 0));
  if (maxb < 1) {
    az_set_error("az_qrw_factor: panel kernel cannot be resident");
    return AZ_ERR_CUDA;
  }
  double* part = (double*)ws;
  double* Tslots = (double*)((char*)ws + (((size_t)qrw_sms() * (1 + QB) * sizeof(double) + 255) & ~(size_t)255));
  for (int64_t j0 = c0; j0 < c1; j0 += QB) {
    const int nbp = (int)std::min<int64_t>(QB, c1 - j0);
    const int64_t p = (*np)++;
    pj0[p] = j0;
    pnb[p] = nbp;
    // recursive panel: QB0-wide base panels factored column by column (the base panel stays
    // L2-resident), each applied to the rest of the QB panel through the blocked update
    for (int b0 = 0; b0 < nbp; b0 += QB0) {
      PanelArgs pa;
      pa.A = A;
      pa.lda = lda;
      pa.m = m;
      pa.j0 = j0 + b0;
      pa.nb = std::min(QB0, nbp - b0);
      const int64_t rows = m - pa.j0;
      const int64_t G = std::max<int64_t>(1, std::min<int64_t>(qrw_sms(), (rows + 127) / 128));
      pa.chunk = (rows + G - 1) / G;
      pa.T = Tslots + (b0 / QB0) * QB * QB;
      pa.part = part;
      void* args[] = {&pa};
      {
        AzTrace tr("qrw_panel", st, rows * pa.nb);
        AZ_CUDA_CHECK(cudaLaunchCooperativeKernel((void*)k_qr_panel, dim3((unsigned)G), dim3(PANEL_THREADS), args, 0, st));
        az_count_launch();
      }
      const int64_t rest = nbp - (b0 + pa.nb);
      if (rest > 0) {
        const int64_t bj0 = pa.j0;
        const int bnb = pa.nb;
        AZ_TRY(az_qrw_apply(A, lda, m, &bj0, &bnb, pa.T, 0, 1, A + (pa.j0 + pa.nb) * lda, lda, rest, ws, ws_bytes, st));
      }
    }
    // T of the whole QB panel from V^T V and the base taus
    {
      UpdArgs u;
      u.applyQ = 0;
      u.V = A;
      u.ldv = lda;
      u.j0 = j0;
      u.nb = nbp;
      u.m = m;
      const int64_t rows = m - j0;
      const int64_t KC = qrw_kc(rows);
      u.kchunk = (rows + KC - 1) / KC;
      u.Wpart = (double*)((char*)ws + qrw_part_bytes());
      AzTrace tr("qrw_tbuild", st);
      k_qr_vtv<<<(unsigned)KC, 256, 0, st>>>(u);
      AZ_LAUNCH_CHECK();
      const size_t tsm = 2 * QB * QB * sizeof(double);
      AZ_CUDA_CHECK(az_smem_attr(k_qr_tbuild, tsm));
      k_qr_tbuild<<<1, 256, tsm, st>>>(u.Wpart, (int)KC, Tslots, nbp, Tbuf + p * QB * QB);
      AZ_LAUNCH_CHECK();
    }
    const int64_t nt = c1 - (j0 + nbp);
    if (nt > 0)
      AZ_TRY(az_qrw_apply(A, lda, m, pj0, pnb, Tbuf, p, p + 1, A + (j0 + nbp) * lda, lda, nt, ws, ws_bytes, st));
  }
  return AZ_OK;
}

// ------------------------------------------------------------------------------------------
// Explicit Q1 in place (dorgqr): with the panels after p already turned into columns of Q, panel p
// is applied to them (rows j0.. of those columns are zero above their own panel start) and its own
// columns become  H_p [I; 0] = [I; 0] - V (T V_top^T)  (V_top = the unit-lower nb x nb top of V):
// row r of the result needs only row r of V, so it overwrites V in place; rows < j0 become zero.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_qr_orgm(const double* A, int64_t lda, int64_t j0, int nb, const double* T,
                                                 double* M) {
  // M[l][c] = sum_i T[l][i] V_top[c][i]  (T column-major QB x QB; M column-major QB x QB)
  for (int e = threadIdx.x; e < QB * QB; e += blockDim.x) {
    const int l = e % QB, c = e / QB;
    double t = 0.0;
    if (l < nb && c < nb)
      for (int i = l; i <= c && i < nb; ++i) {   // T upper (i >= l), V_top[c][i] nonzero for i <= c
        const double vt = (i == c) ? 1.0 : A[(j0 + i) * lda + j0 + c];
        t = fma(T[i * QB + l], vt, t);
      }
    M[c * QB + l] = t;
  }
}

__global__ void __launch_bounds__(256) k_qr_orgrows(double* A, int64_t lda, int64_t m, int64_t j0, int nb,
                                                    const double* M) {
  __shared__ double Vs[32][QB + 1];
  const double* Ms = M;     // 32 KB, warp-uniform reads: served from L1
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t r = j0 + (int64_t)blockIdx.x * 32 + lane;
  for (int l = w; l < nb; l += 8) {
    double v = 0.0;
    if (r < m) v = (r - j0 == l) ? 1.0 : (r - j0 > l ? A[(j0 + l) * lda + r] : 0.0);
    Vs[lane][l] = v;
  }
  __syncthreads();
  double acc[QB / 8];
#pragma unroll
  for (int t = 0; t < QB / 8; ++t) acc[t] = 0.0;
  for (int l = 0; l < nb; ++l) {
    const double v = Vs[lane][l];
#pragma unroll
    for (int t = 0; t < QB / 8; ++t) acc[t] = fma(v, __ldg(Ms + (w + 8 * t) * QB + l), acc[t]);
  }
  if (r < m) {
#pragma unroll
    for (int t = 0; t < QB / 8; ++t) {
      const int c = w + 8 * t;
      if (c < nb) A[(j0 + c) * lda + r] = ((r - j0 == c) ? 1.0 : 0.0) - acc[t];
    }
  }
}

az_status_t az_qrw_form_q(double* A, int64_t lda, int64_t m, const int64_t* pj0, const int* pnb, const double* Tbuf,
                          int64_t np, int64_t kp, void* ws, size_t ws_bytes, cudaStream_t st) {
  int64_t npk = 0;
  while (npk < np && pj0[npk] < kp) ++npk;
  for (int64_t p = 0; p < npk; ++p)
    if (pj0[p] + pnb[p] > kp || (p > 0 && pj0[p] != pj0[p - 1] + pnb[p - 1]) || (p == 0 && pj0[0] != 0)) {
      az_set_error("az_qrw_form_q: panels do not tile columns [0, %lld)", (long long)kp);
      return AZ_ERR_NOT_SUPPORTED;
    }
  if (npk == 0 || pj0[npk - 1] + pnb[npk - 1] != kp) {
    az_set_error("az_qrw_form_q: panels do not tile columns [0, %lld)", (long long)kp);
    return AZ_ERR_NOT_SUPPORTED;
  }
  if (ws_bytes < az_qrw_ws_bytes(m, QB)) {
    az_set_error("az_qrw_form_q: workspace too small");
    return AZ_ERR_WORKSPACE;
  }
  // M lives in the first base-panel T slot of the workspace (unused outside az_qrw_factor)
  double* M = (double*)((char*)ws + (((size_t)qrw_sms() * (1 + QB) * sizeof(double) + 255) & ~(size_t)255));
  for (int64_t p = npk - 1; p >= 0; --p) {
    const int64_t j0 = pj0[p];
    const int nb = pnb[p];
    const int64_t nt = kp - (j0 + nb);
    // the trailing columns: a column block of at most ws-sized width at a time
    for (int64_t c0 = 0; c0 < nt;) {
      int64_t w = nt - c0;
      while (w > QB && ws_bytes < az_qrw_ws_bytes(m, w)) w = (w + 1) / 2;
      AZ_TRY(az_qrw_apply_q(A, lda, m, pj0, pnb, Tbuf, p, p + 1, A + (j0 + nb + c0) * lda, lda, w, ws, ws_bytes, st));
      c0 += w;
    }
    AzTrace tr("qrw_orgqr", st, 2 * (m - j0) * nb * nb);
    k_qr_orgm<<<1, 256, 0, st>>>(A, lda, j0, nb, Tbuf + p * QB * QB, M);
    AZ_LAUNCH_CHECK();
    k_qr_orgrows<<<az_div_up(m - j0, 32), 256, 0, st>>>(A, lda, m, j0, nb, M);
    AZ_LAUNCH_CHECK();
    if (j0 > 0) AZ_CUDA_CHECK(cudaMemset2DAsync(A + j0 * lda, lda * sizeof(double), 0, j0 * sizeof(double), nb, st));
  }
  return AZ_OK;
}

// R (k x k, upper; strict lower zeroed) out of the factored matrix.
__global__ void k_qrw_extract_R(const double* A, int64_t lda, int64_t k, double* R, int64_t ldr) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= k * k) return;
  const int64_t i = e % k, l = e / k;
  R[l * ldr + i] = i <= l ? A[l * lda + i] : 0.0;
}

az_status_t az_qrw_extract_R(const double* A, int64_t lda, int64_t k, double* R, int64_t ldr, cudaStream_t st) {
  k_qrw_extract_R<<<az_div_up(k * k, 256), 256, 0, st>>>(A, lda, k, R, ldr);
  AZ_LAUNCH_CHECK();
  return AZ_OK;
}

int64_t az_qrw_panel_width() { return QB; }
