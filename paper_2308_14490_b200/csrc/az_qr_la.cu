// Split TSQR leaf, pass A, as a blocked Householder QR with look-ahead (the QR that
// reduces the M x (r + p) sketch to its R factor).
//
// Same arithmetic as k_tsqr's pass A (az_qr.cu): each CTA streams its row range in 256-row chunks
// through the structured QR of [R; chunk] (R: the k1 x k1 triangle so far), reflector j being
// H_j = I - tau_j v_j v_j^T with v_j = [e_j ; y_j] (LAPACK dlarfg convention: beta = -sign(alpha)
// ||(alpha, x)||, tau = (beta - alpha) / beta, y = x / (alpha - beta)), and leaves y_j in place of
// column j and tau_j in taus for pass B (k_tsqr_rhs).  Only the ORDER of the work differs: the
// columns are taken in panels of 8, and per panel
//   * two panel warps (on SM sub-partitions 0 and 1, 128 rows each, the panel in registers; AZ_TSQR_LA_NP=4:
//     four, 64 rows each) factorise it column by column -- one 128-thread named barrier per column: the column's norm and its dot products with
//     the panel's other columns are reduced together, the dots taken with the unscaled column and scaled
//     by 1 / (alpha - beta) afterwards -- and form its T (dlarft: H_0 .. H_7 = I - V T V^T);
//   * all eight warps then apply it to the NEXT panel's columns (the look-ahead tile) in compact-WY
//     form on the FP64 tensor cores (DMMA m8n8k4):
//         W = R[J, tile] + Y_J^T X[:, tile],  W <- T^T W,  R[J, tile] -= W,  X[:, tile] -= Y_J W;
//   * and while the panel warps factorise that next panel, the four update warps (on the other two SM
//     sub-partitions, so their DMMA never delays the panel chain) apply the panel to the remaining
//     columns the same way, write its y columns back and refill their shared-memory slots with the
//     same columns of the next chunk (cp.async), so the chunk loads overlap the QR.
// The per-column step of k_tsqr (every warp applies every reflector to its own columns, one 512-thread
// barrier per column) becomes a 4-warp chain per column plus DMMA block updates off the chain: the
// same reflectors up to rounding (the columns right of a panel receive its reflectors as one block).
#include <cstdlib>

#include "az_internal.h"
#include "az_mma.cuh"

namespace {
constexpr int LA_LDR = 65;            // R column stride
constexpr int LA_PW = 8;              // panel width
constexpr int LA_NW = 8;              // warps
constexpr int LA_NU = 4;              // update warps (2, 3, 6, 7: sub-partitions 2 and 3)
// Chunk shape: MC rows per chunk (256: one 175 KB CTA per SM; 128: two 110 KB CTAs per SM, whose
// panel chains interleave), X column stride MC + 4 (== 4 mod 16: conflict-free DMMA fragments)
// NP panel warps: 4 (0, 1, 4, 5: two per sub-partition 0 and 1) or 2 (0 and 1: one per sub-partition,
// twice the rows each; warps 4 and 5 then only join the look-ahead W and the CTA barriers)
template <int MC, int NP = 4>
struct LAShape {
  static constexpr int LDX = MC + 4;
  static constexpr int PR = MC / NP;         // rows of a panel warp
  static constexpr int RPW = PR / 32;        // rows per lane in a panel warp
  static constexpr int MINB = MC == 256 ? 1 : 2;
};

struct LAIn {
  const double* A;     // m x k1 (ld), the probe columns
  double* Y;           // y_j written back (== A for the split leaf)
  int64_t m, ld, ldY, rows_per_cta;
  int64_t rb, bstride;   // merges: stacked row r of A and Y at (r / rb) bstride + r % rb (0 = plain rows)
  int k1, cmax;
  double* Rout;        // per CTA k1 x k1 (ld k1), CTA stride ostride
  int64_t ostride;
  double* taus;        // taus[(cta cmax + chunk) k1 + j]
};

AZ_D void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
enum { BAR_P = 1, BAR_U = 2 };   // panel warps / update warps (128 threads each)

AZ_D void cpa8(double* dst, const double* src, bool in) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(in ? 8 : 0)
               : "memory");
}

// shared-memory layout (doubles)
template <int MC>
struct LASmem {
  static constexpr int X = 0;                          // 64 columns x LDX
  static constexpr int R = X + 64 * LAShape<MC>::LDX;  // 64 columns x LA_LDR
  static constexpr int T = R + 64 * LA_LDR;    // 2 x 64: T[a][m] at a * 8 + m (double-buffered by panel parity)
  static constexpr int RED2 = T + 128;         // 2 x 8 x 4: partial dots, d[l] of warp i at l * 4 + i
  static constexpr int WP = RED2 + 64;         // 8 x 64: the look-ahead tile's partial W (one per warp)
  static constexpr int WSUM = WP + 8 * 64;     // 64: W
  static constexpr int WL = WSUM + 64;         // 64: W' = T^T W
  static constexpr int WS = WL + 64;           // 4 x 64: the update warps' W / W' of a remaining tile
  static constexpr int END = WS + LA_NU * 64;
};

// W'[m][n] = sum_{i <= m} T[i][m] W[i][n]   (W at W[i * 8 + n])
AZ_D double tt_w(const double* T, const double* W, int m, int n) {
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < LA_PW; ++i)
    if (i <= m) t = fma(T[i * 8 + m], W[i * 8 + n], t);
  return t;
}

// X[:, c0 .. c0+8) -= Y_J W' over the row tiles mt0 .. mt1 - 1 (8 rows each; W' at Wp[m * 8 + n])
template <int LDX>
AZ_D void tile_rank_update(double* X, const double* Wp, int j0, int c0, int k1, int mt0, int mt1, int lane) {
  const int r = lane >> 2, q = lane & 3;
  const int ca = c0 + 2 * q, cb = ca + 1;
  const double b0 = Wp[q * 8 + r], b1 = Wp[(q + 4) * 8 + r];   // B(k = panel col, n = tile col)
  for (int mt = mt0; mt < mt1; ++mt) {
    const int row = 8 * mt + r;
    double c[2];
    c[0] = ca < k1 ? X[ca * LDX + row] : 0.0;
    c[1] = cb < k1 ? X[cb * LDX + row] : 0.0;
    dmma(c, -X[(j0 + q) * LDX + row], b0);       // A(m = row, k = panel col)
    dmma(c, -X[(j0 + q + 4) * LDX + row], b1);
    if (ca < k1) X[ca * LDX + row] = c[0];
    if (cb < k1) X[cb * LDX + row] = c[1];
  }
}

// W (8 x 8 C fragment) += Y_J^T X[:, c0..c0+8) over rows [k0, k1r), two accumulators
template <int LDX>
AZ_D void tile_w(double (&acc)[2], const double* X, int j0, int c0, int k1, int k0, int k1r, int lane) {
  const int r = lane >> 2, qd = lane & 3;
  const int cb = c0 + r;
  double a2[2] = {0.0, 0.0};
#pragma unroll 4
  for (int kk = k0; kk < k1r; kk += 8) {
    const double a0 = X[(j0 + r) * LDX + kk + qd];
    const double b0 = cb < k1 ? X[cb * LDX + kk + qd] : 0.0;
    const double a1 = X[(j0 + r) * LDX + kk + 4 + qd];
    const double b1 = cb < k1 ? X[cb * LDX + kk + 4 + qd] : 0.0;
    dmma(acc, a0, b0);
    dmma(a2, a1, b1);
  }
  acc[0] += a2[0];
  acc[1] += a2[1];
}

// Panel factorisation by the four panel warps w = 0..3 (rows 64 w .. 64 w + 63 of the chunk, lane rows
// 64 w + lane + 32 i).
// FULLW = 8: a full panel (every column test resolved at compile time); 0: a last, narrower panel.
// Warp 0 writes R's panel rows, warp 1 forms T (lane a owns row a), warp 2 stores the taus, so that
// no warp carries all the side work between the two barriers of a column.
template <int MC, int NP, int FULLW>
AZ_D void la_panel(double* X, double* R, double* sm, double* Tm, const LAIn& q, int chunk, int j0, int k1, int w,
                   int lane) {
  constexpr int LDX = LAShape<MC, NP>::LDX, RPW = LAShape<MC, NP>::RPW, PR = LAShape<MC, NP>::PR;
  constexpr int TAU_W = NP > 2 ? 2 : 0, TAU_L = NP > 2 ? 0 : 1;   // who stores the taus
  constexpr int T_W = NP > 1 ? 1 : 0;                              // who forms T
  const int PWN = FULLW ? FULLW : min(LA_PW, k1 - j0);
  double* red2 = sm + LASmem<MC>::RED2;
  double x[LA_PW][RPW];   // column j0 + c, row PR w + lane + 32 i
#pragma unroll
  for (int c = 0; c < LA_PW; ++c)
#pragma unroll
    for (int i = 0; i < RPW; ++i) x[c][i] = c < PWN ? X[(j0 + c) * LDX + PR * w + lane + 32 * i] : 0.0;
  double trow[LA_PW];   // warp 1, lane a < 8: row a of T
#pragma unroll
  for (int m = 0; m < LA_PW; ++m) trow[m] = 0.0;
#pragma unroll
  for (int c = 0; c < LA_PW; ++c) {
    if (c >= PWN) break;
    const int jc = j0 + c;
    const double alpha = R[jc * LA_LDR + jc];
    double rl[LA_PW];   // R[jc][j0 + l], read before any warp writes the row (after the barrier)
#pragma unroll
    for (int l = 0; l < LA_PW; ++l) rl[l] = (l > c && l < PWN) ? R[(j0 + l) * LA_LDR + jc] : 0.0;
    // ONE reduction per column: slot c = ||x_c||^2 (the chunk part), slot l != c = x_c . x_l -- the
    // dots are taken with the unscaled column and scaled by the reflector's 1 / (alpha - beta) after,
    // so they need not wait for the reflector (y_c . x_l = scale (x_c . x_l))
    double d[LA_PW];
#pragma unroll
    for (int l = 0; l < LA_PW; ++l) {
      d[l] = 0.0;
      if (l < PWN)
#pragma unroll
        for (int i = 0; i < RPW; ++i) d[l] = fma(x[c][i], x[l][i], d[l]);
    }
    // transpose-reduce: 3 halving levels leave lane L a partial of slot L / 4, 2 more complete it
#pragma unroll
    for (int o = 16, n = LA_PW; n > 1; o >>= 1, n >>= 1) {
      const bool hi = lane & o;
#pragma unroll
      for (int i2 = 0; i2 < n / 2; ++i2) {
        const double send = hi ? d[i2] : d[i2 + n / 2];
        const double keep = hi ? d[i2 + n / 2] : d[i2];
        d[i2] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    double ds = d[0];
    ds += __shfl_xor_sync(0xffffffffu, ds, 2);
    ds += __shfl_xor_sync(0xffffffffu, ds, 1);
    if constexpr (NP == 1) {   // one panel warp: the slot sums are broadcast, no barrier
#pragma unroll
      for (int l = 0; l < LA_PW; ++l) d[l] = __shfl_sync(0xffffffffu, ds, 4 * l);
    } else {
      double* rb = red2 + (c & 1) * 32;   // (double-buffered: one barrier per column)
      if ((lane & 3) == 0) rb[(lane >> 2) * NP + w] = ds;
      bar_sync(BAR_P, 32 * NP);
#pragma unroll
      for (int l = 0; l < LA_PW; ++l) {
        const double2 u = *reinterpret_cast<const double2*>(rb + l * NP);
        if constexpr (NP == 4) {
          const double2 v = *reinterpret_cast<const double2*>(rb + l * 4 + 2);
          d[l] = (u.x + u.y) + (v.x + v.y);
        } else {
          d[l] = u.x + u.y;
        }
      }
    }
    const double sig = d[c];
    double tau = 0.0, scale = 0.0, beta = alpha;
    if (sig > 0.0) {   // (the formulas of k_tsqr)
      const double s2 = fma(alpha, alpha, sig);
      const double rinv = fast_rsqrt(s2);
      const double nrm = s2 * rinv;
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau = fma(fabs(alpha), rinv, 1.0);
      scale = fast_rcp(alpha - beta);
    }
#pragma unroll
    for (int i = 0; i < RPW; ++i) x[c][i] *= scale;   // y_c
#pragma unroll
    for (int l = 0; l < LA_PW; ++l) d[l] *= scale;       // y_c . x_l (l > c), y_c . y_l (l < c)
    if (w == 0 && lane == 0) R[jc * LA_LDR + jc] = beta;
    if (w == TAU_W && lane == TAU_L) q.taus[((int64_t)blockIdx.x * q.cmax + chunk) * k1 + jc] = tau;
    if (w == T_W) {
      // T[a][c] = -tau_c sum_{a <= m < c} T[a][m] (y_m . y_c), T[c][c] = tau_c (lane a owns row a)
      double t = 0.0;
#pragma unroll
      for (int m = 0; m < LA_PW; ++m)
        if (m < c && m >= lane) t = fma(trow[m], d[m], t);
      trow[c] = lane < c ? -tau * t : (lane == c ? tau : 0.0);
    }
    if (tau != 0.0) {
#pragma unroll
      for (int l = 0; l < LA_PW; ++l) {
        if (l > c && l < PWN) {
          const double wl = tau * (rl[l] + d[l]);
#pragma unroll
          for (int i = 0; i < RPW; ++i) x[l][i] = fma(-wl, x[c][i], x[l][i]);
          if (w == 0 && lane == 0) R[(j0 + l) * LA_LDR + jc] = rl[l] - wl;
        }
      }
    }
  }
  // y's in place of the panel columns; T
#pragma unroll
  for (int c = 0; c < LA_PW; ++c)
#pragma unroll
    for (int i = 0; i < RPW; ++i)
      if (c < PWN) X[(j0 + c) * LDX + PR * w + lane + 32 * i] = x[c][i];
  if (w == T_W && lane < LA_PW)
#pragma unroll
    for (int m = 0; m < LA_PW; ++m) Tm[lane * 8 + m] = trow[m];
}

template <int MC, bool STACK, int NP = 4>
__global__ void __launch_bounds__(32 * LA_NW, LAShape<MC, NP>::MINB) k_tsqr_la(LAIn q) {
  constexpr int LDX = LAShape<MC, NP>::LDX;
  using SM = LASmem<MC>;
  extern __shared__ double sm[];
  double* X = sm + SM::X;
  double* R = sm + SM::R;
  const int k1 = q.k1;
  const int np = (k1 + LA_PW - 1) / LA_PW;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int r8 = lane >> 2, qd = lane & 3;
  // warp w runs on SM sub-partition w % 4: the panel warps are 0, 1, 4, 5 (sub-partitions 0 and 1) and
  // the update warps 2, 3, 6, 7, so the panel chain never queues behind the updates' DMMA on its FP64
  // pipe (measured: with the panel and update warps paired on every sub-partition the leaf took 19 %
  // longer than the chain alone)
  const bool panel_w = NP == 4 ? (w & 2) == 0 : w < NP;
  const bool upd_w = (w & 2) != 0;
  const int gi = (w & 1) | ((w >> 2) << 1);   // index within the warp's group (0..3)
  for (int e = tid; e < 64 * LA_LDR; e += 32 * LA_NW) R[e] = 0.0;
  // column slots past k1 are read as (zero) columns of a last, narrower panel or tile
  for (int e = tid; e < (64 - k1) * LDX; e += 32 * LA_NW) X[k1 * LDX + e] = 0.0;
  const int64_t r0 = (int64_t)blockIdx.x * q.rows_per_cta;
  const int64_t r1 = min(q.m, r0 + q.rows_per_cta);
  auto roff = [&](int64_t row) -> int64_t {
    if constexpr (STACK) return (row / q.rb) * q.bstride + row % q.rb;
    return row;
  };
  // first chunk: columns of 256 contiguous rows; rows past r1 zero-filled
  for (int e = tid; e < k1 * MC; e += 32 * LA_NW) {
    const int c = e / MC, i = e % MC;
    const int64_t row = r0 + i;
    cpa8(X + c * LDX + i, q.A + roff(row < r1 ? row : r0) + (int64_t)c * q.ld, row < r1);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();

  // update warps: write panel pp's y columns back, then refill their slots from the next chunk
  auto writeback = [&](int pp, int64_t base, int64_t nbase) {
    const int j0 = pp * LA_PW, pw = min(LA_PW, k1 - j0);
    const int ut = 32 * gi + lane;
    bar_sync(BAR_U, 32 * LA_NU);   // every update of panel pp is done
    for (int e = ut; e < pw * MC; e += 32 * LA_NU) {
      const int c = e / MC, i = e % MC;
      const int64_t row = base + i;
      if (row < r1) q.Y[roff(row) + (int64_t)(j0 + c) * q.ldY] = X[(j0 + c) * LDX + i];
    }
    if (nbase < r1) {
      bar_sync(BAR_U, 32 * LA_NU);   // the slot is read before it is overwritten
      for (int e = ut; e < pw * MC; e += 32 * LA_NU) {
        const int c = e / MC, i = e % MC;
        const int64_t row = nbase + i;
        cpa8(X + (j0 + c) * LDX + i, q.A + roff(row < r1 ? row : r0) + (int64_t)(j0 + c) * q.ld, row < r1);
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
  };

  int chunk = 0;
  for (int64_t base = r0; base < r1; base += MC, ++chunk) {
    const int64_t nbase = base + MC;
    for (int p = 0; p < np; ++p) {
      const int j0 = p * LA_PW, pw = min(LA_PW, k1 - j0);
      double* Tm = sm + SM::T + (p & 1) * 64;
      if (panel_w) {
        // ================= panel p, panel warp gi: rows 64 gi .. 64 gi + 63 =================
        if (pw == LA_PW)
          la_panel<MC, NP, LA_PW>(X, R, sm, Tm, q, chunk, j0, k1, gi, lane);
        else
          la_panel<MC, NP, 0>(X, R, sm, Tm, q, chunk, j0, k1, gi, lane);
      } else if (upd_w && p > 0) {
        // ========= update warps: panel p - 1 on the columns right of panel p (tiles p + 1 ..) =========
        const int uw = gi, pj0 = j0 - LA_PW;
        const double* Tp = sm + SM::T + ((p - 1) & 1) * 64;
        double* WS = sm + SM::WS + uw * 64;
        for (int t = p + 1 + uw; t * LA_PW < k1; t += LA_NU) {
          const int ct = t * LA_PW;
          double acc[2] = {0.0, 0.0};
          tile_w<LDX>(acc, X, pj0, ct, k1, 0, MC, lane);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int n = 2 * qd + e;
            WS[r8 * 8 + n] = acc[e] + ((ct + n < k1) ? R[(ct + n) * LA_LDR + pj0 + r8] : 0.0);
          }
          __syncwarp();
          double wv[2];
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2) {
            const int e = lane + 32 * e2;
            wv[e2] = tt_w(Tp, WS, e >> 3, e & 7);
          }
          __syncwarp();
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2) {
            const int e = lane + 32 * e2, m = e >> 3, n = e & 7;
            WS[e] = wv[e2];
            if (ct + n < k1) R[(ct + n) * LA_LDR + pj0 + m] -= wv[e2];
          }
          __syncwarp();
          tile_rank_update<LDX>(X, WS, pj0, ct, k1, 0, MC / 8, lane);
          __syncwarp();
        }
      }
      __syncthreads();   // panel p factorised; panel p - 1 applied everywhere
      if (p + 1 < np) {
        // ====== look-ahead: panel p on the next panel's columns; W split 8 ways over all warps, then
        // W' = T^T W by warp 0 and each panel warp updates its own 64 rows (so it can go straight on to
        // factorising the next panel); the update warps meanwhile write back panel p - 1 ======
        const int c0 = j0 + LA_PW;
        double* Wp = sm + SM::WP;
        double* Ws = sm + SM::WSUM;
        double* WL = sm + SM::WL;
        double acc[2] = {0.0, 0.0};
        tile_w<LDX>(acc, X, j0, c0, k1, (MC / 8) * w, (MC / 8) * (w + 1), lane);
        Wp[w * 64 + r8 * 8 + 2 * qd] = acc[0];
        Wp[w * 64 + r8 * 8 + 2 * qd + 1] = acc[1];
        __syncthreads();
        if (w == 0) {
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2) {
            const int e = lane + 32 * e2, m = e >> 3, n = e & 7;
            double sum = (c0 + n < k1) ? R[(c0 + n) * LA_LDR + j0 + m] : 0.0;
#pragma unroll
            for (int t = 0; t < LA_NW; ++t) sum += Wp[t * 64 + e];
            Ws[e] = sum;
          }
          __syncwarp();
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2) {
            const int e = lane + 32 * e2, m = e >> 3, n = e & 7;
            const double wv = tt_w(Tm, Ws, m, n);
            WL[e] = wv;
            if (c0 + n < k1) R[(c0 + n) * LA_LDR + j0 + m] -= wv;
          }
        }
        if (panel_w) {
          bar_sync(BAR_P, 32 * NP);
          tile_rank_update<LDX>(X, WL, j0, c0, k1, (MC / NP / 8) * gi, (MC / NP / 8) * (gi + 1), lane);
        } else if (upd_w && p > 0) {
          writeback(p - 1, base, nbase);
        }
      } else if (upd_w && p > 0) {
        writeback(p - 1, base, nbase);
      }
    }
    if (upd_w) {
      writeback(np - 1, base, nbase);   // (the last panel has no columns right of the look-ahead)
      asm volatile("cp.async.wait_all;\n" ::: "memory");
    }
    __syncthreads();   // the next chunk is in place; R holds this chunk's triangle
  }
  // R (k1 x k1, ld k1)
  double* Ro = q.Rout + (int64_t)blockIdx.x * q.ostride;
  for (int e = tid; e < k1 * k1; e += 32 * LA_NW) {
    const int i = e % k1, l = e / k1;
    Ro[e] = i <= l ? R[l * LA_LDR + i] : 0.0;
  }
}
}  // namespace

// AZ_TSQR_LA_NP: 2 (default) panel warps, one per sub-partition 0 and 1 with 128 rows each, or 4 (two
// per sub-partition, 64 rows each).  The chain is partly issue-bound on its sub-partitions: measured
// pass A 1.431 ms (4) against 1.364 ms (2) on c2.
static int la_np() {
  static int v = 0;
  if (!v) {
    const char* e = getenv("AZ_TSQR_LA_NP");
    v = e ? atoi(e) : 2;
    if (v != 1 && v != 4) v = 2;
  }
  return v;
}

// AZ_TSQR_LA_MC=128: 128-row chunks, two CTAs per SM (default 256: one CTA per SM)
int az_tsqr_la_mc() {
  static int v = 0;
  if (!v) {
    const char* e = getenv("AZ_TSQR_LA_MC");
    v = (e && atoi(e) == 128) ? 128 : 256;
  }
  return v;
}

// AZ_TSQR_LA_MERGE=0: the deferred merge levels by the per-column kernel k_tsqr instead
bool az_tsqr_la_merge_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("AZ_TSQR_LA_MERGE");
    v = e ? atoi(e) : 1;
  }
  return v != 0 && az_tsqr_la_enabled() && az_tsqr_la_mc() == 256;
}

size_t az_tsqr_la_smem() {
  return (size_t)(az_tsqr_la_mc() == 128 ? LASmem<128>::END : LASmem<256>::END) * sizeof(double);
}

// AZ_TSQR_LA=0: pass A of the split leaf by the per-column kernel k_tsqr instead
bool az_tsqr_la_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("AZ_TSQR_LA");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

az_status_t az_tsqr_la_leaf(const double* A, int64_t m, int k1, int64_t ld, int64_t rows_per_cta, int P, double* Rout,
                            int64_t ostride, double* Y, int64_t ldY, double* taus, int cmax, cudaStream_t st,
                            int64_t rb, int64_t bstride) {
  if (k1 < 1 || k1 > 64) {
    az_set_error("tsqr_la: k1 = %d not in [1, 64]", k1);
    return AZ_ERR_NOT_SUPPORTED;
  }
  LAIn q;
  q.A = A;
  q.Y = Y;
  q.m = m;
  q.ld = ld;
  q.ldY = ldY;
  q.rows_per_cta = rows_per_cta;
  q.k1 = k1;
  q.cmax = cmax;
  q.Rout = Rout;
  q.ostride = ostride;
  q.taus = taus;
  q.rb = rb;
  q.bstride = bstride;
  const size_t sm = bstride ? (size_t)LASmem<256>::END * sizeof(double) : az_tsqr_la_smem();
  auto kern = bstride ? (la_np() == 4 ? k_tsqr_la<256, true> : k_tsqr_la<256, true, 2>)
                      : (az_tsqr_la_mc() == 128 ? k_tsqr_la<128, false>
                                                : (la_np() == 2   ? k_tsqr_la<256, false, 2>
                                                   : la_np() == 1 ? k_tsqr_la<256, false, 1>
                                                                  : k_tsqr_la<256, false>));
  AZ_CUDA_CHECK(az_smem_attr(kern, sm));
  AzTrace tr(bstride ? "tsqr_merge" : "tsqr_leaf", st, m);
  kern<<<P, 32 * LA_NW, sm, st>>>(q);
  AZ_LAUNCH_CHECK();
  return AZ_OK;
}

