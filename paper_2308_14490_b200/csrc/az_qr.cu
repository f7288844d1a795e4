// R factor of a tall matrix by Householder TSQR (the "SVD of an (r+p)-by-M
// matrix" is computed as QR of the M x (r+p) sketch followed by an SVD of the small R).
//
// Stage 1: each CTA streams its contiguous row range through a structured Householder QR of
// [R; chunk] (R upper triangular, chunk = MC rows held in registers): for column j the
// reflector is H = I - tau v v^T with v = [e_j ; y] (LAPACK dlarfg convention), applied to the
// columns l > j of R and of the chunk.  No Q is formed (only R is needed: the right-hand sides
// ride along as extra columns, so R's last columns hold Q^T b').
// Stage 2..: the per-CTA R factors are stacked and reduced by the same kernel in groups until
// one R remains (a fixed-shape reduction tree: the result does not depend on timing).
//
// Layout inside a CTA: 16 warps; warp w owns columns l = w + 16 c (c < KC); lane owns rows
// lane + 32 r (r < RPL) of the chunk.  R lives in shared memory, packed column-major upper
// triangle; each R column is only ever touched by its owner warp, so the only block-wide
// barrier per column step is the broadcast of the reflector (double-buffered).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "az_internal.h"
#include "az_mma.cuh"

AZ_D int pk(int i, int l) { return (l * (l + 1)) / 2 + i; }   // R[i][l], i <= l

AZ_D double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct QRIn {
  const double* A;
  int64_t m;        // rows
  int k;            // columns
  int k1;           // leading columns to triangularise (the rest are only transformed: Q^T b')
  int64_t ld;       // column stride
  int64_t rb;       // rows per block of the stacked input (row r at (r / rb) * bstride + (r % rb))
  int64_t bstride;
  int64_t rows_per_cta;
  double* Rout;     // per CTA k1 x k column-major (ld = k1), CTA stride ostride
  int64_t ostride;
  // optional (split leaf): the chunk parts y_j of the reflectors and their tau, per chunk
  double* Y;        // y_j of chunk rows written to Y[row + j ldY] (the triangularised columns' storage);
                    // merges: Y[(row / rb) bstride + row % rb + j ldY], the input's block layout
  int64_t ldY;
  double* taus;     // taus[(cta cmax + chunk) k1 + j]
  int cmax;         // chunks per CTA (ceil(rows_per_cta / MC))
};

template <int KC, int RPL, bool YSTACK = false, int NW = 16>
__global__ void __launch_bounds__(32 * NW, NW >= 16 ? 1 : 2) k_tsqr(QRIn q) {
  constexpr int MC = 32 * RPL;
  extern __shared__ double sm[];
  const int k = q.k;
  double* R = sm;                                // k (k+1) / 2
  double* vb = R + (k * (k + 1)) / 2;            // 2 x MC
  double* tb = vb + 2 * MC;                      // 2
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (k * (k + 1)) / 2; i += blockDim.x) R[i] = 0.0;
  const int64_t r0 = (int64_t)blockIdx.x * q.rows_per_cta;
  const int64_t r1 = (q.m < r0 + q.rows_per_cta) ? q.m : r0 + q.rows_per_cta;
  double x[KC][RPL];
  __syncthreads();

  for (int64_t base = r0; base < r1; base += MC) {
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      const int l = w + NW * c;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int64_t row = base + lane + 32 * r;
        double v = 0.0;
        // leaves (bstride == 0) read rows directly; merges read stacked rb-row factors
        const int64_t off = q.bstride ? (row / q.rb) * q.bstride + (row % q.rb) : row;
        if (row < r1 && l < k) v = q.A[off + (int64_t)l * q.ld];
        x[c][r] = v;
      }
    }
    for (int j = 0; j < q.k1; ++j) {
      const int o = j % NW, cj = j / NW;
      double* vj = vb + (j & 1) * MC;
      if (w == o) {
        // everyone waits at the barrier below for this chain, so it is kept short: the slot is
        // picked with a warp-uniform switch (no select chains), alpha is loaded first, and
        // tau = (beta - alpha) / beta = 1 + |alpha| / ||x|| comes from one reciprocal square root
        const double alpha = R[pk(j, j)];
        double xs[RPL];
        switch (cj) {
#define AZ_TSQR_TAKE(C)                                   \
  case C:                                                 \
    if constexpr (C < KC) {                               \
      _Pragma("unroll") for (int r = 0; r < RPL; ++r) {   \
        xs[r] = x[C][r];                                  \
        x[C][r] = 0.0;                                    \
      }                                                   \
    }                                                     \
    break;
          AZ_TSQR_TAKE(0)
          AZ_TSQR_TAKE(1)
          AZ_TSQR_TAKE(2)
          AZ_TSQR_TAKE(3)
          AZ_TSQR_TAKE(4)
          AZ_TSQR_TAKE(5)
          AZ_TSQR_TAKE(6)
          AZ_TSQR_TAKE(7)
#undef AZ_TSQR_TAKE
          default:
#pragma unroll
            for (int r = 0; r < RPL; ++r) xs[r] = 0.0;
        }
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; r += 2) {
          s0 = fma(xs[r], xs[r], s0);
          if (r + 1 < RPL) s1 = fma(xs[r + 1], xs[r + 1], s1);
        }
        const double sig = warp_sum(s0 + s1);
        double tau = 0.0, scale = 0.0, beta = alpha;
        if (sig > 0.0) {
          const double s2 = fma(alpha, alpha, sig);
          const double rinv = fast_rsqrt(s2);
          const double nrm = s2 * rinv;
          beta = alpha >= 0.0 ? -nrm : nrm;
          tau = fma(fabs(alpha), rinv, 1.0);
          scale = fast_rcp(alpha - beta);
        }
#pragma unroll
        for (int r = 0; r < RPL; ++r) vj[lane + 32 * r] = xs[r] * scale;
        if (q.Y) {   // split leaf / merge: keep the reflector for the right-hand-side pass (k_tsqr_rhs)
          if constexpr (YSTACK) {   // merges: Y in the stacked block layout of the input
#pragma unroll
            for (int r = 0; r < RPL; ++r) {
              const int64_t row = base + lane + 32 * r;
              if (row < r1) q.Y[(row / q.rb) * q.bstride + (row % q.rb) + (int64_t)j * q.ldY] = xs[r] * scale;
            }
          } else {
#pragma unroll
            for (int r = 0; r < RPL; ++r) {
              const int64_t row = base + lane + 32 * r;
              if (row < r1) q.Y[row + (int64_t)j * q.ldY] = xs[r] * scale;
            }
          }
          if (lane == 0) q.taus[((int64_t)blockIdx.x * q.cmax + (base - r0) / MC) * q.k1 + j] = tau;
        }
        __syncwarp();
        if (lane == 0) {
          R[pk(j, j)] = beta;
          tb[j & 1] = tau;
        }
      }
      __syncthreads();
      const double tau = tb[j & 1];
      if (tau != 0.0) {
        double v[RPL];
#pragma unroll
        for (int r = 0; r < RPL; ++r) v[r] = vj[lane + 32 * r];
        // all owned live columns at once: KC independent dot products, interleaved warp reductions.
        // A column at or left of j is already triangularised (its registers hold zeros): its dot is
        // skipped (warp-uniform), which removes half of the step's dot-product FMAs on average -- the
        // apply phase is FP64-pipe bound (ncu: math-throttle / not-selected stalls on these DFMAs)
        double p[KC];
#pragma unroll
        for (int c = 0; c < KC; ++c) {
          p[c] = 0.0;
          if (w + NW * c > j) {
#pragma unroll
            for (int r = 0; r < RPL; ++r) p[c] = fma(v[r], x[c][r], p[c]);
          }
        }
        // transpose-reduce: KC - 1 + (5 - log2 KC) shuffles instead of 5 KC; afterwards lane L holds
        // the full dot of column slot L / (32 / KC)
        constexpr int LPC = 32 / KC;   // lanes per column slot after the halving levels
#pragma unroll
        for (int o = 16, n = KC; n > 1; o >>= 1, n >>= 1) {
          const bool hi = lane & o;
#pragma unroll
          for (int i = 0; i < n / 2; ++i) {
            const double send = hi ? p[i] : p[i + n / 2];
            const double keep = hi ? p[i + n / 2] : p[i];
            p[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
        double dsum = p[0];
#pragma unroll
        for (int o = LPC / 2; o > 0; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
        const int cs = lane / LPC;
        const int ls = w + NW * cs;
        const bool live = ls > j && ls < k;
        const double rjs = live ? R[pk(j, ls)] : 0.0;
        const double tws = live ? tau * (rjs + dsum) : 0.0;
        __syncwarp();
        if (live && (lane & (LPC - 1)) == 0) R[pk(j, ls)] = rjs - tws;
#pragma unroll
        for (int c = 0; c < KC; ++c) {
          const int l = w + NW * c;
          const double tw = __shfl_sync(0xffffffffu, tws, c * LPC);
          if (l > j && l < k) {
#pragma unroll
            for (int r = 0; r < RPL; ++r) x[c][r] = fma(-tw, v[r], x[c][r]);
          }
        }
      }
    }
  }
  __syncthreads();
  // top k1 rows of R (k1 x k, ld k1)
  const int k1 = q.k1;
  double* Ro = q.Rout + (int64_t)blockIdx.x * q.ostride;
  for (int e = threadIdx.x; e < k1 * k; e += blockDim.x) {
    const int i = e % k1, l = e / k1;
    Ro[e] = i <= l ? R[pk(i, l)] : 0.0;
  }
}


// ------------------------------------------------------------------------------------------
// Split leaf, pass B: the right-hand-side columns X = b' of a CTA's row range
// are carried through the same chunk sequence as pass A's [R; chunk] QR of the probe columns, but
// each chunk's 64 reflectors are applied at once in compact-WY form.  With V = [I; Y] (the unit
// R-part over the chunk part Y, MC x k1) and T from the dlarft recurrence,
//   H_{k1-1} ... H_0 [R_b; X] :  R_b <- R_b - T^T (R_b + Y^T X)
// (the chunk part of X is not needed afterwards: only R's rows survive a TSQR leaf).  Y^T Y (for T)
// and Y^T X are DMMA Gram products over the chunk rows.  Same values as applying the reflectors one
// by one, up to rounding.
// ------------------------------------------------------------------------------------------
struct QRr {
  int64_t rb, bstride;  // stacked rows (merges): row r at (r / rb) bstride + r % rb; 0 = plain
  const double* Y;      // m x k1 (ld ldY): pass A's reflectors
  int64_t ldY;
  const double* X;      // m x nb (ld ldX): the right-hand-side columns
  int64_t ldX;
  int64_t m, rows_per_cta;
  int k1, nb, MC, cmax;
  const double* taus;
  double* Rout;         // per CTA k1 x (k1 + nb), ld k1, CTA stride ostride: writes columns k1..
  int64_t ostride;
};

constexpr int RR_S2 = 68;  // operand tile stride (== 4 mod 16), 64-row sub-blocks
#ifndef PB_KU
#define PB_KU 16           // pass B: k-steps per unrolled group of the DMMA loop
#endif

__global__ void __launch_bounds__(512, 1) k_tsqr_rhs(QRr q) {
  extern __shared__ double sm[];
  double* Ys = sm;                       // IMAJ [col][row], 64 x RR_S2 (64-row sub-block)
  double* Xs = Ys + 64 * RR_S2;          // IMAJ [col][row]
  double* G = Xs + 64 * RR_S2;           // 64 x 64 (ld 65): Y^T Y, then TG[j][m] = tau_m G[j][m]
  double* P = G + 64 * 65;               // 64 x 64 (ld 65): Y^T X, then W = R_b + P, then d
  double* Rb = P + 64 * 65;              // 64 x 64 (ld 65)
  double* tau_s = Rb + 64 * 65;          // 64
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int k1 = q.k1, nb = q.nb;
  for (int e = tid; e < 64 * 65; e += 512) Rb[e] = 0.0;
  const int64_t r0 = (int64_t)blockIdx.x * q.rows_per_cta;
  const int64_t r1 = min(q.m, r0 + q.rows_per_cta);
  // warps 0-7: G tiles rows (w & 1) 32.., cols (w >> 1) 16..;  warps 8-15: the same tiles of P
  const int ww = w & 7, wm = ww & 1, wn = ww >> 1;
  const bool isG = w < 8;
  // tiles that hold no needed entry skip their MMAs (the DP tensor pipe is the shared limit): G is
  // only read below its diagonal (m < j), and only rows < k1 and columns < k1 (G) / nb (P) exist
  const bool mma_on = 32 * wm < k1 && (isG ? (16 * wn < k1 && 16 * wn < 32 * wm + 31) : 16 * wn < nb);
  double ry[8], rx[8];   // the next 64-row sub-block, in flight during the current MMAs
  auto load = [&](int64_t rr, int64_t cend) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int e = tid + 512 * t, cidx = e >> 6, rl = e & 63;
      const int64_t row = rr + rl;
      const bool in = row < cend;
      const int64_t off = q.bstride ? (row / q.rb) * q.bstride + (row % q.rb) : row;
      ry[t] = (in && cidx < k1) ? q.Y[off + (int64_t)cidx * q.ldY] : 0.0;
      rx[t] = (in && cidx < nb) ? q.X[off + (int64_t)cidx * q.ldX] : 0.0;
    }
  };
  int chunk = 0;
  for (int64_t base = r0; base < r1; base += q.MC, ++chunk) {
    const int64_t cend = min(r1, base + (int64_t)q.MC);
    double acc[4][2][2];
    acc_zero(acc);
    load(base, cend);
    if (tid < 64) tau_s[tid] = tid < k1 ? q.taus[((int64_t)blockIdx.x * q.cmax + chunk) * k1 + tid] : 0.0;
    for (int64_t rr = base; rr < cend; rr += 64) {
      __syncthreads();
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int e = tid + 512 * t, cidx = e >> 6, rl = e & 63;
        Ys[cidx * RR_S2 + rl] = ry[t];
        Xs[cidx * RR_S2 + rl] = rx[t];
      }
      __syncthreads();
      if (rr + 64 < cend) load(rr + 64, cend);
      if (mma_on) warp_mma<4, 2, IMAJ, IMAJ, PB_KU>(acc, Ys, RR_S2, isG ? Ys : Xs, RR_S2, wm * 32, wn * 16, 0, 64, lane);
    }
    double* D = isG ? G : P;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          D[acc_row(wm * 32, i, lane) * 65 + acc_col(wn * 16, jj, e, lane)] = acc[i][jj][e];
    __syncthreads();
    // TG[j][m] = tau_m (y_j . y_m) for m < j;  W = R_b + Y^T X
    for (int e = tid; e < 64 * 64; e += 512) {
      const int j = e >> 6, m = e & 63;
      G[j * 65 + m] = m < j ? tau_s[m] * G[j * 65 + m] : 0.0;
      P[j * 65 + m] += Rb[j * 65 + m];
    }
    __syncthreads();
    // Reflectors in order, per right-hand-side column c (independent): with d_m = v_m^T [R_b; X^(m)]
    // (X^(m): X after reflectors < m; R row j is only touched by reflector j),
    //   d_j = W[j][c] - sum_{m<j} tau_m (y_j . y_m) d_m,   R_b[j][c] -= tau_j d_j
    // in blocks of 8 j: the part over earlier blocks by all threads (one (j, c) each), the
    // triangle inside the block by one thread per column.
    double* S8 = Ys;   // 8 x 64 partial sums (the operand tiles are free now)
    for (int jb = 0; jb < k1; jb += 8) {
      {
        const int r = tid >> 6, c = tid & 63, j = jb + r;
        if (j < k1 && c < nb) {
          double s0 = P[j * 65 + c], s1 = 0.0, s2 = 0.0, s3 = 0.0;
          const double* tg = G + j * 65;
          for (int m = 0; m < jb; m += 4) {   // jb is a multiple of 8
            s0 = fma(-tg[m], P[m * 65 + c], s0);
            s1 = fma(-tg[m + 1], P[(m + 1) * 65 + c], s1);
            s2 = fma(-tg[m + 2], P[(m + 2) * 65 + c], s2);
            s3 = fma(-tg[m + 3], P[(m + 3) * 65 + c], s3);
          }
          S8[r * 64 + c] = (s0 + s1) + (s2 + s3);
        }
      }
      __syncthreads();
      if (tid < nb) {   // the block's triangle, its d values in registers (k1 is a multiple of 8 or
        const int c = tid;   // the rows past k1 have zero sums and are not stored)
        double d[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int j = jb + r;
          double v = (j < k1) ? S8[r * 64 + c] : 0.0;
#pragma unroll
          for (int rr = 0; rr < r; ++rr) v = fma(-G[j * 65 + jb + rr], d[rr], v);
          d[r] = v;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int j = jb + r;
          if (j < k1) {
            P[j * 65 + c] = d[r];
            Rb[j * 65 + c] -= tau_s[j] * d[r];
          }
        }
      }
      __syncthreads();
    }
  }
  double* Ro = q.Rout + (int64_t)blockIdx.x * q.ostride;
  for (int e = tid; e < k1 * nb; e += 512) {
    const int i = e % k1, c = e / k1;
    Ro[(int64_t)(k1 + c) * k1 + i] = Rb[i * 65 + c];
  }
}

static int g_sms = 0;
static int num_sms() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

template <int KC, int RPL, int NW = 16>
static az_status_t tsqr_launch(const QRIn& q, int nblocks, cudaStream_t st) {
  constexpr int MC = 32 * RPL;
  static_assert(KC * NW >= 64 || NW == 16, "KC x NW columns");
  const size_t sm = ((size_t)q.k * (q.k + 1) / 2 + 2 * MC + 2) * sizeof(double);
  // (a separate instantiation for the merges' stacked reflector store keeps the leaf's owner
  // chain free of it)
  auto kern = k_tsqr<KC, RPL, false, NW>;
  if constexpr (RPL == 8 || RPL == 4)   // (merges run the 256- / 128-row shapes only)
    if (q.Y && q.bstride) kern = k_tsqr<KC, RPL, true, NW>;
  AZ_CUDA_CHECK(az_smem_attr(kern, sm));
  AzTrace tr(q.bstride ? "tsqr_merge" : "tsqr_leaf", st, q.m);
  kern<<<nblocks, 32 * NW, sm, st>>>(q);
  AZ_LAUNCH_CHECK();
  return AZ_OK;
}

static az_status_t tsqr_pass(const QRIn& q, int nblocks, cudaStream_t st) {
  if (q.k <= 32) return tsqr_launch<2, 8>(q, nblocks, st);
  if (q.k <= 64) return tsqr_launch<4, 8>(q, nblocks, st);
  if (q.k <= 128) return tsqr_launch<8, 4>(q, nblocks, st);
  az_set_error("tsqr: k = %d > 128 not supported by the single-pass TSQR", q.k);
  return AZ_ERR_NOT_SUPPORTED;
}

static size_t a256q(size_t v) { return (v + 255) & ~(size_t)255; }

size_t az_qr_ws_bytes(int64_t m, int64_t k) {
  if (k > AZ_NARROW_MAX) {   // wide: T factors of every panel + the blocked-update workspace
    const int64_t QBw = az_qrw_panel_width();
    const int64_t np = (k + QBw - 1) / QBw;
    return a256q((size_t)np * QBw * QBw * sizeof(double)) + az_qrw_ws_bytes(m, k);
  }
  const int64_t P = std::max<int64_t>(1, std::min<int64_t>(2 * num_sms(), (m + 127) / 128));
  // leaf / merge factors (two buffers) + the split leaf's reflector taus (per 128-row chunk)
  // + the deferred-rhs merge reflectors of every tree level (az_qr_r_deferred)
  int64_t ylev = 0, tlev = 0;
  for (int64_t cur = P; cur > 1; cur = (cur + 3) / 4) {
    ylev += cur * k * k;
    tlev += (cur + 3) / 4 * k;
  }
  return (size_t)(2 * P * k * k + ((m + 127) / 128 + 2 * P) * k + ylev + tlev) * sizeof(double) + 256;
}

static az_status_t qr_r_wide(double* A, int64_t m, int64_t k, int64_t lda, double* R, int64_t ldr, void* ws,
                             size_t ws_bytes, cudaStream_t st) {
  const int64_t QBw = az_qrw_panel_width();
  const int64_t np = (k + QBw - 1) / QBw;
  const size_t tb = a256q((size_t)np * QBw * QBw * sizeof(double));
  std::vector<int64_t> pj0(np);
  std::vector<int> pnb(np);
  int64_t cnt = 0;
  AZ_TRY(az_qrw_factor(A, lda, m, 0, k, (double*)ws, pj0.data(), pnb.data(), &cnt, (char*)ws + tb, ws_bytes - tb, st));
  return az_qrw_extract_R(A, lda, k, R, ldr, st);
}

__global__ void k_copy_R(const double* Rin, int k1, int k, double* R, int64_t ldr) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < k1 * k) R[(e / k1) * ldr + (e % k1)] = Rin[e];
}

// k1 < k: only the leading k1 columns are triangularised and only the top k1 rows of R are
// returned (R[:k1, k1:] = (Q^T A[:, k1:])[:k1], e.g. Q^T b' for the right-hand sides riding along).
static bool tsqr_split() {   // AZ_TSQR_SPLIT=0 keeps the single-pass leaf for [S | b']
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("AZ_TSQR_SPLIT");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

az_status_t az_qr_r_impl(double* A, int64_t m, int64_t k, int64_t lda, double* R, int64_t ldr,
                         void* ws, size_t ws_bytes, cudaStream_t st, int64_t k1, bool a_scratch,
                         cudaEvent_t after_leaf) {
  if (k1 <= 0 || k1 > k) k1 = k;
  if (ws_bytes < az_qr_ws_bytes(m, k)) {
    az_set_error("az_qr_r: workspace too small");
    return AZ_ERR_WORKSPACE;
  }
  if (k > AZ_NARROW_MAX) {
    if (k > m) {
      az_set_error("az_qr_r: blocked path needs m >= k (m = %lld, k = %lld)", (long long)m, (long long)k);
      return AZ_ERR_NOT_SUPPORTED;
    }
    return qr_r_wide(A, m, k, lda, R, ldr, ws, ws_bytes, st);
  }
  // a sketch of at most 288 rows (c1: 257) is one chunk of one CTA: k1 column steps in all, no
  // merge, the right-hand sides riding along (instead of 3 leaf CTAs, pass B and a merge level)
  const bool one = m <= 288 && k <= 64;
  const int64_t P = one ? 1 : std::max<int64_t>(1, std::min<int64_t>(num_sms(), (m + 127) / 128));
  double* buf[2] = {(double*)ws, (double*)ws + P * k * k};
  QRIn q;
  q.A = A;
  q.m = m;
  q.k = (int)k;
  q.k1 = (int)k1;
  q.ld = lda;
  q.rb = m;
  q.bstride = 0;
  q.rows_per_cta = (m + P - 1) / P;
  q.Rout = buf[0];
  q.ostride = k1 * k;
  q.Y = nullptr;
  q.ldY = 0;
  q.taus = nullptr;
  q.cmax = 0;
  const int64_t nb = k - k1;
  if (one) {
    if (k <= 32)
      AZ_TRY((tsqr_launch<2, 9>(q, 1, st)));
    else
      AZ_TRY((tsqr_launch<4, 9>(q, 1, st)));
  } else if (a_scratch && k1 < k && k1 <= 64 && nb <= 64 && tsqr_split()) {
    // split leaf: pass A triangularises the k1 probe columns alone in 256-row chunks (KC = 4,
    // RPL = 8: half the column steps per row of the 128-column pass) and keeps each chunk's
    // reflectors in place of those columns; pass B applies them to the right-hand sides in
    // compact-WY form (DMMA Gram products)
    constexpr int MC = 256;
    q.k = (int)k1;
    q.Y = A;
    q.ldY = lda;
    q.cmax = (int)((q.rows_per_cta + MC - 1) / MC);
    q.taus = (double*)ws + 2 * P * k * k;
    AZ_TRY((tsqr_launch<4, 8>(q, (int)P, st)));
    QRr r;
    r.rb = 0;
    r.bstride = 0;
    r.Y = A;
    r.ldY = lda;
    r.X = A + k1 * lda;
    r.ldX = lda;
    r.m = m;
    r.rows_per_cta = q.rows_per_cta;
    r.k1 = (int)k1;
    r.nb = (int)nb;
    r.MC = MC;
    r.cmax = q.cmax;
    r.taus = q.taus;
    r.Rout = buf[0];
    r.ostride = k1 * k;
    const size_t rsm = (size_t)(2 * 64 * RR_S2 + 3 * 64 * 65 + 64) * sizeof(double);
    AZ_CUDA_CHECK(az_smem_attr(k_tsqr_rhs, rsm));
    {
      AzTrace tr("tsqr_rhs", st, m);
      k_tsqr_rhs<<<(unsigned)P, 512, rsm, st>>>(r);
      AZ_LAUNCH_CHECK();
    }
  } else {
    AZ_TRY(tsqr_pass(q, (int)P, st));
  }
  if (after_leaf) AZ_CUDA_CHECK(cudaEventRecord(after_leaf, st));
  int64_t cur = P;
  int which = 0;
  // fixed-shape reduction tree: groups of 4 R factors
  while (cur > 1) {
    const int64_t G = 4;
    const int64_t next = (cur + G - 1) / G;
    QRIn t;
    t.A = buf[which];
    t.m = cur * k1;
    t.k = (int)k;
    t.k1 = (int)k1;
    t.ld = k1;
    t.rb = k1;
    t.bstride = k1 * k;
    t.rows_per_cta = G * k1;
    t.Rout = buf[which ^ 1];
    t.ostride = k1 * k;
    t.Y = nullptr;
    t.ldY = 0;
    t.taus = nullptr;
    t.cmax = 0;
    AZ_TRY(tsqr_pass(t, (int)next, st));

    which ^= 1;
    cur = next;
  }
  k_copy_R<<<az_div_up(k1 * k, 256), 256, 0, st>>>(buf[which], (int)k1, (int)k, R, ldr);
  AZ_LAUNCH_CHECK();
  return AZ_OK;
}

// The split leaf with Q^T b' taken off the R factor's critical path (single probe block, k1 <= 64
// probe columns, nb = k - k1 <= 64 right-hand sides; A is scratch), in two enqueue calls:
//   az_qr_r_deferred (st):  pass A (probe columns, reflectors kept in place) -> ev_leaf -> merge
//           tree of the probe columns alone, each level's reflectors kept (in the input's block
//           layout) -> R_S into Rs (k1 x k1, ld ldrs) -> ev_merged
//   az_qr_rhs_deferred (rhs_st, after ev_leaf): pass B, b' through the leaf chunks' reflectors ->
//           (after ev_merged) the same compact-WY pass over each merge level's stacked blocks ->
//           C = (Q^T b')[:k1] (k1 x nb, ld ldc)
// Same R_S and Q^T b' as az_qr_r_impl up to rounding (the same reflectors, applied in the same
// order per column).  The caller may enqueue other work on rhs_st between the two calls.
namespace {
constexpr int DEF_MC = 256;   // merge levels: 4 stacked k1 x k1 blocks per chunk
// Leaf shape of the deferred split leaf.  AZ_TSQR_NW=16 (default): one 512-thread CTA per SM, 256-row
// chunks.  AZ_TSQR_NW=8: two 256-thread CTAs per SM, each a sequence of 128-row chunks (KC = 8 columns
// per warp, RPL = 4 rows per lane) -- measured no faster on c2 (pass A 1.80 vs 1.82 ms) and pass B,
// which must follow the leaf's chunks, slower (1.20 vs 0.90 ms).
static int def_nw() {
  static int v = 0;
  if (!v) {
    const char* e = getenv("AZ_TSQR_NW");
    v = (e && atoi(e) == 8) ? 8 : 16;
  }
  return v;
}
static int def_leaf_mc() {
  if (def_nw() == 8) return 128;
  return az_tsqr_la_enabled() ? az_tsqr_la_mc() : 256;
}
struct DefLev {
  double* Y;
  double* taus;
  int64_t cur, next;
  int which;
};
struct DefLayout {
  int64_t P, rows_per_cta;
  int cmax;
  double* buf[2];
  double* taus0;
  std::vector<DefLev> lev;
  int final_which;
};
DefLayout def_layout(int64_t m, int64_t k, void* ws) {
  DefLayout d;
  // one leaf block fewer than SMs: pass B (one 170 KB CTA per SM and leaf block) then runs in a
  // single wave beside the one-CTA Jacobi, which holds an SM of its own
  const int64_t per_sm = def_leaf_mc() == 128 ? 2 : 1;
  d.P = std::max<int64_t>(1, std::min<int64_t>(per_sm * (num_sms() - 1), (m + 127) / 128));
  d.rows_per_cta = (m + d.P - 1) / d.P;
  d.cmax = (int)((d.rows_per_cta + def_leaf_mc() - 1) / def_leaf_mc());
  d.buf[0] = (double*)ws;
  d.buf[1] = (double*)ws + d.P * k * k;
  d.taus0 = (double*)ws + 2 * d.P * k * k;
  double* yp = d.taus0 + ((m + 127) / 128 + 2 * d.P) * k;
  int which = 0;
  for (int64_t cur = d.P; cur > 1;) {
    const int64_t next = (cur + 3) / 4;
    d.lev.push_back(DefLev{yp, yp + cur * k * k, cur, next, which});
    yp += cur * k * k + next * k;
    which ^= 1;
    cur = next;
  }
  d.final_which = which;
  return d;
}
bool def_ok(int64_t k, int64_t k1) { return k1 >= 1 && k1 <= 64 && k - k1 >= 1 && k - k1 <= 64; }
size_t def_rhs_smem() { return (size_t)(2 * 64 * RR_S2 + 3 * 64 * 65 + 64) * sizeof(double); }
}  // namespace

az_status_t az_qr_r_deferred(double* A, int64_t m, int64_t k, int64_t k1, int64_t lda, double* Rs, int64_t ldrs,
                             void* ws, size_t ws_bytes, cudaStream_t st, cudaEvent_t ev_leaf, cudaEvent_t ev_merged) {
  if (!def_ok(k, k1) || ws_bytes < az_qr_ws_bytes(m, k)) {
    az_set_error("az_qr_r_deferred: needs 1 <= k1 <= 64, 1 <= k - k1 <= 64 and the az_qr workspace");
    return AZ_ERR_INVALID_ARGUMENT;
  }
  const DefLayout d = def_layout(m, k, ws);
  QRIn q;
  q.A = A;
  q.m = m;
  q.k = (int)k1;
  q.k1 = (int)k1;
  q.ld = lda;
  q.rb = m;
  q.bstride = 0;
  q.rows_per_cta = d.rows_per_cta;
  q.Rout = d.buf[0];
  q.ostride = k1 * k;
  q.Y = A;
  q.ldY = lda;
  q.cmax = d.cmax;
  q.taus = d.taus0;
  if (def_nw() == 8)
    AZ_TRY((tsqr_launch<8, 4, 8>(q, (int)d.P, st)));
  else if (az_tsqr_la_enabled())
    AZ_TRY(az_tsqr_la_leaf(A, m, (int)k1, lda, d.rows_per_cta, (int)d.P, d.buf[0], k1 * k, A, lda, d.taus0, d.cmax, st));
  else
    AZ_TRY((tsqr_launch<4, 8>(q, (int)d.P, st)));
  AZ_CUDA_CHECK(cudaEventRecord(ev_leaf, st));
  for (const DefLev& L : d.lev) {   // merge tree of the probe columns, reflectors kept per level
    QRIn t;
    t.A = d.buf[L.which];
    t.m = L.cur * k1;
    t.k = (int)k1;
    t.k1 = (int)k1;
    t.ld = k1;
    t.rb = k1;
    t.bstride = k1 * k;
    t.rows_per_cta = 4 * k1;
    t.Rout = d.buf[L.which ^ 1];
    t.ostride = k1 * k;
    t.Y = L.Y;
    t.ldY = k1;
    t.taus = L.taus;
    t.cmax = 1;
    if (az_tsqr_la_merge_enabled())   // 4 stacked k1 x k1 factors = one chunk of <= 256 rows per CTA
      AZ_TRY(az_tsqr_la_leaf(t.A, t.m, (int)k1, t.ld, t.rows_per_cta, (int)L.next, t.Rout, t.ostride, t.Y, t.ldY,
                             t.taus, 1, st, t.rb, t.bstride));
    else
      AZ_TRY((tsqr_launch<4, 8>(t, (int)L.next, st)));
  }
  k_copy_R<<<az_div_up(k1 * k1, 256), 256, 0, st>>>(d.buf[d.final_which], (int)k1, (int)k1, Rs, ldrs);
  AZ_LAUNCH_CHECK();
  AZ_CUDA_CHECK(cudaEventRecord(ev_merged, st));
  return AZ_OK;
}

az_status_t az_qr_rhs_deferred(double* A, int64_t m, int64_t k, int64_t k1, int64_t lda, double* C, int64_t ldc,
                               void* ws, size_t ws_bytes, cudaStream_t rhs_st, cudaEvent_t ev_leaf,
                               cudaEvent_t ev_merged, cudaEvent_t ev_passb) {
  if (!def_ok(k, k1) || ws_bytes < az_qr_ws_bytes(m, k)) {
    az_set_error("az_qr_rhs_deferred: needs 1 <= k1 <= 64, 1 <= k - k1 <= 64 and the az_qr workspace");
    return AZ_ERR_INVALID_ARGUMENT;
  }
  const int64_t nb = k - k1;
  const DefLayout d = def_layout(m, k, ws);
  const size_t rsm = def_rhs_smem();
  AZ_CUDA_CHECK(az_smem_attr(k_tsqr_rhs, rsm));
  AZ_CUDA_CHECK(cudaStreamWaitEvent(rhs_st, ev_leaf, 0));
  QRr r;   // pass B: the leaf blocks' Q^T b' rows into columns k1.. of buf[0]
  r.rb = 0;
  r.bstride = 0;
  r.Y = A;
  r.ldY = lda;
  r.X = A + k1 * lda;
  r.ldX = lda;
  r.m = m;
  r.rows_per_cta = d.rows_per_cta;
  r.k1 = (int)k1;
  r.nb = (int)nb;
  r.MC = def_leaf_mc();
  r.cmax = d.cmax;
  r.taus = d.taus0;
  r.Rout = d.buf[0];
  r.ostride = k1 * k;
  {
    AzTrace tr("tsqr_rhs", rhs_st, m);
    k_tsqr_rhs<<<(unsigned)d.P, 512, rsm, rhs_st>>>(r);
    AZ_LAUNCH_CHECK();
  }
  if (ev_passb) AZ_CUDA_CHECK(cudaEventRecord(ev_passb, rhs_st));
  AZ_CUDA_CHECK(cudaStreamWaitEvent(rhs_st, ev_merged, 0));
  for (const DefLev& L : d.lev) {   // the stacked blocks' right-hand-side columns, level by level
    QRr c;
    c.rb = k1;
    c.bstride = k1 * k;
    c.Y = L.Y;
    c.ldY = k1;
    c.X = d.buf[L.which] + k1 * k1;
    c.ldX = k1;
    c.m = L.cur * k1;
    c.rows_per_cta = 4 * k1;
    c.k1 = (int)k1;
    c.nb = (int)nb;
    c.MC = DEF_MC;
    c.cmax = 1;
    c.taus = L.taus;
    c.Rout = d.buf[L.which ^ 1];
    c.ostride = k1 * k;
    AzTrace tr("tsqr_rhs_merge", rhs_st, c.m);
    k_tsqr_rhs<<<(unsigned)L.next, 512, rsm, rhs_st>>>(c);
    AZ_LAUNCH_CHECK();
  }
  k_copy_R<<<az_div_up(k1 * nb, 256), 256, 0, rhs_st>>>(d.buf[d.final_which] + k1 * k1, (int)k1, (int)nb, C, ldc);
  AZ_LAUNCH_CHECK();
  return AZ_OK;
}

extern "C" az_status_t az_qr_workspace_size(int64_t m, int64_t k, size_t* bytes) {
  if (!bytes || m < 0 || k < 0) {
    az_set_error("az_qr_workspace_size: bad arguments");
    return AZ_ERR_INVALID_ARGUMENT;
  }
  *bytes = az_qr_ws_bytes(m, k);
  return AZ_OK;
}

extern "C" az_status_t az_qr_r(az_plan_t, double* A, int64_t m, int64_t k, int64_t lda, double* R, int64_t ldr,
                               void* ws, size_t ws_bytes, void* stream) {
  if (!A || !R || m < 1 || k < 1 || lda < m || ldr < k) {
    az_set_error("az_qr_r: bad arguments");
    return AZ_ERR_INVALID_ARGUMENT;
  }
  return az_qr_r_impl(A, m, k, lda, R, ldr, ws, ws_bytes, (cudaStream_t)stream, k);
}

extern "C" az_status_t az_qr_r_partial(az_plan_t, double* A, int64_t m, int64_t k, int64_t k1, int64_t lda, double* R,
                                       int64_t ldr, void* ws, size_t ws_bytes, void* stream) {
  if (!A || !R || m < 1 || k < 1 || k1 < 1 || k1 > k || lda < m || ldr < k1) {
    az_set_error("az_qr_r_partial: bad arguments");
    return AZ_ERR_INVALID_ARGUMENT;
  }
  if (k > AZ_NARROW_MAX && k1 < k) {
    az_set_error("az_qr_r_partial: k1 < k needs k <= %lld", (long long)AZ_NARROW_MAX);
    return AZ_ERR_NOT_SUPPORTED;
  }
  return az_qr_r_impl(A, m, k, lda, R, ldr, ws, ws_bytes, (cudaStream_t)stream, k1);
}

