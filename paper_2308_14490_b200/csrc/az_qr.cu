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
#include <vector>

#include "az_internal.h"

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
  double* Rout;     // per CTA k x k column-major (ld = k)
};

template <int KC, int RPL>
__global__ void __launch_bounds__(512, 1) k_tsqr(QRIn q) {
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
      const int l = w + 16 * c;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int64_t row = base + lane + 32 * r;
        double v = 0.0;
        if (row < r1 && l < k) v = q.A[(row / q.rb) * q.bstride + (row % q.rb) + (int64_t)l * q.ld];
        x[c][r] = v;
      }
    }
    for (int j = 0; j < q.k1; ++j) {
      const int o = j & 15, cj = j >> 4;
      double* vj = vb + (j & 1) * MC;
      if (w == o) {
        double xs[RPL];
#pragma unroll
        for (int r = 0; r < RPL; ++r) xs[r] = 0.0;
#pragma unroll
        for (int c = 0; c < KC; ++c)
          if (c == cj) {
#pragma unroll
            for (int r = 0; r < RPL; ++r) {
              xs[r] = x[c][r];
              x[c][r] = 0.0;
            }
          }
        double sig = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; ++r) sig = fma(xs[r], xs[r], sig);
        sig = warp_sum(sig);
        const double alpha = R[pk(j, j)];
        double tau = 0.0, scale = 0.0, beta = alpha;
        if (sig > 0.0) {
          const double nrm = sqrt(fma(alpha, alpha, sig));
          beta = alpha >= 0.0 ? -nrm : nrm;
          tau = (beta - alpha) / beta;
          scale = 1.0 / (alpha - beta);
        }
#pragma unroll
        for (int r = 0; r < RPL; ++r) vj[lane + 32 * r] = xs[r] * scale;
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
        // all owned columns at once: KC independent dot products, interleaved warp reductions
        double p[KC];
#pragma unroll
        for (int c = 0; c < KC; ++c) {
          p[c] = 0.0;
#pragma unroll
          for (int r = 0; r < RPL; ++r) p[c] = fma(v[r], x[c][r], p[c]);
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
        const int ls = w + 16 * cs;
        const bool live = ls > j && ls < k;
        const double rjs = live ? R[pk(j, ls)] : 0.0;
        const double tws = live ? tau * (rjs + dsum) : 0.0;
        __syncwarp();
        if (live && (lane & (LPC - 1)) == 0) R[pk(j, ls)] = rjs - tws;
#pragma unroll
        for (int c = 0; c < KC; ++c) {
          const int l = w + 16 * c;
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
  double* Ro = q.Rout + (int64_t)blockIdx.x * k1 * k;
  for (int e = threadIdx.x; e < k1 * k; e += blockDim.x) {
    const int i = e % k1, l = e / k1;
    Ro[e] = i <= l ? R[pk(i, l)] : 0.0;
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

template <int KC, int RPL>
static az_status_t tsqr_launch(const QRIn& q, int nblocks, cudaStream_t st) {
  constexpr int MC = 32 * RPL;
  const size_t sm = ((size_t)q.k * (q.k + 1) / 2 + 2 * MC + 2) * sizeof(double);
  auto kern = k_tsqr<KC, RPL>;
  AZ_CUDA_CHECK(az_smem_attr(kern, sm));
  AzTrace tr(q.bstride ? "tsqr_merge" : "tsqr_leaf", st, q.m);
  kern<<<nblocks, 512, sm, st>>>(q);
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
  const int64_t P = std::max<int64_t>(1, std::min<int64_t>(num_sms(), (m + 127) / 128));
  return (size_t)(2 * P * k * k) * sizeof(double) + 256;
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
az_status_t az_qr_r_impl(double* A, int64_t m, int64_t k, int64_t lda, double* R, int64_t ldr,
                         void* ws, size_t ws_bytes, cudaStream_t st, int64_t k1) {
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
  const int64_t P = std::max<int64_t>(1, std::min<int64_t>(num_sms(), (m + 127) / 128));
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
  AZ_TRY(tsqr_pass(q, (int)P, st));
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
    AZ_TRY(tsqr_pass(t, (int)next, st));
    which ^= 1;
    cur = next;
  }
  k_copy_R<<<az_div_up(k1 * k, 256), 256, 0, st>>>(buf[which], (int)k1, (int)k, R, ldr);
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
