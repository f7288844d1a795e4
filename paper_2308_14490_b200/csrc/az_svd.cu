// Truncated least squares on the QR-reduced sketch ("followed by the SVD of an
// (r+p)-by-M matrix"; "threshold-truncated SVD ... solve min ||S y - rhs||").
//
// With Rf = [R_S | c] from the TSQR of [S | b'], R_S = U Sigma V^T and
//   y = V_k Sigma_k^-1 U_k^T c,   k = #{ sigma_i > theta sigma_1 }.
// We run one-sided (Hestenes) Jacobi on B = R_S^T: B W -> columns mutually orthogonal, so
// R_S^T = U' Sigma W^T, R_S = W Sigma U'^T: the rotations W are the LEFT singular vectors of
// R_S and are applied to the rows of c on the fly (c <- W^T c), and the right singular vectors
// are the normalised columns of B W.  Then y = sum_{kept i} (B W)_i (W^T c)_i / sigma_i^2.
// One-sided Jacobi is accurate to high relative precision in the small singular values, which
// is what the threshold decision needs.  Parallel (round-robin) ordering: r/2 disjoint pairs
// per round, one warp per pair.
#include <algorithm>

#include <cstdlib>

#include "az_internal.h"

AZ_D double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ int g_small_sweeps;

// three sums over the 16 lanes of a half warp, the levels interleaved (written out: left to the
// compiler the three reductions ran one after another, a chain of 12 dependent shuffles)
AZ_D void hsum3(double& a, double& b, double& g) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    const double ta = __shfl_xor_sync(0xffffffffu, a, o);
    const double tb = __shfl_xor_sync(0xffffffffu, b, o);
    const double tg = __shfl_xor_sync(0xffffffffu, g, o);
    a += ta;
    b += tb;
    g += tg;
  }
}

// One CTA, r <= 16 EPL.  A pair (p, q) of columns of B = R_S^T is handled by a HALF warp, each lane
// holding EPL entries of both columns in registers for the round: the round is issue-bound on the
// one SM, so the instruction count per pair is what matters (no modulo arithmetic, unrolled
// element loops, 4-level reductions, no shared atomics).
template <int EPL>
__global__ void __launch_bounds__(EPL <= 4 ? 512 : 1024, 1) k_jacobi_small(const double* Rf, int64_t ldr, int r, int nrhs,
                                                          double theta, double* y, int64_t ldy, double* sig_out,
                                                          int64_t* rank_dev, int max_sweeps) {
  extern __shared__ double sm[];
  double* B = sm;                      // r x r, column i at B + i * r
  double* Cm = B + r * r;              // r x nrhs, row p, column c at Cm[p * nrhs + c] (rows contiguous)
  double* nrm2 = Cm + r * nrhs;        // r
  // per-half-warp sweep statistics, reduced once per sweep
  __shared__ int rot_h[64];
  __shared__ int big_h[64];
  __shared__ double smax2_sweep;
  __shared__ unsigned char quiet[AZ_NARROW_MAX];   // column in the sweep's negligible set S
  const double tol = 1.1102230246251565e-16 * sqrt((double)r);   // rotation threshold
  const int tid = threadIdx.x, nth = blockDim.x;
  const int w = tid >> 5, lane = tid & 31, nw = nth >> 5;
  const int hw = tid >> 4, hl = tid & 15, nh = nth >> 4;   // half warps
  for (int e = tid; e < r * r; e += nth) {
    const int i = e / r, t = e % r;    // B[t][i] = R_S[i][t]
    B[e] = Rf[(int64_t)t * ldr + i];
  }
  for (int e = tid; e < r * nrhs; e += nth) {
    const int c = e / r, p = e % r;
    Cm[p * nrhs + c] = Rf[(int64_t)(r + c) * ldr + p];
  }
  __syncthreads();
  const int n = r + (r & 1);           // padded to even
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    // column norms at the start of the sweep: pairs whose smaller column is far below the
    // truncation level (1e-3 theta sigma_1) cannot change the kept part and are skipped
    for (int i = w; i < r; i += nw) {
      double a = 0.0;
      for (int t = lane; t < r; t += 32) a = fma(B[i * r + t], B[i * r + t], a);
      a = wsum(a);
      if (lane == 0) nrm2[i] = a;
    }
    __syncthreads();
    // S = the columns with norm^2 below nu = theta^2 smax^2 / 4.  When their total is below nu as
    // well, every singular value of S's span is below theta sigma_1 / 2 (||X_S||_2 <= ||X_S||_F), so
    // pairs inside S are neither rotated nor counted for convergence this sweep: the rotations against
    // the other columns still make those orthogonal to S, and by Weyl the kept singular values and
    // vectors are those of the other columns alone (reading R34).  The columns of S are not
    // diagonalised among themselves (their reported values are column norms below theta sigma_1 / 2).
    if (w == 0) {
      double m = 0.0;
      for (int i = lane; i < r; i += 32) m = fmax(m, nrm2[i]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      const double nu = 0.25 * theta * theta * m;
      double tail = 0.0;
      for (int i = lane; i < r; i += 32) tail += nrm2[i] < nu ? nrm2[i] : 0.0;
      tail = wsum(tail);
      for (int i = lane; i < r; i += 32) quiet[i] = tail < nu && nrm2[i] < nu;
      if (lane == 0) smax2_sweep = m;
    }
    __syncthreads();
    const double negl = (1e-3 * theta) * (1e-3 * theta) * smax2_sweep;
    int big_me = 0;   // pairs whose cosine exceeds the convergence level 8 tol
    int rot_me = 0;
    for (int round = 0; round < n - 1; ++round) {
      // both halves of a warp run the same trip count (the shuffles span the whole warp)
      for (int base = hw & ~1; base < n / 2; base += nh) {
        const int pi = base + (hw & 1);
        int p = 0, q = r;   // a missing pair (pi >= n / 2) falls through with q = r, i.e. !pair_ok
        if (pi >= n / 2) {
        } else if (pi == 0) {
          p = round;
          q = n - 1;
        } else {
          p = round + pi;
          if (p >= n - 1) p -= n - 1;
          q = round - pi;
          if (q < 0) q += n - 1;
        }
        if (p > q) { const int t = p; p = q; q = t; }
        const bool pair_ok = q < r;
        double* bp = B + (int64_t)p * r;
        double* bq = B + (int64_t)q * r;
        double xp[EPL], xq[EPL];
        double a = 0.0, b = 0.0, g = 0.0;
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          const int t = hl + 16 * e;
          const bool in = pair_ok && t < r;
          xp[e] = in ? bp[t] : 0.0;
          xq[e] = in ? bq[t] : 0.0;
          a = fma(xp[e], xp[e], a);
          b = fma(xq[e], xq[e], b);
          g = fma(xp[e], xq[e], g);
        }
        const bool qq = pair_ok && (quiet[p] & quiet[q]);
        hsum3(a, b, g);
        if (!pair_ok || fmin(a, b) < negl || g == 0.0 || qq) continue;
        const double g2 = g * g, ab = a * b;
        big_me += g2 > (64.0 * tol * tol) * ab;
        if (!(g2 > tol * tol * ab)) continue;
        // tan of the rotation angle, t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (b - a) / 2g,
        // written without the intermediate division: t = 2 g sign(b - a) / (|b - a| + sqrt((b - a)^2 + 4 g^2))
        const double d = b - a;
        // (MUFU-seeded reciprocal / rsqrt with Newton steps: the IEEE division and square root are
        // several times the instructions, and the round is issue-bound)
        const double h = fma(d, d, 4.0 * g2);
        const double tt = (d >= 0.0 ? 2.0 * g : -2.0 * g) * fast_rcp(fabs(d) + h * fast_rsqrt(h));
        const double cs = fast_rsqrt(fma(tt, tt, 1.0)), sn = cs * tt;
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          const int t = hl + 16 * e;
          if (t < r) {
            bp[t] = cs * xp[e] - sn * xq[e];
            bq[t] = sn * xp[e] + cs * xq[e];
          }
        }
        for (int c = hl; c < nrhs; c += 16) {
          const double cp = Cm[p * nrhs + c], cq = Cm[q * nrhs + c];
          Cm[p * nrhs + c] = cs * cp - sn * cq;
          Cm[q * nrhs + c] = sn * cp + cs * cq;
        }
        ++rot_me;
      }
      __syncthreads();
    }
    if (hl == 0) {
      rot_h[hw] = rot_me;
      big_h[hw] = big_me;
    }
    __syncthreads();
    int rots = 0, bigs = 0;
    for (int i = 0; i < nh; ++i) {
      rots += rot_h[i];
      bigs += big_h[i];
    }
    // converged: no rotation, or every measured off-diagonal cosine at the rounding level of the dots
    if (tid == 0) g_small_sweeps = sweep + 1;
    if (rots == 0 || bigs == 0) break;
    __syncthreads();
  }
  // singular values = column norms of B W
  for (int i = w; i < r; i += nw) {
    double a = 0.0;
    for (int t = lane; t < r; t += 32) a = fma(B[i * r + t], B[i * r + t], a);
    a = wsum(a);
    if (lane == 0) nrm2[i] = a;
  }
  __syncthreads();
  double smax2 = 0.0;
  for (int i = 0; i < r; ++i) smax2 = fmax(smax2, nrm2[i]);
  const double thr2 = theta * theta * smax2;
  // y[t][c] = sum_{kept i} B[t][i] C[i][c] / sigma_i^2
  for (int e = tid; e < r * nrhs; e += nth) {
    const int c = e / r, t = e % r;
    double acc = 0.0;
    for (int i = 0; i < r; ++i) {
      const double s2 = nrm2[i];
      if (s2 > thr2 && s2 > 0.0) acc = fma(B[i * r + t], Cm[i * nrhs + c] / s2, acc);
    }
    y[(int64_t)c * ldy + t] = acc;
  }
  // sorted singular values (rank by counting) and the kept count
  for (int i = tid; i < r; i += nth) {
    int pos = 0;
    for (int t = 0; t < r; ++t)
      if (nrm2[t] > nrm2[i] || (nrm2[t] == nrm2[i] && t < i)) ++pos;
    if (sig_out) sig_out[pos] = sqrt(nrm2[i]);
  }
  if (tid == 0) {
    int64_t kk = 0;
    for (int i = 0; i < r; ++i) kk += (nrm2[i] > thr2 && nrm2[i] > 0.0);
    *rank_dev = kk;
  }
}

int az_small_sweeps_last() {
  int v = -1;
  cudaMemcpyFromSymbol(&v, g_small_sweeps, sizeof(int));
  return v;
}

// the single-CTA kernel holds R_S^T and c in shared memory; larger problems go to block Jacobi
static bool small_fits(int64_t r, int64_t nrhs) {
  return r <= AZ_NARROW_MAX && (size_t)(r * r + r * nrhs + r) * sizeof(double) <= 220 * 1024;
}

size_t az_tsvd_ws_bytes(int64_t r, int64_t nrhs) {
  return small_fits(r, nrhs) ? 256 : az_tsvdw_ws_bytes(r, nrhs);
}

az_status_t az_tsvd_impl(const double* Rf, int64_t ldr, int64_t r, int64_t nrhs, double theta, double* y,
                         int64_t ldy, double* sigma_out, int64_t* rank_out, void* ws, size_t ws_bytes,
                         cudaStream_t st, const int64_t** rank_dev) {
  if (!small_fits(r, nrhs))
    return az_tsvdw_impl(Rf, ldr, r, nrhs, theta, y, ldy, sigma_out, rank_out, ws, ws_bytes, st, 40, nullptr,
                         rank_dev);
  size_t sm = (size_t)(r * r + r * nrhs + r) * sizeof(double);
  // the CTA takes an SM to itself (shared memory no other kernel's CTA fits beside): the round is
  // issue-bound, and in az_solve the side stream's column passes run meanwhile
  static const int excl = getenv("AZ_JAC_EXCL") ? atoi(getenv("AZ_JAC_EXCL")) : 1;
  if (excl) sm = std::max<size_t>(sm, 160 * 1024);
  if (ws_bytes < az_tsvd_ws_bytes(r, nrhs)) {
    az_set_error("az_tsvd_solve: workspace too small");
    return AZ_ERR_WORKSPACE;
  }
  int64_t* d_rank = (int64_t*)ws;
  if (rank_dev) *rank_dev = d_rank;
  // one half warp per pair: n / 2 pairs -> 16 (n / 2) threads, whole warps, at most 1024
  const int nth = (int)std::min<int64_t>(1024, std::max<int64_t>(64, 32 * ((r + 3) / 4)));
  AzTrace tr("jacobi_svd", st);
#define AZ_JS(E)                                                                                       \
  {                                                                                                    \
    AZ_CUDA_CHECK(az_smem_attr(k_jacobi_small<E>, sm));                                                \
    k_jacobi_small<E><<<1, nth, sm, st>>>(Rf, ldr, (int)r, (int)nrhs, theta, y, ldy, sigma_out, d_rank, 60); \
  }
  if (r <= 32)
    AZ_JS(2)
  else if (r <= 64)
    AZ_JS(4)
  else
    AZ_JS(8)
#undef AZ_JS
  AZ_LAUNCH_CHECK();
  if (rank_out) {
    AZ_CUDA_CHECK(cudaMemcpyAsync(rank_out, d_rank, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    AZ_CUDA_CHECK(cudaStreamSynchronize(st));
  }
  return AZ_OK;
}

extern "C" az_status_t az_tsvd_workspace_size(int64_t r, int64_t nrhs, size_t* bytes) {
  if (!bytes) return AZ_ERR_INVALID_ARGUMENT;
  *bytes = az_tsvd_ws_bytes(r, nrhs);
  return AZ_OK;
}

extern "C" az_status_t az_tsvd_solve(const double* Rf, int64_t ldr, int64_t r, int64_t nrhs, double theta,
                                     double* y, int64_t ldy, double* sigma_out, int64_t* rank_out, void* ws,
                                     size_t ws_bytes, void* stream) {
  if (!Rf || !y || r < 1 || nrhs < 0 || ldr < r || ldy < r || !(theta >= 0) || !ws) {
    az_set_error("az_tsvd_solve: bad arguments");
    return AZ_ERR_INVALID_ARGUMENT;
  }
  return az_tsvd_impl(Rf, ldr, r, nrhs, theta, y, ldy, sigma_out, rank_out, ws, ws_bytes, (cudaStream_t)stream);
}
