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

#include "az_internal.h"

AZ_D double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ int g_small_sweeps;

__global__ void __launch_bounds__(1024, 1) k_jacobi_small(const double* Rf, int64_t ldr, int r, int nrhs,
                                                          double theta, double* y, int64_t ldy, double* sig_out,
                                                          int64_t* rank_dev, int max_sweeps) {
  extern __shared__ double sm[];
  double* B = sm;                      // r x r, column i at B + i * r
  double* Cm = B + r * r;              // r x nrhs, row p, column c at Cm[p * nrhs + c] (rows contiguous)
  double* nrm2 = Cm + r * nrhs;        // r
  __shared__ int rot_count;
  __shared__ unsigned long long off_bits;   // max |g| / sqrt(a b) over the sweep (double bits)
  const double tol = 1.1102230246251565e-16 * sqrt((double)r);   // rotation threshold
  const int tid = threadIdx.x, nth = blockDim.x;
  const int w = tid >> 5, lane = tid & 31, nw = nth >> 5;
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
  __shared__ double smax2_sweep;
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
    if (tid == 0) {
      double m = 0.0;
      for (int i = 0; i < r; ++i) m = fmax(m, nrm2[i]);
      smax2_sweep = m;
      rot_count = 0;
      off_bits = 0ull;
    }
    __syncthreads();
    const double negl = (1e-3 * theta) * (1e-3 * theta) * smax2_sweep;
    for (int round = 0; round < n - 1; ++round) {
      for (int pi = w; pi < n / 2; pi += nw) {
        int p, q;
        if (pi == 0) {
          p = round;
          q = n - 1;
        } else {
          p = (round + pi) % (n - 1);
          q = (round - pi + (n - 1)) % (n - 1);
        }
        if (p > q) { const int t = p; p = q; q = t; }
        if (q >= r) continue;
        double* bp = B + (int64_t)p * r;
        double* bq = B + (int64_t)q * r;
        double a = 0.0, b = 0.0, g = 0.0;
        for (int t = lane; t < r; t += 32) {
          const double xp = bp[t], xq = bq[t];
          a = fma(xp, xp, a);
          b = fma(xq, xq, b);
          g = fma(xp, xq, g);
        }
        a = wsum(a);
        b = wsum(b);
        g = wsum(g);
        if (fmin(a, b) < negl || g == 0.0) continue;
        const double g2 = g * g, ab = a * b;
        if (lane == 0) atomicMax(&off_bits, (unsigned long long)__double_as_longlong(sqrt(g2 / ab)));
        if (!(g2 > tol * tol * ab)) continue;
        // tan of the rotation angle, t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (b - a) / 2g,
        // written without the intermediate division: t = 2 g sign(b - a) / (|b - a| + sqrt((b - a)^2 + 4 g^2))
        const double d = b - a;
        const double tt = (d >= 0.0 ? 2.0 * g : -2.0 * g) / (fabs(d) + sqrt(fma(d, d, 4.0 * g2)));
        const double cs = rsqrt(fma(tt, tt, 1.0)), sn = cs * tt;
        for (int t = lane; t < r; t += 32) {
          const double xp = bp[t], xq = bq[t];
          bp[t] = cs * xp - sn * xq;
          bq[t] = sn * xp + cs * xq;
        }
        for (int c = lane; c < nrhs; c += 32) {
          const double cp = Cm[p * nrhs + c], cq = Cm[q * nrhs + c];
          Cm[p * nrhs + c] = cs * cp - sn * cq;
          Cm[q * nrhs + c] = sn * cp + cs * cq;
        }
        if (lane == 0) atomicAdd(&rot_count, 1);
      }
      __syncthreads();
    }
    // converged: no rotation, or every measured off-diagonal at the rounding level of the dots
    if (tid == 0) g_small_sweeps = sweep + 1;
    if (rot_count == 0 || __longlong_as_double((long long)off_bits) <= 8.0 * tol) break;
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

extern "C" int az_debug_small_sweeps() {
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
                         cudaStream_t st) {
  if (!small_fits(r, nrhs))
    return az_tsvdw_impl(Rf, ldr, r, nrhs, theta, y, ldy, sigma_out, rank_out, ws, ws_bytes, st, 40, nullptr);
  const size_t sm = (size_t)(r * r + r * nrhs + r) * sizeof(double);
  if (ws_bytes < az_tsvd_ws_bytes(r, nrhs)) {
    az_set_error("az_tsvd_solve: workspace too small");
    return AZ_ERR_WORKSPACE;
  }
  int64_t* d_rank = (int64_t*)ws;
  AZ_CUDA_CHECK(az_smem_attr(k_jacobi_small, sm));
  const int nth = std::min<int64_t>(1024, std::max<int64_t>(64, 32 * ((r + 1) / 2)));
  AzTrace tr("jacobi_svd", st);
  k_jacobi_small<<<1, nth, sm, st>>>(Rf, ldr, (int)r, (int)nrhs, theta, y, ldy, sigma_out, d_rank, 60);
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
