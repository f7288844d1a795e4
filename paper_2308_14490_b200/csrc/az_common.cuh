// Common device helpers for libaz (sm_100a, FP64 / complex128).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/az.h"

#define AZ_HD __host__ __device__ __forceinline__
#define AZ_D __device__ __forceinline__

typedef double2 cplx;

AZ_HD cplx cadd(cplx a, cplx b) { return make_double2(a.x + b.x, a.y + b.y); }
AZ_HD cplx csub(cplx a, cplx b) { return make_double2(a.x - b.x, a.y - b.y); }
AZ_HD cplx cmul(cplx a, cplx b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
AZ_HD cplx cmulc(cplx a, cplx b) {   // a * conj(b)
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
AZ_HD cplx cconj(cplx a) { return make_double2(a.x, -a.y); }
AZ_HD cplx cscale(cplx a, double s) { return make_double2(a.x * s, a.y * s); }
AZ_HD cplx czero() { return make_double2(0.0, 0.0); }

// Shared-memory padding: one 16-byte pad every 8 complex elements makes the Stockham
// stride-8 writes bank-conflict free (8 lanes x 16 B cover all 32 banks).
AZ_HD constexpr int spad(int i) { return i + (i >> 3); }
AZ_HD constexpr int spad_len(int L) { return L + (L >> 3) + 1; }   // +1 staggers consecutive FFT buffers

// 1 / d to within an ulp or so: the MUFU reciprocal seed refined by two Newton steps, for
// latency- or issue-bound chains (the Householder reflector chain of the TSQR, the Jacobi rotation):
// no IEEE division slow-path check.  d must be a nonzero normal number (callers guarantee it)
AZ_D double fast_rcp(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

// 1 / sqrt(x) likewise: MUFU seed, two Newton steps y (3 - x y^2) / 2 (x a positive normal number)
AZ_D double fast_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  double t = fma(-hx * y, y, 0.5);
  y = fma(y, t, y);
  t = fma(-hx * y, y, 0.5);
  return fma(y, t, y);
}

// --------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. SC'11) and the probe generator.
// Independent of oracle/philox.py by construction (task rules); same specification.
// --------------------------------------------------------------------------------------
AZ_D void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c[0];
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]);
    const uint32_t lo1 = 0xCD9E8D57u * c[2];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]);
    const uint32_t n0 = hi1 ^ c[1] ^ k0;
    const uint32_t n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// Two standard normals Omega[2m, j], Omega[2m+1, j] for row pair m and global column j.
AZ_D double2 probe_pair(uint64_t m, uint64_t j, uint64_t seed) {
  uint32_t c[4] = {(uint32_t)m, (uint32_t)(m >> 32), (uint32_t)j, (uint32_t)(j >> 32)};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  const uint64_t a = ((((uint64_t)c[1]) << 32) | c[0]) >> 11;
  const uint64_t b = ((((uint64_t)c[3]) << 32) | c[2]) >> 11;
  const double u1 = (double)(a + 1) * 0x1.0p-53;   // (0, 1]
  const double u2 = (double)b * 0x1.0p-53;         // [0, 1)
  const double r = sqrt(-2.0 * log(u1));
  double sn, cs;
  sincospi(2.0 * u2, &sn, &cs);
  return make_double2(r * cs, r * sn);
}

// Spectral probes of the 1-D four-step layout (reading R35): the column pair
// (Omega[:, 2P], Omega[:, 2P+1]) is Re / Im of u_P = IFFT_n(v_P), where the unnormalised spectrum is
// v_P[k] = sqrt(n) (z0 + i z1), (z0, z1) = probe_pair(k, P + 2^63).  A complex vector of i.i.d.
// circular N(0,1) + i N(0,1) entries has exactly this spectrum (the DFT is sqrt(n) x unitary), so the
// two columns are i.i.d. N(0,1) like every other probe; the sketch then starts from v_P directly.
AZ_D cplx spectral_probe(uint64_t k, uint64_t P, uint64_t seed, double sqn) {
  const double2 z = probe_pair(k, P | (uint64_t(1) << 63), seed);
  return make_double2(sqn * z.x, sqn * z.y);
}

// Complex value of probe pair p (columns col0 + 2p, col0 + 2p + 1) at an even/odd row pair:
// returns z[2m] (in .first) and z[2m+1] for the complex packing z = Omega[:, 2p] + i Omega[:, 2p+1].
struct cpair { cplx a, b; };
AZ_D cpair probe_cplx_pair(uint64_t m, uint64_t col_re, uint64_t col_im, bool has_im, uint64_t seed) {
  const double2 re = probe_pair(m, col_re, seed);
  double2 im = make_double2(0.0, 0.0);
  if (has_im) im = probe_pair(m, col_im, seed);
  cpair r;
  r.a = make_double2(re.x, im.x);
  r.b = make_double2(re.y, im.y);
  return r;
}

// --------------------------------------------------------------------------------------
// Periodised Gaussian (PAPER.md:54 Eq. rbf, :59 Eq. periodic_rbf) and its second derivative
// (PAPER.md:702).  Sums every translate that does not underflow in binary64.
// --------------------------------------------------------------------------------------
AZ_HD double az_phi_per(double x, double eps, double T, int order) {
  const double P = 2.0 * T;
  const double x0 = x - rint(x / P) * P;
  const int mm = 1 + (int)ceil(27.294688127912362 / (P * eps));   // sqrt(745) / (2 T eps)
  const double e2 = eps * eps;
  double acc = 0.0;
  for (int d = -mm; d <= mm; ++d) {
    const double r = x0 - d * P;
    double t = exp(-e2 * r * r);
    if (order == 1) t *= -2.0 * e2 * r;
    if (order == 2) t *= -2.0 * e2 * (1.0 - 2.0 * e2 * r * r);
    acc += t;
  }
  return acc;
}

// --------------------------------------------------------------------------------------
// launch accounting + error plumbing (host side)
// --------------------------------------------------------------------------------------
void az_count_launch();
void az_set_error(const char* fmt, ...);

#define AZ_CUDA_CHECK(expr)                                                    \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      az_set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return AZ_ERR_CUDA;                                                      \
    }                                                                          \
  } while (0)

#define AZ_LAUNCH_CHECK()                                                      \
  do {                                                                         \
    az_count_launch();                                                         \
    cudaError_t _e = cudaGetLastError();                                       \
    if (_e != cudaSuccess) {                                                   \
      az_set_error("%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
      return AZ_ERR_CUDA;                                                      \
    }                                                                          \
  } while (0)

// Opt a kernel into > 48 KB of dynamic shared memory (idempotent).  The attribute call is made once
// per (kernel, size): it is a driver round trip, and the small solves (c1) are host-latency bound.
template <class K>
inline cudaError_t az_smem_attr(K kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  static thread_local const void* last_k[64];
  static thread_local size_t last_b[64];
  const size_t h = (((size_t)(const void*)kernel) >> 4) & 63;
  if (last_k[h] == (const void*)kernel && last_b[h] >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) {
    last_k[h] = (const void*)kernel;
    last_b[h] = bytes;
  }
  return e;
}

#define AZ_TRY(...)                                                            \
  do {                                                                         \
    az_status_t _s = (__VA_ARGS__);                                            \
    if (_s != AZ_OK) return _s;                                                \
  } while (0)

// --------------------------------------------------------------------------------------
// Bulk asynchronous copies (the TMA engine's 1-D form, cp.async.bulk -> SASS UBLKCP) into shared
// memory, completion tracked by an mbarrier's transaction count.  Addresses and sizes must be
// multiples of 16 bytes.
// --------------------------------------------------------------------------------------
namespace bulk {
AZ_D uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
AZ_D void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count));
}
// make the initialised barriers visible to the async proxy (the copy engine)
AZ_D void fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::); }
// order this thread's earlier generic-proxy shared-memory accesses before later async-proxy writes
AZ_D void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::); }
AZ_D void arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
AZ_D void copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
AZ_D void wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
  } while (!done);
}
}  // namespace bulk
