// libaz: plan creation (step 0 of PAPER.md Sec. 3.2.3), C ABI entry points and dispatch.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <vector>

#include "az_fft.cuh"
#include "az_internal.h"

// ---------------------------------------------------------------------------------------
// error / instrumentation plumbing
// ---------------------------------------------------------------------------------------
static thread_local char g_err[1024] = "";
static std::atomic<int64_t> g_launches{0};

void az_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
void az_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

extern "C" const char* az_last_error(void) { return g_err; }

// ---- tracing ----
#include <map>
#include <mutex>
#include <string>
namespace {
struct TraceRec {
  std::string name;
  cudaEvent_t e0, e1;
  int64_t units;
};
std::mutex g_tr_mu;
bool g_tr_on = false;
std::vector<TraceRec> g_tr;
size_t g_tr_used = 0;
}  // namespace

bool az_trace_active() { return g_tr_on; }

AzTrace::AzTrace(const char* name, cudaStream_t s, int64_t units) : slot(-1), st(s) {
  if (!g_tr_on) return;
  std::lock_guard<std::mutex> lk(g_tr_mu);
  if (g_tr_used == g_tr.size()) {
    TraceRec r;
    cudaEventCreate(&r.e0);
    cudaEventCreate(&r.e1);
    g_tr.push_back(r);
  }
  slot = (int)g_tr_used++;
  g_tr[slot].name = name;
  g_tr[slot].units = units;
  cudaEventRecord(g_tr[slot].e0, st);
}
AzTrace::~AzTrace() {
  if (slot >= 0) cudaEventRecord(g_tr[slot].e1, st);
}

extern "C" int az_trace_enable(int on) {
  std::lock_guard<std::mutex> lk(g_tr_mu);
  g_tr_on = on != 0;
  g_tr_used = 0;
  return 0;
}

extern "C" int az_trace_report(char* buf, int len) {
  std::lock_guard<std::mutex> lk(g_tr_mu);
  struct Agg {
    int64_t count = 0, units = 0;
    double ms = 0.0;
  };
  std::map<std::string, Agg> agg;
  // diagnostics: per-launch start / end (printed by the filling call only, not by the size query)
  const bool timeline = buf && getenv("AZ_TRACE_TIMELINE") != nullptr;
  for (size_t i = 0; i < g_tr_used; ++i) {
    cudaEventSynchronize(g_tr[i].e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, g_tr[i].e0, g_tr[i].e1);
    if (timeline) {
      float t0 = 0.f;
      cudaEventElapsedTime(&t0, g_tr[0].e0, g_tr[i].e0);
      fprintf(stderr, "timeline %-24s %9.3f %9.3f\n", g_tr[i].name.c_str(), t0, t0 + ms);
    }
    auto& a = agg[g_tr[i].name];
    a.count += 1;
    a.ms += ms;
    a.units += g_tr[i].units;
  }
  std::string out;
  char line[256];
  for (auto& kv : agg) {
    snprintf(line, sizeof(line), "%s %lld %.6f %lld\n", kv.first.c_str(), (long long)kv.second.count, kv.second.ms,
             (long long)kv.second.units);
    out += line;
  }
  if (buf && len > 0) {
    const size_t n = std::min<size_t>(out.size(), (size_t)len - 1);
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return (int)out.size();
}
int az_small_sweeps_last();
int az_bjac_sweeps_last();
extern "C" int az_svd_sweeps_last(int which) {
  return which == 0 ? az_small_sweeps_last() : az_bjac_sweeps_last();
}
extern "C" int64_t az_launch_count(int reset) {
  return reset ? g_launches.exchange(0) : g_launches.load();
}
extern "C" const char* az_status_string(az_status_t s) {
  switch (s) {
    case AZ_OK: return "AZ_OK";
    case AZ_ERR_INVALID_ARGUMENT: return "AZ_ERR_INVALID_ARGUMENT";
    case AZ_ERR_OVERSAMPLING: return "AZ_ERR_OVERSAMPLING";
    case AZ_ERR_SINGULAR_SYMBOL: return "AZ_ERR_SINGULAR_SYMBOL";
    case AZ_ERR_OUT_OF_MEMORY: return "AZ_ERR_OUT_OF_MEMORY";
    case AZ_ERR_CUDA: return "AZ_ERR_CUDA";
    case AZ_ERR_NOT_SUPPORTED: return "AZ_ERR_NOT_SUPPORTED";
    case AZ_ERR_WORKSPACE: return "AZ_ERR_WORKSPACE";
    case AZ_ERR_NCCL: return "AZ_ERR_NCCL";
    case AZ_WARN_SKETCH_SATURATED: return "AZ_WARN_SKETCH_SATURATED";
  }
  return "AZ_UNKNOWN";
}

#define AZ_ARG(cond, ...)                 \
  do {                                    \
    if (!(cond)) {                        \
      az_set_error(__VA_ARGS__);          \
      return AZ_ERR_INVALID_ARGUMENT;     \
    }                                     \
  } while (0)

// ---------------------------------------------------------------------------------------
// generic batched in-place FFT of contiguous vectors (symbol tables)
// ---------------------------------------------------------------------------------------
template <int L, int DIR>
__global__ void k_fft_rows(cplx* data, int64_t count, const cplx* __restrict__ tw) {
  extern __shared__ cplx sm[];
  constexpr int TPF = L / 8;
  const int nf = blockDim.x / TPF;
  const int f = threadIdx.x / TPF, j = threadIdx.x % TPF;
  const int64_t row = (int64_t)blockIdx.x * nf + f;
  cplx* buf = sm + f * spad_len(L);
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int i = j + t * TPF;
    buf[spad(i)] = row < count ? data[row * L + i] : czero();
  }
  __syncthreads();
  fft_smem<L, DIR>(buf, j, tw, TWN);
  if (row < count) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int i = j + t * TPF;
      data[row * L + i] = buf[spad(i)];
    }
  }
}

template <int L>
static az_status_t fft_rows_launch(const cplx* tw, cplx* data, int64_t count, int dir, cudaStream_t st) {
  constexpr int TPF = L / 8;
  const int nf = TPF >= 256 ? 1 : 256 / TPF;
  const size_t sm = (size_t)nf * spad_len(L) * sizeof(cplx);
  if (dir < 0)
    k_fft_rows<L, -1><<<az_div_up(count, nf), nf * TPF, sm, st>>>(data, count, tw);
  else
    k_fft_rows<L, 1><<<az_div_up(count, nf), nf * TPF, sm, st>>>(data, count, tw);
  AZ_LAUNCH_CHECK();
  return AZ_OK;
}

az_status_t az_fft_batch(const cplx* tw, cplx* data, int64_t len, int64_t count, int dir, cudaStream_t st) {
  switch (len) {
    case 8: return fft_rows_launch<8>(tw, data, count, dir, st);
    case 16: return fft_rows_launch<16>(tw, data, count, dir, st);
    case 32: return fft_rows_launch<32>(tw, data, count, dir, st);
    case 64: return fft_rows_launch<64>(tw, data, count, dir, st);
    case 128: return fft_rows_launch<128>(tw, data, count, dir, st);
    case 256: return fft_rows_launch<256>(tw, data, count, dir, st);
    case 512: return fft_rows_launch<512>(tw, data, count, dir, st);
    case 1024: return fft_rows_launch<1024>(tw, data, count, dir, st);
    case 2048: return fft_rows_launch<2048>(tw, data, count, dir, st);
  }
  az_set_error("az_fft_batch: unsupported length %lld", (long long)len);
  return AZ_ERR_NOT_SUPPORTED;
}

// ---------------------------------------------------------------------------------------
// step-0 kernels: twiddles, kernel samples, sigma^2, thresholded pseudo-inverse weights
// ---------------------------------------------------------------------------------------
__global__ void k_twiddles(cplx* tw, int twn, cplx* hi, cplx* lo, int64_t Lbig, int nhi, int nlo) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double s, c;
  if (i < twn) {
    sincospi(-2.0 * (double)i / (double)twn, &s, &c);
    tw[i] = make_double2(c, s);
  }
  if (hi && i < nhi) {   // e^{-2 pi i (h 2^TW4B) / Lbig}
    const int64_t t = (i << TW4B) % Lbig;
    sincospi(-2.0 * (double)t / (double)Lbig, &s, &c);
    hi[i] = make_double2(c, s);
  }
  if (lo && i < nlo) {
    sincospi(-2.0 * (double)i / (double)Lbig, &s, &c);
    lo[i] = make_double2(c, s);
  }
}

// Lemma 3 on the fine grid: w[q] = phi^per(q h_L) (order 0 or 2), q in [0, L).
// real part of the row symbol (the imaginary part of the DFT of the real even kernel samples is
// rounding noise)
__global__ void k_real_sym(double* Wr, const cplx* W0, const cplx* W2, int lap, double alpha, double k0sq, int64_t L) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < L) Wr[i] = lap ? alpha * fma(k0sq, W0[i].x, W2[i].x) : W0[i].x;
}

__global__ void k_samples(cplx* out, int64_t L, double hL, double eps, double T, int order) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < L) out[q] = make_double2(az_phi_per((double)q * hL, eps, T, order), 0.0);
}

// Boundary stencils (CS1 step 6): for boundary point b and axis d, the window of centres
// j = j0 .. j0 + win - 1 (mod n) around x_b and the weights phi^per(x_b - c_j).
__global__ void k_stencil(const double* bxy, int64_t Mb, int dim, int d, int n, double T, double h, double eps,
                          int win, double* bw, int32_t* bj) {
  const int b = blockIdx.x, t = threadIdx.x;
  if (b >= Mb) return;
  const double x = bxy[dim * b + d];
  const int half = (win - 1) / 2;
  const int j0 = (int)rint((x + T) / h) - half;
  if (t == 0) bj[2 * b + d] = j0;
  if (t < 64) {
    double w = 0.0;
    if (t < win) {
      const int j = ((j0 + t) % n + n) % n;
      w = az_phi_per(x - (-T + j * h), eps, T, 0);
    }
    bw[(2 * b + d) * 64 + t] = w;
  }
}

// 2-D boundary rows in Robin form beta (a phi_j + b n . grad phi_j)(x_b) (PAPER.md:736-737 Dirichlet,
// 839-846 Neumann): per point the x window [jx0, jx0 + win) and y window [jy0, jy0 + win_y) and four
// separable weight vectors, row value = sum_t sum_l w[jx][jy] (P[t] Y0[l] + Q[t] Y1[l]) with
//   P = a phi(x - c_x) + b n_x phi'(x - c_x),  Y0 = phi(y - c_y),  Q = phi(x - c_x),  Y1 = b n_y phi'(y - c_y).
__global__ void k_stencil2(const double* bxy, const double* coef, int64_t Mb, int nx, int ny, double Tx, double Ty,
                           double eps, int winx, int winy, double* bw, int32_t* bj) {
  const int b = blockIdx.x, t = threadIdx.x;
  if (b >= Mb) return;
  const double x = bxy[2 * b], y = bxy[2 * b + 1];
  const double ca = coef ? coef[4 * b] : 1.0, cb = coef ? coef[4 * b + 1] : 0.0;
  const double nxv = coef ? coef[4 * b + 2] : 0.0, nyv = coef ? coef[4 * b + 3] : 0.0;
  const double hx = 2.0 * Tx / nx, hy = 2.0 * Ty / ny;
  const int jx0 = (int)rint((x + Tx) / hx) - (winx - 1) / 2;
  const int jy0 = (int)rint((y + Ty) / hy) - (winy - 1) / 2;
  if (t == 0) {
    bj[2 * b] = jx0;
    bj[2 * b + 1] = jy0;
  }
  if (t < 64) {
    double P = 0.0, Q = 0.0, Y0 = 0.0, Y1 = 0.0;
    if (t < winx) {
      const int j = ((jx0 + t) % nx + nx) % nx;
      const double r = x - (-Tx + j * hx);
      const double f0 = az_phi_per(r, eps, Tx, 0);
      Q = f0;
      P = ca * f0 + (cb != 0.0 ? cb * nxv * az_phi_per(r, eps, Tx, 1) : 0.0);
    }
    if (t < winy) {
      const int j = ((jy0 + t) % ny + ny) % ny;
      const double r = y - (-Ty + j * hy);
      Y0 = az_phi_per(r, eps, Ty, 0);
      Y1 = cb != 0.0 ? cb * nyv * az_phi_per(r, eps, Ty, 1) : 0.0;
    }
    bw[(4 * b + 0) * 64 + t] = P;
    bw[(4 * b + 1) * 64 + t] = Y0;
    bw[(4 * b + 2) * 64 + t] = Q;
    bw[(4 * b + 3) * 64 + t] = Y1;
  }
}

struct SymArgs {
  const cplx* W0;
  const cplx* W2;
  int lap;
  double alpha;
  double k0sq;
  const cplx* W0y;   // 2-D: the y axis' tables
  const cplx* W2y;
};

// row symbols: VALUE rows W0; LAPLACIAN rows alpha (W2 + k0^2 W0) in 1-D and
// alpha (W2x W0y + W0x W2y + k0^2 W0x W0y) in 2-D
AZ_D cplx sym_1d(const SymArgs& a, int64_t kf) {
  return a.lap ? cscale(cadd(a.W2[kf], cscale(a.W0[kf], a.k0sq)), a.alpha) : a.W0[kf];
}
AZ_D cplx sym_2d(const SymArgs& a, int64_t kx, int64_t ky) {
  if (!a.lap) return cmul(a.W0[kx], a.W0y[ky]);
  const cplx w00 = cmul(a.W0[kx], a.W0y[ky]);
  return cscale(cadd(cadd(cmul(a.W2[kx], a.W0y[ky]), cmul(a.W0[kx], a.W2y[ky])), cscale(w00, a.k0sq)), a.alpha);
}

AZ_D void atomic_max_pos(double* addr, double v) {   // v >= 0
  atomicMax((unsigned long long*)addr, (unsigned long long)__double_as_longlong(v));
}
AZ_D void atomic_min_pos(double* addr, double v) {
  atomicMin((unsigned long long*)addr, (unsigned long long)__double_as_longlong(v));
}

// sigma^2(k) = sum over the s^d aliases of |W(k + m n)|^2 (diag of B*B)
__global__ void k_sigma2(double* sig2, double* smax, SymArgs a, int layout, int64_t n, int64_t s,
                         int64_t N1, int64_t N2, int64_t L2, int64_t ny) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  int64_t N = layout == AZ_LAYOUT_2D ? n * ny : n;
  if (k < N) {
    if (layout == AZ_LAYOUT_1D_SMALL) {
      for (int64_t m = 0; m < s; ++m) {
        const cplx w = sym_1d(a, k + m * n);
        acc += w.x * w.x + w.y * w.y;
      }
    } else if (layout == AZ_LAYOUT_1D_FOURSTEP) {
      const int64_t k1 = k / N2, k2 = k % N2;
      for (int64_t m = 0; m < s; ++m) {
        const cplx w = sym_1d(a, k1 * L2 + k2 + m * N2);
        acc += w.x * w.x + w.y * w.y;
      }
    } else {
      const int64_t kx = k / ny, ky = k % ny;
      for (int64_t mx = 0; mx < s; ++mx)
        for (int64_t my = 0; my < s; ++my) {
          const cplx w = sym_2d(a, kx + mx * n, ky + my * ny);
          acc += w.x * w.x + w.y * w.y;
        }
    }
    sig2[k] = acc;
  }
  // block max
  __shared__ double red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) atomic_max_pos(smax, red[0]);
}

// Thresholded pseudo-inverse weight (PAPER.md:190-209 + the eigenvalue threshold):
// zinv(k) = 1/sigma^2(k) if sigma(k) > rcond * sigma_max else 0.
__global__ void k_zinv(double* zinv, const double* sig2, int64_t N, const double* smax, double rcond,
                       unsigned long long* ndrop, double* smin) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  const double thr = rcond * rcond * (*smax);
  const double v = sig2[k];
  if (v > thr && v > 0.0) {
    zinv[k] = 1.0 / v;
    atomic_min_pos(smin, v);
  } else {
    zinv[k] = 0.0;
    atomicAdd(ndrop, 1ull);
  }
}

// ---------------------------------------------------------------------------------------
// plan create / destroy / query
// ---------------------------------------------------------------------------------------
static bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
static int ilog2(int64_t v) { int k = 0; while ((int64_t(1) << k) < v) ++k; return k; }

static void plan_free(az_plan_s* p) {
  if (p) az_pipe_destroy(p);
  if (!p) return;
  az_graphs_free(p);
  if (p->side) {
    cudaStreamSynchronize(p->side);
    cudaStreamDestroy(p->side);
    for (auto& e : p->side_ev)
      if (e) cudaEventDestroy(e);
  }
  if (p->side2) {
    cudaStreamSynchronize(p->side2);
    cudaStreamDestroy(p->side2);
    for (auto& e : p->side2_ev)
      if (e) cudaEventDestroy(e);
  }
  if (p->hi) {
    cudaStreamSynchronize(p->hi);
    cudaStreamDestroy(p->hi);
  }
  if (p->d_W0y == p->d_W0) p->d_W0y = nullptr;   // aliases of the x tables (square boxes)
  if (p->d_W2y == p->d_W2) p->d_W2y = nullptr;
  void* ptrs[] = {p->d_mask, p->d_pos, p->d_W0, p->d_W2, p->d_W0y, p->d_W2y, p->d_Wr, p->d_zinv, p->d_tw,
                  p->d_tw4hi, p->d_tw4lo, p->d_bxy, p->d_bw, p->d_bj, p->d_C1, p->d_Z2, p->d_G, p->d_solve_ws, p->d_satflag};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  if (p->h_stage) cudaFreeHost(p->h_stage);
  delete p;
}

template <class T>
static az_status_t dalloc(T** ptr, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)ptr, count * sizeof(T));
  if (e != cudaSuccess) {
    az_set_error("cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
    return AZ_ERR_OUT_OF_MEMORY;
  }
  return AZ_OK;
}

static az_status_t plan_build(az_plan_s* p, const az_plan_desc_t* d, cudaStream_t st) {
  // ---- mask -> row index map (pos) ----
  std::vector<int32_t> pos(p->G);
  int64_t M = 0;
  for (int64_t g = 0; g < p->G; ++g) pos[g] = d->mask[g] ? (int32_t)(M++) : -1;
  p->M = M;
  {
    int64_t first = -1, last = -1;
    for (int64_t g = 0; g < p->G; ++g)
      if (d->mask[g]) {
        if (first < 0) first = g;
        last = g;
      }
    if (first >= 0 && last - first + 1 == M) {
      p->run0 = first;
      p->run1 = last + 1;
    }
  }
  if (p->M + p->Mb <= p->N) {
    az_set_error("oversampling insufficient: M + Mb = %lld <= N = %lld (PAPER.md:124)",
                 (long long)(p->M + p->Mb), (long long)p->N);
    return AZ_ERR_OVERSAMPLING;
  }
  AZ_TRY(dalloc(&p->d_mask, p->G));
  AZ_TRY(dalloc(&p->d_pos, p->G));
  AZ_CUDA_CHECK(cudaMemcpyAsync(p->d_mask, d->mask, p->G, cudaMemcpyHostToDevice, st));
  AZ_CUDA_CHECK(cudaMemcpyAsync(p->d_pos, pos.data(), p->G * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  if (p->Mb) {
    AZ_TRY(dalloc(&p->d_bxy, p->Mb * 2));
    AZ_CUDA_CHECK(cudaMemcpyAsync(p->d_bxy, d->boundary_xy, p->Mb * p->dim * sizeof(double),
                                  cudaMemcpyHostToDevice, st));
    // phi(r) < e^-40 beyond r = sqrt(40)/eps: window of 2 ceil(sqrt(40)/(eps h)) + 3 centres per axis
    auto window = [&](int64_t nn, double TT) {
      const double h = 2.0 * TT / (double)nn;
      const int half = (int)std::ceil(std::sqrt(40.0) / (p->eps * h)) + 1;
      return (int)std::min<int64_t>(2 * half + 1, nn);   // all centres when the window wraps
    };
    p->win = window(p->n, p->T);
    p->win_y = p->dim == 2 ? window(p->ny, p->Ty) : 0;
    if (p->win > 64 || p->win_y > 64) {
      az_set_error("boundary stencil wider than 64 centres (eps*h too small)");
      return AZ_ERR_NOT_SUPPORTED;
    }
    if (p->dim == 2) {
      AZ_TRY(dalloc(&p->d_bw, p->Mb * 4 * 64));
      AZ_TRY(dalloc(&p->d_bj, p->Mb * 2));
      double* d_coef = nullptr;
      if (d->boundary_coef) {
        AZ_TRY(dalloc(&d_coef, p->Mb * 4));
        AZ_CUDA_CHECK(cudaMemcpyAsync(d_coef, d->boundary_coef, p->Mb * 4 * sizeof(double), cudaMemcpyHostToDevice, st));
      }
      k_stencil2<<<(unsigned)p->Mb, 64, 0, st>>>(p->d_bxy, d_coef, p->Mb, (int)p->n, (int)p->ny, p->T, p->Ty, p->eps,
                                                 p->win, p->win_y, p->d_bw, p->d_bj);
      AZ_LAUNCH_CHECK();
      if (d_coef) {
        AZ_CUDA_CHECK(cudaStreamSynchronize(st));
        cudaFree(d_coef);
      }
    } else {
      AZ_TRY(dalloc(&p->d_bw, p->Mb * 2 * 64));
      AZ_TRY(dalloc(&p->d_bj, p->Mb * 2));
      k_stencil<<<(unsigned)p->Mb, 64, 0, st>>>(p->d_bxy, p->Mb, p->dim, 0, (int)p->n, p->T, 2.0 * p->T / (double)p->n,
                                                p->eps, p->win, p->d_bw, p->d_bj);
      AZ_LAUNCH_CHECK();
    }
  }
  // ---- twiddles ----
  AZ_TRY(dalloc(&p->d_tw, TWN));
  int nhi = 0, nlo = 0;
  if (p->layout == AZ_LAYOUT_1D_FOURSTEP) {
    nlo = 1 << TW4B;
    nhi = (int)((p->L + nlo - 1) >> TW4B);
    AZ_TRY(dalloc(&p->d_tw4hi, nhi));
    AZ_TRY(dalloc(&p->d_tw4lo, nlo));
  }
  {
    const int64_t cnt = std::max<int64_t>(TWN, std::max(nhi, nlo));
    k_twiddles<<<az_div_up(cnt, 256), 256, 0, st>>>(p->d_tw, TWN, p->d_tw4hi, p->d_tw4lo, p->L, nhi, nlo);
    AZ_LAUNCH_CHECK();
  }
  // ---- scratch for the multi-pass layouts ----
  if (p->layout != AZ_LAYOUT_1D_SMALL) {
    const int64_t per_pair = (p->G + p->N) * (int64_t)sizeof(cplx);
    int64_t scratch_mb = 1600;   // up to 32 vector pairs per launch: fewer, fuller waves (measured on c2)
    if (const char* e = getenv("AZ_SCRATCH_MB")) scratch_mb = std::max<int64_t>(1, atoll(e));
    int64_t B = (scratch_mb << 20) / per_pair;
    B = std::max<int64_t>(1, std::min<int64_t>(B, 32));
    p->Bmax = B;
    AZ_TRY(dalloc(&p->d_C1, B * p->N));
    if (p->layout == AZ_LAYOUT_1D_FOURSTEP) AZ_TRY(dalloc(&p->d_Z2, B * p->N));
    AZ_TRY(dalloc(&p->d_G, B * p->G));
  }
  // ---- symbol tables: fine-grid kernel samples and their DFT (Lemma 3), per axis ----
  const int lap = p->op == AZ_ROW_LAPLACIAN;
  const bool aniso = p->dim == 2 && (p->ny != p->n || p->Ty != p->T);
  for (int axis = 0; axis < (aniso ? 2 : 1); ++axis) {
    const int64_t LL = axis == 0 ? p->L : p->Ly;
    const double TT = axis == 0 ? p->T : p->Ty;
    const double hL = 2.0 * TT / (double)LL;
    cplx** W0 = axis == 0 ? &p->d_W0 : &p->d_W0y;
    cplx** W2 = axis == 0 ? &p->d_W2 : &p->d_W2y;
    AZ_TRY(dalloc(W0, LL));
    if (lap) AZ_TRY(dalloc(W2, LL));
    for (int order = 0; order <= (lap ? 2 : 0); order += 2) {
      cplx* W = order == 0 ? *W0 : *W2;
      k_samples<<<az_div_up(LL, 256), 256, 0, st>>>(W, LL, hL, p->eps, TT, order);
      AZ_LAUNCH_CHECK();
      if (p->layout == AZ_LAYOUT_1D_FOURSTEP)
        AZ_TRY(az1f_fft_fine_forward(p, W, st));
      else
        AZ_TRY(az_fft_batch(p->d_tw, W, LL, 1, -1, st));
    }
  }
  if (!aniso) {
    p->d_W0y = p->d_W0;
    p->d_W2y = p->d_W2;
  }
  if (p->layout == AZ_LAYOUT_1D_FOURSTEP) {
    AZ_TRY(dalloc(&p->d_Wr, p->L));
    k_real_sym<<<az_div_up(p->L, 256), 256, 0, st>>>(p->d_Wr, p->d_W0, p->d_W2, lap, p->alpha, p->k0sq, p->L);
    AZ_LAUNCH_CHECK();
  }
  // ---- sigma^2, max, thresholded inverse ----
  double* d_sig2;
  double* d_red;   // [0] smax, [1] smin, [2] ndrop (as u64)
  AZ_TRY(dalloc(&p->d_zinv, p->N));
  AZ_TRY(dalloc(&d_sig2, p->N));
  AZ_TRY(dalloc(&d_red, 3));
  double init[3] = {0.0, INFINITY, 0.0};
  unsigned long long z = 0;
  memcpy(&init[2], &z, sizeof(z));
  AZ_CUDA_CHECK(cudaMemcpyAsync(d_red, init, sizeof(init), cudaMemcpyHostToDevice, st));
  SymArgs a{p->d_W0, p->d_W2, lap, p->alpha, p->k0sq, p->d_W0y, p->d_W2y};
  k_sigma2<<<az_div_up(p->N, 256), 256, 0, st>>>(d_sig2, d_red, a, p->layout, p->n, p->s, p->N1, p->N2, p->L2,
                                                 p->ny);
  AZ_LAUNCH_CHECK();
  k_zinv<<<az_div_up(p->N, 256), 256, 0, st>>>(p->d_zinv, d_sig2, p->N, d_red, p->rcond,
                                               (unsigned long long*)(d_red + 2), d_red + 1);
  AZ_LAUNCH_CHECK();
  double out[3];
  AZ_CUDA_CHECK(cudaMemcpyAsync(out, d_red, sizeof(out), cudaMemcpyDeviceToHost, st));
  AZ_CUDA_CHECK(cudaStreamSynchronize(st));
  cudaFree(d_sig2);
  cudaFree(d_red);
  unsigned long long nd;
  memcpy(&nd, &out[2], sizeof(nd));
  p->sigma_max2 = out[0];
  p->sigma_min_kept2 = out[1];
  p->n_dropped = (int64_t)nd;
  if (!(p->sigma_max2 > 0.0)) {
    az_set_error("singular symbol: max sigma = 0");
    return AZ_ERR_SINGULAR_SYMBOL;
  }
  return AZ_OK;
}

extern "C" az_status_t az_plan_create(const az_plan_desc_t* d, void* stream, az_plan_t* out) {
  AZ_ARG(d && out, "null descriptor or output");
  *out = nullptr;
  AZ_ARG(d->dim == 1 || d->dim == 2, "dim must be 1 or 2");
  AZ_ARG(is_pow2(d->n), "n must be a power of two");
  AZ_ARG(d->L == 1 || d->L == 2 || d->L == 4, "L (oversampling) must be 1, 2 or 4");
  AZ_ARG(d->T > 0 && d->eps > 0, "T and eps must be positive");
  AZ_ARG(d->mask, "mask is required");
  AZ_ARG(d->op == AZ_ROW_VALUE || d->op == AZ_ROW_LAPLACIAN, "unknown row op");
  AZ_ARG(d->n_boundary >= 0, "n_boundary < 0");
  AZ_ARG(d->n_boundary == 0 || d->boundary_xy, "boundary points missing");
  AZ_ARG(d->zstar_rcond >= 0 && d->zstar_rcond < 1, "zstar_rcond must be in [0, 1)");
  AZ_ARG(!d->boundary_coef || d->dim == 2, "boundary_coef (Robin / Neumann rows) is supported in 2-D only");
  const int64_t L = d->n * d->L;
  if (d->dim == 1) {
    if (d->n < 16 || d->n > (1 << 21) || (d->n_boundary != 0 && L > 2048)) {
      az_set_error("1-D: need 16 <= n <= 2^21; boundary rows (ODE) need L n <= 2048");
      return AZ_ERR_NOT_SUPPORTED;
    }
  } else {
    if (d->n < 8 || L > 2048 || d->L != 2) {
      az_set_error("2-D: need n >= 8, L = 2 and L*n <= 2048");
      return AZ_ERR_NOT_SUPPORTED;
    }
    AZ_ARG(d->n_y >= 0 && d->T_y >= 0, "n_y and T_y must be >= 0");
    const int64_t ny = d->n_y ? d->n_y : d->n;
    AZ_ARG(is_pow2(ny), "n_y must be a power of two");
    if (ny < 8 || ny * d->L > 2048 || 2 * ny < d->n || ny > 2 * d->n) {
      az_set_error("2-D: need n_y >= 8, L*n_y <= 2048 and n/2 <= n_y <= 2n");
      return AZ_ERR_NOT_SUPPORTED;
    }
  }
  az_plan_s* p = new az_plan_s();
  p->dim = d->dim;
  p->n = d->n;
  p->s = d->L;
  p->L = L;
  p->ny = d->dim == 2 && d->n_y ? d->n_y : d->n;
  p->Ly = p->ny * d->L;
  p->Ty = d->dim == 2 && d->T_y > 0 ? d->T_y : d->T;
  p->N = d->dim == 1 ? d->n : d->n * p->ny;
  p->G = d->dim == 1 ? L : L * p->Ly;
  p->Mb = d->n_boundary;
  p->T = d->T;
  p->eps = d->eps;
  p->alpha = d->op == AZ_ROW_LAPLACIAN ? d->row_scale : 1.0;
  p->k0sq = d->op == AZ_ROW_LAPLACIAN ? d->k0sq : 0.0;
  p->beta = d->boundary_weight;
  p->rcond = d->zstar_rcond;
  p->seed = d->seed;
  p->op = d->op;
  if (d->dim == 2) {
    p->layout = AZ_LAYOUT_2D;
  } else if (L <= 2048) {
    p->layout = AZ_LAYOUT_1D_SMALL;
  } else {
    p->layout = AZ_LAYOUT_1D_FOURSTEP;
    const int k = ilog2(d->n);
    p->N1 = int64_t(1) << ((k + 1) / 2);
    p->N2 = d->n / p->N1;
    p->L2 = p->N2 * p->s;
    if (p->L2 > 2048 || p->N1 > 2048 || p->N2 < 8 || p->N1 < 8) {
      delete p;
      az_set_error("1-D four-step: unsupported factorisation");
      return AZ_ERR_NOT_SUPPORTED;
    }
  }
  az_status_t s = plan_build(p, d, (cudaStream_t)stream);
  if (s != AZ_OK) {
    plan_free(p);
    return s;
  }
  *out = p;
  return AZ_OK;
}

extern "C" az_status_t az_plan_destroy(az_plan_t p) {
  plan_free(p);
  return AZ_OK;
}

extern "C" az_status_t az_plan_query(az_plan_t p, az_plan_info_t* info) {
  AZ_ARG(p && info, "null plan or info");
  // unitary normalisation of Lemma 3: singular values of A^c are sqrt(sigma^2_fine / s^d)
  // with the fine-grid DFT W.
  const double sd = p->dim == 1 ? (double)p->s : (double)(p->s * p->s);
  info->N = p->N;
  info->M = p->M;
  info->Mb = p->Mb;
  info->sigma_max = std::sqrt(p->sigma_max2 / sd);
  info->sigma_min_kept = std::sqrt(p->sigma_min_kept2 / sd);
  info->n_dropped = p->n_dropped;
  info->zstar_norm = 1.0 / info->sigma_min_kept;
  return AZ_OK;
}

// ---------------------------------------------------------------------------------------
// operator entry points
// ---------------------------------------------------------------------------------------
static az_status_t dispatch(az_plan_s* p, int op, int src, const double* in, int64_t ldin, double* out,
                            int64_t ldout, int64_t nvec, int64_t col0, cudaStream_t st) {
  if (nvec == 0) return AZ_OK;
  switch (p->layout) {
    case AZ_LAYOUT_1D_SMALL: return az1s_apply(p, op, src, in, ldin, out, ldout, nvec, col0, st);
    case AZ_LAYOUT_1D_FOURSTEP: return az1f_apply(p, op, src, in, ldin, out, ldout, nvec, col0, st);
    default: return az2_apply(p, op, src, in, ldin, out, ldout, nvec, col0, st);
  }
}

az_status_t az_apply_op(az_plan_s* p, int op, const double* in, int64_t ldin, double* out, int64_t ldout,
                        int64_t nvec, cudaStream_t st) {
  return dispatch(p, op, SRC_VEC, in, ldin, out, ldout, nvec, 0, st);
}

static az_status_t check_io(az_plan_s* p, const void* in, int64_t ldin, int64_t rin, const void* out,
                            int64_t ldout, int64_t rout, int64_t nvec) {
  AZ_ARG(p, "null plan");
  AZ_ARG(nvec >= 0, "nvec < 0");
  if (nvec == 0) return AZ_OK;
  AZ_ARG(in && out, "null vector pointer");
  AZ_ARG(ldin >= rin && ldout >= rout, "leading dimension too small (ldin %lld < %lld or ldout %lld < %lld)",
         (long long)ldin, (long long)rin, (long long)ldout, (long long)rout);
  return AZ_OK;
}

extern "C" az_status_t az_apply_A(az_plan_t p, const double* x, int64_t ldx, double* y, int64_t ldy,
                                  int64_t nvec, void* stream) {
  AZ_TRY(check_io(p, x, ldx, p ? p->N : 0, y, ldy, p ? p->M + p->Mb : 0, nvec));
  return dispatch(p, OP_A, SRC_VEC, x, ldx, y, ldy, nvec, 0, (cudaStream_t)stream);
}
extern "C" az_status_t az_apply_At(az_plan_t p, const double* y, int64_t ldy, double* x, int64_t ldx,
                                   int64_t nvec, void* stream) {
  AZ_TRY(check_io(p, y, ldy, p ? p->M + p->Mb : 0, x, ldx, p ? p->N : 0, nvec));
  return dispatch(p, OP_AT, SRC_VEC, y, ldy, x, ldx, nvec, 0, (cudaStream_t)stream);
}
extern "C" az_status_t az_apply_Zstar(az_plan_t p, const double* y, int64_t ldy, double* x, int64_t ldx,
                                      int64_t nvec, void* stream) {
  AZ_TRY(check_io(p, y, ldy, p ? p->M + p->Mb : 0, x, ldx, p ? p->N : 0, nvec));
  return dispatch(p, OP_ZSTAR, SRC_VEC, y, ldy, x, ldx, nvec, 0, (cudaStream_t)stream);
}
extern "C" az_status_t az_apply_step1(az_plan_t p, const double* v, int64_t ldv, double* y, int64_t ldy,
                                      int64_t nvec, void* stream) {
  AZ_TRY(check_io(p, v, ldv, p ? p->N : 0, y, ldy, p ? p->M + p->Mb : 0, nvec));
  return dispatch(p, OP_STEP1, SRC_VEC, v, ldv, y, ldy, nvec, 0, (cudaStream_t)stream);
}
extern "C" az_status_t az_apply_resid(az_plan_t p, const double* b, int64_t ldb, double* y, int64_t ldy,
                                      int64_t nvec, void* stream) {
  AZ_TRY(check_io(p, b, ldb, p ? p->M + p->Mb : 0, y, ldy, p ? p->M + p->Mb : 0, nvec));
  AZ_ARG(b != y, "az_apply_resid: in-place (b == y) is not supported");
  return dispatch(p, OP_RESID, SRC_VEC, b, ldb, y, ldy, nvec, 0, (cudaStream_t)stream);
}
extern "C" az_status_t az_sketch(az_plan_t p, int64_t col0, int64_t ncols, double* S, int64_t ldS,
                                 void* stream) {
  AZ_ARG(p, "null plan");
  AZ_ARG(col0 >= 0 && ncols >= 0, "negative column range");
  if (ncols == 0) return AZ_OK;
  AZ_ARG(S && ldS >= p->M + p->Mb, "bad S / ldS");
  return dispatch(p, OP_STEP1, SRC_PROBE, nullptr, 0, S, ldS, ncols, col0, (cudaStream_t)stream);
}
