// The AZ solve (Alg. 1) and the probe-regeneration GEMM x = Omega y.
//
//   b'  = (I - A Z*) b                                    (az_apply_resid)
//   S   = (A - A Z* A) Omega, Omega in blocks of R probes (az_sketch, Philox on the fly)
//   Rf  = R factor of [S | b']                            (TSQR; rows never permuted)
//   y   = V_k Sigma_k^-1 U_k^T (Q^T b')                   (one-sided Jacobi on R_S)
//   x2  = Omega y                                         (this file, Omega regenerated)
//   x   = x2 + Z* (b - A x2)                              (step 2 + step 3)
// Probe blocks are added while the sketch is saturated, rank > probes - p (p = 10),
// up to max_blocks (reading R5).
// Four-step narrow solves with one probe block (c2) reorganise the same algebra:
//   x = Z* b + M y, M = Omega - Z* A Omega (reading R30), both from the b' / sketch chains;
//   y = P (Q^T b'), P = pinv_theta(R_S) from the SVD of [R_S | I], with Q^T b' carried through the
//   kept TSQR reflectors on a side stream while the merge tree and the SVD run at high priority.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <vector>

#include "az_internal.h"
#include "az_mma.cuh"

// ------------------------------------------------------------------------------------------
// x (+)= Omega[:, col0 : col0 + ncols] y   (a9 of SURVEY.md §8(a))
// CTA tile: 128 rows (64 row pairs) x all nrhs <= 64 columns; Omega tile generated into smem.
// ------------------------------------------------------------------------------------------
constexpr int OM_ROWS = 128;
constexpr int OM_JT = 16;

__global__ void __launch_bounds__(256) k_omega_apply(int64_t N, int64_t col0, int ncols, const double* y, int64_t ldy,
                                                     int nrhs, double* x, int64_t ldx, int accumulate, uint64_t seed) {
  __shared__ double om[OM_JT][OM_ROWS + 1];
  __shared__ double ys[OM_JT][64];
  const int tid = threadIdx.x;
  const int64_t row0 = (int64_t)blockIdx.x * OM_ROWS;
  // thread -> (4 rows, up to 8 rhs): 32 row groups x 8 rhs groups
  const int rg = tid & 31, cg = tid >> 5;
  double acc[4][8];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[a][c] = 0.0;
  for (int j0 = 0; j0 < ncols; j0 += OM_JT) {
    __syncthreads();
    // Omega tile: OM_ROWS/2 row pairs x OM_JT columns
    for (int e = tid; e < (OM_ROWS / 2) * OM_JT; e += blockDim.x) {
      const int pr = e % (OM_ROWS / 2), jj = e / (OM_ROWS / 2);
      const int64_t i = row0 + 2 * pr;
      double2 z = make_double2(0.0, 0.0);
      if (j0 + jj < ncols && i < N) z = probe_pair((uint64_t)(i >> 1), (uint64_t)(col0 + j0 + jj), seed);
      om[jj][2 * pr] = z.x;
      om[jj][2 * pr + 1] = (i + 1 < N) ? z.y : 0.0;
    }
    for (int e = tid; e < OM_JT * 64; e += blockDim.x) {
      const int jj = e / 64, c = e % 64;
      ys[jj][c] = (j0 + jj < ncols && c < nrhs) ? y[(int64_t)c * ldy + j0 + jj] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int jj = 0; jj < OM_JT; ++jj) {
      double o[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) o[a] = om[jj][rg + 32 * a];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double yv = ys[jj][cg + 8 * c];
#pragma unroll
        for (int a = 0; a < 4; ++a) acc[a][c] = fma(o[a], yv, acc[a][c]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t i = row0 + rg + 32 * a;
    if (i >= N) continue;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int cc = cg + 8 * c;
      if (cc < nrhs) {
        double* px = x + (int64_t)cc * ldx + i;
        *px = accumulate ? *px + acc[a][c] : acc[a][c];
      }
    }
  }
}

static az_status_t omega_apply_spectral(az_plan_s* p, int64_t col0, int64_t ncols, const double* y, int64_t ldy,
                                        int64_t nrhs, double* x, int64_t ldx, int accumulate, cudaStream_t st);

static az_status_t omega_apply(az_plan_s* p, int64_t col0, int64_t ncols, const double* y, int64_t ldy,
                               int64_t nrhs, double* x, int64_t ldx, int accumulate, cudaStream_t st) {
  if (p->layout == AZ_LAYOUT_1D_FOURSTEP) return omega_apply_spectral(p, col0, ncols, y, ldy, nrhs, x, ldx, accumulate, st);
  for (int64_t c0 = 0; c0 < nrhs; c0 += 64) {
    const int nr = (int)std::min<int64_t>(64, nrhs - c0);
    AzTrace tr("omega_apply", st, p->N * ncols * nr);
    k_omega_apply<<<az_div_up(p->N, OM_ROWS), 256, 0, st>>>(p->N, col0, (int)ncols, y + c0 * ldy, ldy, nr,
                                                            x + c0 * ldx, ldx, accumulate, p->seed);
    AZ_LAUNCH_CHECK();
  }
  return AZ_OK;
}

extern "C" az_status_t az_omega_apply(az_plan_t p, int64_t col0, int64_t ncols, const double* y, int64_t ldy,
                                      int64_t nrhs, double* x, int64_t ldx, int accumulate, void* stream) {
  if (!p || col0 < 0 || ncols < 0 || nrhs < 0 || (nrhs && (!x || ldx < p->N)) || (ncols && nrhs && (!y || ldy < ncols))) {
    az_set_error("az_omega_apply: bad arguments");
    return AZ_ERR_INVALID_ARGUMENT;
  }
  return omega_apply(p, col0, ncols, y, ldy, nrhs, x, ldx, accumulate, (cudaStream_t)stream);
}

// ------------------------------------------------------------------------------------------
// small elementwise kernels
// ------------------------------------------------------------------------------------------
__global__ void k_copy_cols(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int64_t cols) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const int64_t r = e % rows, c = e / rows;
  dst[c * ldd + r] = src[c * lds + r];
}
__global__ void k_sub_cols(const double* b, int64_t ldb, double* y, int64_t ldy, int64_t rows, int64_t cols) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const int64_t r = e % rows, c = e / rows;
  y[c * ldy + r] = b[c * ldb + r] - y[c * ldy + r];       // y <- b - y
}
__global__ void k_add_cols(const double* a, int64_t lda, double* x, int64_t ldx, int64_t rows, int64_t cols) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const int64_t r = e % rows, c = e / rows;
  x[c * ldx + r] += a[c * lda + r];
}

// ------------------------------------------------------------------------------------------
// workspace layout
// ------------------------------------------------------------------------------------------
struct SolveWS {
  double* S;     // rows x (Rmax + nrhs)
  double* bp;    // rows x nrhs : b'
  double* Rf;    // kt x kt
  double* y;     // Rmax x nrhs
  double* sig;   // Rmax
  double* tmp;   // rows x nrhs
  double* x2;    // N x nrhs
  double* Zb;    // N x nrhs: Z* b from the b' chain (four-step narrow path), else null
  cplx* Zs;      // the b' chain's Z* b spectra (N x ceil(nrhs / 2) complex), same condition
  double* Om;    // N x Rmax: M = Omega - Z* A Omega from the sketch (same condition)
  double* Rp;    // Rmax x 2 Rmax: [R_S | I] for P = pinv_theta(R_S) (deferred Q^T b', same condition)
  double* Pm;    // Rmax x Rmax: P
  double* cq;    // Rmax x nrhs: Q^T b' from the right-hand-side stream
  void* qrws;
  size_t qrbytes;
  void* svdws;
  size_t svdbytes;
  double* Tb;    // wide path: T factors of every panel
  int64_t maxpanels;
  bool wide;
  size_t total;
};

static size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

// Y = A B (or C - A B), DMMA tiles; defined with the factored-solve kernels below
__global__ void k_gemm_mn(const double* A, int64_t lda, const double* Bm, int64_t ldb, double* Y, int64_t ldy, int64_t m,
                          int64_t k, int64_t n, const double* C = nullptr, int64_t ldc = 0, double sgn = -1.0);
__global__ void k_gemm_mn_small(const double* A, int64_t lda, const double* Bm, int64_t ldb, double* Y, int64_t ldy,
                                int64_t m, int k, int n, const double* C, int64_t ldc, double sgn = -1.0);
__global__ void k_identity_cols(double* Rf, int64_t ld, int64_t k, int64_t col0);

// 1-D narrow solves (four-step and one-CTA layouts): step 2 as x = Z* b + M y from the b' and sketch
// chains (reading R30; AZ_STEP2_LINEAR=0 disables).  Its rounding error is of the order
// u ||Z*|| ||b|| (Z* b and (Z* A Omega) y cancel), against u ||Z*|| ||b - A x2|| for the residual form
// x2 + Z* (b - A x2): it is used only while ||Z*|| <= 1e5 (c1 / c2: 2.7e3; the paper's own eps regime
// reaches 1e9, where the residual form is kept)
static bool step2_linear(const az_plan_s* p) {
  static int k = -1;
  if (k < 0) {
    const char* e = getenv("AZ_STEP2_LINEAR");
    k = e ? atoi(e) : 1;
  }
  const double sd = p->dim == 1 ? (double)p->s : (double)(p->s * p->s);
  const double zstar_norm = p->sigma_min_kept2 > 0 ? 1.0 / std::sqrt(p->sigma_min_kept2 / sd) : 1e300;
  return k != 0 && zstar_norm <= 1e5;
}

// AZ_QR_DEFER=0: Q^T b' rides along in the TSQR merges (on the R factor's critical path) instead of
// following on the side stream while the SVD computes P = pinv_theta(R_S)
static bool qr_defer() {
  static int k = -1;
  if (k < 0) {
    const char* e = getenv("AZ_QR_DEFER");
    k = e ? atoi(e) : 1;
  }
  return k != 0;
}

// AZ_SOLVE_HI=0: the QR and the SVD stay on the caller's stream while the side stream runs
// AZ_SIDE_PRIO=0: the side stream at default priority (like the second side stream)
static bool side_prio_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("AZ_SIDE_PRIO");
    v = (e && *e == '0') ? 0 : 1;
  }
  return v != 0;
}

// AZ_SIDE2: 2 (default) the Z* b column pass on a second side stream right after the TSQR leaf, beside
// the M pass and the merges; 1: on that stream after pass B; 3: the M pass on it too (the side stream
// then starts pass B at once); 0: on the side stream before the M pass (the former order).  Measured
// c2 ms per step (two 20-step runs each): 2: 9.21 / 9.22, 1: 9.30 / 9.30, 0: 9.28 / 9.33; later, with
// the look-ahead merges: 2: 9.02 / 8.96, 3: 9.04 / 9.01.
static int side2_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("AZ_SIDE2");
    v = e ? atoi(e) : 2;
    if (v < 0 || v > 3) v = 2;
  }
  return v;
}

static bool no_hi() {
  static int k = -1;
  if (k < 0) {
    const char* e = getenv("AZ_SOLVE_HI");
    k = e ? atoi(e) : 1;
  }
  return k == 0;
}

// k_gemm_mn_small walks its 64-row tiles grid-stride: one wave of exactly the resident CTAs (126
// registers per thread allow two per SM, not the three its shared memory would), or the CTAs past
// the first wave run alone at the end
static unsigned gemm_small_grid(int64_t m) {
  static int per_sm = 0, sms = 0;
  if (!per_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gemm_mn_small, 256, 2 * 64 * 68 * sizeof(double)) !=
            cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
  }
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(az_div_up(m, 64), (int64_t)per_sm * sms));
}

// The single-pass TSQR / one-CTA Jacobi (narrow) path takes the sketch while probes + nrhs <= 128;
// the blocked Householder / block-Jacobi (wide) path beyond.  The choice follows the probes a solve
// actually draws: an adaptive solve whose first block fits the narrow path runs it first and moves to
// the wide path (drawing its blocks afresh) only if that block saturated (reading R5).
static bool narrow_first(int64_t nrhs, int64_t R, int32_t max_blocks) {
  return max_blocks > 1 && R + nrhs <= AZ_NARROW_MAX && R * max_blocks + nrhs > AZ_NARROW_MAX;
}

static SolveWS layout(az_plan_s* p, int64_t nrhs, int64_t R, int32_t max_blocks, char* base) {
  SolveWS w;
  const int64_t rows = p->M + p->Mb;
  const int64_t Rmax = R * max_blocks;
  const int64_t kt = Rmax + nrhs;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* ptr = base ? base + off : nullptr;
    off += align256(bytes);
    return ptr;
  };
  w.S = (double*)take(sizeof(double) * rows * kt);
  w.bp = (double*)take(sizeof(double) * rows * nrhs);
  w.Rf = (double*)take(sizeof(double) * kt * kt);
  w.y = (double*)take(sizeof(double) * Rmax * nrhs);
  w.sig = (double*)take(sizeof(double) * Rmax);
  w.tmp = (double*)take(sizeof(double) * rows * nrhs);
  w.x2 = (double*)take(sizeof(double) * p->N * nrhs);
  w.wide = kt > AZ_NARROW_MAX;
  const bool four = p->layout == AZ_LAYOUT_1D_FOURSTEP;
  const bool keep = !w.wide && (four || p->layout == AZ_LAYOUT_1D_SMALL) && step2_linear(p);
  w.Zb = keep ? (double*)take(sizeof(double) * p->N * nrhs) : nullptr;
  w.Zs = keep && four ? (cplx*)take(sizeof(cplx) * p->N * ((nrhs + 1) / 2)) : nullptr;
  w.Om = keep ? (double*)take(sizeof(double) * p->N * Rmax) : nullptr;
  w.Rp = keep && four ? (double*)take(sizeof(double) * Rmax * 2 * Rmax) : nullptr;
  w.Pm = keep && four ? (double*)take(sizeof(double) * Rmax * Rmax) : nullptr;
  w.cq = keep && four ? (double*)take(sizeof(double) * Rmax * nrhs) : nullptr;
  if (w.wide) {
    const int64_t QBw = az_qrw_panel_width();
    w.maxpanels = max_blocks * ((R + QBw - 1) / QBw);
    w.Tb = (double*)take(sizeof(double) * w.maxpanels * QBw * QBw);
    w.qrbytes = az_qrw_ws_bytes(rows, std::max<int64_t>(R, nrhs));
  } else {
    w.maxpanels = 0;
    w.Tb = nullptr;
    w.qrbytes = az_qr_ws_bytes(rows, kt);
  }
  w.qrws = take(w.qrbytes);
  w.svdbytes = az_tsvd_ws_bytes(Rmax, nrhs);
  w.svdws = take(w.svdbytes);
  w.total = off;
  return w;
}

extern "C" az_status_t az_solve_workspace_size(az_plan_t p, int64_t nrhs, int64_t R, int32_t max_blocks, size_t* bytes) {
  if (!p || !bytes || nrhs < 1 || R < 1 || max_blocks < 1) {
    az_set_error("az_solve_workspace_size: bad arguments");
    return AZ_ERR_INVALID_ARGUMENT;
  }
  *bytes = layout(p, nrhs, R, max_blocks, nullptr).total;
  if (narrow_first(nrhs, R, max_blocks)) *bytes = std::max(*bytes, layout(p, nrhs, R, 1, nullptr).total);
  return AZ_OK;
}

// Stage-timing events, drawn from a per-thread pool (created once: event creation is a driver
// round trip, and the small solves are host-latency bound).  Nested users take the next set.
struct Ev {
  cudaEvent_t* e;
  static constexpr int kDepth = 4;
  static thread_local cudaEvent_t pool[kDepth][8];
  static thread_local int depth;
  Ev() {
    const int d = depth < kDepth ? depth : kDepth - 1;
    ++depth;
    e = pool[d];
    if (!e[0])
      for (int i = 0; i < 8; ++i) cudaEventCreate(&e[i]);
  }
  ~Ev() { --depth; }
};
thread_local cudaEvent_t Ev::pool[Ev::kDepth][8] = {};
thread_local int Ev::depth = 0;

static double ms_between(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return (double)ms;
}

az_status_t az_apply_op(az_plan_s* p, int op, const double* in, int64_t ldin, double* out, int64_t ldout,
                        int64_t nvec, cudaStream_t st);

// Step 2 + 3 of Alg. 1: x = x2 + Z* (b - A x2).  Four-step layout: one fused
// five-pass chain (az1f_step2); otherwise A, b - A x2, Z*, + x2.  tmp: (M + Mb) x nrhs scratch.
static az_status_t step2(az_plan_s* p, const double* x2, const double* b, int64_t ldb, double* x, int64_t ldx,
                         double* tmp, int64_t nrhs, cudaStream_t st, int64_t ldx2 = 0) {
  if (!ldx2) ldx2 = p->N;
  if (p->layout == AZ_LAYOUT_1D_FOURSTEP) return az1f_step2(p, x2, ldx2, b, ldb, x, ldx, nrhs, st);
  const int64_t rows = p->M + p->Mb;
  AZ_TRY(az_apply_op(p, OP_A, x2, ldx2, tmp, rows, nrhs, st));
  {
    AzTrace tr("elementwise", st);
    k_sub_cols<<<az_div_up(rows * nrhs, 256), 256, 0, st>>>(b, ldb, tmp, rows, rows, nrhs);
  }
  AZ_LAUNCH_CHECK();
  AZ_TRY(az_apply_op(p, OP_ZSTAR, tmp, rows, x, ldx, nrhs, st));
  {
    AzTrace tr("elementwise", st);
    k_add_cols<<<az_div_up(p->N * nrhs, 256), 256, 0, st>>>(x2, ldx2, x, ldx, p->N, nrhs);
  }
  AZ_LAUNCH_CHECK();
  return AZ_OK;
}

extern "C" az_status_t az_step2_workspace_size(az_plan_t p, int64_t nrhs, size_t* bytes) {
  if (!p || !bytes || nrhs < 0) {
    az_set_error("az_step2_workspace_size: bad arguments");
    return AZ_ERR_INVALID_ARGUMENT;
  }
  *bytes = p->layout == AZ_LAYOUT_1D_FOURSTEP ? 0 : sizeof(double) * (size_t)(p->M + p->Mb) * (size_t)nrhs;
  return AZ_OK;
}

extern "C" az_status_t az_step2(az_plan_t p, const double* x2, int64_t ldx2, const double* b, int64_t ldb, double* x,
                                int64_t ldx, int64_t nrhs, void* workspace, size_t ws_bytes, void* stream) {
  size_t need = 0;
  if (!p || nrhs < 0 || (nrhs > 0 && (!x2 || !b || !x)) || ldx2 < p->N || ldb < p->M + p->Mb || ldx < p->N ||
      az_step2_workspace_size(p, nrhs, &need) != AZ_OK) {
    az_set_error("az_step2: bad arguments");
    return AZ_ERR_INVALID_ARGUMENT;
  }
  if (nrhs == 0) return AZ_OK;
  if (ws_bytes < need || (need && !workspace)) {
    az_set_error("az_step2: workspace too small (%zu < %zu)", ws_bytes, need);
    return AZ_ERR_WORKSPACE;
  }
  return step2(p, x2, b, ldb, x, ldx, (double*)workspace, nrhs, (cudaStream_t)stream, ldx2);
}

__global__ void k_flag_saturated(const int64_t* rank, int64_t limit, int* flag) {
  if (*rank > limit) atomicOr(flag, 1);
}

// One solve on a workspace laid out for (nrhs, R, max_blocks).  async (max_blocks == 1 only): the
// solve is enqueued without any host synchronisation and no report; if sat_flag (DEVICE) is given,
// a saturated sketch sets it (az_solve_host_pipelined / az_plan_sync).
// Where an async solve left its results (for a captured solve's report).
struct SolveTail {
  const int64_t* rank_dev = nullptr;
  const double* sig = nullptr;
  int64_t kp = 0;
};

static az_status_t solve_impl(az_plan_s* p, const double* b, int64_t ldb, double* x, int64_t ldx, int64_t nrhs,
                              double theta, int64_t R, int32_t max_blocks, void* workspace,
                              az_solve_report_t* report, cudaStream_t st, bool async_mode, int* sat_flag,
                              cudaEvent_t* graph_ev = nullptr, SolveTail* tail = nullptr) {
  SolveWS w = layout(p, nrhs, R, max_blocks, (char*)workspace);
  const int64_t rows = p->M + p->Mb;
  const int pfix = 10;
  // the rank is needed on the host mid-solve only to decide on another probe block; with one block
  // it is read after the last kernel, so step 2 is enqueued without waiting for the SVD
  const bool host_rank = max_blocks > 1;
  const int64_t* rank_dev = nullptr;
  static const bool dbg_host = getenv("AZ_DEBUG_HOST") != nullptr;
  auto hnow = []() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double th0 = dbg_host ? hnow() : 0.0;
  Ev ev_pool;
  // stage events: the pool's, or -- while a solve is captured into a graph -- the graph's own, recorded
  // as external event nodes so that their times can be read after each replay
  struct {
    cudaEvent_t* e;
    bool ext;
  } ev{graph_ev ? graph_ev : ev_pool.e, graph_ev != nullptr};
  auto rec = [&](cudaEvent_t e, cudaStream_t s) {
    if (ev.ext) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    else cudaEventRecord(e, s);
  };
  rec(ev.e[0], st);
  // ---- right-hand side b' = (I - A Z*) b (narrow single-block solve: straight into S) ----
  const bool bp_in_S = !w.wide && max_blocks == 1;
  // the Z* b and M column passes are only needed by step 2: with one probe block and one batch per
  // chain they run on a side stream beside the TSQR merges and the SVD (which leave most SMs idle)
  const bool side = w.Zb && max_blocks == 1 && (nrhs + 1) / 2 <= p->Bmax && (R + 1) / 2 <= p->Bmax;
  if (side && !p->side) {
    int lo = 0, top = 0;
    AZ_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &top));
    // priorities: the QR / SVD stream (hi) first, then the side stream (pass B and the merge-level passes,
    // whose few CTAs must not queue behind the second side stream's column pass), then side2
    const int side_prio = (side_prio_on() && top < lo) ? std::min(lo, top + 1) : lo;
    AZ_CUDA_CHECK(cudaStreamCreateWithPriority(&p->side, cudaStreamNonBlocking, side_prio));
    for (auto& e : p->side_ev) AZ_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    AZ_CUDA_CHECK(cudaStreamCreateWithPriority(&p->hi, cudaStreamNonBlocking, top));
    AZ_CUDA_CHECK(cudaStreamCreateWithFlags(&p->side2, cudaStreamNonBlocking));
    for (auto& e : p->side2_ev) AZ_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // the QR and the SVD: on the high-priority stream beside the side stream (joined back below)
  cudaStream_t qs = side && !no_hi() ? p->hi : st;
  // Q^T b' off the R factor's critical path: R_S alone through the merge tree, P = pinv_theta(R_S) by
  // the SVD of [R_S | I], while b' follows the kept reflectors on the side stream; y = P (Q^T b')
  const bool defer = side && qr_defer() && R <= 64 && nrhs <= 64 && w.Rp;
  const int s2mode = side2_mode();
  const bool use_side2 = side && defer && s2mode != 0;
  if (w.Zb && w.Zs) {   // b' and, for step 2, Z* b (one extra column pass)
    AZ_TRY(az1f_resid_z(p, b, ldb, bp_in_S ? w.S + R * rows : w.bp, rows, w.Zb, p->N, nrhs, st, w.Zs, side));
  } else if (w.Zb) {    // one-CTA layout: Z* b from the chain's spectrum of it (one more transform)
    AZ_TRY(az1s_apply(p, OP_RESID, SRC_VEC, b, ldb, bp_in_S ? w.S + R * rows : w.bp, rows, nrhs, 0, st, w.Zb, p->N));
  } else {
    AZ_TRY(az_apply_op(p, OP_RESID, b, ldb, bp_in_S ? w.S + R * rows : w.bp, rows, nrhs, st));
  }
  rec(ev.e[1], st);
  if (dbg_host) fprintf(stderr, "az_solve host: resid issued +%.2f ms\n", hnow() - th0);
  double ms_sketch = 0, ms_qr = 0, ms_svd = 0;
  int64_t rank = 0, nb = 0;
  bool saturated = false;
  // wide path (2-D): incremental blocked Householder; panels of earlier blocks are applied to
  // each new block, and every panel is applied to b' (which becomes Q^T b' in its top rows)
  std::vector<int64_t> pj0(w.maxpanels);
  std::vector<int> pnb(w.maxpanels);
  int64_t np = 0;
  double s1lo = 0.0;   // lower bound on sigma_1 of the sketch's R factor
  for (nb = 1; nb <= max_blocks; ++nb) {
    const int64_t kp = nb * R;                 // probe columns
    const int64_t kt = kp + nrhs;
    cudaEvent_t e0 = ev.e[2], e1 = ev.e[3], e2 = ev.e[4], e3 = ev.e[5];
    rec(e0, st);
    if (w.Om && w.Zs) {   // the sketch and M = Omega - Z* A Omega for step 2
      AZ_TRY(az1f_sketch_m(p, (nb - 1) * R, R, w.S + (nb - 1) * R * rows, rows, w.Om + (nb - 1) * R * p->N, p->N, st,
                           nullptr, side));
    } else if (w.Om) {
      AZ_TRY(az1s_apply(p, OP_STEP1, SRC_PROBE, nullptr, 0, w.S + (nb - 1) * R * rows, rows, R, (nb - 1) * R, st,
                        w.Om + (nb - 1) * R * p->N, p->N));
    } else
      AZ_TRY(az_sketch(p, (nb - 1) * R, R, w.S + (nb - 1) * R * rows, rows, st));
    if (!w.wide && !bp_in_S) {
      AzTrace tr("elementwise", st);
      k_copy_cols<<<az_div_up(rows * nrhs, 256), 256, 0, st>>>(w.bp, rows, w.S + kp * rows, rows, rows, nrhs);
      AZ_LAUNCH_CHECK();
    }
    rec(e1, st);
    if (qs != st) AZ_CUDA_CHECK(cudaStreamWaitEvent(qs, e1, 0));
    if (dbg_host) fprintf(stderr, "az_solve host: sketch issued +%.2f ms\n", hnow() - th0);
    if (!w.wide) {
      // a single probe block: the sketch columns are not needed after this QR (split leaf allowed)
      if (defer) {
        AZ_TRY(az_qr_r_deferred(w.S, rows, kt, kp, rows, w.Rp, kp, w.qrws, w.qrbytes, qs, p->side_ev[0],
                                p->side_ev[1]));
      } else {
        AZ_TRY(az_qr_r_impl(w.S, rows, kt, rows, w.Rf, kt, w.qrws, w.qrbytes, qs, kp, max_blocks == 1,
                            side ? p->side_ev[0] : nullptr));
      }
      if (side) {
        // side stream: the deferred Z* b and M passes beside the merges (whose CTAs take freed SMs
        // first), then -- deferred -- Q^T b' through the kept reflectors beside the SVD
        AZ_CUDA_CHECK(cudaStreamWaitEvent(p->side, p->side_ev[0], 0));
        if (!use_side2) AZ_TRY(az1f_out_z(p, w.Zs, w.Zb, p->N, nrhs, p->side));
        if (!(use_side2 && s2mode == 3)) AZ_TRY(az1f_out_z(p, p->d_Z2, w.Om, p->N, R, p->side));
        // Z* b on a second side stream: after pass B (mode 1; it then runs beside the right-hand-side
        // merge passes and the SVD, which leave most SMs idle) or right after the leaf (mode 2)
        if (use_side2 && s2mode >= 2) {
          AZ_CUDA_CHECK(cudaStreamWaitEvent(p->side2, p->side_ev[0], 0));
          AZ_TRY(az1f_out_z(p, w.Zs, w.Zb, p->N, nrhs, p->side2, side_prio_on()));
          // mode 3: the M pass too, so the side stream starts pass B right after the leaf
          if (s2mode == 3) AZ_TRY(az1f_out_z(p, p->d_Z2, w.Om, p->N, R, p->side2));
        }
        if (defer)
          AZ_TRY(az_qr_rhs_deferred(w.S, rows, kt, kp, rows, w.cq, kp, w.qrws, w.qrbytes, p->side, p->side_ev[0],
                                    p->side_ev[1], use_side2 && s2mode == 1 ? p->side2_ev[0] : nullptr));
        if (use_side2) {
          if (s2mode == 1) {
            AZ_CUDA_CHECK(cudaStreamWaitEvent(p->side2, p->side2_ev[0], 0));
            AZ_TRY(az1f_out_z(p, w.Zs, w.Zb, p->N, nrhs, p->side2));
          }
          AZ_CUDA_CHECK(cudaEventRecord(p->side2_ev[1], p->side2));
        }
        AZ_CUDA_CHECK(cudaEventRecord(p->side_ev[2], p->side));
      }
    } else {
      if (kp > rows) {
        az_set_error("az_solve: %lld probe columns exceed the %lld rows", (long long)kp, (long long)rows);
        return AZ_ERR_NOT_SUPPORTED;
      }
      double* Snew = w.S + (nb - 1) * R * rows;
      AZ_TRY(az_qrw_apply(w.S, rows, rows, pj0.data(), pnb.data(), w.Tb, 0, np, Snew, rows, R, w.qrws, w.qrbytes, st));
      const int64_t np0 = np;
      AZ_TRY(az_qrw_factor(w.S, rows, rows, (nb - 1) * R, kp, w.Tb, pj0.data(), pnb.data(), &np, w.qrws, w.qrbytes, st));
      AZ_TRY(az_qrw_apply(w.S, rows, rows, pj0.data(), pnb.data(), w.Tb, np0, np, w.bp, rows, nrhs, w.qrws, w.qrbytes, st));
      AZ_TRY(az_qrw_extract_R(w.S, rows, kp, w.Rf, kt, st));
      AzTrace tr("elementwise", st);
      k_copy_cols<<<az_div_up(kp * nrhs, 256), 256, 0, st>>>(w.bp, rows, w.Rf + kp * kt, kt, kp, nrhs);
      AZ_LAUNCH_CHECK();
    }
    rec(e2, qs);
    if (dbg_host) fprintf(stderr, "az_solve host: qr issued +%.2f ms\n", hnow() - th0);
    bool full_svd = true;
    if (w.wide && nb >= 2 && nb < max_blocks) {
      // Cheap saturation pre-test (reading R5): with R_b = [[R11, R12], [0, R22]] and
      // R22 the new block's R x R corner, sigma_{kp-R+j}(R_b) <= sigma_j(R22) (R_b minus a rank
      // kp - R matrix), so rank_t(S) <= kp - R + rank_t(R22) for any threshold t.  With
      // t = theta * s1lo, s1lo <= sigma_1(R_b) (singular values of the leading block and of R22
      // are lower bounds), k22 <= R - p proves the sketch unsaturated; otherwise the full SVD is
      // skipped and another block is drawn (a possibly extra block, never a missing one).
      const int64_t off = (nb - 1) * R;
      int64_t k22 = 0;
      AZ_TRY(az_tsvd_impl(w.Rf + off * kt + off, kt, R, 0, theta, w.y, R, w.sig, &k22, w.svdws, w.svdbytes, st));
      std::vector<double> s22(R);
      AZ_CUDA_CHECK(cudaMemcpyAsync(s22.data(), w.sig, sizeof(double) * R, cudaMemcpyDeviceToHost, st));
      AZ_CUDA_CHECK(cudaStreamSynchronize(st));
      s1lo = std::max(s1lo, s22[0]);
      k22 = 0;
      for (int64_t i = 0; i < R; ++i) k22 += s22[i] > theta * s1lo;
      full_svd = k22 <= R - pfix;
      rank = kp;   // not computed: treated as saturated unless the full SVD runs
    }
    if (full_svd && defer) {
      // [R_S | I]: the truncated SVD solve of the identity is P = V_k Sigma_k^-1 U_k^T
      k_identity_cols<<<az_div_up(kp * kp, 256), 256, 0, qs>>>(w.Rp, kp, kp, kp);
      AZ_LAUNCH_CHECK();
      AZ_TRY(az_tsvd_impl(w.Rp, kp, kp, kp, theta, w.Pm, kp, w.sig, host_rank ? &rank : nullptr, w.svdws,
                          w.svdbytes, qs, &rank_dev));
    } else if (full_svd) {
      AZ_TRY(az_tsvd_impl(w.Rf, kt, kp, nrhs, theta, w.y, kp, w.sig, host_rank ? &rank : nullptr, w.svdws,
                          w.svdbytes, qs, &rank_dev));
      if (w.wide && nb < max_blocks) {   // sigma_1 lower bound for the next block's pre-test
        double s1 = 0.0;
        AZ_CUDA_CHECK(cudaMemcpyAsync(&s1, w.sig, sizeof(double), cudaMemcpyDeviceToHost, st));
        AZ_CUDA_CHECK(cudaStreamSynchronize(st));
        s1lo = std::max(s1lo, s1);
      }
    }
    rec(e3, qs);
    if (qs != st) AZ_CUDA_CHECK(cudaStreamWaitEvent(st, e3, 0));
    if (host_rank) {
      cudaEventSynchronize(e3);
      ms_sketch += ms_between(e0, e1);
      ms_qr += ms_between(e1, e2);
      ms_svd += ms_between(e2, e3);
    }
    saturated = host_rank && rank > kp - pfix;
    if (!saturated || nb == max_blocks) break;
  }
  if (nb > max_blocks) nb = max_blocks;
  const int64_t kp = nb * R;
  if (dbg_host) fprintf(stderr, "az_solve host: svd issued +%.2f ms\n", hnow() - th0);
  rec(ev.e[6], st);
  // ---- x2 = Omega y ; x = x2 + Z* (b - A x2) ----
  if (w.Om) {
    // by linearity of Z* (PAPER.md:229-230): x = Omega y + Z* b - (Z* A Omega) y = Z* b + M y, with
    // Z* b and M = Omega - Z* A Omega produced by the b' and sketch chains: one DMMA pass, no FFT
    if (side) AZ_CUDA_CHECK(cudaStreamWaitEvent(st, p->side_ev[2], 0));   // Z* b, M (and Q^T b') are ready
    if (use_side2) AZ_CUDA_CHECK(cudaStreamWaitEvent(st, p->side2_ev[1], 0));
    if (defer) {   // y = P (Q^T b')
      AzTrace tr("y_pc", st);
      k_gemm_mn<<<dim3(az_div_up(kp, 64), az_div_up(nrhs, 64)), 256, 0, st>>>(w.Pm, kp, w.cq, kp, w.y, kp, kp, kp,
                                                                             nrhs);
      AZ_LAUNCH_CHECK();
    }
    AzTrace tr("step2_gemm", st, 2 * p->N * kp * nrhs);
    if (kp <= 64) {
      const size_t gs = 2 * 64 * 68 * sizeof(double);
      AZ_CUDA_CHECK(az_smem_attr(k_gemm_mn_small, gs));
      for (int64_t c0 = 0; c0 < nrhs; c0 += 64)
        k_gemm_mn_small<<<gemm_small_grid(p->N), 256, gs, st>>>(
            w.Om, p->N, w.y + c0 * kp, kp, x + c0 * ldx, ldx, p->N, (int)kp, (int)std::min<int64_t>(64, nrhs - c0),
            w.Zb + c0 * p->N, p->N, 1.0);
    } else {
      k_gemm_mn<<<dim3(az_div_up(p->N, 64), az_div_up(nrhs, 64)), 256, 0, st>>>(w.Om, p->N, w.y, kp, x, ldx, p->N, kp,
                                                                                nrhs, w.Zb, p->N, 1.0);
    }
    AZ_LAUNCH_CHECK();
  } else {
    AZ_TRY(omega_apply(p, 0, kp, w.y, kp, nrhs, w.x2, p->N, 0, st));
    AZ_TRY(step2(p, w.x2, b, ldb, x, ldx, w.tmp, nrhs, st));
  }
  rec(ev.e[7], st);
  if (dbg_host) fprintf(stderr, "az_solve host: all issued +%.2f ms\n", hnow() - th0);
  if (tail) {
    tail->rank_dev = rank_dev;
    tail->sig = w.sig;
    tail->kp = kp;
  }
  if (async_mode) {
    if (sat_flag && rank_dev) {
      k_flag_saturated<<<1, 1, 0, st>>>(rank_dev, kp - pfix, sat_flag);
      AZ_LAUNCH_CHECK();
    }
    return AZ_OK;
  }
  AZ_CUDA_CHECK(cudaEventSynchronize(ev.e[7]));
  if (!host_rank) {
    if (rank_dev) AZ_CUDA_CHECK(cudaMemcpy(&rank, rank_dev, sizeof(int64_t), cudaMemcpyDeviceToHost));
    ms_sketch = ms_between(ev.e[2], ev.e[3]);
    ms_qr = ms_between(ev.e[3], ev.e[4]);
    ms_svd = ms_between(ev.e[4], ev.e[5]);
    saturated = rank > kp - pfix;
  }
  if (report) {
    report->rank_used = rank;
    report->probes_used = kp;
    report->saturated = saturated ? 1 : 0;
    report->sigma_first = 0;
    report->sigma_last_kept = 0;
    if (kp <= 256) {   // one copy of the (short) spectrum: both values from it
      double sg[256];
      AZ_CUDA_CHECK(cudaMemcpy(sg, w.sig, sizeof(double) * kp, cudaMemcpyDeviceToHost));
      report->sigma_first = sg[0];
      if (rank > 0) report->sigma_last_kept = sg[rank - 1];
    } else {
      AZ_CUDA_CHECK(cudaMemcpy(&report->sigma_first, w.sig, sizeof(double), cudaMemcpyDeviceToHost));
      if (rank > 0)
        AZ_CUDA_CHECK(cudaMemcpy(&report->sigma_last_kept, w.sig + rank - 1, sizeof(double), cudaMemcpyDeviceToHost));
    }
    report->ms_rhs = ms_between(ev.e[0], ev.e[1]);
    report->ms_sketch = ms_sketch;
    report->ms_qr = ms_qr;
    report->ms_svd = ms_svd;
    report->ms_step2 = ms_between(ev.e[6], ev.e[7]);
    report->ms_total = ms_between(ev.e[0], ev.e[7]);
    report->sigma = w.sig;
    report->n_sigma = kp;
  }
  return saturated ? AZ_WARN_SKETCH_SATURATED : AZ_OK;
}

// ------------------------------------------------------------------------------------------
// CUDA graphs of single-block narrow solves (one-CTA 1-D and narrow 2-D layouts): a solve whose
// arguments repeat (same b, x, workspace, theta, R, nrhs) is captured on its second call and replayed
// from then on -- one graph launch instead of a dozen kernel launches and stage-event records, which
// for a c1-sized solve are a fifth of its time.  The report (rank, spectrum, stage times) comes from
// pinned copies and external event nodes inside the graph.  AZ_SOLVE_GRAPH=0 disables; tracing
// (az_trace_enable) runs solves eagerly.
// ------------------------------------------------------------------------------------------
namespace {
struct SolveKey {
  const double* b = nullptr;
  int64_t ldb = 0;
  double* x = nullptr;
  int64_t ldx = 0, nrhs = 0;
  double theta = 0;
  int64_t R = 0;
  void* ws = nullptr;
  bool operator==(const SolveKey& o) const {
    return b == o.b && ldb == o.ldb && x == o.x && ldx == o.ldx && nrhs == o.nrhs && theta == o.theta && R == o.R &&
           ws == o.ws;
  }
};
struct GraphEntry {
  SolveKey key;
  cudaGraphExec_t exec = nullptr;
  int64_t* h_rank = nullptr;   // pinned
  double* h_sig = nullptr;     // pinned, kp values
  int64_t kp = 0;
  cudaEvent_t ev[8] = {};
};
void entry_free(GraphEntry& g) {
  if (g.exec) cudaGraphExecDestroy(g.exec);
  if (g.h_rank) cudaFreeHost(g.h_rank);
  if (g.h_sig) cudaFreeHost(g.h_sig);
  for (auto& e : g.ev)
    if (e) cudaEventDestroy(e);
  g = GraphEntry{};
}
bool graphs_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("AZ_SOLVE_GRAPH");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}
}  // namespace

struct az_graphs_s {
  static constexpr int kMax = 4;
  GraphEntry e[kMax];
  int n = 0, next = 0;
  SolveKey last;
  bool has_last = false;
  bool broken = false;   // a capture failed: this plan's solves stay eager
  cudaStream_t cap = nullptr;
};

void az_graphs_free(az_plan_s* p) {
  if (!p->graphs) return;
  for (int i = 0; i < p->graphs->n; ++i) entry_free(p->graphs->e[i]);
  if (p->graphs->cap) cudaStreamDestroy(p->graphs->cap);
  delete p->graphs;
  p->graphs = nullptr;
}

static bool graph_eligible(const az_plan_s* p, int64_t nrhs, int64_t R) {
  return graphs_on() && !az_trace_active() && p->layout != AZ_LAYOUT_1D_FOURSTEP && R + nrhs <= AZ_NARROW_MAX;
}

static az_status_t graph_capture(az_plan_s* p, const SolveKey& k, GraphEntry& g) {
  az_graphs_s* G = p->graphs;
  if (!G->cap) AZ_CUDA_CHECK(cudaStreamCreateWithFlags(&G->cap, cudaStreamNonBlocking));
  for (auto& e : g.ev) AZ_CUDA_CHECK(cudaEventCreate(&e));
  AZ_CUDA_CHECK(cudaHostAlloc((void**)&g.h_rank, sizeof(int64_t), cudaHostAllocDefault));
  AZ_CUDA_CHECK(cudaHostAlloc((void**)&g.h_sig, sizeof(double) * k.R, cudaHostAllocDefault));
  SolveTail tail;
  AZ_CUDA_CHECK(cudaStreamBeginCapture(G->cap, cudaStreamCaptureModeThreadLocal));
  az_status_t s = solve_impl(p, k.b, k.ldb, k.x, k.ldx, k.nrhs, k.theta, k.R, 1, k.ws, nullptr, G->cap, true, nullptr,
                             g.ev, &tail);
  if (s == AZ_OK && tail.rank_dev && tail.kp == k.R) {
    cudaMemcpyAsync(g.h_rank, tail.rank_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, G->cap);
    cudaMemcpyAsync(g.h_sig, tail.sig, sizeof(double) * tail.kp, cudaMemcpyDeviceToHost, G->cap);
  }
  cudaGraph_t graph = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(G->cap, &graph);
  if (s != AZ_OK || ce != cudaSuccess || !graph || !tail.rank_dev || tail.kp != k.R) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    az_set_error("az_solve: graph capture failed (%s)", cudaGetErrorString(ce));
    return s != AZ_OK ? s : AZ_ERR_CUDA;
  }
  const cudaError_t ie = cudaGraphInstantiate(&g.exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) {
    cudaGetLastError();
    g.exec = nullptr;
    az_set_error("az_solve: graph instantiation failed (%s)", cudaGetErrorString(ie));
    return AZ_ERR_CUDA;
  }
  g.key = k;
  g.kp = tail.kp;
  return AZ_OK;
}

// One single-block narrow solve from a graph; *used = false: the caller solves eagerly (first sighting
// of these arguments, or graphs unavailable).
static az_status_t graph_solve(az_plan_s* p, const SolveKey& k, az_solve_report_t* report, cudaStream_t st,
                               bool* used) {
  *used = false;
  if (!p->graphs) p->graphs = new az_graphs_s();
  az_graphs_s* G = p->graphs;
  if (G->broken) return AZ_OK;
  GraphEntry* g = nullptr;
  for (int i = 0; i < G->n; ++i)
    if (G->e[i].key == k) g = &G->e[i];
  if (!g) {
    if (!(G->has_last && G->last == k)) {
      G->last = k;
      G->has_last = true;
      return AZ_OK;
    }
    const int slot = G->n < az_graphs_s::kMax ? G->n++ : (G->next++ % az_graphs_s::kMax);
    entry_free(G->e[slot]);
    if (graph_capture(p, k, G->e[slot]) != AZ_OK) {
      entry_free(G->e[slot]);
      if (slot == G->n - 1) --G->n;
      G->broken = true;
      return AZ_OK;
    }
    g = &G->e[slot];
  }
  AZ_CUDA_CHECK(cudaGraphLaunch(g->exec, st));
  AZ_CUDA_CHECK(cudaStreamSynchronize(st));
  *used = true;
  const int64_t rank = *g->h_rank, kp = g->kp;
  const bool saturated = rank > kp - 10;
  if (report) {
    report->rank_used = rank;
    report->probes_used = kp;
    report->saturated = saturated ? 1 : 0;
    report->sigma_first = g->h_sig[0];
    report->sigma_last_kept = rank > 0 ? g->h_sig[rank - 1] : 0.0;
    report->ms_rhs = ms_between(g->ev[0], g->ev[1]);
    report->ms_sketch = ms_between(g->ev[2], g->ev[3]);
    report->ms_qr = ms_between(g->ev[3], g->ev[4]);
    report->ms_svd = ms_between(g->ev[4], g->ev[5]);
    report->ms_step2 = ms_between(g->ev[6], g->ev[7]);
    report->ms_total = ms_between(g->ev[0], g->ev[7]);
    report->sigma = layout(p, k.nrhs, k.R, 1, (char*)k.ws).sig;
    report->n_sigma = kp;
  }
  return saturated ? AZ_WARN_SKETCH_SATURATED : AZ_OK;
}

extern "C" int32_t az_solve_graph_count(az_plan_t p) { return p && p->graphs ? p->graphs->n : 0; }

// the single-block (first) attempt of az_solve: from a graph when eligible, else eagerly
static az_status_t solve_single(az_plan_s* p, const double* b, int64_t ldb, double* x, int64_t ldx, int64_t nrhs,
                                double theta, int64_t R, void* workspace, az_solve_report_t* report, cudaStream_t st) {
  if (graph_eligible(p, nrhs, R)) {
    SolveKey k;
    k.b = b;
    k.ldb = ldb;
    k.x = x;
    k.ldx = ldx;
    k.nrhs = nrhs;
    k.theta = theta;
    k.R = R;
    k.ws = workspace;
    bool used = false;
    const az_status_t s = graph_solve(p, k, report, st, &used);
    if (used || (s != AZ_OK && s != AZ_WARN_SKETCH_SATURATED)) return s;
  }
  return solve_impl(p, b, ldb, x, ldx, nrhs, theta, R, 1, workspace, report, st, false, nullptr);
}

extern "C" az_status_t az_solve(az_plan_t p, const double* b, int64_t ldb, double* x, int64_t ldx, int64_t nrhs,
                                double theta, int64_t R, int32_t max_blocks, void* workspace, size_t ws_bytes,
                                az_solve_report_t* report, void* stream) {
  if (!p || !b || !x || nrhs < 1 || R < 1 || max_blocks < 1 || !(theta >= 0.0) || ldb < p->M + p->Mb || ldx < p->N) {
    az_set_error("az_solve: bad arguments");
    return AZ_ERR_INVALID_ARGUMENT;
  }
  size_t need = 0;
  AZ_TRY(az_solve_workspace_size(p, nrhs, R, max_blocks, &need));
  if (!workspace || ws_bytes < need) {
    az_set_error("az_solve: workspace too small (%zu < %zu)", ws_bytes, need);
    return AZ_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  az_solve_report_t rep;
  memset(&rep, 0, sizeof(rep));
  double ms_first = 0.0;
  if (max_blocks == 1) {
    const az_status_t s = solve_single(p, b, ldb, x, ldx, nrhs, theta, R, workspace, &rep, st);
    if (s != AZ_OK && s != AZ_WARN_SKETCH_SATURATED) return s;
    if (report) *report = rep;
    return s;
  }
  if (narrow_first(nrhs, R, max_blocks)) {
    // the first probe block on the narrow path; kept unless it saturated
    const az_status_t s = solve_single(p, b, ldb, x, ldx, nrhs, theta, R, workspace, &rep, st);
    if (s != AZ_WARN_SKETCH_SATURATED) {
      if (report) *report = rep;
      return s;
    }
    ms_first = rep.ms_total;
    memset(&rep, 0, sizeof(rep));
  }
  const az_status_t s = solve_impl(p, b, ldb, x, ldx, nrhs, theta, R, max_blocks, workspace, &rep, st, false, nullptr);
  if (s != AZ_OK && s != AZ_WARN_SKETCH_SATURATED) return s;
  rep.ms_total += ms_first;
  if (report) *report = rep;
  return s;
}

// Host-buffer convenience (end-to-end timing: host->device copy of b, solve, device->host x).
extern "C" az_status_t az_solve_host(az_plan_t p, const double* b_host, double* x_host, int64_t nrhs, double theta,
                                     int64_t R, int32_t max_blocks, az_solve_report_t* report, void* stream) {
  if (!p || !b_host || !x_host || nrhs < 1) {
    az_set_error("az_solve_host: bad arguments");
    return AZ_ERR_INVALID_ARGUMENT;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rows = p->M + p->Mb;
  size_t need = 0;
  AZ_TRY(az_solve_workspace_size(p, nrhs, R, max_blocks, &need));
  const size_t bbytes = sizeof(double) * rows * nrhs, xbytes = sizeof(double) * p->N * nrhs;
  const size_t total = align256(need) + align256(bbytes) + align256(xbytes);
  if (p->d_solve_ws_bytes < total) {
    if (p->d_solve_ws) cudaFree(p->d_solve_ws);
    p->d_solve_ws = nullptr;
    p->d_solve_ws_bytes = 0;
    if (cudaMalloc(&p->d_solve_ws, total) != cudaSuccess) {
      az_set_error("az_solve_host: cudaMalloc(%zu) failed", total);
      return AZ_ERR_OUT_OF_MEMORY;
    }
    p->d_solve_ws_bytes = total;
  }
  char* base = (char*)p->d_solve_ws;
  double* db = (double*)(base + align256(need));
  double* dx = (double*)(base + align256(need) + align256(bbytes));
  // direct DMA when the caller's buffers are pinned (cudaHostAlloc / torch pin_memory)
  AZ_CUDA_CHECK(cudaMemcpyAsync(db, b_host, bbytes, cudaMemcpyHostToDevice, st));
  az_status_t s = az_solve(p, db, rows, dx, p->N, nrhs, theta, R, max_blocks, base, need, report, stream);
  if (s != AZ_OK && s != AZ_WARN_SKETCH_SATURATED) return s;
  AZ_CUDA_CHECK(cudaMemcpyAsync(x_host, dx, xbytes, cudaMemcpyDeviceToHost, st));
  AZ_CUDA_CHECK(cudaStreamSynchronize(st));
  return s;
}

// ==========================================================================================
// Factorisation reuse across right-hand sides (the
// step-1 matrix (A - A Z* A) Omega does not depend on b).  az_factorize draws and factors the
// sketch once -- blocked Householder with the panels (V, T) kept in place, and the truncated
// pseudo-inverse P = V_k Sigma_k^-1 U_k^T of R_S (the truncated SVD solve applied to c = I).
// az_solve_factored then costs b' = (I - A Z*) b, Q^T b' (the stored panels), y = P (Q^T b')[:k],
// x2 = Omega y and step 2 -- no sketch, no QR, no SVD.
// ==========================================================================================
struct az_factor_s {
  az_plan_s* p = nullptr;
  int64_t rows = 0, R = 0, kp = 0, kpmax = 0, rank = 0;
  bool saturated = false;
  double theta = 0.0, sigma_first = 0.0, sigma_last_kept = 0.0;
  double* S = nullptr;     // rows x kpmax, factored in place
  double* Tb = nullptr;    // panel T factors
  double* P = nullptr;     // kp x kp (ld kpmax)
  az_vbuf_s* Svb = nullptr;   // S's virtual range (physical HBM mapped per probe block), else cudaMalloc
  double* Q1 = nullptr;    // explicit leading kp columns of Q (rows x kp): S's own columns, in place
  double* Om = nullptr;    // explicit probes Omega (N x kp), the same Philox values as on the fly
  double* Mm = nullptr;    // four-step layout, <= 64 probes: M = Omega - Z* A Omega (N x kpmax), so a
                           // factored solve is x = Z* b + M y (no x2 = Omega y, no step-2 passes)
  std::vector<int64_t> pj0;
  std::vector<int> pnb;
  int64_t np = 0;
  double ms_sketch = 0, ms_qr = 0, ms_svd = 0;
};

__global__ void k_identity_cols(double* Rf, int64_t ld, int64_t k, int64_t col0) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= k * k) return;
  const int64_t i = e % k, c = e / k;
  Rf[(col0 + c) * ld + i] = (i == c) ? 1.0 : 0.0;
}

// Omega[:, col0 .. col0 + ncols) explicitly (N x ncols, ld N): the probe generator of a1
__global__ void k_omega_fill(int64_t N, int64_t col0, int64_t ncols, double* Om, uint64_t seed) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t npair = (N + 1) / 2;
  if (e >= npair * ncols) return;
  const int64_t m = e % npair, j = e / npair;
  const double2 z = probe_pair((uint64_t)m, (uint64_t)(col0 + j), seed);
  Om[j * N + 2 * m] = z.x;
  if (2 * m + 1 < N) Om[j * N + 2 * m + 1] = z.y;
}

// Omega of a four-step plan is not pointwise (spectral probes, reading R35): x (+)= Omega y by batches of
// whole probe pairs, each made explicit in the plan's C1 scratch (2 Bmax columns of N) and multiplied
// by the DMMA GEMM.
static az_status_t omega_apply_spectral(az_plan_s* p, int64_t col0, int64_t ncols, const double* y, int64_t ldy,
                                        int64_t nrhs, double* x, int64_t ldx, int accumulate, cudaStream_t st) {
  if (ncols <= 0 || nrhs <= 0) {
    if (!accumulate && nrhs > 0) {
      for (int64_t c = 0; c < nrhs; ++c) AZ_CUDA_CHECK(cudaMemsetAsync(x + c * ldx, 0, sizeof(double) * p->N, st));
    }
    return AZ_OK;
  }
  double* Om = reinterpret_cast<double*>(p->d_C1);
  const int64_t cap = 2 * p->Bmax, c0e = col0 & ~int64_t(1), cend = col0 + ncols;
  for (int64_t g0 = c0e; g0 < cend; g0 += cap) {
    const int64_t a0 = std::max(g0, col0), g1 = std::min(g0 + cap, cend);
    AZ_TRY(az1f_omega_fill(p, a0, g1 - a0, Om, p->N, st));
    const bool acc = accumulate || g0 > c0e;
    AzTrace tr("omega_apply", st, p->N * (g1 - a0) * nrhs);
    k_gemm_mn<<<dim3(az_div_up(p->N, 64), az_div_up(nrhs, 64)), 256, 0, st>>>(Om, p->N, y + (a0 - col0), ldy, x, ldx, p->N,
                                                                              g1 - a0, nrhs, acc ? x : nullptr, ldx, 1.0);
    AZ_LAUNCH_CHECK();
  }
  return AZ_OK;
}

// The two factored-solve products for many right-hand sides on the FP64 tensor path (DMMA
// m8n8k4; same FP64 peak as DFMA on B200, but 256 multiply-adds per warp instruction).
//
// Y (m x n) = A (m x k, ld lda) B (k x n, ld ldb): CTA tile 64 rows x 64 columns, k in steps of 32;
// warps 2 (rows) x 4 (columns), 32 x 16 each.
constexpr int GS = 36;   // operand tile stride (== 4 mod 16: conflict-free fragments)
__global__ void __launch_bounds__(256) k_gemm_mn(const double* A, int64_t lda, const double* Bm, int64_t ldb, double* Y,
                                                 int64_t ldy, int64_t m, int64_t k, int64_t n, const double* C,
                                                 int64_t ldc, double sgn) {   // C non-null: Y = C + sgn A B
  __shared__ double As[32 * 68];   // KMAJ [k][row], stride 68 (== 4 mod 16)
  __shared__ double Bs[32 * 68];   // KMAJ [k][col]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wm = w & 1, wn = w >> 1;
  const int64_t r0 = (int64_t)blockIdx.x * 64, c0 = (int64_t)blockIdx.y * 64;
  double acc[4][2][2];
  acc_zero(acc);
  for (int64_t k0 = 0; k0 < k; k0 += 32) {
    __syncthreads();
    for (int e = tid; e < 32 * 64; e += 256) {
      const int kk = e >> 6, i = e & 63;      // A: rows contiguous in memory
      As[kk * 68 + i] = (r0 + i < m && k0 + kk < k) ? A[(k0 + kk) * lda + r0 + i] : 0.0;
      const int cc = e >> 5, k2 = e & 31;     // B: k contiguous in memory
      Bs[k2 * 68 + cc] = (c0 + cc < n && k0 + k2 < k) ? Bm[(c0 + cc) * ldb + k0 + k2] : 0.0;
    }
    __syncthreads();
    warp_mma<4, 2, KMAJ, KMAJ>(acc, As, 68, Bs, 68, wm * 32, wn * 16, 0, 32, lane);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t r = r0 + acc_row(wm * 32, i, lane), cc = c0 + acc_col(wn * 16, j, e, lane);
        if (r < m && cc < n) Y[cc * ldy + r] = C ? fma(sgn, acc[i][j][e], C[cc * ldc + r]) : acc[i][j][e];
      }
}

// Y = C - A B for a tall A (m x k) and a small B (k x n), k <= 64, n <= 64 (step 2 of the four-step
// narrow solve: r = b - (A Omega) y): B is staged in shared memory once per CTA and the CTA walks
// row tiles of 64 (grid-stride), so the small operand is not re-read per tile.
__global__ void __launch_bounds__(256) k_gemm_mn_small(const double* A, int64_t lda, const double* Bm, int64_t ldb,
                                                       double* Y, int64_t ldy, int64_t m, int k, int n, const double* C,
                                                       int64_t ldc, double sgn) {
  extern __shared__ double gsm[];
  double* As = gsm;                // KMAJ [k][row], 64 x 68
  double* Bs = gsm + 64 * 68;      // KMAJ [k][col]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wm = w & 1, wn = w >> 1;
  const int kp = (k + 3) & ~3;
  for (int e = tid; e < 64 * 64; e += 256) {
    const int cc = e >> 6, kk = e & 63;
    Bs[kk * 68 + cc] = (cc < n && kk < k) ? Bm[(int64_t)cc * ldb + kk] : 0.0;
  }
  // the next row tile's A values and this tile's C fragments are fetched into registers while the
  // current tile's MMAs run
  double va[16], cf[4][2][2];
  const int li = tid & 63, lk0 = tid >> 6;   // A element (row li, k = lk0 + 4 t)
  auto load_a = [&](int64_t r0) {
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int kk = lk0 + 4 * t;
      va[t] = (r0 + li < m && kk < k) ? A[(int64_t)kk * lda + r0 + li] : 0.0;
    }
  };
  auto load_c = [&](int64_t r0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t r = r0 + acc_row(wm * 32, i, lane);
          const int cc = acc_col(wn * 16, j, e, lane);
          cf[i][j][e] = (C && r < m && cc < n) ? C[(int64_t)cc * ldc + r] : 0.0;
        }
  };
  const int64_t stride = (int64_t)gridDim.x * 64;
  int64_t r0 = (int64_t)blockIdx.x * 64;
  if (r0 < m) load_a(r0);
  for (; r0 < m; r0 += stride) {
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 16; ++t) As[(lk0 + 4 * t) * 68 + li] = va[t];
    __syncthreads();
    load_c(r0);
    if (r0 + stride < m) load_a(r0 + stride);
    double acc[4][2][2];
    acc_zero(acc);
    warp_mma<4, 2, KMAJ, KMAJ>(acc, As, 68, Bs, 68, wm * 32, wn * 16, 0, kp, lane);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t r = r0 + acc_row(wm * 32, i, lane);
          const int cc = acc_col(wn * 16, j, e, lane);
          if (r < m && cc < n) Y[(int64_t)cc * ldy + r] = C ? fma(sgn, acc[i][j][e], cf[i][j][e]) : acc[i][j][e];
        }
  }
}

// Wpart[kc] (k x n) = A[rows of chunk kc]^T B[rows of chunk kc]  (A: m x k, B: m x n, column-major):
// CTA tile 64 (A columns) x 64 (B columns); warps 2 x 2 x 2 (the last splits each 32-row step in
// halves, reduced through shared memory at the end)
__global__ void __launch_bounds__(256) k_gemm_tn_part(const double* A, int64_t lda, const double* Bm, int64_t ldb,
                                                      double* Wpart, int64_t m, int64_t k, int64_t n, int64_t kchunk) {
  __shared__ double smv[2 * 64 * GS];
  double* As = smv;                 // IMAJ [A column][row]
  double* Bs = smv + 64 * GS;       // IMAJ [B column][row]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wm = w & 1, wn = (w >> 1) & 1, wk = w >> 2;
  const int64_t i0 = (int64_t)blockIdx.x * 64, n0 = (int64_t)blockIdx.y * 64;
  const int64_t rb = (int64_t)blockIdx.z * kchunk, re = min(m, rb + kchunk);
  double acc[4][4][2];
  acc_zero(acc);
  const int lk = tid & 31, li = tid >> 5;   // load slots: element (column li + 8 t, row lk)
  double va[8], vb[8];
  auto load = [&](int64_t rr) {
    const int64_t r = rr + lk;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int i = li + 8 * t;
      va[t] = (r < re && i0 + i < k) ? A[(i0 + i) * lda + r] : 0.0;
      vb[t] = (r < re && n0 + i < n) ? Bm[(n0 + i) * ldb + r] : 0.0;
    }
  };
  if (rb < re) load(rb);
  for (int64_t rr = rb; rr < re; rr += 32) {
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      As[(li + 8 * t) * GS + lk] = va[t];
      Bs[(li + 8 * t) * GS + lk] = vb[t];
    }
    __syncthreads();
    if (rr + 32 < re) load(rr + 32);   // next tile in flight during the MMAs
    warp_mma<4, 4, IMAJ, IMAJ>(acc, As, GS, Bs, GS, wm * 32, wn * 32, wk * 16, 16, lane);
  }
  __syncthreads();
  double* rs = smv + (w & 3) * 32 * 33;   // reduce the two row halves (scratch reuses the tiles)
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
    double* W = Wpart + (int64_t)blockIdx.z * k * n;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int ml = acc_row(0, i, lane), nl = acc_col(0, j, e, lane);
          const int64_t ii = i0 + wm * 32 + ml, nn = n0 + wn * 32 + nl;
          if (ii < k && nn < n) W[nn * k + ii] = acc[i][j][e] + rs[ml * 33 + nl];
        }
  }
}

// Memory-bound forms of the two factored-solve products for few right-hand sides (NR <= 8 per
// pass): every element of the tall factor is read once per pass, the small operand is staged in
// shared memory, and the split over the long dimension is summed in a fixed order (k_sum_parts).
//
// part[z][r][i] = sum_{q in row chunk z} A[q, i] B[q, r]      (A: m x k, B: m x NR, col-major)
template <int NR>
__global__ void __launch_bounds__(256, 2) k_tsgemv_tn(const double* A, int64_t lda, const double* Bm, int64_t ldb,
                                                   double* part, int64_t m, int64_t k, int64_t nrhs_total, int rc) {
  extern __shared__ double bs[];                 // rc x NR, column r at bs + r * rc
  const int64_t q0 = (int64_t)blockIdx.y * rc;
  const int rn = (int)(m - q0 < rc ? m - q0 : (int64_t)rc);
  for (int e = threadIdx.x; e < rc * NR; e += 256) {
    const int r = e / rc, q = e % rc;
    bs[e] = q < rn ? Bm[(int64_t)r * ldb + q0 + q] : 0.0;
  }
  __syncthreads();
  // a warp takes 4 columns at a time, so each staged b' value read from shared memory feeds 4
  // loaded elements (one read per element would make the pass shared-memory bound at NR = 8)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t cend = (k < (int64_t)blockIdx.x * 64 + 64 ? k : (int64_t)blockIdx.x * 64 + 64);
  for (int64_t i0 = (int64_t)blockIdx.x * 64 + 4 * w; i0 < cend; i0 += 32) {
    const double* a[4];
    bool ok[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      ok[c] = i0 + c < cend;
      a[c] = A + (ok[c] ? i0 + c : i0) * lda + q0;
    }
    double acc[4][NR];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int r = 0; r < NR; ++r) acc[c][r] = 0.0;
    int q = lane;
    for (; q + 3 * 32 < rn; q += 4 * 32) {
      double v[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < 4; ++c) v[u][c] = ok[c] ? __ldcs(a[c] + q + 32 * u) : 0.0;   // streamed once
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const double bv = bs[r * rc + q + 32 * u];
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[c][r] = fma(v[u][c], bv, acc[c][r]);
        }
    }
    for (; q < rn; q += 32) {
      double v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = ok[c] ? __ldcs(a[c] + q) : 0.0;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const double bv = bs[r * rc + q];
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[c][r] = fma(v[c], bv, acc[c][r]);
      }
    }
    // warp reduction of the V = 4 NRP partial sums by recursive halving: each step trades half of
    // the values with the partner lane, so V - 1 + (5 - log2 V) shuffles instead of 5 V
    constexpr int NRP = NR <= 1 ? 1 : NR <= 2 ? 2 : NR <= 4 ? 4 : 8, V = 4 * NRP;
    constexpr int LV = V == 4 ? 2 : V == 8 ? 3 : V == 16 ? 4 : 5;
    double vals[V];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int r = 0; r < NRP; ++r) vals[c * NRP + r] = r < NR ? acc[c][r] : 0.0;
#pragma unroll
    for (int t = 0; t < LV; ++t) {
      const int sft = 16 >> t, h = V >> (t + 1);
      const bool up = (lane & sft) != 0;
#pragma unroll
      for (int i = 0; i < h; ++i) {
        const double send = up ? vals[i] : vals[i + h];
        const double keep = up ? vals[i + h] : vals[i];
        vals[i] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
      }
    }
#pragma unroll
    for (int o = (16 >> LV); o > 0; o >>= 1) vals[0] += __shfl_xor_sync(0xffffffffu, vals[0], o);
    if ((lane & ((32 >> LV) - 1)) == 0) {
      const int idx = lane >> (5 - LV), c = idx / NRP, r = idx % NRP;
      if (r < NR && ok[c]) part[((int64_t)blockIdx.y * nrhs_total + r) * k + i0 + c] = vals[0];
    }
  }
}

// part[z][r][j] = sum_{i in column chunk z} A[j, i] y[i, r]   (A: m x k col-major, y: k x NR)
template <int NR>
__global__ void __launch_bounds__(256) k_tsgemv_nn(const double* A, int64_t lda, const double* y, int64_t ldy,
                                                   double* part, int64_t m, int64_t k, int64_t nrhs_total, int kc) {
  extern __shared__ double ys[];                 // kc x NR, row i at ys + i * NR
  const int64_t i0 = (int64_t)blockIdx.y * kc;
  const int kn = (int)(k - i0 < kc ? k - i0 : (int64_t)kc);
  for (int e = threadIdx.x; e < kc * NR; e += 256) {
    const int i = e / NR, r = e % NR;
    ys[e] = i < kn ? y[(int64_t)r * ldy + i0 + i] : 0.0;
  }
  __syncthreads();
  const int64_t j0 = (int64_t)blockIdx.x * 512 + threadIdx.x;
  const bool ok0 = j0 < m, ok1 = j0 + 256 < m;
  double acc0[NR], acc1[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc0[r] = acc1[r] = 0.0;
  const double* a = A + i0 * lda;
  int i = 0;
  for (; i + 4 <= kn; i += 4) {
    double v0[4], v1[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      v0[u] = ok0 ? __ldcs(a + (int64_t)(i + u) * lda + j0) : 0.0;
      v1[u] = ok1 ? __ldcs(a + (int64_t)(i + u) * lda + j0 + 256) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const double yy = ys[(i + u) * NR + r];
        acc0[r] = fma(v0[u], yy, acc0[r]);
        acc1[r] = fma(v1[u], yy, acc1[r]);
      }
  }
  for (; i < kn; ++i) {
    const double v0 = ok0 ? a[(int64_t)i * lda + j0] : 0.0, v1 = ok1 ? a[(int64_t)i * lda + j0 + 256] : 0.0;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      acc0[r] = fma(v0, ys[i * NR + r], acc0[r]);
      acc1[r] = fma(v1, ys[i * NR + r], acc1[r]);
    }
  }
  double* pz = part + (int64_t)blockIdx.y * nrhs_total * m;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    if (ok0) pz[r * m + j0] = acc0[r];
    if (ok1) pz[r * m + j0 + 256] = acc1[r];
  }
}

__global__ void k_sum_parts(const double* Wpart, int64_t KC, int64_t len, double* out, int64_t k, int64_t ldo) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= len) return;
  double t = 0.0;
  for (int64_t kc = 0; kc < KC; ++kc) t += Wpart[kc * len + e];   // fixed order
  out[(e / k) * ldo + (e % k)] = t;
}

extern "C" az_status_t az_factorize(az_plan_t p, double theta, int64_t R, int32_t max_blocks, az_factor_t* out,
                                    az_solve_report_t* report, void* stream) {
  if (!p || !out || R < 1 || max_blocks < 1 || !(theta >= 0.0)) {
    az_set_error("az_factorize: bad arguments");
    return AZ_ERR_INVALID_ARGUMENT;
  }
  *out = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  az_factor_s* f = new az_factor_s();
  f->p = p;
  f->rows = p->M + p->Mb;
  f->R = R;
  f->theta = theta;
  max_blocks = (int32_t)std::min<int64_t>(max_blocks, std::max<int64_t>(1, f->rows / R));   // probes <= rows
  f->kpmax = R * max_blocks;
  const int64_t rows = f->rows, kpmax = f->kpmax;
  if (kpmax > rows) {
    delete f;
    az_set_error("az_factorize: %lld probe columns exceed the %lld rows", (long long)kpmax, (long long)rows);
    return AZ_ERR_NOT_SUPPORTED;
  }
  const int64_t QBw = az_qrw_panel_width();
  const int64_t maxpanels = max_blocks * ((R + QBw - 1) / QBw);
  f->pj0.resize(maxpanels);
  f->pnb.resize(maxpanels);
  const size_t qrbytes = az_qrw_ws_bytes(rows, R);
  const size_t svdbytes = az_tsvd_ws_bytes(kpmax, kpmax);
  double *Rf = nullptr, *sig = nullptr;
  void *qrws = nullptr, *svdws = nullptr;
  auto fail = [&](az_status_t s) {
    cudaFree(Rf);
    cudaFree(sig);
    cudaFree(qrws);
    cudaFree(svdws);
    az_factor_destroy(f);
    return s;
  };
  // S grows by one probe block at a time: reserve the address range for kpmax columns and map HBM
  // per block, so a factorisation that stops early never holds the unused tail
  f->Svb = az_vbuf_reserve(sizeof(double) * rows * kpmax);
  if (f->Svb) f->S = (double*)az_vbuf_ptr(f->Svb);
  if ((!f->Svb && cudaMalloc(&f->S, sizeof(double) * rows * kpmax) != cudaSuccess) ||
      cudaMalloc(&f->Tb, sizeof(double) * maxpanels * QBw * QBw) != cudaSuccess ||
      cudaMalloc(&f->P, sizeof(double) * kpmax * kpmax) != cudaSuccess ||
      cudaMalloc(&Rf, sizeof(double) * kpmax * 2 * kpmax) != cudaSuccess ||
      cudaMalloc(&sig, sizeof(double) * kpmax) != cudaSuccess || cudaMalloc(&qrws, qrbytes) != cudaSuccess ||
      cudaMalloc(&svdws, svdbytes) != cudaSuccess) {
    az_set_error("az_factorize: out of device memory");
    return fail(AZ_ERR_OUT_OF_MEMORY);
  }
  // four-step layout with at most 64 probes: keep A Omega (step 2 of a factored solve is then one
  // small GEMM and three FFT passes)
  if (p->layout == AZ_LAYOUT_1D_FOURSTEP && kpmax <= 64 && step2_linear(p) &&
      cudaMalloc(&f->Mm, sizeof(double) * p->N * kpmax) != cudaSuccess) {
    cudaGetLastError();
    f->Mm = nullptr;
  }
  const int pfix = 10;
  double s1lo = 0.0;
  int64_t nb = 0, rank = 0;
  bool saturated = true;
  Ev ev;
  for (nb = 1; nb <= max_blocks; ++nb) {
    const int64_t kp = nb * R;
    cudaEventRecord(ev.e[2], st);
    double* Snew = f->S + (nb - 1) * R * rows;
    if (f->Svb && !az_vbuf_ensure(f->Svb, sizeof(double) * rows * kp)) {
      az_set_error("az_factorize: out of device memory (probe block %lld)", (long long)nb);
      return fail(AZ_ERR_OUT_OF_MEMORY);
    }
    az_status_t s = f->Mm ? az1f_sketch_m(p, (nb - 1) * R, R, Snew, rows, f->Mm + (nb - 1) * R * p->N, p->N, st)
                          : az_sketch(p, (nb - 1) * R, R, Snew, rows, st);
    if (s != AZ_OK) return fail(s);
    cudaEventRecord(ev.e[3], st);
    if ((s = az_qrw_apply(f->S, rows, rows, f->pj0.data(), f->pnb.data(), f->Tb, 0, f->np, Snew, rows, R, qrws, qrbytes, st)) != AZ_OK ||
        (s = az_qrw_factor(f->S, rows, rows, (nb - 1) * R, kp, f->Tb, f->pj0.data(), f->pnb.data(), &f->np, qrws,
                           qrbytes, st)) != AZ_OK ||
        (s = az_qrw_extract_R(f->S, rows, kp, Rf, kpmax, st)) != AZ_OK)
      return fail(s);
    cudaEventRecord(ev.e[4], st);
    bool full_svd = true;
    if (nb >= 2 && nb < max_blocks) {   // the R22 pre-test of az_solve (reading R5)
      const int64_t off = (nb - 1) * R;
      int64_t k22 = 0;
      if ((s = az_tsvd_impl(Rf + off * kpmax + off, kpmax, R, 0, theta, f->P, R, sig, &k22, svdws, svdbytes, st)) != AZ_OK)
        return fail(s);
      std::vector<double> s22(R);
      if (cudaMemcpyAsync(s22.data(), sig, sizeof(double) * R, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
          cudaStreamSynchronize(st) != cudaSuccess)
        return fail(AZ_ERR_CUDA);
      s1lo = std::max(s1lo, s22[0]);
      k22 = 0;
      for (int64_t i = 0; i < R; ++i) k22 += s22[i] > theta * s1lo;
      full_svd = k22 <= R - pfix;
      rank = kp;
    }
    if (full_svd) {
      // [R_S | I]: the truncated SVD solve of the identity is P = V_k Sigma_k^-1 U_k^T
      k_identity_cols<<<az_div_up(kp * kp, 256), 256, 0, st>>>(Rf, kpmax, kp, kp);
      if (cudaGetLastError() != cudaSuccess) return fail(AZ_ERR_CUDA);
      if ((s = az_tsvd_impl(Rf, kpmax, kp, kp, theta, f->P, kpmax, sig, &rank, svdws, svdbytes, st)) != AZ_OK)
        return fail(s);
      double sv[2] = {0, 0};
      cudaMemcpyAsync(&sv[0], sig, sizeof(double), cudaMemcpyDeviceToHost, st);
      if (rank > 0) cudaMemcpyAsync(&sv[1], sig + rank - 1, sizeof(double), cudaMemcpyDeviceToHost, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) return fail(AZ_ERR_CUDA);
      s1lo = std::max(s1lo, sv[0]);
      f->sigma_first = sv[0];
      f->sigma_last_kept = sv[1];
    }
    cudaEventRecord(ev.e[5], st);
    cudaEventSynchronize(ev.e[5]);
    f->ms_sketch += ms_between(ev.e[2], ev.e[3]);
    f->ms_qr += ms_between(ev.e[3], ev.e[4]);
    f->ms_svd += ms_between(ev.e[4], ev.e[5]);
    saturated = rank > kp - pfix;
    if (!saturated || nb == max_blocks) break;
  }
  if (nb > max_blocks) nb = max_blocks;
  f->kp = nb * R;
  f->rank = rank;
  f->saturated = saturated;
  cudaFree(Rf);
  cudaFree(sig);
  cudaFree(svdws);
  Rf = sig = nullptr;
  svdws = nullptr;
  // explicit Q1 = Q [I_kp; 0], formed in place of S's first kp columns (the panels' V and T are not
  // needed afterwards), and Omega (N x kp): a factored solve then streams each once instead of
  // re-applying every Householder panel and regenerating the probes.  S's unused tail is returned
  // first; Omega is kept only if it fits, else it is regenerated per solve.
  {
    const char* fe = getenv("AZ_FACTOR_EXPLICIT");
    if (!(fe && fe[0] == '0')) {
      const int64_t kp = f->kp;
      if (cudaStreamSynchronize(st) != cudaSuccess) return fail(AZ_ERR_CUDA);
      if (f->Svb) az_vbuf_trim(f->Svb, sizeof(double) * rows * kp);
      az_status_t s2 = az_qrw_form_q(f->S, rows, rows, f->pj0.data(), f->pnb.data(), f->Tb, f->np, kp, qrws, qrbytes, st);
      if (s2 != AZ_OK) return fail(s2);
      f->Q1 = f->S;
      cudaFree(f->Tb);
      f->Tb = nullptr;
      if (!f->Mm && cudaMalloc(&f->Om, sizeof(double) * p->N * kp) == cudaSuccess) {
        AzTrace tr("omega_fill", st);
        if (p->layout == AZ_LAYOUT_1D_FOURSTEP) {   // spectral probes (reading R35)
          const az_status_t s3 = az1f_omega_fill(p, 0, kp, f->Om, p->N, st);
          if (s3 != AZ_OK) return fail(s3);
        } else {
          k_omega_fill<<<az_div_up(((p->N + 1) / 2) * kp, 256), 256, 0, st>>>(p->N, 0, kp, f->Om, p->seed);
        }
        if (cudaGetLastError() != cudaSuccess) return fail(AZ_ERR_CUDA);
      } else {
        cudaGetLastError();
        f->Om = nullptr;
      }
      if (cudaStreamSynchronize(st) != cudaSuccess) return fail(AZ_ERR_CUDA);
    }
  }
  cudaFree(qrws);
  if (report) {
    memset(report, 0, sizeof(*report));
    report->rank_used = f->rank;
    report->probes_used = f->kp;
    report->saturated = f->saturated ? 1 : 0;
    report->sigma_first = f->sigma_first;
    report->sigma_last_kept = f->sigma_last_kept;
    report->ms_sketch = f->ms_sketch;
    report->ms_qr = f->ms_qr;
    report->ms_svd = f->ms_svd;
    report->ms_total = f->ms_sketch + f->ms_qr + f->ms_svd;
  }
  *out = f;
  return saturated ? AZ_WARN_SKETCH_SATURATED : AZ_OK;
}

extern "C" az_status_t az_factor_destroy(az_factor_t f) {
  if (!f) return AZ_OK;
  if (f->Svb)
    az_vbuf_free(f->Svb);
  else
    cudaFree(f->S);
  cudaFree(f->Tb);
  cudaFree(f->P);
  cudaFree(f->Om);
  cudaFree(f->Mm);
  delete f;
  return AZ_OK;
}

extern "C" az_status_t az_factor_query(az_factor_t f, int64_t* probes, int64_t* rank) {
  if (!f) return AZ_ERR_INVALID_ARGUMENT;
  if (probes) *probes = f->kp;
  if (rank) *rank = f->rank;
  return AZ_OK;
}

// the memory-bound tsgemv passes below this many right-hand sides, tiled FMA GEMMs above
static bool fac_small(int64_t nrhs) { return nrhs <= 16; }      // Q1^T b'
static bool fac_small_nn(int64_t nrhs) { return nrhs <= 40; }   // P c, Omega y

static int nr_slots(int64_t nrhs) {
  const int64_t r = std::min<int64_t>(8, nrhs);
  return r <= 1 ? 1 : r <= 2 ? 2 : r <= 4 ? 4 : 8;
}

// split of the tsgemv_nn product Y (m x nrhs) = A (m x k) y: column chunk kc (y chunk staged in
// <= 32 KB of shared memory), enough chunks to give ~4 CTAs per SM
static int64_t nn_kc(int64_t m, int64_t k, int64_t nrhs) {
  const int64_t zc = std::max<int64_t>(1, az_div_up(4 * 148, az_div_up(m, 512)));
  return std::min<int64_t>(4096 / nr_slots(nrhs), std::max<int64_t>(32, az_div_up(az_div_up(k, zc), 32) * 32));
}
static int64_t nn_part_elems(int64_t m, int64_t k, int64_t nrhs) {
  return fac_small_nn(nrhs) ? az_div_up(k, nn_kc(m, k, nrhs)) * m * nrhs : 0;
}

// Y (m x nrhs, ld ldo) = A (m x k, ld lda) y (k x nrhs, ld ldy)
static az_status_t nn_product(const double* A, int64_t lda, int64_t m, int64_t k, const double* y, int64_t ldy,
                              double* Y, int64_t ldo, int64_t nrhs, double* part, cudaStream_t st) {
  if (!fac_small_nn(nrhs)) {
    k_gemm_mn<<<dim3(az_div_up(m, 64), az_div_up(nrhs, 64)), 256, 0, st>>>(A, lda, y, ldy, Y, ldo, m, k, nrhs);
    AZ_LAUNCH_CHECK();
    return AZ_OK;
  }
  const int64_t kc = nn_kc(m, k, nrhs), KCn = az_div_up(k, kc);
  for (int64_t g0 = 0; g0 < nrhs; g0 += 8) {
    const int nr = (int)std::min<int64_t>(8, nrhs - g0);
    const size_t smn = sizeof(double) * kc * nr;
    const dim3 gn(az_div_up(m, 512), (unsigned)KCn);
#define AZ_TSGEMV_NN(NR)                                                                                    \
  case NR:                                                                                                  \
    AZ_CUDA_CHECK(az_smem_attr(k_tsgemv_nn<NR>, smn));                                                      \
    k_tsgemv_nn<NR><<<gn, 256, smn, st>>>(A, lda, y + g0 * ldy, ldy, part + g0 * m, m, k, nrhs, (int)kc); \
    break;
    switch (nr) {
      AZ_TSGEMV_NN(1)
      AZ_TSGEMV_NN(2)
      AZ_TSGEMV_NN(3)
      AZ_TSGEMV_NN(4)
      AZ_TSGEMV_NN(5)
      AZ_TSGEMV_NN(6)
      AZ_TSGEMV_NN(7)
      AZ_TSGEMV_NN(8)
    }
#undef AZ_TSGEMV_NN
    AZ_LAUNCH_CHECK();
  }
  k_sum_parts<<<az_div_up(m * nrhs, 256), 256, 0, st>>>(part, KCn, m * nrhs, Y, m, ldo);
  AZ_LAUNCH_CHECK();
  return AZ_OK;
}

struct FacWS {
  double *bp, *y, *x2, *tmp, *c, *part;
  int64_t KC, rc, KCt;   // tiled split-K count; tsgemv row chunk and count
  void* qrws;
  size_t qrbytes, total;
};

static FacWS fac_layout(az_factor_s* f, int64_t nrhs, char* base) {
  FacWS w;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* ptr = base ? base + off : nullptr;
    off += align256(bytes);
    return ptr;
  };
  w.bp = (double*)take(sizeof(double) * f->rows * nrhs);
  w.y = (double*)take(sizeof(double) * f->kp * nrhs);
  w.x2 = (double*)take(sizeof(double) * f->p->N * nrhs);
  w.tmp = (double*)take(sizeof(double) * f->rows * nrhs);
  w.c = (double*)take(sizeof(double) * f->kp * nrhs);
  // tiled split-K: enough row chunks for ~2 CTAs per SM over the (kp / 64) x (nrhs / 64) output tiles
  const int64_t tiles = (int64_t)az_div_up(f->kp, 64) * az_div_up(nrhs, 64);
  w.KC = std::max<int64_t>(1, std::min<int64_t>(az_div_up(2 * 148, tiles), f->rows / 1024));
  w.rc = 8192 / nr_slots(nrhs);                        // 64 KB of staged b' per CTA
  w.KCt = az_div_up(f->rows, w.rc);
  const int64_t parts = std::max({(fac_small(nrhs) ? w.KCt : w.KC) * f->kp * nrhs,
                                  nn_part_elems(f->kp, f->kp, nrhs), nn_part_elems(f->p->N, f->kp, nrhs)});
  w.part = (double*)take(sizeof(double) * parts);
  w.qrbytes = f->Q1 ? 0 : az_qrw_ws_bytes(f->rows, nrhs);
  w.qrws = f->Q1 ? nullptr : take(w.qrbytes);
  w.total = off;
  return w;
}

extern "C" az_status_t az_factor_workspace_size(az_factor_t f, int64_t nrhs, size_t* bytes) {
  if (!f || !bytes || nrhs < 1) return AZ_ERR_INVALID_ARGUMENT;
  *bytes = fac_layout(f, nrhs, nullptr).total;
  return AZ_OK;
}

extern "C" az_status_t az_solve_factored(az_factor_t f, const double* b, int64_t ldb, double* x, int64_t ldx,
                                         int64_t nrhs, void* workspace, size_t ws_bytes, az_solve_report_t* report,
                                         void* stream) {
  if (!f || !b || !x || nrhs < 1 || ldb < f->rows || ldx < f->p->N) {
    az_set_error("az_solve_factored: bad arguments");
    return AZ_ERR_INVALID_ARGUMENT;
  }
  FacWS w = fac_layout(f, nrhs, nullptr);
  if (!workspace || ws_bytes < w.total) {
    az_set_error("az_solve_factored: workspace too small (%zu < %zu)", ws_bytes, w.total);
    return AZ_ERR_WORKSPACE;
  }
  w = fac_layout(f, nrhs, (char*)workspace);
  az_plan_s* p = f->p;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rows = f->rows, kp = f->kp;
  Ev ev;
  cudaEventRecord(ev.e[0], st);
  const bool use_m = f->Mm && kp <= 64;
  if (use_m)   // b' = (I - A Z*) b and Z* b (into the x2 slot)
    AZ_TRY(az1f_resid_z(p, b, ldb, w.bp, rows, w.x2, p->N, nrhs, st));
  else
    AZ_TRY(az_apply_op(p, OP_RESID, b, ldb, w.bp, rows, nrhs, st));          // b' = (I - A Z*) b
  cudaEventRecord(ev.e[1], st);
  if (!f->Q1) {
    // compact form: Q^T b' through the Householder panels, y = P (Q^T b')[:kp], x2 = Omega y regenerated
    AZ_TRY(az_qrw_apply(f->S, rows, rows, f->pj0.data(), f->pnb.data(), f->Tb, 0, f->np, w.bp, rows, nrhs, w.qrws,
                        w.qrbytes, st));
    {
      AzTrace tr("factored_y", st, 2 * kp * kp * nrhs);
      AZ_TRY(nn_product(f->P, f->kpmax, kp, kp, w.bp, rows, w.y, kp, nrhs, w.part, st));   // y = P (Q^T b')[:kp]
    }
    cudaEventRecord(ev.e[2], st);
    if (!use_m) AZ_TRY(omega_apply(p, 0, kp, w.y, kp, nrhs, w.x2, p->N, 0, st));
  } else {
    // c = Q1^T b' (split-K over the rows, ordered reduction), y = P c, x2 = Omega y
    {
    AzTrace tr("fac_qtb", st, sizeof(double) * (rows + kp) * kp);
    if (fac_small(nrhs)) {
      for (int64_t g0 = 0; g0 < nrhs; g0 += 8) {
        const int nr = (int)std::min<int64_t>(8, nrhs - g0);
        const size_t smt = sizeof(double) * w.rc * nr;
        const dim3 gt(az_div_up(kp, 64), w.KCt);
#define AZ_TSGEMV_TN(NR)                                                                                         \
  case NR:                                                                                                       \
    AZ_CUDA_CHECK(az_smem_attr(k_tsgemv_tn<NR>, smt));                                                           \
    k_tsgemv_tn<NR><<<gt, 256, smt, st>>>(f->Q1, rows, w.bp + g0 * rows, rows, w.part + g0 * kp, rows, kp, nrhs, \
                                          (int)w.rc);                                                           \
    break;
        switch (nr) {
          AZ_TSGEMV_TN(1)
          AZ_TSGEMV_TN(2)
          AZ_TSGEMV_TN(3)
          AZ_TSGEMV_TN(4)
          AZ_TSGEMV_TN(5)
          AZ_TSGEMV_TN(6)
          AZ_TSGEMV_TN(7)
          AZ_TSGEMV_TN(8)
        }
#undef AZ_TSGEMV_TN
        AZ_LAUNCH_CHECK();
      }
      k_sum_parts<<<az_div_up(kp * nrhs, 256), 256, 0, st>>>(w.part, w.KCt, kp * nrhs, w.c, kp, kp);
      AZ_LAUNCH_CHECK();
    } else {
      const int64_t kchunk = (rows + w.KC - 1) / w.KC;
      k_gemm_tn_part<<<dim3(az_div_up(kp, 64), az_div_up(nrhs, 64), (unsigned)w.KC), 256, 0, st>>>(
          f->Q1, rows, w.bp, rows, w.part, rows, kp, nrhs, kchunk);
      AZ_LAUNCH_CHECK();
      k_sum_parts<<<az_div_up(kp * nrhs, 256), 256, 0, st>>>(w.part, w.KC, kp * nrhs, w.c, kp, kp);
      AZ_LAUNCH_CHECK();
    }
    AZ_TRY(nn_product(f->P, f->kpmax, kp, kp, w.c, kp, w.y, kp, nrhs, w.part, st));   // y = P c
    }
    cudaEventRecord(ev.e[2], st);
    const int64_t N = p->N;
    if (!use_m) {
      AzTrace tr2("fac_omega_y", st, sizeof(double) * N * kp);
      if (!f->Om)
        AZ_TRY(omega_apply(p, 0, kp, w.y, kp, nrhs, w.x2, N, 0, st));   // Omega did not fit: regenerated
      else
        AZ_TRY(nn_product(f->Om, N, N, kp, w.y, kp, w.x2, N, nrhs, w.part, st));
    }
  }
  if (use_m) {
    // x = Z* b + M y  (M = Omega - Z* A Omega kept at factorisation, Z* b from the b' chain)
    AzTrace tr("step2_gemm", st, 2 * p->N * kp * nrhs);
    const size_t gs = 2 * 64 * 68 * sizeof(double);
    AZ_CUDA_CHECK(az_smem_attr(k_gemm_mn_small, gs));
    for (int64_t c0 = 0; c0 < nrhs; c0 += 64)
      k_gemm_mn_small<<<gemm_small_grid(p->N), 256, gs, st>>>(
          f->Mm, p->N, w.y + c0 * kp, kp, x + c0 * ldx, ldx, p->N, (int)kp, (int)std::min<int64_t>(64, nrhs - c0),
          w.x2 + c0 * p->N, p->N, 1.0);
    AZ_LAUNCH_CHECK();
  } else {
    AZ_TRY(step2(p, w.x2, b, ldb, x, ldx, w.tmp, nrhs, st));
  }
  cudaEventRecord(ev.e[3], st);
  AZ_CUDA_CHECK(cudaEventSynchronize(ev.e[3]));
  if (report) {
    memset(report, 0, sizeof(*report));
    report->rank_used = f->rank;
    report->probes_used = kp;
    report->saturated = f->saturated ? 1 : 0;
    report->sigma_first = f->sigma_first;
    report->sigma_last_kept = f->sigma_last_kept;
    report->ms_rhs = ms_between(ev.e[0], ev.e[1]);
    report->ms_qr = ms_between(ev.e[1], ev.e[2]);
    report->ms_step2 = ms_between(ev.e[2], ev.e[3]);
    report->ms_total = ms_between(ev.e[0], ev.e[3]);
  }
  return AZ_OK;
}

// ==========================================================================================
// Pipelined host-buffer solves: az_solve_host_pipelined enqueues H2D of b (upload stream),
// the solve (caller's stream) and D2H of x (download stream) and returns; consecutive calls
// overlap one step's upload and the previous step's download with the current solve (two device
// slots).  x_host holds the result once az_plan_sync returns.  Host buffers should be pinned.
// ==========================================================================================
struct az_pipe_s {
  cudaStream_t up = nullptr, down = nullptr;
  double* bdev[2] = {nullptr, nullptr};
  double* xdev[2] = {nullptr, nullptr};
  void* ws = nullptr;
  size_t ws_bytes = 0;
  cudaEvent_t ev_up[2], ev_solved[2], ev_down[2];
  int slot = 0;
  int64_t nrhs = 0, R = 0;
  int32_t mb = 0;
};

static void pipe_free(az_pipe_s* q) {
  if (!q) return;
  if (q->up) cudaStreamSynchronize(q->up);
  if (q->down) cudaStreamSynchronize(q->down);
  for (int i = 0; i < 2; ++i) {
    cudaFree(q->bdev[i]);
    cudaFree(q->xdev[i]);
    cudaEventDestroy(q->ev_up[i]);
    cudaEventDestroy(q->ev_solved[i]);
    cudaEventDestroy(q->ev_down[i]);
  }
  cudaFree(q->ws);
  if (q->up) cudaStreamDestroy(q->up);
  if (q->down) cudaStreamDestroy(q->down);
  delete q;
}

void az_pipe_destroy(az_plan_s* p) {
  pipe_free(p->pipe);
  p->pipe = nullptr;
}

extern "C" az_status_t az_solve_host_pipelined(az_plan_t p, const double* b_host, double* x_host, int64_t nrhs,
                                               double theta, int64_t R, int32_t max_blocks, void* stream) {
  if (!p || !b_host || !x_host || nrhs < 1 || R < 1 || max_blocks < 1) {
    az_set_error("az_solve_host_pipelined: bad arguments");
    return AZ_ERR_INVALID_ARGUMENT;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rows = p->M + p->Mb;
  az_pipe_s* q = p->pipe;
  if (!q || q->nrhs != nrhs || q->R != R || q->mb != max_blocks) {
    az_pipe_destroy(p);
    q = new az_pipe_s();
    p->pipe = q;
    q->nrhs = nrhs;
    q->R = R;
    q->mb = max_blocks;
    AZ_TRY(az_solve_workspace_size(p, nrhs, R, max_blocks, &q->ws_bytes));
    bool ok = cudaStreamCreateWithFlags(&q->up, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&q->down, cudaStreamNonBlocking) == cudaSuccess &&
              cudaMalloc(&q->ws, q->ws_bytes) == cudaSuccess;
    for (int i = 0; i < 2 && ok; ++i)
      ok = cudaMalloc(&q->bdev[i], sizeof(double) * rows * nrhs) == cudaSuccess &&
           cudaMalloc(&q->xdev[i], sizeof(double) * p->N * nrhs) == cudaSuccess &&
           cudaEventCreateWithFlags(&q->ev_up[i], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&q->ev_solved[i], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&q->ev_down[i], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
      az_pipe_destroy(p);
      az_set_error("az_solve_host_pipelined: out of device memory");
      return AZ_ERR_OUT_OF_MEMORY;
    }
  }
  const int sl = q->slot;
  q->slot ^= 1;
  // upload after the solve that last read this slot has finished
  AZ_CUDA_CHECK(cudaStreamWaitEvent(q->up, q->ev_solved[sl], 0));
  AZ_CUDA_CHECK(cudaMemcpyAsync(q->bdev[sl], b_host, sizeof(double) * rows * nrhs, cudaMemcpyHostToDevice, q->up));
  AZ_CUDA_CHECK(cudaEventRecord(q->ev_up[sl], q->up));
  // solve once the upload is in and the slot's previous result has been downloaded
  AZ_CUDA_CHECK(cudaStreamWaitEvent(st, q->ev_up[sl], 0));
  AZ_CUDA_CHECK(cudaStreamWaitEvent(st, q->ev_down[sl], 0));
  if (!p->d_satflag) {
    AZ_CUDA_CHECK(cudaMalloc(&p->d_satflag, sizeof(int)));
    AZ_CUDA_CHECK(cudaMemsetAsync(p->d_satflag, 0, sizeof(int), st));
  }
  // one probe block: enqueued without a host synchronisation (saturation lands in the plan's device
  // flag, read by az_plan_sync); adaptive solves need the rank on the host and synchronise
  az_status_t s = max_blocks == 1
                      ? solve_impl(p, q->bdev[sl], rows, q->xdev[sl], p->N, nrhs, theta, R, 1, q->ws, nullptr, st,
                                   true, p->d_satflag)
                      : az_solve(p, q->bdev[sl], rows, q->xdev[sl], p->N, nrhs, theta, R, max_blocks, q->ws,
                                 q->ws_bytes, nullptr, stream);
  if (s != AZ_OK && s != AZ_WARN_SKETCH_SATURATED) return s;
  AZ_CUDA_CHECK(cudaEventRecord(q->ev_solved[sl], st));
  AZ_CUDA_CHECK(cudaStreamWaitEvent(q->down, q->ev_solved[sl], 0));
  AZ_CUDA_CHECK(cudaMemcpyAsync(x_host, q->xdev[sl], sizeof(double) * p->N * nrhs, cudaMemcpyDeviceToHost, q->down));
  AZ_CUDA_CHECK(cudaEventRecord(q->ev_down[sl], q->down));
  return s;
}

extern "C" az_status_t az_plan_sync(az_plan_t p) {
  if (!p) return AZ_ERR_INVALID_ARGUMENT;
  if (p->pipe) {
    AZ_CUDA_CHECK(cudaStreamSynchronize(p->pipe->up));
    AZ_CUDA_CHECK(cudaStreamSynchronize(p->pipe->down));
  }
  AZ_CUDA_CHECK(cudaDeviceSynchronize());
  if (p->d_satflag) {
    int f = 0;
    AZ_CUDA_CHECK(cudaMemcpy(&f, p->d_satflag, sizeof(int), cudaMemcpyDeviceToHost));
    AZ_CUDA_CHECK(cudaMemset(p->d_satflag, 0, sizeof(int)));
    if (f) return AZ_WARN_SKETCH_SATURATED;
  }
  return AZ_OK;
}
