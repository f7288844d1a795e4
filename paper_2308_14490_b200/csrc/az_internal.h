// Internal plan structure and cross-file declarations of libaz.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "az_common.cuh"

enum az_layout_t {
  AZ_LAYOUT_1D_SMALL = 0,   // 1-D, L = s n <= 2048: whole chain per vector pair in one CTA
  AZ_LAYOUT_1D_FOURSTEP = 1,// 1-D, n > 1024: four-step [N1][N2] / [N1][L2] layout, 5 HBM passes
  AZ_LAYOUT_2D = 2          // 2-D, [x][y] row-major, y contiguous
};

// Operation selectors shared by the pass kernels.
enum az_op_t { OP_A = 0, OP_AT = 1, OP_ZSTAR = 2, OP_STEP1 = 3, OP_RESID = 4, OP_STEP2 = 5 };

// Input sources for coefficient-space entry.
enum az_src_t { SRC_VEC = 0, SRC_PROBE = 1 };

struct az_pipe_s;   // az_solve_host_pipelined state (az_solve.cu)
void az_pipe_destroy(struct az_plan_s* p);

struct az_plan_s {
  // geometry
  int dim;
  int64_t n, s, L;          // L = s n grid points per axis (2-D: the x axis)
  int64_t ny = 0, Ly = 0;   // 2-D: centres / grid points along y (== n, L for square boxes)
  int64_t N, G;             // n (1-D) or n ny; L (1-D) or L Ly
  int64_t M, Mb;
  double T, eps, alpha, beta, rcond;
  double Ty = 0.0;          // 2-D: half-period along y
  double k0sq = 0.0;            // Helmholtz term of LAPLACIAN rows
  uint64_t seed;
  int op;
  int layout;
  // four-step factorisation (1-D large): n = N1 N2, L = N1 L2
  int64_t N1, N2, L2;
  // device tables
  uint8_t* d_mask = nullptr;    // G
  int32_t* d_pos = nullptr;     // G: row index of an interior grid point, -1 outside
  int64_t run0 = -1, run1 = -1; // the mask is the single run [run0, run1) of the natural grid order
                                // (1-D intervals): row = g - run0, no table lookups
  cplx* d_W0 = nullptr;         // fine symbol, order 0 (per axis length L; four-step: [N1][L2])
  cplx* d_W2 = nullptr;         // fine symbol, order 2 (Laplacian)
  cplx* d_W0y = nullptr;        // 2-D: the y axis' symbols (alias d_W0 / d_W2 when the box is square)
  cplx* d_W2y = nullptr;
  double* d_Wr = nullptr;       // four-step layout: the row symbol (W0, or alpha W2) as a real table
                                // (phi^per samples are real and even, so W is real up to rounding)
  double* d_zinv = nullptr;     // N: 1/sigma^2(k) if kept else 0 (coefficient spectrum order)
  cplx* d_tw = nullptr;         // TWN-point twiddle table e^{-2 pi i t / TWN}
  cplx* d_tw4hi = nullptr;      // four-step twiddles e^{-2 pi i (h 2^TW4B) / L}
  cplx* d_tw4lo = nullptr;      // e^{-2 pi i l / L}
  double* d_bxy = nullptr;      // Mb x 2 boundary points
  int win = 0;                  // boundary stencil width (centres along x; 1-D: the axis), <= 64
  int win_y = 0;                // 2-D: along y
  double* d_bw = nullptr;       // Mb x 2 x 64 separable stencil weights phi^per(x_b - c_j)
  int32_t* d_bj = nullptr;      // Mb x 2 first centre index of the window (mod n on use)
  // scratch for the pass kernels
  int64_t Bmax = 0;             // max vector PAIRS per batch
  cplx* d_C1 = nullptr;         // Bmax * N complex
  cplx* d_Z2 = nullptr;         // four-step: Bmax * N complex (Z* outputs of the b' / sketch chains)
  cplx* d_G = nullptr;          // Bmax * G complex
  // host-side info
  double sigma_max2 = 0, sigma_min_kept2 = 0;
  int64_t n_dropped = 0;
  // pinned host staging for az_solve_host
  double* h_stage = nullptr;
  size_t h_stage_bytes = 0;
  void* d_solve_ws = nullptr;
  size_t d_solve_ws_bytes = 0;
  az_pipe_s* pipe = nullptr;
  int* d_satflag = nullptr;     // set by pipelined solves whose sketch saturated; read by az_plan_sync
  // side stream of az_solve: the Z* b / M column passes (and, deferred, Q^T b') run beside the TSQR
  // merges and the SVD; side_ev: [0] TSQR leaf done, [1] R_S merged, [2] the side stream's work done
  cudaStream_t side = nullptr;
  cudaEvent_t side_ev[3] = {nullptr, nullptr, nullptr};
  // second side stream: the Z* b column pass beside the right-hand-side merge passes, once pass B is
  // done (side2_ev: [0] pass B done, [1] Z* b done)
  cudaStream_t side2 = nullptr;
  cudaEvent_t side2_ev[2] = {nullptr, nullptr};
  // high-priority stream for the TSQR and the SVD while the side stream runs: the block scheduler
  // then hands freed SMs to the merge tree (the critical path) before the side stream's passes
  cudaStream_t hi = nullptr;
  // CUDA graphs of repeated single-block narrow solves (az_solve.cu)
  struct az_graphs_s* graphs = nullptr;
};
void az_graphs_free(az_plan_s* p);
bool az_trace_active();

constexpr int TWN = 2048;
constexpr int TW4B = 11;

// --- 1-D small layout (az_ops1d.cu)
// zout (OP_STEP1 / OP_RESID only): also write M = Omega - Z* A Omega / Z* b (N x nvec, ld ldz)
az_status_t az1s_apply(az_plan_s* p, int op, int src, const double* in, int64_t ldin, double* out,
                       int64_t ldout, int64_t nvec, int64_t col0, cudaStream_t st, double* zout = nullptr,
                       int64_t ldz = 0);
az_status_t az1s_fft_table(az_plan_s* p, cplx* data, int64_t len, cudaStream_t st);

// --- 1-D four-step layout (az_ops1f.cu)
az_status_t az1f_apply(az_plan_s* p, int op, int src, const double* in, int64_t ldin, double* out,
                       int64_t ldout, int64_t nvec, int64_t col0, cudaStream_t st);
az_status_t az1f_fft_fine_forward(az_plan_s* p, cplx* data, cudaStream_t st);
az_status_t az1f_step2(az_plan_s* p, const double* x2, int64_t ldx2, const double* b, int64_t ldb, double* x,
                       int64_t ldx, int64_t nvec, cudaStream_t st);
// b' = (I - A Z*) b that also returns Z* b (N x nvec); the sketch that also returns
// M = Omega - Z* A Omega (N x ncols, written over the kept Omega)
// Zspec: the spectrum buffer (B x N complex; null = the plan's d_Z2); defer: leave the closing column
// pass to az1f_out_z (single batch only), so it can run on another stream
az_status_t az1f_resid_z(az_plan_s* p, const double* b, int64_t ldb, double* bp, int64_t ldbp, double* Zb, int64_t ldz,
                         int64_t nvec, cudaStream_t st, cplx* Zspec = nullptr, bool defer = false);
az_status_t az1f_sketch_m(az_plan_s* p, int64_t col0, int64_t ncols, double* S, int64_t ldS, double* Om, int64_t ldOm,
                          cudaStream_t st, cplx* Zspec = nullptr, bool defer = false);
az_status_t az1f_out_z(az_plan_s* p, const cplx* Zspec, double* out, int64_t ldout, int64_t nvec, cudaStream_t st,
                       bool background = false);
// Omega[:, col0 .. col0 + ncols) of a four-step plan's spectral probes (reading R35), N x ncols, ld ldOm
az_status_t az1f_omega_fill(az_plan_s* p, int64_t col0, int64_t ncols, double* Om, int64_t ldOm, cudaStream_t st);

// --- 2-D layout (az_ops2d.cu)
az_status_t az2_apply(az_plan_s* p, int op, int src, const double* in, int64_t ldin, double* out,
                      int64_t ldout, int64_t nvec, int64_t col0, cudaStream_t st);

// generic FFT of `count` contiguous vectors of length len (len <= 2048) in place
az_status_t az_fft_batch(const cplx* tw, cplx* data, int64_t len, int64_t count, int dir, cudaStream_t st);

// --- QR / SVD / solve
// a_scratch: A may be overwritten (the solve's sketch buffer), which enables the split TSQR leaf
// after_leaf (optional): recorded once the leaf passes are enqueued (before the merge tree)
az_status_t az_qr_r_impl(double* A, int64_t m, int64_t k, int64_t lda, double* R, int64_t ldr,
                         void* ws, size_t ws_bytes, cudaStream_t st, int64_t k1 = 0, bool a_scratch = false,
                         cudaEvent_t after_leaf = nullptr);
size_t az_qr_ws_bytes(int64_t m, int64_t k);
// pass A of the split leaf as a blocked QR with look-ahead (az_qr_la.cu): 256-row chunks, P CTAs of
// rows_per_cta rows; Y (in place of A's k1 columns), taus and the per-CTA R factors as k_tsqr's pass A
bool az_tsqr_la_enabled();
int az_tsqr_la_mc();   // chunk rows of the look-ahead leaf (AZ_TSQR_LA_MC: 256 or 128)
az_status_t az_tsqr_la_leaf(const double* A, int64_t m, int k1, int64_t ld, int64_t rows_per_cta, int P, double* Rout,
                            int64_t ostride, double* Y, int64_t ldY, double* taus, int cmax, cudaStream_t st,
                            int64_t rb = 0, int64_t bstride = 0);
bool az_tsqr_la_merge_enabled();   // AZ_TSQR_LA_MERGE (default 1): merge levels by the look-ahead kernel
// R_S of the k1 probe columns on st (ev_leaf / ev_merged recorded there), then (Q^T b')[:k1] of the
// k - k1 right-hand-side columns on rhs_st (k1, k - k1 <= 64; A is scratch) (az_qr.cu)
az_status_t az_qr_r_deferred(double* A, int64_t m, int64_t k, int64_t k1, int64_t lda, double* Rs, int64_t ldrs,
                             void* ws, size_t ws_bytes, cudaStream_t st, cudaEvent_t ev_leaf, cudaEvent_t ev_merged);
az_status_t az_qr_rhs_deferred(double* A, int64_t m, int64_t k, int64_t k1, int64_t lda, double* C, int64_t ldc,
                               void* ws, size_t ws_bytes, cudaStream_t rhs_st, cudaEvent_t ev_leaf,
                               cudaEvent_t ev_merged, cudaEvent_t ev_passb = nullptr);
// rank_out: HOST, filled synchronously (may be null); rank_dev (optional): receives the DEVICE
// address where the rank lands on `st` (valid while ws is)
az_status_t az_tsvd_impl(const double* Rf, int64_t ldr, int64_t r, int64_t nrhs, double theta,
                         double* y, int64_t ldy, double* sigma_out, int64_t* rank_out,
                         void* ws, size_t ws_bytes, cudaStream_t st, const int64_t** rank_dev = nullptr);
size_t az_tsvd_ws_bytes(int64_t r, int64_t nrhs);

// --- wide (2-D) dense path: blocked Householder QR (az_qrw.cu), block Jacobi SVD (az_svdw.cu)
constexpr int64_t AZ_NARROW_MAX = 128;    // k <= this: single-pass TSQR / single-CTA Jacobi
int64_t az_qrw_panel_width();
size_t az_qrw_ws_bytes(int64_t m, int64_t ncols_max);
az_status_t az_qrw_apply(const double* V, int64_t ldv, int64_t m, const int64_t* pj0, const int* pnb,
                         const double* Tbuf, int64_t p0, int64_t p1, double* C, int64_t ldc, int64_t nt, void* ws,
                         size_t ws_bytes, cudaStream_t st);
az_status_t az_qrw_apply_q(const double* V, int64_t ldv, int64_t m, const int64_t* pj0, const int* pnb,
                           const double* Tbuf, int64_t p0, int64_t p1, double* C, int64_t ldc, int64_t nt, void* ws,
                           size_t ws_bytes, cudaStream_t st);
az_status_t az_qrw_factor(double* A, int64_t lda, int64_t m, int64_t c0, int64_t c1, double* Tbuf, int64_t* pj0,
                          int* pnb, int64_t* np, void* ws, size_t ws_bytes, cudaStream_t st);
az_status_t az_qrw_extract_R(const double* A, int64_t lda, int64_t k, double* R, int64_t ldr, cudaStream_t st);
// Q1 = Q [I_kp; 0] formed in place of the factored columns [0, kp) (LAPACK dorgqr order: panels
// from the last to the first); every panel must start below kp and end at or before it
az_status_t az_qrw_form_q(double* A, int64_t lda, int64_t m, const int64_t* pj0, const int* pnb, const double* Tbuf,
                          int64_t np, int64_t kp, void* ws, size_t ws_bytes, cudaStream_t st);

// growable device buffer on the virtual-memory API (az_vmm.cu); nullptr when unavailable
struct az_vbuf_s;
az_vbuf_s* az_vbuf_reserve(size_t max_bytes);
void* az_vbuf_ptr(az_vbuf_s* v);
bool az_vbuf_ensure(az_vbuf_s* v, size_t bytes);
void az_vbuf_trim(az_vbuf_s* v, size_t bytes);
size_t az_vbuf_mapped(az_vbuf_s* v);
void az_vbuf_free(az_vbuf_s* v);
size_t az_tsvdw_ws_bytes(int64_t r, int64_t nrhs);
az_status_t az_tsvdw_impl(const double* Rf, int64_t ldr, int64_t r, int64_t nrhs, double theta, double* y,
                          int64_t ldy, double* sigma_out, int64_t* rank_out, void* ws, size_t ws_bytes,
                          cudaStream_t st, int max_sweeps, int* sweeps_out, const int64_t** rank_dev = nullptr);


// Optional per-launch CUDA-event tracing (az_trace_enable): records an event pair around each
// traced launch on the launching stream; az_trace_report sums the durations per kernel name.
struct AzTrace {
  AzTrace(const char* name, cudaStream_t st, int64_t units = 0);
  ~AzTrace();
  int slot;
  cudaStream_t st;
};

inline unsigned az_div_up(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }
