/*
 * az.h -- C ABI of libaz: the data-parallel hot path of the AZ algorithm for
 * oversampled periodised-Gaussian RBF collocation (arXiv:2308.14490, PAPER.md),
 * hand-written for NVIDIA B200 (sm_100a), FP64 / complex128 throughout.
 *
 * The path (Alg. 1, with Z* = F B^dag P E):
 *   step 1   solve (I - A Z*) A x2 = (I - A Z*) b with the randomized low-rank solver
 *            (PAPER.md:257, 269): S = (A - A Z* A) Omega, truncated SVD, x2 = Omega y
 *   step 2   x1 = Z* (b - A x2)
 *   step 3   x  = x1 + x2
 *
 * Conventions (all entry points):
 *   - Every vector/matrix argument is a caller-owned DEVICE pointer to float64 data,
 *     column-major, `nvec` columns with leading dimension ld >= rows, unless stated.
 *   - Coefficient vectors (length N = n^dim) are in natural row-major order of the
 *     centres, j = jx*n + jy.
 *   - Row vectors (length M + Mb) hold the M interior collocation rows in natural
 *     row-major order of the oversampled grid (x outer), then the Mb boundary rows
 *     in the caller's order.  The paper orders the
 *     interior rows like Pi X~; a row permutation does not change
 *     the least-squares problem, and the polyphase order is internal only.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     All calls are asynchronous on `stream` unless stated; the library never
 *     synchronises the device except where a host result is returned.
 *   - A plan owns scratch that its calls share: calls on one plan must be ordered by the
 *     caller (one stream, or explicit stream dependencies); different plans are independent.
 *     az_solve may run parts of a solve on internal streams of the plan (a side stream and a
 *     high-priority stream); their work is joined back into `stream` by events before the
 *     solve's last kernel, so stream order on `stream` still holds.
 *   - Errors are status codes; no C++ exception crosses the ABI.  Arguments are
 *     validated before any launch and outputs are untouched on argument errors.
 *     az_last_error() returns a thread-local detail string for the last failure.
 *   - There is no CPU fallback: every arithmetic step runs in libaz's kernels.
 */
#ifndef AZ_H_
#define AZ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct az_plan_s* az_plan_t;

typedef enum {
  AZ_OK = 0,
  AZ_ERR_INVALID_ARGUMENT = 1,
  AZ_ERR_OVERSAMPLING = 2,      /* M + Mb <= N: "choose s large enough such that M > N" */
  AZ_ERR_SINGULAR_SYMBOL = 3,   /* max_k sigma(k) == 0 (SPEC.md:188 singular-symbol)                */
  AZ_ERR_OUT_OF_MEMORY = 4,
  AZ_ERR_CUDA = 5,
  AZ_ERR_NOT_SUPPORTED = 6,     /* size/oversampling outside the supported FFT lengths              */
  AZ_ERR_WORKSPACE = 7,         /* workspace too small                                              */
  AZ_ERR_NCCL = 8,              /* a collective of the multi-GPU solve failed (NCCL error or async error) */
  AZ_WARN_SKETCH_SATURATED = 100 /* rank == probes - p after max_blocks probe blocks (x still written) */
} az_status_t;

typedef enum {
  AZ_ROW_VALUE = 0,      /* interior rows phi_j(x_i) (function approximation) */
  AZ_ROW_LAPLACIAN = 1   /* interior rows row_scale * (d2/dx2 + d2/dy2) phi_j(x_i), PAPER.md:741-752 with k0^2 = 0 */
} az_row_op_t;

/* Plan descriptor.  Box [-T, T)^dim, n centres per axis c_j = -T + j 2T/n,
 * oversampled grid of L*n points per axis x_q = -T + q 2T/(L n).
 * Supported: dim = 1 with n a power of two in [16, 2^21]; dim = 2 with n a power of two in
 * [8, 1024] (and n_y, see below); L in {1, 2, 4} (2-D: L = 2) with L*n <= 2048 per 2-D axis. */
typedef struct {
  int32_t dim;                 /* 1 or 2 */
  int64_t n;                   /* centres per axis (paper N, N^x = N^y) */
  int32_t L;                   /* oversampling factor per axis (paper s; BASELINE "L") */
  double T;                    /* half-period of the box (paper T) */
  double eps;                  /* Gaussian shape parameter */
  int32_t op;                  /* az_row_op_t */
  double row_scale;            /* alpha: interior rows and data scaled by it (-1/(2 eps^2)) */
  const uint8_t* mask;         /* HOST, (L n)^dim bytes, natural row-major (x outer); 1 = collocation point
                                  (PAPER.md:121-123, 587-589).  Deep-copied. */
  int64_t n_boundary;          /* Mb (0 if none) */
  const double* boundary_xy;   /* HOST, Mb x dim row-major points; deep-copied */
  double boundary_weight;      /* beta: boundary rows are beta * phi_j(x_b) */
  double zstar_rcond;          /* Z* keeps modes with sigma(k) > rcond * max sigma (reading R3) */
  uint64_t seed;               /* Philox key of the probe matrix Omega */
  double k0sq;                 /* Helmholtz term: LAPLACIAN rows are alpha (Delta + k0^2) phi_j
                                  (PAPER.md:694-722 1-D ODE, 730-806 2-D; 0 = Poisson).  Ignored for VALUE. */
  int64_t n_y;                 /* 2-D anisotropic boxes ("N = N^x N^y", 644-647): centres along y,
                                  a power of two with n/2 <= n_y <= 2n and L*n_y <= 2048; 0 = n.  The box is
                                  [-T, T) x [-T_y, T_y), centres c_j = (-T + jx 2T/n, -T_y + jy 2T_y/n_y),
                                  column j = jx n_y + jy; the mask is (L n) x (L n_y), x outer.  Ignored in 1-D. */
  double T_y;                  /* half-period along y (0 = T).  eps is one isotropic shape parameter. */
  const double* boundary_coef; /* HOST, Mb x 4 row-major [a, b, n_x, n_y] (2-D only): boundary row k is
                                  beta (a phi_j + b n . grad phi_j)(x_k) -- Dirichlet (a = 1, b = 0), Neumann
                                  (a = 0) or Robin rows (the flower of PAPER.md:839-846: Neumann on the outer,
                                  Dirichlet on the inner boundary).  NULL = all Dirichlet.  Deep-copied. */
} az_plan_desc_t;

typedef struct {
  int64_t N;          /* columns n^dim */
  int64_t M;          /* interior rows */
  int64_t Mb;         /* boundary rows */
  double sigma_max;   /* largest singular value of the periodic A^c (unitary normalisation, Lemma 3) */
  double sigma_min_kept;
  int64_t n_dropped;  /* Z* modes below the threshold */
  double zstar_norm;  /* ||Z*||_2 = 1 / sigma_min_kept */
} az_plan_info_t;

/* Build the plan (step 0): kernel samples and their DFTs (Lemma 3,
 * PAPER.md:344-353) for the symbol of B, sigma(k)^2 = sum_i |d_i(k)|^2 and the thresholded
 * pseudo-inverse diagonals, mask packing, device scratch.
 * Synchronises `stream` once (reads back sigma_max).  *out receives the plan. */
az_status_t az_plan_create(const az_plan_desc_t* desc, void* stream, az_plan_t* out);
az_status_t az_plan_destroy(az_plan_t plan);
az_status_t az_plan_query(az_plan_t plan, az_plan_info_t* info);

/* y (M+Mb x nvec) = A x (N x nvec).  A = [R P* B F* ; beta A^b].  */
az_status_t az_apply_A(az_plan_t plan, const double* x, int64_t ldx, double* y, int64_t ldy,
                       int64_t nvec, void* stream);
/* x (N x nvec) = A^T y (M+Mb x nvec).  The adjoint of az_apply_A.            */
az_status_t az_apply_At(az_plan_t plan, const double* y, int64_t ldy, double* x, int64_t ldx,
                        int64_t nvec, void* stream);
/* x (N x nvec) = Z* y.  Z* = [F B^dag P E, 0_{N x Mb}]:
 * the boundary rows of y are ignored.                                                        */
az_status_t az_apply_Zstar(az_plan_t plan, const double* y, int64_t ldy, double* x, int64_t ldx,
                           int64_t nvec, void* stream);
/* y (M+Mb x nvec) = (A - A Z* A) v  -- the step-1 operator.                */
az_status_t az_apply_step1(az_plan_t plan, const double* v, int64_t ldv, double* y, int64_t ldy,
                           int64_t nvec, void* stream);
/* y (M+Mb x nvec) = (I - A Z*) b  -- the step-1 right-hand side.              */
az_status_t az_apply_resid(az_plan_t plan, const double* b, int64_t ldb, double* y, int64_t ldy,
                           int64_t nvec, void* stream);

/* S[:, 0:ncols] = (A - A Z* A) Omega[:, col0 : col0+ncols] with Omega generated on the fly
 * (Philox4x32-10 keyed by plan seed and GLOBAL column index; probes never stored).
 * PAPER.md:269 "r+p matrix vector products".  Used by az_solve and by multi-GPU drivers that
 * shard probe columns.  S is (M+Mb) x ncols, leading dimension ldS.
 * Probe definition (reading R35): 1-D plans with s n > 2048 (the four-step layout) draw
 * column pair P = (2P, 2P+1) in the frequency domain -- Re / Im of IFFT_n(v_P), v_P[k] =
 * sqrt(n) (z0 + i z1), (z0, z1) = Box-Muller of Philox counter (k, P + 2^63) -- i.i.d. N(0,1)
 * columns like the entrywise probes (Omega[2m, j], Omega[2m+1, j] from counter (m, j)) of every
 * other plan.  Any col0 (an odd col0 computes its first pair and discards the real column).   */
az_status_t az_sketch(az_plan_t plan, int64_t col0, int64_t ncols, double* S, int64_t ldS,
                      void* stream);
/* x (N x nrhs) (+)= Omega[:, col0 : col0+ncols] y  (y: ncols x nrhs, DEVICE).  accumulate = 0
 * overwrites x.  Regenerates Omega (a9 of SURVEY.md §8(a)); spectral probes (four-step plans)
 * are made explicit per batch of pairs in the plan's scratch and applied by a DMMA GEMM.      */
az_status_t az_omega_apply(az_plan_t plan, int64_t col0, int64_t ncols, const double* y, int64_t ldy,
                           int64_t nrhs, double* x, int64_t ldx, int accumulate, void* stream);

/* Steps 2 and 3 of Alg. 1 for a given step-1 solution: x = x2 + Z* (b - A x2).
 * x2: N x nrhs (ld ldx2), b: (M+Mb) x nrhs (ld ldb), x: N x nrhs (ld ldx), all DEVICE; x must not
 * alias x2 or b.  Used by multi-GPU drivers for their right-hand-side shard (az_solve does the same
 * internally).  workspace: az_step2_workspace_size bytes of DEVICE scratch (0 for the 1-D four-step
 * layout, which runs the correction as one fused five-pass chain).  Asynchronous on stream.       */
az_status_t az_step2_workspace_size(az_plan_t plan, int64_t nrhs, size_t* bytes);
az_status_t az_step2(az_plan_t plan, const double* x2, int64_t ldx2, const double* b, int64_t ldb, double* x,
                     int64_t ldx, int64_t nrhs, void* workspace, size_t ws_bytes, void* stream);

/* R factor of a tall matrix by Householder TSQR (no Q is formed; "SVD of an
 * (r+p)-by-M matrix" done as QR + small SVD).  A: m x k DEVICE column-major (ld lda), k <= 128
 * for the single-pass TSQR; larger k uses blocked Householder (A is overwritten, needs m >= k).
 * Rout: k x k upper-triangular DEVICE, leading dimension ldr (strict lower part zeroed).
 * Rows may be in any order (QR is row-permutation equivariant).                              */
az_status_t az_qr_r(az_plan_t plan, double* A, int64_t m, int64_t k, int64_t lda,
                    double* Rout, int64_t ldr, void* workspace, size_t ws_bytes, void* stream);
az_status_t az_qr_workspace_size(int64_t m, int64_t k, size_t* bytes);
/* Same, triangularising only the leading k1 <= k columns (k <= 128, single-pass TSQR): Rout is
 * k1 x k = [R_11 | (Q_1^T A[:, k1:])[:k1]], i.e. the right-hand sides riding along in the last
 * k - k1 columns come out as Q^T b' (the multi-GPU solve merges such factors from row blocks).
 * Workspace as for az_qr_r(m, k).  AZ_ERR_NOT_SUPPORTED if k > 128 and k1 < k.                 */
az_status_t az_qr_r_partial(az_plan_t plan, double* A, int64_t m, int64_t k, int64_t k1, int64_t lda,
                            double* Rout, int64_t ldr, void* workspace, size_t ws_bytes, void* stream);

/* Truncated least squares on the QR-reduced sketch: with Rf = [R_S | c] (R_S: r x r upper
 * triangular, c: r x nrhs = (Q^T b')[:r]), compute R_S = U Sigma V^T (one-sided Jacobi SVD),
 * keep sigma_i > theta * sigma_1, y = V_k Sigma_k^-1 U_k^T c.  All DEVICE.  rank_out (HOST,
 * may be NULL) receives k and sigma_out (DEVICE, may be NULL) the r singular values
 * (descending).  Synchronises the stream when rank_out != NULL.                              */
az_status_t az_tsvd_solve(const double* Rf, int64_t ldr, int64_t r, int64_t nrhs, double theta,
                          double* y, int64_t ldy, double* sigma_out, int64_t* rank_out,
                          void* workspace, size_t ws_bytes, void* stream);
az_status_t az_tsvd_workspace_size(int64_t r, int64_t nrhs, size_t* bytes);

typedef struct {
  int64_t rank_used;        /* k: kept singular values of the sketch */
  int64_t probes_used;      /* number of probe columns drawn (multiple of R) */
  int32_t saturated;        /* 1 if k > probes_used - p after max_blocks blocks */
  double sigma_first, sigma_last_kept;
  double ms_rhs, ms_sketch, ms_qr, ms_svd, ms_step2, ms_total;   /* CUDA-event stage times */
  const double* sigma;      /* az_solve: DEVICE pointer INTO the caller's workspace to the n_sigma
                               singular values of the sketch's R factor, descending (the spectrum the
                               truncation at theta sigma_1 is taken on); valid until the
                               workspace is reused or freed.  NULL from the factored entry points. */
  int64_t n_sigma;          /* = probes_used */
} az_solve_report_t;

/* Bytes of DEVICE workspace az_solve needs for nrhs right-hand sides, probe block R and at
 * most max_blocks probe blocks. */
az_status_t az_solve_workspace_size(az_plan_t plan, int64_t nrhs, int64_t R, int32_t max_blocks,
                                    size_t* bytes);
/* The whole AZ solve (Alg. 1).  b: (M+Mb) x nrhs, x: N x nrhs (DEVICE).
 * theta: sketch truncation threshold relative to sigma_1 of the sketch (R4).
 * R: probe block size; blocks are added until rank <= probes - p (p = 10) or
 * max_blocks is reached (R5; max_blocks = 1 is the literal single-block sketch).
 * The dense stage follows the probes actually drawn: while probes + nrhs <= 128 the single-pass
 * TSQR and one-CTA Jacobi take the sketch; an adaptive solve whose first block fits runs it that
 * way and moves to the blocked path (drawing its blocks afresh) only if that block saturated.
 * report: HOST, may be NULL.  ALWAYS synchronises the stream before returning (whether or not a
 * report is requested), so x, the workspace and the status are final on return.  Returns
 * AZ_WARN_SKETCH_SATURATED (x still written) if the last block saturated.
 * CUDA graphs: a single-block narrow solve (max_blocks = 1, or the first block of an adaptive solve;
 * one-CTA 1-D and 2-D layouts) whose arguments (b, ldb, x, ldx, nrhs, theta, R, workspace) repeat
 * those of the plan's previous such call is captured into a graph owned by the plan (at most 4 per
 * plan) and replayed on later calls with the same arguments: same kernels, same results; b and the
 * workspace are read at replay, so their contents may change between calls, but b, x and the
 * workspace must stay allocated at those addresses while the plan lives (az_plan_destroy frees the
 * graphs).  Disabled by AZ_SOLVE_GRAPH=0 and while tracing is on.                             */
az_status_t az_solve(az_plan_t plan, const double* b, int64_t ldb, double* x, int64_t ldx,
                     int64_t nrhs, double theta, int64_t R, int32_t max_blocks,
                     void* workspace, size_t ws_bytes, az_solve_report_t* report, void* stream);
/* Number of solve graphs the plan holds (diagnostics / tests). */
int32_t az_solve_graph_count(az_plan_t plan);

/* Host-buffer convenience: b (HOST, (M+Mb) x nrhs) -> x (HOST, N x nrhs), including the
 * host<->device copies (pinned staging owned by the plan).  Used for end-to-end timing.      */
az_status_t az_solve_host(az_plan_t plan, const double* b_host, double* x_host, int64_t nrhs,
                          double theta, int64_t R, int32_t max_blocks, az_solve_report_t* report,
                          void* stream);

const char* az_status_string(az_status_t s);
const char* az_last_error(void);
/* Number of libaz kernel launches issued by this thread since the last reset (instrumentation
 * for the bench's gpu_launches field). */
int64_t az_launch_count(int reset);

/* Pipelined host-buffer solves (the e2e path): enqueue H2D of b_host (an internal upload stream),
 * the solve on `stream` and D2H into x_host (an internal download stream), then return.  With
 * max_blocks == 1 nothing is synchronised (the solve's saturation test runs on the device and sets
 * a plan flag); max_blocks > 1 needs the rank on the host and synchronises like az_solve.  Two
 * internal device slots let a call's upload and the previous call's download overlap the current
 * solve.  x_host is valid after az_plan_sync.  Host buffers should be pinned (cudaHostAlloc / torch
 * pin_memory); b_host must not be modified until az_plan_sync.  Same shapes as az_solve_host.
 * Returns errors of the enqueue only.                                                         */
az_status_t az_solve_host_pipelined(az_plan_t plan, const double* b_host, double* x_host, int64_t nrhs,
                                    double theta, int64_t R, int32_t max_blocks, void* stream);
/* Waits for every pipelined solve of the plan (and the device).  Returns AZ_WARN_SKETCH_SATURATED
 * if any single-block pipelined solve since the last az_plan_sync saturated (rank > probes - p), and
 * clears that flag.                                                                            */
az_status_t az_plan_sync(az_plan_t plan);

/* ---- multi-GPU: NCCL over NVLink / NVSwitch, one process per GPU ----------------
 * NCCL is loaded at run time (the libnccl.so.2 already in the process, else the system one); without
 * it these entry points return AZ_ERR_NOT_SUPPORTED.  Bootstrap: rank 0 calls az_comm_unique_id, the
 * caller broadcasts the 128 bytes (e.g. over torch.distributed), every rank calls az_comm_create
 * (collective, blocking).  world must divide 8 (the leaves of the fixed TSQR tree).               */
typedef struct az_comm_s* az_comm_t;
az_status_t az_comm_unique_id(void* id128);          /* HOST, 128 bytes out (an ncclUniqueId) */
az_status_t az_comm_create(int32_t world, int32_t rank, const void* id128, az_comm_t* out);
az_status_t az_comm_destroy(az_comm_t comm);
/* The sharded AZ solve, collective over comm (every rank calls it with the same plan descriptor,
 * b, theta, R, max_blocks; b and x are replicated DEVICE arrays, shapes as az_solve).  Rank g
 * computes b' for its pair-aligned share of the right-hand sides and the sketch of its share of
 * every probe block (Philox keyed by the global column); an all-to-all (grouped ncclSend/ncclRecv)
 * re-blocks each new block by rows; the rows are cut into 8 fixed leaves, each leaf is reduced by
 * the single-pass TSQR to [R_l | c_l], the 8 factors are all-gathered and merged on every rank;
 * every rank runs the truncated SVD; x2 = Omega y and step 2 run per right-hand-side shard and x is
 * all-gathered (Alg. 1, :222-232).  x is bitwise identical at world
 * sizes 1, 2, 4 and 8.  Scratch is stream-ordered device memory (cudaMallocAsync) of the call.
 * Synchronises the stream; the report (HOST, may be NULL) has rank, probes, saturation and sigma.  */
az_status_t az_solve_sharded(az_plan_t plan, az_comm_t comm, const double* b, int64_t ldb, double* x, int64_t ldx,
                             int64_t nrhs, double theta, int64_t R, int32_t max_blocks,
                             az_solve_report_t* report, void* stream);

/* ---- factorisation reuse --------------------------------------------
 * The step-1 matrix (A - A Z* A) Omega does not depend on b (Alg. 1, :228, :283): factor
 * it once, then solve for any number of right-hand sides at the cost of b' = (I - A Z*) b, Q^T b'
 * (the stored Householder panels), y = P (Q^T b')[:k] with P the truncated pseudo-inverse of R_S
 * (V_k Sigma_k^-1 U_k^T, sigma > theta sigma_1), x2 = Omega y and step 2.  The factor owns its
 * DEVICE memory (the factored sketch, rows x probes, and P, probes x probes).  az_factorize
 * draws probe blocks exactly as az_solve (reading R5) and returns AZ_WARN_SKETCH_SATURATED (with a
 * usable factor) if max_blocks is exhausted.  The plan must outlive the factor.               */
typedef struct az_factor_s* az_factor_t;
az_status_t az_factorize(az_plan_t plan, double theta, int64_t R, int32_t max_blocks, az_factor_t* out,
                         az_solve_report_t* report, void* stream);
az_status_t az_factor_destroy(az_factor_t f);
az_status_t az_factor_query(az_factor_t f, int64_t* probes, int64_t* rank);
/* b: (M+Mb) x nrhs, x: N x nrhs, DEVICE column-major; workspace from az_factor_workspace_size. */
az_status_t az_factor_workspace_size(az_factor_t f, int64_t nrhs, size_t* bytes);
az_status_t az_solve_factored(az_factor_t f, const double* b, int64_t ldb, double* x, int64_t ldx,
                              int64_t nrhs, void* workspace, size_t ws_bytes,
                              az_solve_report_t* report, void* stream);

/* Per-kernel CUDA-event tracing for measurement (bench.py roofline): when enabled, every libaz
 * launch is bracketed by two events on its stream.  az_trace_report synchronises those events
 * and writes "name count total_ms\n" lines into buf (NUL-terminated, truncated to len).
 * Tracing adds two event records per launch; it is off by default. */
int az_trace_enable(int on);
int az_trace_report(char* buf, int len);

/* Diagnostics (tests and tools): Jacobi sweeps of the last truncated SVD.  which = 0: the one-CTA
 * one-sided Jacobi (r <= 128; reads a device counter, synchronising); which = 1: the block Jacobi
 * (r > 128; outer sweeps, host counter).  PAPER.md:269 (the SVD of the sketch).               */
int az_svd_sweeps_last(int which);

#ifdef __cplusplus
}
#endif
#endif /* AZ_H_ */
