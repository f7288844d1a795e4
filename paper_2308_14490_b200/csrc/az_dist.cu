// Multi-GPU AZ solve inside libaz: NCCL over NVLink / NVSwitch, one process per
// GPU.  The schedule is the one of paper_2308_14490_b200/dist.py (whose host logic is tested with the
// gloo backend on CPU), with every arithmetic step and every collective issued here:
//
//   1. rank g computes b' = (I - A Z*) b for its pair-aligned share of the right-hand sides and the
//      sketch S = (A - A Z* A) Omega for its share of each new probe block (Philox keyed by the
//      GLOBAL column: the probes are the single-GPU ones);
//   2. an all-to-all (grouped ncclSend / ncclRecv) re-blocks the NEW columns into row blocks;
//   3. TSQR over a FIXED tree of NLEAF = 8 row leaves (rank g owns 8 / G consecutive leaves): each
//      leaf gives [R_l | c_l]; a binary tree of pairwise merges (left over right, by the owner of the
//      left child; ncclSend/ncclRecv where the children live on different ranks -- one factor per
//      rank and level) ends in [R_S | Q^T b'] on rank 0;
//   4. the truncated SVD solve on rank 0; y and the rank are broadcast (ncclBroadcast);
//   5. x2 = Omega y and x = x2 + Z* (b - A x2) for the rank's right-hand sides, then an all-gather of
//      x (b and x replicated on every rank).
// Pair-aligned shards and the fixed tree make every operation see the same operands at G = 1, 2, 4
// and 8, so x is bitwise identical across world sizes (hard part H6).
//
// NCCL is loaded at run time (libnccl.so.2: the copy PyTorch already loaded, else the system one),
// so libaz has no link-time dependency on it; without NCCL the entry points return
// AZ_ERR_NOT_SUPPORTED.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "az_internal.h"

namespace {

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // the copy already in the process
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW);
    if (!h) return;
    auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name)); };
    sym(n.GetUniqueId, "ncclGetUniqueId");
    sym(n.CommInitRank, "ncclCommInitRank");
    sym(n.CommDestroy, "ncclCommDestroy");
    sym(n.AllGather, "ncclAllGather");
    sym(n.Broadcast, "ncclBroadcast");
    sym(n.Send, "ncclSend");
    sym(n.Recv, "ncclRecv");
    sym(n.CommGetAsyncError, "ncclCommGetAsyncError");
    sym(n.GroupStart, "ncclGroupStart");
    sym(n.GroupEnd, "ncclGroupEnd");
    sym(n.GetErrorString, "ncclGetErrorString");
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.AllGather && n.Broadcast && n.Send && n.Recv &&
           n.GroupStart &&
           n.GroupEnd && n.GetErrorString;
  });
  return n;
}

#define AZ_NCCL(call)                                                                    \
  do {                                                                                   \
    ncclResult_t _r = (call);                                                            \
    if (_r != ncclSuccess) {                                                             \
      az_set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, nccl().GetErrorString(_r)); \
      return AZ_ERR_NCCL;                                                                \
    }                                                                                    \
  } while (0)

constexpr int NLEAF = 8;

std::vector<int64_t> split(int64_t n, int parts) {
  std::vector<int64_t> b(parts + 1);
  for (int g = 0; g <= parts; ++g) b[g] = (n * g) / parts;
  return b;
}
std::vector<int64_t> split_pairs(int64_t n, int parts) {
  std::vector<int64_t> b = split((n + 1) / 2, parts);
  for (auto& v : b) v = std::min<int64_t>(n, 2 * v);
  return b;
}

// stream-ordered device scratch, freed at scope exit (after the stream's work: cudaFreeAsync)
struct DBuf {
  double* p = nullptr;
  cudaStream_t st;
  explicit DBuf(cudaStream_t s) : st(s) {}
  cudaError_t alloc(size_t n) { return cudaMallocAsync((void**)&p, std::max<size_t>(n, 1) * sizeof(double), st); }
  ~DBuf() {
    if (p) cudaFreeAsync(p, st);
  }
};

}  // namespace

struct az_comm_s {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0;
};

az_status_t az_apply_op(az_plan_s* p, int op, const double* in, int64_t ldin, double* out, int64_t ldout,
                        int64_t nvec, cudaStream_t st);
extern "C" az_status_t az_sketch(az_plan_t p, int64_t col0, int64_t ncols, double* S, int64_t ldS, void* stream);
extern "C" az_status_t az_omega_apply(az_plan_t p, int64_t col0, int64_t ncols, const double* y, int64_t ldy,
                                      int64_t nrhs, double* x, int64_t ldx, int accumulate, void* stream);
extern "C" az_status_t az_step2_workspace_size(az_plan_t p, int64_t nrhs, size_t* bytes);
extern "C" az_status_t az_step2(az_plan_t p, const double* x2, int64_t ldx2, const double* b, int64_t ldb, double* x,
                                int64_t ldx, int64_t nrhs, void* workspace, size_t ws_bytes, void* stream);

extern "C" az_status_t az_comm_unique_id(void* id128) {
  if (!id128) return AZ_ERR_INVALID_ARGUMENT;
  if (!nccl().ok) {
    az_set_error("az_comm_unique_id: NCCL (libnccl.so.2) not available");
    return AZ_ERR_NOT_SUPPORTED;
  }
  ncclUniqueId id;
  AZ_NCCL(nccl().GetUniqueId(&id));
  memcpy(id128, &id, sizeof(id));
  return AZ_OK;
}

extern "C" az_status_t az_comm_create(int32_t world, int32_t rank, const void* id128, az_comm_t* out) {
  if (!out || !id128 || world < 1 || rank < 0 || rank >= world || NLEAF % world) {
    az_set_error("az_comm_create: bad arguments (world must divide %d)", NLEAF);
    return AZ_ERR_INVALID_ARGUMENT;
  }
  if (!nccl().ok) {
    az_set_error("az_comm_create: NCCL (libnccl.so.2) not available");
    return AZ_ERR_NOT_SUPPORTED;
  }
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  auto* c = new az_comm_s();
  c->world = world;
  c->rank = rank;
  const ncclResult_t r = nccl().CommInitRank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    az_set_error("az_comm_create: ncclCommInitRank: %s", nccl().GetErrorString(r));
    delete c;
    return AZ_ERR_NCCL;
  }
  *out = c;
  return AZ_OK;
}

extern "C" az_status_t az_comm_destroy(az_comm_t c) {
  if (!c) return AZ_ERR_INVALID_ARGUMENT;
  if (c->comm) nccl().CommDestroy(c->comm);
  delete c;
  return AZ_OK;
}

// all-to-all re-block: `local` holds this rank's columns (rows x c_me, ld rows) of a k-column
// matrix whose rank g owns the contiguous columns [cols[g], cols[g + 1]); `out` (rows_me x k, ld ldo)
// receives this rank's rows [rs[me], rs[me + 1]) of every column.  send: scratch of rows * c_me.
static az_status_t reblock(az_comm_s* c, const double* local, int64_t rows, const std::vector<int64_t>& cols,
                           const std::vector<int64_t>& rs, double* out, int64_t ldo, double* send, cudaStream_t st) {
  const int G = c->world, me = c->rank;
  const int64_t cme = cols[me + 1] - cols[me];
  const int64_t rme = rs[me + 1] - rs[me];
  // pack: for every destination h, my columns restricted to h's rows, contiguous (column-major, ld rb[h])
  std::vector<int64_t> soff(G + 1, 0);
  for (int h = 0; h < G; ++h) {
    const int64_t rb = rs[h + 1] - rs[h];
    soff[h + 1] = soff[h] + rb * cme;
    if (rb && cme)
      AZ_CUDA_CHECK(cudaMemcpy2DAsync(send + soff[h], rb * sizeof(double), local + rs[h], rows * sizeof(double),
                                      rb * sizeof(double), cme, cudaMemcpyDeviceToDevice, st));
  }
  // rank g's columns for my rows land column-major (ld rme) at their place in out when ldo == rme
  AZ_NCCL(nccl().GroupStart());
  for (int h = 0; h < G; ++h) {
    const int64_t ns = soff[h + 1] - soff[h];
    if (ns) AZ_NCCL(nccl().Send(send + soff[h], ns, ncclFloat64, h, c->comm, st));
    const int64_t nr = rme * (cols[h + 1] - cols[h]);
    if (nr) AZ_NCCL(nccl().Recv(out + cols[h] * ldo, nr, ncclFloat64, h, c->comm, st));
  }
  AZ_NCCL(nccl().GroupEnd());
  return AZ_OK;
}

extern "C" az_status_t az_solve_sharded(az_plan_t p, az_comm_t c, const double* b, int64_t ldb, double* x,
                                        int64_t ldx, int64_t nrhs, double theta, int64_t R, int32_t max_blocks,
                                        az_solve_report_t* report, void* stream) {
  if (!p || !c || !b || !x || nrhs < 1 || R < 1 || max_blocks < 1 || !(theta >= 0.0) || ldb < p->M + p->Mb ||
      ldx < p->N) {
    az_set_error("az_solve_sharded: bad arguments");
    return AZ_ERR_INVALID_ARGUMENT;
  }
  if (!nccl().ok) {
    az_set_error("az_solve_sharded: NCCL not available");
    return AZ_ERR_NOT_SUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int G = c->world, me = c->rank, lpr = NLEAF / G;
  const int64_t rows = p->M + p->Mb, N = p->N;
  const int pfix = 10;
  const std::vector<int64_t> qs = split_pairs(nrhs, G), ps = split_pairs(R, G), leaves = split(rows, NLEAF);
  std::vector<int64_t> rs(G + 1);
  for (int g = 0; g <= G; ++g) rs[g] = leaves[g * lpr];
  const int64_t q0 = qs[me], q1 = qs[me + 1], qme = q1 - q0;
  const int64_t rme = rs[me + 1] - rs[me];
  const int64_t kpmax = R * max_blocks, kmax = kpmax + nrhs;
  int64_t leafmax = 0;
  for (int l = 0; l < NLEAF; ++l) leafmax = std::max(leafmax, leaves[l + 1] - leaves[l]);
  int64_t qmax = 0;
  for (int g = 0; g < G; ++g) qmax = std::max(qmax, qs[g + 1] - qs[g]);
  // scratch: my b' / new probe columns (rows x max(q_me, R_me)), the send buffer, my rows of [S | b']
  // (rows_me x kmax, S in columns [0, kpmax), b' in [kpmax, kmax)), a leaf [S | b'] (>= k rows), the
  // leaf factors (NLEAF x kp x k), the stacked factors, the merged R, y, sigma, x2 / x shards
  DBuf loc(st), snd(st), Ame(st), leaf(st), fac(st), stk(st), Rm(st), yb(st), sg(st), xs(st), x2(st), wq(st), ws2(st),
      wsv(st);
  const int64_t pme_max = std::max<int64_t>(qme, ps[me + 1] - ps[me]);
  const int64_t leafrows = std::max(leafmax, kmax);
  const int64_t stkrows = std::max<int64_t>(2 * kpmax, kmax);
  size_t qrw = 0, svw = 0;
  for (int64_t b2 = 1; b2 <= max_blocks; ++b2) {   // the QR / SVD workspaces of every block's shapes
    const int64_t k2 = b2 * R + nrhs;
    qrw = std::max({qrw, az_qr_ws_bytes(leafrows, k2), az_qr_ws_bytes(stkrows, k2)});
    svw = std::max(svw, az_tsvd_ws_bytes(b2 * R, nrhs));
  }
  size_t s2bytes = 0;
  AZ_TRY(az_step2_workspace_size(p, std::max<int64_t>(qme, 1), &s2bytes));
  if (loc.alloc(rows * std::max<int64_t>(pme_max, 1)) || snd.alloc(rows * std::max<int64_t>(pme_max, 1)) ||
      Ame.alloc(rme * kmax) || leaf.alloc(leafrows * kmax) || fac.alloc((size_t)NLEAF * kpmax * kmax) ||
      stk.alloc(stkrows * kmax) || Rm.alloc(kmax * kmax) || yb.alloc(kpmax * nrhs) || sg.alloc(kpmax + 1) ||
      xs.alloc(N * qmax * G) || x2.alloc(N * std::max<int64_t>(qme, 1)) || wq.alloc(qrw / sizeof(double) + 1) ||
      ws2.alloc(s2bytes / sizeof(double) + 1) || wsv.alloc(svw / sizeof(double) + 1)) {
    az_set_error("az_solve_sharded: out of device memory");
    return AZ_ERR_OUT_OF_MEMORY;
  }
  double* Bme = Ame.p + kpmax * rme;   // my rows of b' (ld rme)
  // 1-2. b' for my right-hand sides, re-blocked once
  if (qme) AZ_TRY(az_apply_op(p, OP_RESID, b + q0 * ldb, ldb, loc.p, rows, qme, st));
  AZ_TRY(reblock(c, loc.p, rows, qs, rs, Bme, rme, snd.p, st));
  int64_t rank = 0, kp = 0, nb = 0;
  bool saturated = false;
  for (nb = 1; nb <= max_blocks; ++nb) {
    const int64_t c0 = (nb - 1) * R;
    kp = nb * R;
    const int64_t k = kp + nrhs;
    const int64_t pme = ps[me + 1] - ps[me];
    if (pme) AZ_TRY(az_sketch(p, c0 + ps[me], pme, loc.p, rows, st));
    // the new block's columns land at columns c0 + ps[g] of my rows of S
    std::vector<int64_t> cols(G + 1);
    for (int g = 0; g <= G; ++g) cols[g] = ps[g];
    AZ_TRY(reblock(c, loc.p, rows, cols, rs, Ame.p + c0 * rme, rme, snd.p, st));
    // 3. my leaves: [S(:, :kp) | b'] rows -> [R_l | c_l] (kp x k, ld kp) at fac + leaf kp k
    for (int l = me * lpr; l < (me + 1) * lpr; ++l) {
      const int64_t a0 = leaves[l] - rs[me], ml = leaves[l + 1] - leaves[l];
      const int64_t mpad = std::max(ml, k);   // fewer rows than columns: zero rows leave R unchanged
      if (mpad > ml) AZ_CUDA_CHECK(cudaMemsetAsync(leaf.p, 0, sizeof(double) * mpad * k, st));
      AZ_CUDA_CHECK(cudaMemcpy2DAsync(leaf.p, mpad * sizeof(double), Ame.p + a0, rme * sizeof(double),
                                      ml * sizeof(double), kp, cudaMemcpyDeviceToDevice, st));
      AZ_CUDA_CHECK(cudaMemcpy2DAsync(leaf.p + kp * mpad, mpad * sizeof(double), Bme + a0, rme * sizeof(double),
                                      ml * sizeof(double), nrhs, cudaMemcpyDeviceToDevice, st));
      double* fl = fac.p + (size_t)l * kp * k;
      if (k <= AZ_NARROW_MAX) {
        AZ_TRY(az_qr_r_impl(leaf.p, mpad, k, mpad, fl, kp, wq.p, qrw, st, kp));
      } else {   // blocked path: the full R (k x k); its top kp rows are [R_l | c_l]
        AZ_TRY(az_qr_r_impl(leaf.p, mpad, k, mpad, Rm.p, k, wq.p, qrw, st));
        AZ_CUDA_CHECK(cudaMemcpy2DAsync(fl, kp * sizeof(double), Rm.p, k * sizeof(double), kp * sizeof(double), k,
                                        cudaMemcpyDeviceToDevice, st));
      }
    }
    // binary tree of pairwise merges over the 8 leaves (fixed shape: bitwise identical across G)
    const size_t fsz = (size_t)kp * k;
    const int64_t mrows = std::max<int64_t>(2 * kp, k);   // stacked pair (zero rows pad m < k)
    for (int width = 1; width < NLEAF; width *= 2) {
      AZ_NCCL(nccl().GroupStart());
      for (int i = 0; i < NLEAF / width; i += 2) {
        const int ol = (i * width) / lpr, orr = ((i + 1) * width) / lpr;
        double* rf = fac.p + (size_t)(i + 1) * width * fsz;   // node (i + 1)'s factor, at its first leaf's slot
        if (ol != orr && me == orr) AZ_NCCL(nccl().Send(rf, fsz, ncclFloat64, ol, c->comm, st));
        if (ol != orr && me == ol) AZ_NCCL(nccl().Recv(rf, fsz, ncclFloat64, orr, c->comm, st));
      }
      AZ_NCCL(nccl().GroupEnd());
      for (int i = 0; i < NLEAF / width; i += 2) {
        if ((i * width) / lpr != me) continue;
        double* lf = fac.p + (size_t)i * width * fsz;
        double* rf = fac.p + (size_t)(i + 1) * width * fsz;
        if (mrows > 2 * kp) AZ_CUDA_CHECK(cudaMemsetAsync(stk.p, 0, sizeof(double) * mrows * k, st));
        AZ_CUDA_CHECK(cudaMemcpy2DAsync(stk.p, mrows * sizeof(double), lf, kp * sizeof(double), kp * sizeof(double), k,
                                        cudaMemcpyDeviceToDevice, st));
        AZ_CUDA_CHECK(cudaMemcpy2DAsync(stk.p + kp, mrows * sizeof(double), rf, kp * sizeof(double),
                                        kp * sizeof(double), k, cudaMemcpyDeviceToDevice, st));
        // the parent's factor replaces the left child's (kp x k, ld kp)
        if (k <= AZ_NARROW_MAX) {
          AZ_TRY(az_qr_r_impl(stk.p, mrows, k, mrows, lf, kp, wq.p, qrw, st, kp));
        } else {
          AZ_TRY(az_qr_r_impl(stk.p, mrows, k, mrows, Rm.p, k, wq.p, qrw, st));
          AZ_CUDA_CHECK(cudaMemcpy2DAsync(lf, kp * sizeof(double), Rm.p, k * sizeof(double), kp * sizeof(double), k,
                                          cudaMemcpyDeviceToDevice, st));
        }
      }
    }
    // 4. truncated SVD solve on rank 0 (the root factor, kp x k at fac), y and the rank broadcast
    double* info = sg.p + kpmax;   // one double beside sigma: the rank, as a value
    if (me == 0) {
      AZ_TRY(az_tsvd_impl(fac.p, kp, kp, nrhs, theta, yb.p, kp, sg.p, &rank, wsv.p, svw, st));
      const double rv = (double)rank;
      AZ_CUDA_CHECK(cudaMemcpyAsync(info, &rv, sizeof(double), cudaMemcpyHostToDevice, st));
    }
    AZ_NCCL(nccl().GroupStart());
    AZ_NCCL(nccl().Broadcast(yb.p, yb.p, (size_t)kp * nrhs, ncclFloat64, 0, c->comm, st));
    AZ_NCCL(nccl().Broadcast(sg.p, sg.p, (size_t)kpmax + 1, ncclFloat64, 0, c->comm, st));
    AZ_NCCL(nccl().GroupEnd());
    if (me != 0) {
      double rv = 0.0;
      AZ_CUDA_CHECK(cudaMemcpyAsync(&rv, info, sizeof(double), cudaMemcpyDeviceToHost, st));
      AZ_CUDA_CHECK(cudaStreamSynchronize(st));
      rank = (int64_t)rv;
    }
    saturated = rank > kp - pfix;
    if (!saturated || nb == max_blocks) break;
  }
  if (nb > max_blocks) nb = max_blocks;
  // 5. x2 = Omega y and steps 2-3 for my right-hand sides; all-gather of x
  double* xme = xs.p + (size_t)me * N * qmax;
  if (qme) {
    AZ_TRY(az_omega_apply(p, 0, kp, yb.p + q0 * kp, kp, qme, x2.p, N, 0, st));
    AZ_TRY(az_step2(p, x2.p, N, b + q0 * ldb, ldb, xme, N, qme, ws2.p, s2bytes, st));
  }
  if (qmax) AZ_NCCL(nccl().AllGather(xme, xs.p, (size_t)N * qmax, ncclFloat64, c->comm, st));
  for (int g = 0; g < G; ++g) {
    const int64_t cg = qs[g + 1] - qs[g];
    if (cg)
      AZ_CUDA_CHECK(cudaMemcpy2DAsync(x + qs[g] * ldx, ldx * sizeof(double), xs.p + (size_t)g * N * qmax,
                                      N * sizeof(double), N * sizeof(double), cg, cudaMemcpyDeviceToDevice, st));
  }
  AZ_CUDA_CHECK(cudaStreamSynchronize(st));
  if (nccl().CommGetAsyncError) {   // a peer failing mid-collective surfaces here, not as a hang later
    ncclResult_t ae = ncclSuccess;
    if (nccl().CommGetAsyncError(c->comm, &ae) == ncclSuccess && ae != ncclSuccess) {
      az_set_error("az_solve_sharded: NCCL async error: %s", nccl().GetErrorString(ae));
      return AZ_ERR_NCCL;
    }
  }
  if (report) {
    memset(report, 0, sizeof(*report));
    report->rank_used = rank;
    report->probes_used = kp;
    report->saturated = saturated ? 1 : 0;
    double s1 = 0.0;
    AZ_CUDA_CHECK(cudaMemcpy(&s1, sg.p, sizeof(double), cudaMemcpyDeviceToHost));
    report->sigma_first = s1;
    if (rank > 0) AZ_CUDA_CHECK(cudaMemcpy(&report->sigma_last_kept, sg.p + rank - 1, sizeof(double), cudaMemcpyDeviceToHost));
  }
  return saturated ? AZ_WARN_SKETCH_SATURATED : AZ_OK;
}
