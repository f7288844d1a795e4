// 1-D operators for large n (c2: n = 2^20, fine grid L = 2^21) with the four-step layout.
//
// Coefficient vector x[n1 N2 + n2] is an N1 x N2 row-major matrix, the fine grid an N1 x L2 one
// (L2 = s N2).  A length-n DFT is: column FFTs (length N1, along n1), twiddle e^{-2 pi i n2 k1/n},
// row FFTs (length N2) -> spectrum X[k1][k2] at frequency k = k1 + N1 k2 ("transposed order").
// The fine spectrum is kept in the same order, kf = k1 + N1 k2', so the s aliases k + m n of a
// coefficient frequency sit in the SAME row k1 (k2' = k2 + m N2): expansion and folding are
// row-local and no transpose pass is ever needed.  W and zinv are stored in these orders.
//
// Passes (one kernel each, over a batch of vector pairs packed as complex):
//   C1  cols (N1):  coefficient input -> FFT_N1 -> twiddle                    -> C1 buffer
//   R2  rows:       FFT_N2 -> [keep v^] -> expand x W/L -> IFFT_L2 -> twiddle   -> G
//   C3  cols (N1):  IFFT_N1 -> E R (mask) -> FFT_N1 -> twiddle                -> G
//   R4  rows:       FFT_L2 -> fold conj(W) x zinv -> (r^ = v^ - w^) -> expand -> IFFT_L2 -> twiddle
//                   (Z*, A^T: fold -> IFFT_N2 -> twiddle -> C1)
//   C5  cols (N1):  IFFT_N1 -> R (gather rows) [b - . for I - A Z*]
//   Z1  cols (N1):  E (scatter rows) -> FFT_N1 -> twiddle                     -> G
//   Z3  cols (N1):  IFFT_N1 -> coefficient output
#include <algorithm>
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "az_fftr.cuh"
#include "az_internal.h"

struct P1f {
  const cplx* W0;
  const cplx* W2;
  const double* zinv;
  const double* Wr;      // real row symbol (plan d_Wr)
  const int32_t* pos;
  const uint8_t* mask;
  int64_t run0, run1;    // single-run mask (plan run0/run1), else run0 < 0
  const cplx* tw;
  const cplx* t4hi;
  const cplx* t4lo;
  int lap;
  double alpha;
  int64_t n, L;
  int N1, N2, L2, s;
  int64_t M;
  uint64_t seed;
  cplx* C1;
  cplx* G;
  const double* in;
  int64_t ldin;
  const double* in2;     // second input (the right-hand sides b of the fused step-2 chain)
  int64_t ldin2;
  double* out;
  int64_t ldout;
  cplx* Z2;              // FR_STEP1 / FR_RESID: optional Z*-part output (coefficient spectrum after IFFT_N2)
  double* out2;          // FC_OUT_Z output (N x nvec)
  int64_t ldout2;
  bool defer_z;          // skip the closing FC_OUT_Z pass (az1f_out_z runs it later)
  int64_t nvec, col0, pair0;
  int lead;              // spectral probes from an odd col0: the first pair's real column precedes the call
  double sqn;            // sqrt(n): scale of the spectral probes
  const char* trace_name;   // trace label override (null: the pass kind's name)
};

// row of the fine grid point g (natural order), -1 outside Omega
AZ_D int row_of(const P1f& a, int64_t g) {
  if (a.run0 >= 0) return (g >= a.run0 && g < a.run1) ? (int)(g - a.run0) : -1;
  return a.pos[g];
}

// e^{DIR 2 pi i t / L} for t in [0, L)
template <int DIR>
AZ_D cplx tw4(const P1f& a, int64_t t) {
  cplx w = cmul(__ldg(&a.t4hi[t >> TW4B]), __ldg(&a.t4lo[t & ((1 << TW4B) - 1)]));
  if (DIR > 0) w.y = -w.y;
  return w;
}

struct Cols1 {
  int64_t cre, cim;
  bool has_re, has_im;
};
AZ_D Cols1 pcols(const P1f& a, int b) {
  Cols1 c;
  c.cre = 2 * (a.pair0 + b) - a.lead;
  c.cim = c.cre + 1;
  c.has_re = c.cre >= 0;
  c.has_im = c.cim < a.nvec;
  return c;
}

// global probe pair of the batch's vector pair b (spectral probes, reading R35)
AZ_D uint64_t probe_pair_index(const P1f& a, int b) { return (uint64_t)((a.col0 >> 1) + a.pair0 + b); }

// ------------------------------------------------------------------------------------------
// column passes: a CTA owns TC adjacent columns of an N1-row matrix; each column FFT is computed
// by T = NC / 16 threads holding 16 values each (az_fftr.cuh), element e of thread j = row j + e T.
// Thread t -> (column c = t mod TC, j = t / TC): a warp reads TC consecutive complex values of
// 32 / TC rows per access.
// ------------------------------------------------------------------------------------------
enum { FC_IN_COEF = 0, FC_FINE_MASK = 1, FC_OUT_GATHER = 2, FC_OUT_RESID = 3, FC_IN_ROWS = 4, FC_OUT_COEF = 5,
       FC_FWD_G = 6, FC_RESID_MID = 7, FC_OUT_COEF_ADD = 8, FC_OUT_Z = 9 };
// FC_OUT_Z: IFFT_N1 of the Z2 buffer -> out2 = (.) / n  (Z* b from the b' chain; M = Omega - Z* A Omega
//           from the sketch, whose row pass wrote the spectrum r^ = v^ - w^)
// FC_RESID_MID: IFFT_N1 -> r = b - (A x) on Omega, 0 outside -> FFT_N1 -> twiddle  (the A -> b - A x ->
//               Z* junction of step 2 in one pass, no row vector written or read)
// FC_OUT_COEF_ADD: IFFT_N1 -> x = x2 + (.) / n  (the closing addition of step 2)

// Per-column exchange buffers (complex slots apart): a quarter warp (8 lanes, one 128-byte wavefront
// of a 128-bit shared access) holds TC adjacent columns x 8 / TC consecutive rows j; consecutive j
// already fall in consecutive 16-byte bank groups (az_fftr.cuh padE), so the column buffers are
// offset by 8 / TC groups (an odd number of groups for TC >= 8): all 8 lanes in distinct groups.
template <int NC, int TC, int EC>
AZ_HD constexpr int col_stride() {
  constexpr int base = fftr::padded_lenE<EC>(NC) - 1;
  constexpr int want = TC >= 8 ? 1 : 8 / TC;
  return base + ((want - base % 8) % 8 + 8) % 8;
}

// EC = values per thread in the column FFTs (16: fewer exchanges; 8: half the registers, more
// resident warps); MINB = CTAs per SM the register budget is sized for.
// The transform and store of a column pass on the values v (element e: row j + e T of column col,
// vector pair b), shared by the one-tile kernel (k1f_cols) and the persistent TMA-fed one (k1f_cols_p).
template <int NC, int TC, int KIND, int EC>
AZ_D void cols_body(const P1f& a, cplx (&v)[EC], int j, int col, int b, cplx* buf, double cout) {
  constexpr int T = NC / EC;
  const Cols1 cc = pcols(a, b);
  const bool coef = (KIND == FC_IN_COEF || KIND == FC_OUT_COEF || KIND == FC_OUT_COEF_ADD || KIND == FC_OUT_Z);
  const int W = coef ? a.N2 : a.L2;                    // row length of the matrix
  cplx* C1b = (KIND == FC_OUT_Z) ? a.Z2 + (int64_t)b * a.n : a.C1 + (int64_t)b * a.n;
  cplx* Gb = a.G + (int64_t)b * a.L;
  const int64_t tmul = coef ? a.s : 1;                 // e^{-2 pi i n2 k1 / n} = e^{-2 pi i (s n2 k1) / L}
  uint32_t mbits = 0;   // FC_FINE_MASK: the 16 mask bytes of this thread, packed
  if constexpr (KIND == FC_FINE_MASK) {
#pragma unroll
    for (int e = 0; e < EC; ++e) {
      const int64_t g = (int64_t)(j + e * T) * W + col;
      const bool in = a.run0 >= 0 ? (g >= a.run0 && g < a.run1) : a.mask[g] != 0;
      mbits |= (in ? 1u : 0u) << e;
    }
    static_assert(EC <= 32, "mask bits");
  }

  // ---- transforms ----
  if constexpr (KIND == FC_IN_COEF || KIND == FC_IN_ROWS || KIND == FC_FWD_G) {
    fftr::fft<NC, EC, -1, 4>(v, j, buf, a.tw, TWN);
  } else if constexpr (KIND == FC_RESID_MID) {
    fftr::fft<NC, EC, 1, 4>(v, j, buf, a.tw, TWN);
#pragma unroll
    for (int e = 0; e < EC; ++e) {
      const int r = row_of(a, (int64_t)(j + e * T) * W + col);
      v[e] = r >= 0 ? make_double2(a.in2[r + cc.cre * a.ldin2] - v[e].x,
                                   cc.has_im ? a.in2[r + cc.cim * a.ldin2] - v[e].y : 0.0)
                    : czero();
    }
    fftr::fft<NC, EC, -1, 4>(v, j, buf, a.tw, TWN);
  } else if constexpr (KIND == FC_FINE_MASK) {
    fftr::fft<NC, EC, 1, 4>(v, j, buf, a.tw, TWN);
#pragma unroll
    for (int e = 0; e < EC; ++e)
      if (!((mbits >> e) & 1u)) v[e] = czero();
    fftr::fft<NC, EC, -1, 4>(v, j, buf, a.tw, TWN);
  } else {
    fftr::fft<NC, EC, 1, 4>(v, j, buf, a.tw, TWN);
  }

  // ---- store ----
  if constexpr (KIND == FC_IN_COEF || KIND == FC_IN_ROWS || KIND == FC_FINE_MASK || KIND == FC_FWD_G ||
                KIND == FC_RESID_MID) {
    cplx* dst = (KIND == FC_IN_COEF) ? C1b : Gb;
    // twiddle e^{-2 pi i k1 col tmul / L} for k1 = j + e T by recurrence in e (<= EC - 1 products)
    cplx w = tw4<-1>(a, ((int64_t)j * col * tmul) & (a.L - 1));
    const cplx ws = tw4<-1>(a, ((int64_t)T * col * tmul) & (a.L - 1));
#pragma unroll
    for (int e = 0; e < EC; ++e) {
      const int k1 = j + e * T;
      dst[(int64_t)k1 * W + col] = cmul(v[e], w);
      w = cmul(w, ws);
    }
  } else if constexpr (KIND == FC_OUT_GATHER || KIND == FC_OUT_RESID) {
#pragma unroll
    for (int e = 0; e < EC; ++e) {
      const int r = row_of(a, (int64_t)(j + e * T) * W + col);
      if (r >= 0) {
        if constexpr (KIND == FC_OUT_RESID) {
          a.out[r + cc.cre * a.ldout] = a.in[r + cc.cre * a.ldin] - v[e].x;
          if (cc.has_im) a.out[r + cc.cim * a.ldout] = a.in[r + cc.cim * a.ldin] - v[e].y;
        } else {
          if (cc.has_re) a.out[r + cc.cre * a.ldout] = v[e].x;
          if (cc.has_im) a.out[r + cc.cim * a.ldout] = v[e].y;
        }
      }
    }
  } else if constexpr (KIND == FC_OUT_COEF_ADD) {
#pragma unroll
    for (int e = 0; e < EC; ++e) {
      const int64_t i = (int64_t)(j + e * T) * W + col;
      a.out[i + cc.cre * a.ldout] = fma(v[e].x, cout, a.in[i + cc.cre * a.ldin]);
      if (cc.has_im) a.out[i + cc.cim * a.ldout] = fma(v[e].y, cout, a.in[i + cc.cim * a.ldin]);
    }
  } else if constexpr (KIND == FC_OUT_Z) {
#pragma unroll
    for (int e = 0; e < EC; ++e) {
      const int64_t i = (int64_t)(j + e * T) * W + col;
      if (cc.has_re) a.out2[i + cc.cre * a.ldout2] = v[e].x * cout;
      if (cc.has_im) a.out2[i + cc.cim * a.ldout2] = v[e].y * cout;
    }
  } else {   // FC_OUT_COEF
#pragma unroll
    for (int e = 0; e < EC; ++e) {
      const int64_t i = (int64_t)(j + e * T) * W + col;
      a.out[i + cc.cre * a.ldout] = v[e].x * cout;
      if (cc.has_im) a.out[i + cc.cim * a.ldout] = v[e].y * cout;
    }
  }
}

template <int NC, int TC, int KIND, int SRC, int EC, int MINB>
__global__ void __launch_bounds__(TC * (NC / EC), MINB) k1f_cols(P1f a, double cout) {
  extern __shared__ cplx sm[];
  constexpr int T = NC / EC;
  const int tid = threadIdx.x, c = tid % TC, j = tid / TC;
  const int b = blockIdx.y;
  const int c0 = blockIdx.x * TC;
  const int col = c0 + c;
  const Cols1 cc = pcols(a, b);
  const bool coef = (KIND == FC_IN_COEF || KIND == FC_OUT_COEF || KIND == FC_OUT_COEF_ADD || KIND == FC_OUT_Z);
  const int W = coef ? a.N2 : a.L2;                    // row length of the matrix
  cplx* C1b = (KIND == FC_OUT_Z) ? a.Z2 + (int64_t)b * a.n : a.C1 + (int64_t)b * a.n;
  cplx* Gb = a.G + (int64_t)b * a.L;
  cplx* buf = sm + c * col_stride<NC, TC, EC>();
  cplx v[EC];

  // ---- load (element e: row j + e T) ----
  if constexpr (KIND == FC_IN_COEF && SRC == SRC_PROBE) {
    // lanes (2m, 2m+1) hold columns (col, col + 1), col even: the even lane draws the real-part
    // probe pair of the two columns, the odd lane the imaginary-part pair, and they swap halves.
    const bool odd = c & 1;
#pragma unroll
    for (int e = 0; e < EC; ++e) {
      const int64_t i = (int64_t)(j + e * T) * W + (col & ~1);
      double2 z = make_double2(0.0, 0.0);
      if (!odd || cc.has_im) z = probe_pair((uint64_t)(i >> 1), (uint64_t)(a.col0 + (odd ? cc.cim : cc.cre)), a.seed);
      const double send = odd ? z.x : z.y;
      const double recv = __shfl_xor_sync(0xffffffffu, send, 1);
      v[e] = odd ? make_double2(recv, z.y) : make_double2(z.x, recv);
    }
  } else if constexpr (KIND == FC_IN_COEF) {
#pragma unroll
    for (int e = 0; e < EC; ++e) {
      const int64_t i = (int64_t)(j + e * T) * W + col;
      v[e] = make_double2(a.in[i + cc.cre * a.ldin], cc.has_im ? a.in[i + cc.cim * a.ldin] : 0.0);
    }
  } else if constexpr (KIND == FC_IN_ROWS) {
#pragma unroll
    for (int e = 0; e < EC; ++e) {
      const int r = row_of(a, (int64_t)(j + e * T) * W + col);
      v[e] = r >= 0 ? make_double2(a.in[r + cc.cre * a.ldin], cc.has_im ? a.in[r + cc.cim * a.ldin] : 0.0) : czero();
    }
  } else {
    const cplx* src = coef ? C1b : Gb;
#pragma unroll
    for (int e = 0; e < EC; ++e) v[e] = src[(int64_t)(j + e * T) * W + col];
  }
  cols_body<NC, TC, KIND, EC>(a, v, j, col, b, buf, cout);
}

// ------------------------------------------------------------------------------------------
// Persistent column passes over plan-owned tiles (default; AZ_COLS_PERSIST=0 selects k1f_cols): a CTA
// owns TC adjacent columns and walks a range of the batch's vector pairs; the next pair's TC x NC
// tile is brought in by the TMA engine (cp.async.bulk.tensor.3d, SASS UTMALDG, boxes of TC complex x
// 256 rows of the [pair][row][column] tensor) into a shared-memory stage tracked by an mbarrier while
// the current pair is transformed.  Same arithmetic as k1f_cols (cols_body).
// ------------------------------------------------------------------------------------------
template <int NC, int TC, int EC>
struct ColsP {
  static constexpr int T = NC / EC;
  static constexpr int NT = TC * T;
  static constexpr int BOXR = NC < 256 ? NC : 256;     // rows per TMA box
  static constexpr size_t stage_bytes = sizeof(cplx) * TC * NC;
  static constexpr size_t smem = 1024 + stage_bytes + sizeof(cplx) * TC * col_stride<NC, TC, EC>();
};

template <int NC, int TC, int KIND, int EC, int MINB>
__global__ void __launch_bounds__(TC * (NC / EC), MINB)
    k1f_cols_p(P1f a, double cout, const __grid_constant__ CUtensorMap tmap, int npairs, int pgroups) {
  using C = ColsP<NC, TC, EC>;
  constexpr int T = C::T;
  extern __shared__ __align__(1024) unsigned char smraw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smraw);
  cplx* stage = reinterpret_cast<cplx*>(smraw + 1024);   // [row][TC] complex, as the box lands
  cplx* xbuf = stage + TC * NC;
  const int tid = threadIdx.x, c = tid % TC, j = tid / TC;
  const int c0 = blockIdx.x * TC;
  const int col = c0 + c;
  const int b0 = (int)(((int64_t)npairs * blockIdx.y) / pgroups);
  const int b1 = (int)(((int64_t)npairs * (blockIdx.y + 1)) / pgroups);
  cplx* buf = xbuf + c * col_stride<NC, TC, EC>();
  auto issue = [&](int b) {
    bulk::arrive_expect_tx(bar, (uint32_t)C::stage_bytes);
#pragma unroll
    for (int r0 = 0; r0 < NC; r0 += C::BOXR) {
      const uint32_t dst = bulk::smem_addr(stage + r0 * TC);
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
              dst),
          "l"(&tmap), "r"(2 * c0), "r"(r0), "r"(b), "r"(bulk::smem_addr(bar))
          : "memory");
    }
  };
  if (tid == 0) {
    bulk::mbar_init(bar, 1);
    bulk::fence_init();
  }
  __syncthreads();
  if (tid == 0 && b0 < b1) issue(b0);
  uint32_t ph = 0;
  for (int b = b0; b < b1; ++b) {
    cplx v[EC];
    bulk::wait(bar, ph);
    ph ^= 1;
#pragma unroll
    for (int e = 0; e < EC; ++e) v[e] = stage[(j + e * T) * TC + c];
    __syncthreads();   // the stage is free: the next pair's tile may land
    if (tid == 0 && b + 1 < b1) {
      bulk::fence_proxy_async();
      issue(b + 1);
    }
    cols_body<NC, TC, KIND, EC>(a, v, j, col, b, buf, cout);
  }
}

// ------------------------------------------------------------------------------------------
// row passes: a CTA owns RPC rows k1; T = LR2 / 16 = NR2 / 8 threads per row.  Length-LR2
// transforms hold 16 values per thread, length-NR2 ones 8, so element e of the coefficient
// spectrum (k2 = j + e T) and its alias k2 + NR2 (element e + 8 of the fine spectrum) are in the
// same thread: fold, expand, the symbol multiply and the v^ - w^ update are all thread-local.
// ------------------------------------------------------------------------------------------
template <int NR2, int LR2, int EL>
AZ_HD constexpr int row_buf() {
  return fftr::padded_lenE<EL>(LR2) > fftr::padded_lenE<EL / 2>(NR2) ? fftr::padded_lenE<EL>(LR2)
                                                                      : fftr::padded_lenE<EL / 2>(NR2);
}

enum { FR_EXPAND = 0, FR_EXPAND_KEEP = 1, FR_STEP1 = 2, FR_RESID = 3, FR_ZSTAR = 4, FR_AT = 5, FR_EXPAND_PROBE = 6,
       FR_PROBE_Z = 7 };
// FR_EXPAND_PROBE: the spectral probes v^ drawn in the row (reading R35) -> keep v^ -> expand x W/L -> IFFT_L2
//                  (the sketch's first pass: no coefficient-side column pass, no FFT_N2)
// FR_PROBE_Z:      v^ drawn in the row -> IFFT_N2 -> twiddle -> Z2 (FC_OUT_Z then gives Omega explicitly)
template <int KIND>
struct RowGen {
  static constexpr bool on = KIND == FR_EXPAND_PROBE || KIND == FR_PROBE_Z;
};
// v^[k1 + N1 (j + e T)] of probe pair P, element e of thread j
template <int EN, int T>
AZ_D void gen_row(const P1f& a, int k1, uint64_t P, int j, cplx (&vn)[EN]) {
#pragma unroll
  for (int e = 0; e < EN; ++e)
    vn[e] = spectral_probe((uint64_t)k1 + (uint64_t)a.N1 * (uint64_t)(j + e * T), P, a.seed, a.sqn);
}

template <int NR2, int LR2, int RPC, int KIND, int EL, int MINB>
__global__ void __launch_bounds__(RPC * (LR2 / EL), MINB) k1f_rows(P1f a, int nrows) {
  extern __shared__ cplx sm[];
  static_assert(LR2 == 2 * NR2, "four-step rows: L = 2 only");
  constexpr int EN = EL / 2;            // values per thread of the length-NR2 transforms
  constexpr int T = LR2 / EL;
  const int f = threadIdx.x / T, j = threadIdx.x % T;
  const int k1 = blockIdx.x * RPC + f;
  const bool live = k1 < nrows;
  const int b = blockIdx.y;
  // one buffer serves the length-LR2 (EL values per thread) and length-NR2 (EN) transforms
  constexpr int PB = row_buf<NR2, LR2, EL>();
  cplx* buf = sm + f * PB;
  cplx* C1b = a.C1 + (int64_t)b * a.n;
  cplx* Gb = a.G + (int64_t)b * a.L;
  const double invL = 1.0 / (double)a.L;
  const int64_t rowW = (int64_t)(live ? k1 : 0) * LR2;     // row offset in W / G
  const int64_t rowC = (int64_t)(live ? k1 : 0) * NR2;     // row offset in C1 / zinv
  cplx vn[EN];
  cplx vl[EL];
  // the row's symbol / 1/sigma^2 / v^ inputs are copied into shared memory with cp.async at kernel
  // start, so their DRAM latency overlaps the first transform instead of stalling the fold
  constexpr bool NEED_Z = (KIND == FR_STEP1 || KIND == FR_RESID || KIND == FR_ZSTAR);
  constexpr bool NEED_C = (KIND == FR_STEP1);
  double* pre = reinterpret_cast<double*>(sm + RPC * PB) + f * (LR2 + 3 * NR2);
  double* Ws = pre;                 // LR2 real symbol values of the row
  double* Zs = pre + LR2;           // NR2 values of 1/sigma^2
  cplx* Cs = reinterpret_cast<cplx*>(pre + LR2 + NR2);   // NR2 values of v^
  if (live) {
    auto cp16 = [](void* dst, const void* src) {
      const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
    };
    for (int i = j; i < LR2 / 2; i += T) cp16(Ws + 2 * i, a.Wr + rowW + 2 * i);
    if constexpr (NEED_Z)
      for (int i = j; i < NR2 / 2; i += T) cp16(Zs + 2 * i, a.zinv + rowC + 2 * i);
    if constexpr (NEED_C)
      for (int i = j; i < NR2; i += T) cp16(Cs + i, C1b + rowC + i);
  }
  asm volatile("cp.async.commit_group;\n" ::);

  if constexpr (KIND == FR_EXPAND || KIND == FR_EXPAND_KEEP || RowGen<KIND>::on) {
    if constexpr (RowGen<KIND>::on) {
      gen_row<EN, T>(a, live ? k1 : 0, probe_pair_index(a, b), j, vn);
    } else {
#pragma unroll
      for (int e = 0; e < EN; ++e) vn[e] = live ? C1b[rowC + j + e * T] : czero();
      fftr::fft<NR2, EN, -1>(vn, j, buf, a.tw, TWN);
    }
    if ((KIND == FR_EXPAND_KEEP || KIND == FR_EXPAND_PROBE) && live)
#pragma unroll
      for (int e = 0; e < EN; ++e) C1b[rowC + j + e * T] = vn[e];
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
  } else {
#pragma unroll
    for (int e = 0; e < EL; ++e) vl[e] = live ? Gb[rowW + j + e * T] : czero();
    fftr::fft<LR2, EL, -1>(vl, j, buf, a.tw, TWN);
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
#pragma unroll
    for (int e = 0; e < EN; ++e) {
      const int k2 = j + e * T;
      cplx acc = cadd(cscale(vl[e], Ws[k2]), cscale(vl[e + EN], Ws[k2 + NR2]));
      if constexpr (KIND != FR_AT) acc = cscale(acc, Zs[k2]);
      vn[e] = acc;
    }
    if constexpr (KIND == FR_STEP1) {   // r^ = v^ - w^  (the spectrum of M = v - Z* A v)
#pragma unroll
      for (int e = 0; e < EN; ++e) vn[e] = csub(Cs[j + e * T], vn[e]);
    }
    if constexpr (KIND == FR_STEP1 || KIND == FR_RESID) {
      if (a.Z2) {   // r^ (STEP1: M = v - Z* A v) or w^ (RESID: Z* b) on to the coefficient side: IFFT_N2 + twiddle
        cplx wz[EN];
#pragma unroll
        for (int e = 0; e < EN; ++e) wz[e] = vn[e];
        fftr::fft<NR2, EN, 1>(wz, j, buf, a.tw, TWN);
        if (live) {
          cplx* Zb = a.Z2 + (int64_t)b * a.n;
          cplx w = tw4<1>(a, ((int64_t)j * k1 * 2) & (a.L - 1));
          const cplx ws = tw4<1>(a, ((int64_t)T * k1 * 2) & (a.L - 1));
#pragma unroll
          for (int e = 0; e < EN; ++e) {
            Zb[rowC + j + e * T] = cmul(wz[e], w);
            w = cmul(w, ws);
          }
        }
      }
    }
  }
  if constexpr (KIND == FR_PROBE_Z) {
    fftr::fft<NR2, EN, 1>(vn, j, buf, a.tw, TWN);
    if (live) {
      cplx* Zb = a.Z2 + (int64_t)b * a.n;
      cplx w = tw4<1>(a, ((int64_t)j * k1 * 2) & (a.L - 1));
      const cplx ws = tw4<1>(a, ((int64_t)T * k1 * 2) & (a.L - 1));
#pragma unroll
      for (int e = 0; e < EN; ++e) {
        Zb[rowC + j + e * T] = cmul(vn[e], w);
        w = cmul(w, ws);
      }
    }
  } else if constexpr (KIND == FR_ZSTAR || KIND == FR_AT) {
    fftr::fft<NR2, EN, 1>(vn, j, buf, a.tw, TWN);
    if (live) {
      // e^{+2 pi i n2 k1 / n} = e^{+2 pi i (2 n2 k1) / L}, n2 = j + e T, by recurrence in e
      cplx w = tw4<1>(a, ((int64_t)j * k1 * 2) & (a.L - 1));
      const cplx ws = tw4<1>(a, ((int64_t)T * k1 * 2) & (a.L - 1));
#pragma unroll
      for (int e = 0; e < EN; ++e) {
        C1b[rowC + j + e * T] = cmul(vn[e], w);
        w = cmul(w, ws);
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < EL; ++e) vl[e] = cscale(vn[e & (EN - 1)], Ws[j + e * T] * invL);
    fftr::fft<LR2, EL, 1>(vl, j, buf, a.tw, TWN);
    if (live) {
      // e^{+2 pi i n2' k1 / L}, n2' = j + e T, by recurrence in e
      cplx w = tw4<1>(a, ((int64_t)j * k1) & (a.L - 1));
      const cplx ws = tw4<1>(a, ((int64_t)T * k1) & (a.L - 1));
#pragma unroll
      for (int e = 0; e < EL; ++e) {
        Gb[rowW + j + e * T] = cmul(vl[e], w);
        w = cmul(w, ws);
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// Persistent row passes (default; AZ_ROWS_PERSIST=0 selects k1f_rows): a CTA owns one row k1 and
// walks a contiguous range of the batch's vector pairs (grid.y splits the pairs).  The row's symbol
// and 1/sigma^2 tables come in once per CTA instead of once per pair, and the NEXT pair's input row
// is in flight -- a bulk asynchronous copy (cp.async.bulk, the TMA engine's 1-D form) into a
// shared-memory stage tracked by an mbarrier -- while the current pair is transformed, so the HBM
// latency that stalled the one-pair CTAs (ncu: 35-39 % of their warp samples on long-scoreboard
// waits) overlaps the FFTs.  The step-1 pass's v^ row has its own stage, requested at the start of
// the pair and waited for only at the fold.  Same arithmetic, in the same order, as k1f_rows.
// ------------------------------------------------------------------------------------------
template <int NR2, int LR2, int KIND>
struct RowsP {
  static constexpr int EL = 16, EN = 8, T = LR2 / EL;
  static constexpr bool GEN = RowGen<KIND>::on;         // no input row: the spectral probes are drawn
  static constexpr bool IN_FINE = !(KIND == FR_EXPAND || KIND == FR_EXPAND_KEEP || GEN);
  static constexpr int INLEN = GEN ? 0 : (IN_FINE ? LR2 : NR2);   // complex values of the input row
  static constexpr bool NEED_W = KIND != FR_PROBE_Z;
  static constexpr bool NEED_Z = (KIND == FR_STEP1 || KIND == FR_RESID || KIND == FR_ZSTAR);
  static constexpr bool NEED_C = (KIND == FR_STEP1);
  static constexpr int PB = row_buf<NR2, LR2, EL>();
  // [3 mbarriers, 64 B][W row: LR2 doubles][1/sigma^2 row: NR2 doubles][v^ row: NR2 complex if NEED_C]
  // [input stage: INLEN complex][exchange buffer: PB complex]
  static constexpr size_t smem = 64 + sizeof(double) * (LR2 + NR2) + sizeof(cplx) * ((NEED_C ? NR2 : 0) + INLEN + PB);
};

template <int NR2, int LR2, int KIND>
__global__ void __launch_bounds__(LR2 / 16, 2) k1f_rows_p(P1f a, int npairs, int pgroups) {
  using C = RowsP<NR2, LR2, KIND>;
  constexpr int EL = C::EL, EN = C::EN, T = C::T, INLEN = C::INLEN;
  static_assert(LR2 == 2 * NR2, "four-step rows: L = 2 only");
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smraw);   // 0: tables, 1: input stage, 2: v^ row
  double* Ws = reinterpret_cast<double*>(smraw + 64);
  double* Zs = Ws + LR2;
  cplx* Cs = reinterpret_cast<cplx*>(Zs + NR2);
  cplx* stage = Cs + (C::NEED_C ? NR2 : 0);
  cplx* buf = stage + INLEN;
  const int j = threadIdx.x;
  const int k1 = blockIdx.x;
  const int b0 = (int)(((int64_t)npairs * blockIdx.y) / pgroups);
  const int b1 = (int)(((int64_t)npairs * (blockIdx.y + 1)) / pgroups);
  const int64_t rowW = (int64_t)k1 * LR2, rowC = (int64_t)k1 * NR2;
  const double invL = 1.0 / (double)a.L;
  auto in_row = [&](int b) -> const cplx* {
    return C::IN_FINE ? a.G + (int64_t)b * a.L + rowW : a.C1 + (int64_t)b * a.n + rowC;
  };
  if (j == 0) {
    bulk::mbar_init(&bars[0], 1);
    bulk::mbar_init(&bars[1], 1);
    bulk::mbar_init(&bars[2], 1);
    bulk::fence_init();
  }
  __syncthreads();
  if (j == 0 && b0 < b1) {
    if constexpr (C::NEED_W) {
      bulk::arrive_expect_tx(&bars[0], (uint32_t)(sizeof(double) * (LR2 + (C::NEED_Z ? NR2 : 0))));
      bulk::copy_g2s(Ws, a.Wr + rowW, sizeof(double) * LR2, &bars[0]);
      if constexpr (C::NEED_Z) bulk::copy_g2s(Zs, a.zinv + rowC, sizeof(double) * NR2, &bars[0]);
    }
    if constexpr (!C::GEN) {
      bulk::arrive_expect_tx(&bars[1], sizeof(cplx) * INLEN);
      bulk::copy_g2s(stage, in_row(b0), sizeof(cplx) * INLEN, &bars[1]);
    }
  }
  uint32_t ph_in = 0, ph_c = 0;
  bool tables = false;
  for (int b = b0; b < b1; ++b) {
    cplx* C1b = a.C1 + (int64_t)b * a.n;
    cplx* Gb = a.G + (int64_t)b * a.L;
    cplx vn[EN];
    cplx vl[EL];
    if constexpr (C::GEN) {
      gen_row<EN, T>(a, k1, probe_pair_index(a, b), j, vn);
      __syncthreads();   // the previous pair's last exchange is read before this pair's first one writes
    } else {
      bulk::wait(&bars[1], ph_in);
      ph_in ^= 1;
      if constexpr (C::IN_FINE) {
#pragma unroll
        for (int e = 0; e < EL; ++e) vl[e] = stage[j + e * T];
      } else {
#pragma unroll
        for (int e = 0; e < EN; ++e) vn[e] = stage[j + e * T];
      }
      __syncthreads();   // every thread holds its input: the stage (and the v^ row) may be refilled
    }
    if (j == 0) {
      bulk::fence_proxy_async();
      if (!C::GEN && b + 1 < b1) {
        bulk::arrive_expect_tx(&bars[1], sizeof(cplx) * INLEN);
        bulk::copy_g2s(stage, in_row(b + 1), sizeof(cplx) * INLEN, &bars[1]);
      }
      if constexpr (C::NEED_C) {
        bulk::arrive_expect_tx(&bars[2], sizeof(cplx) * NR2);
        bulk::copy_g2s(Cs, C1b + rowC, sizeof(cplx) * NR2, &bars[2]);
      }
    }
    if constexpr (KIND == FR_PROBE_Z) {
      // (nothing to fold or expand: the drawn spectrum goes straight to the coefficient side below)
    } else if constexpr (KIND == FR_EXPAND || KIND == FR_EXPAND_KEEP || KIND == FR_EXPAND_PROBE) {
      if constexpr (!C::GEN) fftr::fft<NR2, EN, -1>(vn, j, buf, a.tw, TWN);
      if constexpr (KIND == FR_EXPAND_KEEP || KIND == FR_EXPAND_PROBE) {
#pragma unroll
        for (int e = 0; e < EN; ++e) C1b[rowC + j + e * T] = vn[e];
      }
      if (!tables) {
        bulk::wait(&bars[0], 0);
        tables = true;
      }
    } else {
      fftr::fft<LR2, EL, -1>(vl, j, buf, a.tw, TWN);
      if (!tables) {
        bulk::wait(&bars[0], 0);
        tables = true;
      }
#pragma unroll
      for (int e = 0; e < EN; ++e) {
        const int k2 = j + e * T;
        cplx acc = cadd(cscale(vl[e], Ws[k2]), cscale(vl[e + EN], Ws[k2 + NR2]));
        if constexpr (KIND != FR_AT) acc = cscale(acc, Zs[k2]);
        vn[e] = acc;
      }
      if constexpr (KIND == FR_STEP1) {   // r^ = v^ - w^  (the spectrum of M = v - Z* A v)
        bulk::wait(&bars[2], ph_c);
        ph_c ^= 1;
#pragma unroll
        for (int e = 0; e < EN; ++e) vn[e] = csub(Cs[j + e * T], vn[e]);
      }
      if constexpr (KIND == FR_STEP1 || KIND == FR_RESID) {
        if (a.Z2) {   // r^ (STEP1) or w^ (RESID) on to the coefficient side: IFFT_N2 + twiddle
          cplx wz[EN];
#pragma unroll
          for (int e = 0; e < EN; ++e) wz[e] = vn[e];
          fftr::fft<NR2, EN, 1>(wz, j, buf, a.tw, TWN);
          cplx* Zb = a.Z2 + (int64_t)b * a.n;
          cplx w = tw4<1>(a, ((int64_t)j * k1 * 2) & (a.L - 1));
          const cplx ws = tw4<1>(a, ((int64_t)T * k1 * 2) & (a.L - 1));
#pragma unroll
          for (int e = 0; e < EN; ++e) {
            Zb[rowC + j + e * T] = cmul(wz[e], w);
            w = cmul(w, ws);
          }
        }
      }
    }
    if constexpr (KIND == FR_PROBE_Z) {
      fftr::fft<NR2, EN, 1>(vn, j, buf, a.tw, TWN);
      cplx* Zb = a.Z2 + (int64_t)b * a.n;
      cplx w = tw4<1>(a, ((int64_t)j * k1 * 2) & (a.L - 1));
      const cplx ws = tw4<1>(a, ((int64_t)T * k1 * 2) & (a.L - 1));
#pragma unroll
      for (int e = 0; e < EN; ++e) {
        Zb[rowC + j + e * T] = cmul(vn[e], w);
        w = cmul(w, ws);
      }
    } else if constexpr (KIND == FR_ZSTAR || KIND == FR_AT) {
      fftr::fft<NR2, EN, 1>(vn, j, buf, a.tw, TWN);
      cplx w = tw4<1>(a, ((int64_t)j * k1 * 2) & (a.L - 1));
      const cplx ws = tw4<1>(a, ((int64_t)T * k1 * 2) & (a.L - 1));
#pragma unroll
      for (int e = 0; e < EN; ++e) {
        C1b[rowC + j + e * T] = cmul(vn[e], w);
        w = cmul(w, ws);
      }
    } else {
#pragma unroll
      for (int e = 0; e < EL; ++e) vl[e] = cscale(vn[e & (EN - 1)], Ws[j + e * T] * invL);
      fftr::fft<LR2, EL, 1>(vl, j, buf, a.tw, TWN);
      cplx w = tw4<1>(a, ((int64_t)j * k1) & (a.L - 1));
      const cplx ws = tw4<1>(a, ((int64_t)T * k1) & (a.L - 1));
#pragma unroll
      for (int e = 0; e < EL; ++e) {
        Gb[rowW + j + e * T] = cmul(vl[e], w);
        w = cmul(w, ws);
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// host orchestration
// ------------------------------------------------------------------------------------------
static int fft_e() {   // tuning knob: AZ_FFT_E=8 (8 values per thread), 17 (16 values, 8 columns per CTA)
  static int e = 0;
  if (!e) {
    const char* v = getenv("AZ_FFT_E");
    e = v ? atoi(v) : 16;
    if (e != 8 && e != 17) e = 16;
  }
  return e;
}

static int fft_er() {   // rows: AZ_FFT_ER=8 (8 values per thread), default 16
  static int e = 0;
  if (!e) {
    const char* v = getenv("AZ_FFT_ER");
    e = v ? atoi(v) : 16;
    if (e != 8) e = 16;
  }
  return e;
}

template <int NC, int KIND, int SRC, int EC, int MINB>
static az_status_t fcols_e(const P1f& a, int ncols, int nb, double cout, cudaStream_t st) {
  constexpr int T = NC / EC;
  constexpr int TC0 = (MINB == 1 ? 512 : 256) / T;
  constexpr int TC = TC0 < 2 ? 2 : (TC0 > 16 ? 16 : TC0);
  const size_t sm = (size_t)TC * col_stride<NC, TC, EC>() * sizeof(cplx);
  auto kern = k1f_cols<NC, TC, KIND, SRC, EC, MINB>;
  AZ_CUDA_CHECK(az_smem_attr(kern, sm));
  static const char* names[] = {"1f_cols_in_coef", "1f_cols_fine_mask", "1f_cols_out_gather", "1f_cols_out_resid",
                                "1f_cols_in_rows", "1f_cols_out_coef", "1f_cols_fwd", "1f_cols_resid_mid",
                                "1f_cols_out_coef_add", "1f_cols_out_z"};
  AzTrace tr(a.trace_name ? a.trace_name : names[KIND], st, nb);
  kern<<<dim3(az_div_up(ncols, TC), nb), TC * T, sm, st>>>(a, cout);
  AZ_LAUNCH_CHECK();
  return AZ_OK;
}

static bool cols_persist() {   // AZ_COLS_PERSIST=0: one CTA per (column tile, pair), no prefetch
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("AZ_COLS_PERSIST");
    v = (e && *e == '0') ? 0 : 1;
  }
  return v != 0;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency)
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    else
      cudaGetLastError();
  }
  return fn;
}

// the [pair][row][column] complex tensor of a column pass's input: rows N1, row length W complex,
// pair stride pstride complex; boxes of TC complex x BOXR rows x 1 pair
static bool make_cols_tmap(CUtensorMap* m, const cplx* base, int N1, int W, int64_t pstride, int nb, int TC, int BOXR) {
  auto enc = tmap_encode();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)(2 * W), (cuuint64_t)N1, (cuuint64_t)nb};
  const cuuint64_t strides[2] = {(cuuint64_t)W * sizeof(cplx), (cuuint64_t)pstride * sizeof(cplx)};
  const cuuint32_t box[3] = {(cuuint32_t)(2 * TC), (cuuint32_t)BOXR, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<cplx*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NC, int KIND>
static az_status_t fcols_p(const P1f& a, int ncols, int nb, double cout, cudaStream_t st, bool* done) {
  constexpr int EC = 16, TC = 4, MINB = 1;
  using C = ColsP<NC, TC, EC>;
  *done = false;
  const bool coef = (KIND == FC_OUT_COEF || KIND == FC_OUT_COEF_ADD || KIND == FC_OUT_Z);
  const cplx* base = KIND == FC_OUT_Z ? a.Z2 : (coef ? a.C1 : a.G);
  const int W = coef ? a.N2 : a.L2;
  const int64_t pstride = coef ? a.n : a.L;
  if (ncols % TC || ((uintptr_t)base & 15)) return AZ_OK;
  CUtensorMap m;
  if (!make_cols_tmap(&m, base + (int64_t)a.pair0 * 0, a.N1, W, pstride, nb, TC, C::BOXR)) return AZ_OK;
  auto kern = k1f_cols_p<NC, TC, KIND, EC, MINB>;
  AZ_CUDA_CHECK(az_smem_attr(kern, C::smem));
  static int resident = 0;
  if (!resident) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, C::NT, C::smem) != cudaSuccess || per < 1) {
      cudaGetLastError();
      per = 1;
    }
    resident = per * sms;
  }
  const int tiles = ncols / TC;
  const int pg = std::max(1, std::min(nb, (4 * resident + tiles - 1) / tiles));
  static const char* names[] = {"1f_cols_in_coef", "1f_cols_fine_mask", "1f_cols_out_gather", "1f_cols_out_resid",
                                "1f_cols_in_rows", "1f_cols_out_coef", "1f_cols_fwd", "1f_cols_resid_mid",
                                "1f_cols_out_coef_add", "1f_cols_out_z"};
  AzTrace tr(a.trace_name ? a.trace_name : names[KIND], st, nb);
  kern<<<dim3(tiles, pg), C::NT, C::smem, st>>>(a, cout, m, nb, pg);
  AZ_LAUNCH_CHECK();
  *done = true;
  return AZ_OK;
}

template <int NC, int KIND, int SRC>
static az_status_t fcols(const P1f& a, int ncols, int nb, double cout, cudaStream_t st) {
  // measured on c2 (ms per step, one-tile -> persistent): out_z 0.644 -> 0.612, out_gather 0.460 ->
  // 0.441, fine_mask 0.762 -> 0.779, out_resid 0.893 -> 1.407 (its gather of b stalls the one 8-warp
  // CTA per SM): the persistent form is used where the tile is the pass's only input
  constexpr bool tile_in = KIND == FC_OUT_GATHER || KIND == FC_OUT_COEF || KIND == FC_OUT_Z;
  if constexpr (tile_in && NC >= 256 && ColsP<NC, 4, 16>::smem <= 227 * 1024) {
    if (cols_persist() && fft_e() == 16) {
      bool done = false;
      AZ_TRY((fcols_p<NC, KIND>(a, ncols, nb, cout, st, &done)));
      if (done) return AZ_OK;
    }
  }
  if (fft_e() == 8) return fcols_e<NC, KIND, SRC, 8, 3>(a, ncols, nb, cout, st);
  if (fft_e() == 17) return fcols_e<NC, KIND, SRC, 16, 1>(a, ncols, nb, cout, st);
  return fcols_e<NC, KIND, SRC, 16, 2>(a, ncols, nb, cout, st);
}

template <int NR2, int KIND, int EL, int MINB>
static az_status_t frows_e(const P1f& a, int nb, cudaStream_t st) {
  constexpr int LR2 = 2 * NR2;
  constexpr int T = LR2 / EL;
  constexpr int RPC0 = 128 / T;
  constexpr int RPC = RPC0 < 1 ? 1 : (RPC0 > 64 ? 64 : RPC0);
  const size_t sm = (size_t)RPC * (row_buf<NR2, LR2, EL>() * sizeof(cplx) + (LR2 + 3 * NR2) * sizeof(double));
  auto kern = k1f_rows<NR2, LR2, RPC, KIND, EL, MINB>;
  AZ_CUDA_CHECK(az_smem_attr(kern, sm));
  static const char* names[] = {"1f_rows_expand", "1f_rows_expand_keep", "1f_rows_step1", "1f_rows_resid",
                                "1f_rows_zstar", "1f_rows_at", "1f_rows_expand_probe", "1f_rows_probe_z"};
  AzTrace tr(names[KIND], st, nb);
  kern<<<dim3(az_div_up(a.N1, RPC), nb), RPC * T, sm, st>>>(a, a.N1);
  AZ_LAUNCH_CHECK();
  return AZ_OK;
}

static bool rows_persist() {   // AZ_ROWS_PERSIST=0: one CTA per (row, pair), no prefetch (k1f_rows)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("AZ_ROWS_PERSIST");
    v = (e && *e == '0') ? 0 : 1;
  }
  return v != 0;
}

template <int NR2, int KIND>
static az_status_t frows_p(const P1f& a, int nb, cudaStream_t st) {
  constexpr int LR2 = 2 * NR2;
  using C = RowsP<NR2, LR2, KIND>;
  auto kern = k1f_rows_p<NR2, LR2, KIND>;
  AZ_CUDA_CHECK(az_smem_attr(kern, C::smem));
  static int resident = 0;   // CTAs the GPU holds at once (2 per SM by the launch bound / shared memory)
  if (!resident) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, C::T, C::smem) != cudaSuccess || per < 1) {
      cudaGetLastError();
      per = 1;
    }
    resident = per * sms;
  }
  // split the pairs so that the grid is >= 4 waves (tails) while each CTA still walks several pairs
  const int pg = std::max(1, std::min(nb, (4 * resident + a.N1 - 1) / a.N1));
  static const char* names[] = {"1f_rows_expand", "1f_rows_expand_keep", "1f_rows_step1", "1f_rows_resid",
                                "1f_rows_zstar", "1f_rows_at", "1f_rows_expand_probe", "1f_rows_probe_z"};
  AzTrace tr(names[KIND], st, nb);
  kern<<<dim3(a.N1, pg), C::T, C::smem, st>>>(a, nb, pg);
  AZ_LAUNCH_CHECK();
  return AZ_OK;
}

template <int NR2, int KIND>
static az_status_t frows(const P1f& a, int nb, cudaStream_t st) {
  if (fft_er() == 8) return frows_e<NR2, KIND, 8, 3>(a, nb, st);
  // the persistent form needs 16-byte aligned rows of at least 16 values (NR2 >= 64 here)
  if (rows_persist() && NR2 >= 64) return frows_p<NR2, KIND>(a, nb, st);
  return frows_e<NR2, KIND, 16, 3>(a, nb, st);
}

template <int NC, int NR2>
static az_status_t run1f(const P1f& a0, int op, int src, int64_t npairs, int64_t Bmax, cudaStream_t st) {
  const int N2 = NR2, L2 = 2 * NR2;
  for (int64_t p0 = 0; p0 < npairs; p0 += Bmax) {
    P1f a = a0;
    a.pair0 = p0;
    const int nb = (int)std::min<int64_t>(Bmax, npairs - p0);
    switch (op) {
      case OP_A:
        AZ_TRY(fcols<NC, FC_IN_COEF, SRC_VEC>(a, N2, nb, 1.0, st));
        AZ_TRY(frows<NR2, FR_EXPAND>(a, nb, st));
        AZ_TRY(fcols<NC, FC_OUT_GATHER, SRC_VEC>(a, L2, nb, 1.0, st));
        break;
      case OP_STEP1:
        if (src == SRC_PROBE) {   // spectral probes (reading R35): v^ drawn in the first row pass
          AZ_TRY(frows<NR2, FR_EXPAND_PROBE>(a, nb, st));
        } else {
          AZ_TRY(fcols<NC, FC_IN_COEF, SRC_VEC>(a, N2, nb, 1.0, st));
          AZ_TRY(frows<NR2, FR_EXPAND_KEEP>(a, nb, st));
        }
        AZ_TRY(fcols<NC, FC_FINE_MASK, SRC_VEC>(a, L2, nb, 1.0, st));
        AZ_TRY(frows<NR2, FR_STEP1>(a, nb, st));
        AZ_TRY(fcols<NC, FC_OUT_GATHER, SRC_VEC>(a, L2, nb, 1.0, st));
        if (a.Z2 && !a.defer_z) AZ_TRY(fcols<NC, FC_OUT_Z, SRC_VEC>(a, N2, nb, 1.0 / (double)a.n, st));   // M
        break;
      case OP_RESID:
        AZ_TRY(fcols<NC, FC_IN_ROWS, SRC_VEC>(a, L2, nb, 1.0, st));
        AZ_TRY(frows<NR2, FR_RESID>(a, nb, st));
        AZ_TRY(fcols<NC, FC_OUT_RESID, SRC_VEC>(a, L2, nb, 1.0, st));
        if (a.Z2 && !a.defer_z) AZ_TRY(fcols<NC, FC_OUT_Z, SRC_VEC>(a, N2, nb, 1.0 / (double)a.n, st));
        break;
      case OP_ZSTAR:
        AZ_TRY(fcols<NC, FC_IN_ROWS, SRC_VEC>(a, L2, nb, 1.0, st));
        AZ_TRY(frows<NR2, FR_ZSTAR>(a, nb, st));
        AZ_TRY(fcols<NC, FC_OUT_COEF, SRC_VEC>(a, N2, nb, 1.0 / (double)a.n, st));
        break;
      case OP_STEP2:   // x = x2 + Z* (b - A x2): in = x2, in2 = b, out = x
        AZ_TRY(fcols<NC, FC_IN_COEF, SRC_VEC>(a, N2, nb, 1.0, st));
        AZ_TRY(frows<NR2, FR_EXPAND>(a, nb, st));
        AZ_TRY(fcols<NC, FC_RESID_MID, SRC_VEC>(a, L2, nb, 1.0, st));
        AZ_TRY(frows<NR2, FR_ZSTAR>(a, nb, st));
        AZ_TRY(fcols<NC, FC_OUT_COEF_ADD, SRC_VEC>(a, N2, nb, 1.0 / (double)a.n, st));
        break;
      case OP_AT:
        AZ_TRY(fcols<NC, FC_IN_ROWS, SRC_VEC>(a, L2, nb, 1.0, st));
        AZ_TRY(frows<NR2, FR_AT>(a, nb, st));
        AZ_TRY(fcols<NC, FC_OUT_COEF, SRC_VEC>(a, N2, nb, 1.0 / (double)a.L, st));
        break;
    }
  }
  return AZ_OK;
}

static P1f make_p1f(az_plan_s* p) {
  P1f a;
  a.W0 = p->d_W0;
  a.W2 = p->d_W2;
  a.zinv = p->d_zinv;
  a.Wr = p->d_Wr;
  a.pos = p->d_pos;
  a.run0 = p->run0;
  a.run1 = p->run1;
  a.mask = p->d_mask;
  a.tw = p->d_tw;
  a.t4hi = p->d_tw4hi;
  a.t4lo = p->d_tw4lo;
  a.lap = p->op == AZ_ROW_LAPLACIAN;
  a.alpha = p->alpha;
  a.n = p->n;
  a.L = p->L;
  a.N1 = (int)p->N1;
  a.N2 = (int)p->N2;
  a.L2 = (int)p->L2;
  a.s = (int)p->s;
  a.M = p->M;
  a.seed = p->seed;
  a.C1 = p->d_C1;
  a.G = p->d_G;
  a.in = nullptr;
  a.in2 = nullptr;
  a.ldin2 = 0;
  a.out = nullptr;
  a.Z2 = nullptr;
  a.out2 = nullptr;
  a.ldout2 = 0;
  a.defer_z = false;
  a.ldin = a.ldout = 0;
  a.nvec = a.col0 = a.pair0 = 0;
  a.lead = 0;
  a.sqn = sqrt((double)p->n);
  a.trace_name = nullptr;
  return a;
}

#define AZ_1F_DISPATCH(FN, ...)                                                        \
  switch (p->N1 * 4096 + p->N2) {                                                      \
    case 64 * 4096 + 32: return FN<64, 32>(__VA_ARGS__);                               \
    case 128 * 4096 + 64: return FN<128, 64>(__VA_ARGS__);                             \
    case 256 * 4096 + 128: return FN<256, 128>(__VA_ARGS__);                           \
    case 512 * 4096 + 256: return FN<512, 256>(__VA_ARGS__);                           \
    case 1024 * 4096 + 512: return FN<1024, 512>(__VA_ARGS__);                         \
    case 2048 * 4096 + 1024: return FN<2048, 1024>(__VA_ARGS__);                       \
    case 64 * 4096 + 64: return FN<64, 64>(__VA_ARGS__);                               \
    case 128 * 4096 + 128: return FN<128, 128>(__VA_ARGS__);                           \
    case 256 * 4096 + 256: return FN<256, 256>(__VA_ARGS__);                           \
    case 512 * 4096 + 512: return FN<512, 512>(__VA_ARGS__);                           \
    case 1024 * 4096 + 1024: return FN<1024, 1024>(__VA_ARGS__);                       \
  }                                                                                    \
  az_set_error("four-step: unsupported N1 x N2 = %lld x %lld", (long long)p->N1, (long long)p->N2); \
  return AZ_ERR_NOT_SUPPORTED;

az_status_t az1f_apply(az_plan_s* p, int op, int src, const double* in, int64_t ldin, double* out,
                       int64_t ldout, int64_t nvec, int64_t col0, cudaStream_t st) {
  if (p->s != 2) {
    az_set_error("four-step layout supports L = 2 only");
    return AZ_ERR_NOT_SUPPORTED;
  }
  P1f a = make_p1f(p);
  a.in = in;
  a.ldin = ldin;
  a.out = out;
  a.ldout = ldout;
  a.nvec = nvec;
  a.col0 = col0;
  if (src == SRC_PROBE) a.lead = (int)(col0 & 1);
  const int64_t npairs = (nvec + a.lead + 1) / 2;
  AZ_1F_DISPATCH(run1f, a, op, src, npairs, p->Bmax, st)
}

// Forward length-L DFT of the fine-grid samples stored in natural order, result in the
// transposed four-step order [k1][k2'] (the symbol table W, step 0).
__global__ void k1f_copy(cplx* dst, const cplx* src, int64_t L) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < L) dst[i] = src[i];
}

template <int NC, int NR2>
static az_status_t fine_forward(az_plan_s* p, cplx* W, cudaStream_t st) {
  P1f a = make_p1f(p);
  k1f_copy<<<az_div_up(p->L, 256), 256, 0, st>>>(a.G, W, p->L);
  AZ_LAUNCH_CHECK();
  AZ_TRY(fcols<NC, FC_FWD_G, SRC_VEC>(a, 2 * NR2, 1, 1.0, st));      // FFT_N1 + twiddle
  AZ_TRY(az_fft_batch(p->d_tw, a.G, 2 * NR2, p->N1, -1, st));        // FFT_L2 along rows
  k1f_copy<<<az_div_up(p->L, 256), 256, 0, st>>>(W, a.G, p->L);
  AZ_LAUNCH_CHECK();
  return AZ_OK;
}

az_status_t az1f_fft_fine_forward(az_plan_s* p, cplx* W, cudaStream_t st) {
  AZ_1F_DISPATCH(fine_forward, p, W, st)
}

// Step 2 of Alg. 1 for the four-step layout in five passes:
//   x = x2 + Z* (b - A x2)
az_status_t az1f_step2(az_plan_s* p, const double* x2, int64_t ldx2, const double* b, int64_t ldb, double* x,
                       int64_t ldx, int64_t nvec, cudaStream_t st) {
  P1f a = make_p1f(p);
  a.in = x2;
  a.ldin = ldx2;
  a.in2 = b;
  a.ldin2 = ldb;
  a.out = x;
  a.ldout = ldx;
  a.nvec = nvec;
  a.col0 = 0;
  const int64_t npairs = (nvec + 1) / 2;
  AZ_1F_DISPATCH(run1f, a, OP_STEP2, SRC_VEC, npairs, p->Bmax, st)
}

// b' = (I - A Z*) b (out = bp) and Z* b (out2 = Zb, N x nvec) in one chain: the row pass also takes
// its Z* b spectrum to the coefficient side, one extra column pass finishes it.
az_status_t az1f_resid_z(az_plan_s* p, const double* b, int64_t ldb, double* bp, int64_t ldbp, double* Zb, int64_t ldz,
                         int64_t nvec, cudaStream_t st, cplx* Zspec, bool defer) {
  P1f a = make_p1f(p);
  a.in = b;
  a.ldin = ldb;
  a.out = bp;
  a.ldout = ldbp;
  a.Z2 = Zspec ? Zspec : p->d_Z2;
  a.defer_z = defer && (nvec + 1) / 2 <= p->Bmax;
  a.out2 = Zb;
  a.ldout2 = ldz;
  a.nvec = nvec;
  a.col0 = 0;
  const int64_t npairs = (nvec + 1) / 2;
  AZ_1F_DISPATCH(run1f, a, OP_RESID, SRC_VEC, npairs, p->Bmax, st)
}

// S = (A - A Z* A) Omega[:, col0 ..) and M = Omega - Z* A Omega (Om, N x ncols): the step-1 row
// pass already forms M's spectrum r^ = v^ - w^ and takes it to the coefficient side; one column pass
// finishes it.  Step 2 of the solve is then x = Z* b + M y (PAPER.md:229-230 by linearity of Z*).
az_status_t az1f_sketch_m(az_plan_s* p, int64_t col0, int64_t ncols, double* S, int64_t ldS, double* Om, int64_t ldOm,
                          cudaStream_t st, cplx* Zspec, bool defer) {
  P1f a = make_p1f(p);
  a.out = S;
  a.ldout = ldS;
  a.Z2 = Zspec ? Zspec : p->d_Z2;
  a.defer_z = defer && (col0 & 1) == 0 && (ncols + 1) / 2 <= p->Bmax;
  a.out2 = Om;
  a.ldout2 = ldOm;
  a.nvec = ncols;
  a.col0 = col0;
  a.lead = (int)(col0 & 1);
  const int64_t npairs = (ncols + a.lead + 1) / 2;
  AZ_1F_DISPATCH(run1f, a, OP_STEP1, SRC_PROBE, npairs, p->Bmax, st)
}

// Omega[:, col0 .. col0 + ncols) explicitly (N x ncols, ld ldOm) for the spectral probes of this layout
// (reading R35): per batch of probe pairs, the drawn spectrum -> IFFT_N2 -> twiddle (row pass, into the
// plan's Z2 buffer) -> IFFT_N1 / n (column pass).  Uses the plan's scratch: stream-ordered like every pass.
template <int NC, int NR2>
static az_status_t omega_run(P1f a, int64_t npairs, int64_t Bmax, cudaStream_t st) {
  for (int64_t p0 = 0; p0 < npairs; p0 += Bmax) {
    a.pair0 = p0;
    const int nb = (int)std::min<int64_t>(Bmax, npairs - p0);
    AZ_TRY(frows<NR2, FR_PROBE_Z>(a, nb, st));
    AZ_TRY(fcols<NC, FC_OUT_Z, SRC_VEC>(a, NR2, nb, 1.0 / (double)a.n, st));
  }
  return AZ_OK;
}

az_status_t az1f_omega_fill(az_plan_s* p, int64_t col0, int64_t ncols, double* Om, int64_t ldOm, cudaStream_t st) {
  if (ncols <= 0) return AZ_OK;
  P1f a = make_p1f(p);
  a.Z2 = p->d_Z2;
  a.out2 = Om;
  a.ldout2 = ldOm;
  a.nvec = ncols;
  a.col0 = col0;
  a.lead = (int)(col0 & 1);
  const int64_t npairs = (ncols + a.lead + 1) / 2;
  AZ_1F_DISPATCH(omega_run, a, npairs, p->Bmax, st)
}

// The closing column pass of az1f_resid_z / az1f_sketch_m (deferred, single batch): IFFT_N1 of the
// spectra in Zspec -> out (N x nvec)
template <int NC, int NR2>
static az_status_t out_z_run(const P1f& a, int64_t npairs, cudaStream_t st) {
  return fcols<NC, FC_OUT_Z, SRC_VEC>(a, NR2, (int)npairs, 1.0 / (double)a.n, st);
}

az_status_t az1f_out_z(az_plan_s* p, const cplx* Zspec, double* out, int64_t ldout, int64_t nvec, cudaStream_t st,
                       bool background) {
  P1f a = make_p1f(p);
  // (a background pass on the lowest-priority stream yields SMs to the others: its event-timed
  // duration is not its cost, so it is traced under its own label)
  if (background) a.trace_name = "1f_cols_out_z_bg";
  a.Z2 = const_cast<cplx*>(Zspec);
  a.out2 = out;
  a.ldout2 = ldout;
  a.nvec = nvec;
  a.col0 = 0;
  a.pair0 = 0;
  const int64_t npairs = (nvec + 1) / 2;
  if (npairs > p->Bmax) {
    az_set_error("az1f_out_z: more than one batch");
    return AZ_ERR_NOT_SUPPORTED;
  }
  AZ_1F_DISPATCH(out_z_run, a, npairs, st)
}
