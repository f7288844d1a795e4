// 1-D operators for L = s n <= 2048: the whole operator chain for one vector pair runs in one
// CTA with the data resident in shared memory (only the compulsory bytes touch HBM).
//
// Fine-grid formulation (equivalent to PAPER.md Sec. 3.1):
//   A^c a    = IFFT_L( W . FFT_L(a_up) ) / L,   a_up = a zero-stuffed onto the fine grid
//              (FFT_L(a_up)(kf) = a^(kf mod n): the s aliases of the coefficient spectrum),
//   W        = FFT_L( phi^per(q h_L) )  (Lemma 3 on the fine grid: W(k + m n) are the s
//              diagonals d_i of B up to the polyphase phase factors),
//   Z* y     = IFFT_n( zinv . sum_m conj(W(k+mn)) FFT_L(E y)(k+mn) ) / n   (B^dag P E, then F),
//   A^T y    = IFFT_n( sum_m conj(W(k+mn)) FFT_L(y)(k+mn) ) / L.
// IFFT_n of a spectrum f is read off the fine grid: IFFT_L(extend f)[s j] = s IFFT_n(f)[j].
// Two real vectors are processed together as one complex vector (real part = column 2p,
// imaginary part = column 2p+1): every operator here is real, so it acts on both at once.
#include "az_fft.cuh"
#include "az_internal.h"

struct P1s {
  const cplx* W0;
  const cplx* W2;
  const double* zinv;
  const int32_t* pos;
  const cplx* tw;
  int lap;
  double k0sq;
  double alpha;
  int n, s;
  uint64_t seed;
  const double* in;
  int64_t ldin;
  double* out;
  int64_t ldout;
  int64_t nvec;
  int64_t col0;
  // boundary rows (1-D ODE): rows M .. M + Mb - 1 are beta phi_j(x_b);
  // window of win centres starting at bj[2 b] with weights bw[2 b * 64 + t]
  int64_t M, Mb;
  double beta;
  int win;
  const double* bw;
  const int32_t* bj;
  // optional (OP_STEP1 / OP_RESID, step 2 by linearity, reading R30): the coefficient vector whose
  // spectrum the chain forms anyway -- M = Omega - Z* A Omega (step 1) or Z* b (resid) -- to zout
  double* zout;
  int64_t ldz;
};

// beta sum_t bw[b][t] coef[(j0_b + t) mod n] for boundary point b, by one thread (win <= 64 terms;
// the CTA of a short transform can be smaller than a warp); coef(j) callable
template <class F>
AZ_D cplx boundary_dot(const P1s& a, int b, F coef) {
  cplx acc = czero();
  const int j0 = a.bj[2 * b];
  for (int t = 0; t < a.win; ++t) {
    const int j = ((j0 + t) % a.n + a.n) % a.n;
    acc = cadd(acc, cscale(coef(j), a.bw[2 * b * 64 + t]));
  }
  return cscale(acc, a.beta);
}

AZ_D void cpa16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

// shared memory of one chain CTA: the transform buffer, the n-point spectrum, and the plan tables
// (symbol W, and W'' for the Laplacian rows; 1/sigma^2; the row map), staged once per CTA by one
// batch of cp.async -- a CTA of L/8 threads has no other warps to hide a table load's latency,
// and the loops that read them would otherwise wait on one round trip per iteration
template <int L>
AZ_HD size_t chain1s_smem(int n, int lap) {
  return (size_t)(spad_len(L) + n + L * (lap ? 2 : 1)) * sizeof(cplx) + (size_t)n * sizeof(double) +
         (size_t)L * sizeof(int32_t);
}

template <int L, int OP, int SRC>
__global__ void __launch_bounds__(L / 8) k_chain1s(P1s a) {
  extern __shared__ cplx sm[];
  cplx* buf = sm;                       // spad_len(L)
  cplx* aux = sm + spad_len(L);         // n
  constexpr int NT = L / 8;
  const int tid = threadIdx.x;
  const int n = a.n, s = a.s;
  cplx* W0s = aux + n;                  // L
  cplx* W2s = W0s + L;                  // L (Laplacian rows only)
  double* zs = (double*)(W0s + L * (a.lap ? 2 : 1));   // n
  int32_t* ps = (int32_t*)(zs + n);     // L
  for (int i = tid; i < L; i += NT) {
    cpa16(W0s + i, a.W0 + i);
    if (a.lap) cpa16(W2s + i, a.W2 + i);
  }
  for (int i = tid; 2 * i < n; i += NT) cpa16(zs + 2 * i, a.zinv + 2 * i);
  for (int i = tid; 4 * i < L; i += NT) cpa16(ps + 4 * i, a.pos + 4 * i);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  auto sym = [&](int kf) { return a.lap ? cscale(cadd(W2s[kf], cscale(W0s[kf], a.k0sq)), a.alpha) : W0s[kf]; };
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  const int64_t cre = 2 * (int64_t)blockIdx.x, cim = cre + 1;
  const bool has_im = cim < a.nvec;
  const double invL = 1.0 / (double)L;

  // boundary rows that only need the coefficient input
  if constexpr (OP == OP_A) {
    for (int bp = tid; bp < a.Mb; bp += NT) {
      const cplx yb = boundary_dot(a, bp, [&](int j) {
        return make_double2(a.in[j + cre * a.ldin], has_im ? a.in[j + cim * a.ldin] : 0.0);
      });
      a.out[a.M + bp + cre * a.ldout] = yb.x;
      if (has_im) a.out[a.M + bp + cim * a.ldout] = yb.y;
    }
  }
  if constexpr (OP == OP_A || OP == OP_STEP1) {
    // ---- coefficient input, zero-stuffed onto the fine grid ----
    for (int q = tid; q < L; q += NT) buf[spad(q)] = czero();
    __syncthreads();
    if constexpr (SRC == SRC_PROBE) {
      for (int m = tid; m < n / 2; m += NT) {
        const cpair pr = probe_cplx_pair((uint64_t)m, (uint64_t)(a.col0 + cre), (uint64_t)(a.col0 + cim),
                                         has_im, a.seed);
        buf[spad(2 * m * s)] = pr.a;
        buf[spad((2 * m + 1) * s)] = pr.b;
      }
    } else {
      for (int j = tid; j < n; j += NT) {
        const double re = a.in[j + cre * a.ldin];
        const double im = has_im ? a.in[j + cim * a.ldin] : 0.0;
        buf[spad(j * s)] = make_double2(re, im);
      }
    }
    __syncthreads();
    fft_smem<L, -1>(buf, tid, a.tw, TWN);          // FFT_L(a_up)(kf) = a^(kf mod n)
    if constexpr (OP == OP_STEP1) {
      for (int k = tid; k < n; k += NT) aux[k] = buf[spad(k)];   // v^ kept for r^ = v^ - w^
    }
    for (int kf = tid; kf < L; kf += NT) buf[spad(kf)] = cscale(cmul(buf[spad(kf)], sym(kf)), invL);
    __syncthreads();
    fft_smem<L, 1>(buf, tid, a.tw, TWN);           // A^c a on the full grid
    if constexpr (OP == OP_STEP1) {
      // E R: keep the collocation points only
      for (int q = tid; q < L; q += NT)
        if (ps[q] < 0) buf[spad(q)] = czero();
      __syncthreads();
      fft_smem<L, -1>(buf, tid, a.tw, TWN);
      // B^dag P fold + spectral division, then r^ = v^ - w^
      for (int k = tid; k < n; k += NT) {
        cplx acc = czero();
        for (int m = 0; m < s; ++m) {
          const int kf = k + m * n;
          acc = cadd(acc, cmulc(buf[spad(kf)], sym(kf)));
        }
        aux[k] = csub(aux[k], cscale(acc, zs[k]));
      }
      __syncthreads();
      if (a.Mb > 0 || a.zout) {
        // r = v - Z* A v from its spectrum r^ (aux), IFFT_L(extend r^)[s j] / L = r_j: the boundary
        // rows of (A - A Z* A) v = A^b r, and M's column pair
        for (int kf = tid; kf < L; kf += NT) buf[spad(kf)] = aux[kf & (n - 1)];
        __syncthreads();
        fft_smem<L, 1>(buf, tid, a.tw, TWN);
        if (a.zout)
          for (int j = tid; j < n; j += NT) {
            const cplx v = cscale(buf[spad(j * s)], invL);
            a.zout[j + cre * a.ldz] = v.x;
            if (has_im) a.zout[j + cim * a.ldz] = v.y;
          }
        for (int bp = tid; bp < a.Mb; bp += NT) {
          const cplx yb = boundary_dot(a, bp, [&](int j) { return cscale(buf[spad(j * s)], invL); });
          a.out[a.M + bp + cre * a.ldout] = yb.x;
          if (has_im) a.out[a.M + bp + cim * a.ldout] = yb.y;
        }
        __syncthreads();
      }
      for (int kf = tid; kf < L; kf += NT) buf[spad(kf)] = cscale(cmul(aux[kf & (n - 1)], sym(kf)), invL);
      __syncthreads();
      fft_smem<L, 1>(buf, tid, a.tw, TWN);
    }
    // ---- R: gather the collocation rows ----
    for (int q = tid; q < L; q += NT) {
      const int r = ps[q];
      if (r >= 0) {
        const cplx v = buf[spad(q)];
        a.out[r + cre * a.ldout] = v.x;
        if (has_im) a.out[r + cim * a.ldout] = v.y;
      }
    }
  } else {
    // ---- row input, E: zero padding onto the fine grid ----
    for (int q = tid; q < L; q += NT) {
      const int r = ps[q];
      cplx v = czero();
      if (r >= 0) v = make_double2(a.in[r + cre * a.ldin], has_im ? a.in[r + cim * a.ldin] : 0.0);
      buf[spad(q)] = v;
    }
    __syncthreads();
    fft_smem<L, -1>(buf, tid, a.tw, TWN);
    for (int k = tid; k < n; k += NT) {
      cplx acc = czero();
      for (int m = 0; m < s; ++m) {
        const int kf = k + m * n;
        acc = cadd(acc, cmulc(buf[spad(kf)], sym(kf)));
      }
      aux[k] = (OP == OP_AT) ? acc : cscale(acc, zs[k]);
    }
    __syncthreads();
    if constexpr (OP == OP_RESID) {
      if (a.Mb > 0 || a.zout) {
        // w = Z* b from its spectrum (aux): the boundary rows of (I - A Z*) b, b_b - A^b w, and Z* b
        for (int kf = tid; kf < L; kf += NT) buf[spad(kf)] = aux[kf & (n - 1)];
        __syncthreads();
        fft_smem<L, 1>(buf, tid, a.tw, TWN);
        if (a.zout)
          for (int j = tid; j < n; j += NT) {
            const cplx v = cscale(buf[spad(j * s)], invL);
            a.zout[j + cre * a.ldz] = v.x;
            if (has_im) a.zout[j + cim * a.ldz] = v.y;
          }
        for (int bp = tid; bp < a.Mb; bp += NT) {
          const cplx yb = boundary_dot(a, bp, [&](int j) { return cscale(buf[spad(j * s)], invL); });
          const int64_t r = a.M + bp;
          a.out[r + cre * a.ldout] = a.in[r + cre * a.ldin] - yb.x;
          if (has_im) a.out[r + cim * a.ldout] = a.in[r + cim * a.ldin] - yb.y;
        }
        __syncthreads();
      }
      for (int kf = tid; kf < L; kf += NT) buf[spad(kf)] = cscale(cmul(aux[kf & (n - 1)], sym(kf)), invL);
    } else {
      for (int kf = tid; kf < L; kf += NT) buf[spad(kf)] = aux[kf & (n - 1)];
    }
    __syncthreads();
    fft_smem<L, 1>(buf, tid, a.tw, TWN);
    if constexpr (OP == OP_RESID) {
      for (int q = tid; q < L; q += NT) {
        const int r = ps[q];
        if (r >= 0) {
          const cplx v = buf[spad(q)];
          a.out[r + cre * a.ldout] = a.in[r + cre * a.ldin] - v.x;
          if (has_im) a.out[r + cim * a.ldout] = a.in[r + cim * a.ldin] - v.y;
        }
      }
    } else {
      const double c = (OP == OP_ZSTAR) ? invL : invL / (double)s;
      for (int j = tid; j < n; j += NT) {
        cplx v = cscale(buf[spad(j * s)], c);
        if (OP == OP_AT)   // + (A^b)^T y_b: beta phi_j(x_b) y_b over the boundary windows covering j
          for (int bp = 0; bp < a.Mb; ++bp) {
            const int t = ((j - a.bj[2 * bp]) % n + n) % n;
            if (t < a.win) {
              const double wgt = a.beta * a.bw[2 * bp * 64 + t];
              const int64_t r = a.M + bp;
              v = cadd(v, make_double2(wgt * a.in[r + cre * a.ldin], has_im ? wgt * a.in[r + cim * a.ldin] : 0.0));
            }
          }
        a.out[j + cre * a.ldout] = v.x;
        if (has_im) a.out[j + cim * a.ldout] = v.y;
      }
    }
  }
}

template <int L>
static az_status_t launch1s(const P1s& a, int op, int src, int64_t npairs, cudaStream_t st) {
  const size_t sm = chain1s_smem<L>(a.n, a.lap);
  const dim3 grid((unsigned)npairs), block(L / 8);
  AzTrace tr("1d_chain", st, npairs);
#define AZ_L1S(OPV, SRCV) (az_smem_attr(k_chain1s<L, OPV, SRCV>, sm), k_chain1s<L, OPV, SRCV><<<grid, block, sm, st>>>(a))
  if (op == OP_A) AZ_L1S(OP_A, SRC_VEC);
  else if (op == OP_STEP1 && src == SRC_PROBE) AZ_L1S(OP_STEP1, SRC_PROBE);
  else if (op == OP_STEP1) AZ_L1S(OP_STEP1, SRC_VEC);
  else if (op == OP_AT) AZ_L1S(OP_AT, SRC_VEC);
  else if (op == OP_ZSTAR) AZ_L1S(OP_ZSTAR, SRC_VEC);
  else AZ_L1S(OP_RESID, SRC_VEC);
#undef AZ_L1S
  AZ_LAUNCH_CHECK();
  return AZ_OK;
}

az_status_t az1s_apply(az_plan_s* p, int op, int src, const double* in, int64_t ldin, double* out,
                       int64_t ldout, int64_t nvec, int64_t col0, cudaStream_t st, double* zout, int64_t ldz) {
  P1s a;
  a.zout = (op == OP_STEP1 || op == OP_RESID) ? zout : nullptr;
  a.ldz = ldz;
  a.W0 = p->d_W0;
  a.W2 = p->d_W2;
  a.zinv = p->d_zinv;
  a.pos = p->d_pos;
  a.tw = p->d_tw;
  a.lap = p->op == AZ_ROW_LAPLACIAN;
  a.k0sq = p->k0sq;
  a.alpha = p->alpha;
  a.n = (int)p->n;
  a.s = (int)p->s;
  a.seed = p->seed;
  a.in = in;
  a.ldin = ldin;
  a.out = out;
  a.ldout = ldout;
  a.nvec = nvec;
  a.col0 = col0;
  a.M = p->M;
  a.Mb = p->Mb;
  a.beta = p->beta;
  a.win = p->win;
  a.bw = p->d_bw;
  a.bj = p->d_bj;
  const int64_t npairs = (nvec + 1) / 2;
  switch (p->L) {
    case 16: return launch1s<16>(a, op, src, npairs, st);
    case 32: return launch1s<32>(a, op, src, npairs, st);
    case 64: return launch1s<64>(a, op, src, npairs, st);
    case 128: return launch1s<128>(a, op, src, npairs, st);
    case 256: return launch1s<256>(a, op, src, npairs, st);
    case 512: return launch1s<512>(a, op, src, npairs, st);
    case 1024: return launch1s<1024>(a, op, src, npairs, st);
    case 2048: return launch1s<2048>(a, op, src, npairs, st);
  }
  az_set_error("1-D small layout: unsupported L = %lld", (long long)p->L);
  return AZ_ERR_NOT_SUPPORTED;
}
