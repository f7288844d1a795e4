// Shared-memory Stockham FFT (FP64 complex), CTA-cooperative, radix 8 with a final
// radix-4/2 stage.  Length L = 2^k, 8 <= L <= 2048, unnormalised:
//   DIR = -1:  X[q] = sum_r x[r] e^{-2 pi i q r / L}
//   DIR = +1:  X[q] = sum_r x[r] e^{+2 pi i q r / L}
// Layout: one FFT per buffer of spad_len(L) complex values, element i at buf[spad(i)].
// Threads: each FFT uses L/8 threads (index j in [0, L/8)); each thread owns exactly 8
// complex values per stage (1 radix-8, 2 radix-4 or 4 radix-2 butterflies).
// Twiddles come from a table tw[t] = e^{-2 pi i t / twn} (twn >= L, power of two), read
// through the read-only path (L1 resident).
//
// Stockham autosort iteration (Govindaraju et al., SC'08, "FftIteration"):
//   k = j mod Ns;  v_r = in[j + r L/R] * w^{k r},  w = e^{DIR 2 pi i / (Ns R)};
//   V = DFT_R(v);  out[(j / Ns) Ns R + k + r Ns] = V_r;   Ns *= R.
#pragma once
#include "az_common.cuh"

template <int DIR>
AZ_D cplx mul_dir_i(cplx a) {   // a * (DIR * i)
  return DIR < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}

template <int DIR>
AZ_D void dft2(cplx* v) {
  const cplx t = v[0];
  v[0] = cadd(t, v[1]);
  v[1] = csub(t, v[1]);
}

template <int DIR>
AZ_D void dft4(cplx* v) {
  const cplx t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
  const cplx t2 = cadd(v[1], v[3]), t3 = mul_dir_i<DIR>(csub(v[1], v[3]));
  v[0] = cadd(t0, t2);
  v[2] = csub(t0, t2);
  v[1] = cadd(t1, t3);
  v[3] = csub(t1, t3);
}

template <int DIR>
AZ_D void dft8(cplx* v) {
  const double c = 0.70710678118654752440;
  cplx e[4] = {v[0], v[2], v[4], v[6]};
  cplx o[4] = {v[1], v[3], v[5], v[7]};
  dft4<DIR>(e);
  dft4<DIR>(o);
  // w^q o_q, w = e^{DIR i pi / 4}
  const cplx o1 = cscale(cadd(o[1], mul_dir_i<DIR>(o[1])), c);
  const cplx o2 = mul_dir_i<DIR>(o[2]);
  const cplx o3 = cscale(csub(mul_dir_i<DIR>(o[3]), o[3]), c);
  v[0] = cadd(e[0], o[0]);
  v[4] = csub(e[0], o[0]);
  v[1] = cadd(e[1], o1);
  v[5] = csub(e[1], o1);
  v[2] = cadd(e[2], o2);
  v[6] = csub(e[2], o2);
  v[3] = cadd(e[3], o3);
  v[7] = csub(e[3], o3);
}

template <int R, int DIR>
AZ_D void dftR(cplx* v) {
  if constexpr (R == 8) dft8<DIR>(v);
  else if constexpr (R == 4) dft4<DIR>(v);
  else dft2<DIR>(v);
}

template <int L, int DIR, int R, int NS, int TPF>
AZ_D void stockham_stage(cplx* buf, int j, const cplx* __restrict__ tw, int twn) {
  constexpr int NB = L / (R * TPF);     // butterflies per thread
  constexpr int SIN = L / R;
  static_assert(NB >= 1 && NB * R * TPF == L, "bad thread split");
  cplx v[NB * R];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int jj = j + b * TPF;
    const int k = jj & (NS - 1);
#pragma unroll
    for (int r = 0; r < R; ++r) v[b * R + r] = buf[spad(jj + r * SIN)];
    if constexpr (NS > 1) {
      const int tstep = k * (twn / (NS * R));
#pragma unroll
      for (int r = 1; r < R; ++r) {
        cplx w = __ldg(&tw[tstep * r]);
        if (DIR > 0) w.y = -w.y;
        v[b * R + r] = cmul(v[b * R + r], w);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    dftR<R, DIR>(v + b * R);
    const int jj = j + b * TPF;
    const int k = jj & (NS - 1);
    const int idxD = (jj / NS) * NS * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) buf[spad(idxD + r * NS)] = v[b * R + r];
  }
  __syncthreads();
}

template <int L, int DIR, int NS, int TPF>
AZ_D void fft_stages(cplx* buf, int j, const cplx* __restrict__ tw, int twn) {
  if constexpr (NS * 8 <= L) {
    stockham_stage<L, DIR, 8, NS, TPF>(buf, j, tw, twn);
    fft_stages<L, DIR, NS * 8, TPF>(buf, j, tw, twn);
  } else if constexpr (NS * 4 == L) {
    stockham_stage<L, DIR, 4, NS, TPF>(buf, j, tw, twn);
  } else if constexpr (NS * 2 == L) {
    stockham_stage<L, DIR, 2, NS, TPF>(buf, j, tw, twn);
  }
}

// All threads of the CTA must call this (it contains __syncthreads); every thread always
// computes (ragged tails run on scratch slots whose results are not stored).
// TPF = threads per FFT (default L/8: 8 values per thread per stage; L/16: 16 values, ...).
template <int L, int DIR, int TPF = L / 8>
AZ_D void fft_smem(cplx* buf, int j, const cplx* __restrict__ tw, int twn) {
  static_assert(L >= 8 && (L & (L - 1)) == 0, "L must be a power of two >= 8");
  static_assert(TPF >= 1 && L % (8 * TPF) == 0, "TPF must divide L/8");
  fft_stages<L, DIR, 1, TPF>(buf, j, tw, twn);
}

// Number of Stockham stages (for sanity checks).
constexpr int fft_num_stages(int L) {
  int k = 0;
  while ((1 << k) < L) ++k;
  return k / 3 + (k % 3 ? 1 : 0);
}
