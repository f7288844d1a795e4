// Register-resident Stockham FFT (FP64 complex) for the HBM-bound operator passes.
//
// One FFT of length L is computed by T = L / E threads, each holding E complex values in registers
// in the "strided" distribution
//        v[e] = x[j + e T],   j in [0, T), e in [0, E).
// Input and output use the same distribution, so pointwise operations between transforms (the
// symbol multiply, polyphase fold / expand, mask) are thread-local whenever the index maps of the
// two transforms agree (e.g. length-2048 with E = 16 and length-1024 with E = 8 both have T = 128:
// x[j + 128 e] and its alias x[j + 128 e + 1024] sit in the same thread).  Only the exchanges
// between radix stages go through shared memory (a length-2048 transform with E = 16 has stages
// 16 x 16 x 8: two exchanges instead of the four of a radix-8 shared-memory FFT).
//
// Stockham stage (Govindaraju et al. SC'08), radix R, span NS (virtual thread jj in [0, L / R)):
//   k = jj mod NS;  u_r = in[jj + r L / R] w^{k r},  w = e^{DIR 2 pi i / (NS R)};  U = DFT_R(u);
//   out[(jj / NS) NS R + k + r NS] = U_r.
// A thread runs the E / R butterflies jj = j + b T (b < E / R) of a stage; butterfly b's inputs and
// (for the last stage) outputs are registers v[b + r E / R].  Unnormalised:
//   DIR = -1:  X[q] = sum x[p] e^{-2 pi i p q / L},   DIR = +1: e^{+...}.
#pragma once
#include "az_common.cuh"

namespace fftr {

template <int DIR>
AZ_D cplx mul_i(cplx a) {   // a * (DIR i)
  return DIR < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}

template <int DIR>
AZ_D void bf2(cplx& a, cplx& b) {
  const cplx t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

// in-place DFT of 4 values x[s0], x[s0 + st], x[s0 + 2 st], x[s0 + 3 st] (natural order out)
template <int DIR, int N>
AZ_D void dft4s(cplx (&x)[N], int s0, int st) {
  const cplx a0 = x[s0], a1 = x[s0 + st], a2 = x[s0 + 2 * st], a3 = x[s0 + 3 * st];
  const cplx t0 = cadd(a0, a2), t1 = csub(a0, a2);
  const cplx t2 = cadd(a1, a3), t3 = mul_i<DIR>(csub(a1, a3));
  x[s0] = cadd(t0, t2);
  x[s0 + 2 * st] = csub(t0, t2);
  x[s0 + st] = cadd(t1, t3);
  x[s0 + 3 * st] = csub(t1, t3);
}

template <int DIR>
AZ_D void dft2(cplx (&u)[2]) {
  bf2<DIR>(u[0], u[1]);
}

template <int DIR>
AZ_D void dft4(cplx (&u)[4]) {
  dft4s<DIR, 4>(u, 0, 1);
}

template <int DIR>
AZ_D void dft8(cplx (&u)[8]) {
  const double c = 0.70710678118654752440;
  cplx e[4] = {u[0], u[2], u[4], u[6]};
  cplx o[4] = {u[1], u[3], u[5], u[7]};
  dft4s<DIR, 4>(e, 0, 1);
  dft4s<DIR, 4>(o, 0, 1);
  const cplx o1 = cscale(cadd(o[1], mul_i<DIR>(o[1])), c);
  const cplx o2 = mul_i<DIR>(o[2]);
  const cplx o3 = cscale(csub(mul_i<DIR>(o[3]), o[3]), c);
  u[0] = cadd(e[0], o[0]);
  u[4] = csub(e[0], o[0]);
  u[1] = cadd(e[1], o1);
  u[5] = csub(e[1], o1);
  u[2] = cadd(e[2], o2);
  u[6] = csub(e[2], o2);
  u[3] = cadd(e[3], o3);
  u[7] = csub(e[3], o3);
}

// 16-point DFT as 4 x 4: columns (stride 4), twiddles w16^{n1 k2}, rows, transpose.
template <int DIR>
AZ_D void dft16(cplx (&u)[16]) {
  const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173, h = 0.70710678118654752440;
  // DFT over n2 (u[n1 + 4 n2], stride 4) for each n1
#pragma unroll
  for (int n1 = 0; n1 < 4; ++n1) dft4s<DIR, 16>(u, n1, 4);
  // now u[n1 + 4 k2]; multiply by w16^{n1 k2}, w16 = e^{DIR 2 pi i / 16}
  const double sd = DIR < 0 ? -1.0 : 1.0;
  const cplx w1 = make_double2(c1, sd * s1), w2 = make_double2(h, sd * h), w3 = make_double2(s1, sd * c1);
  const cplx w6 = make_double2(-h, sd * h), w9 = make_double2(-c1, -sd * s1);
  u[1 + 4] = cmul(u[1 + 4], w1);
  u[1 + 8] = cmul(u[1 + 8], w2);
  u[1 + 12] = cmul(u[1 + 12], w3);
  u[2 + 4] = cmul(u[2 + 4], w2);
  u[2 + 8] = mul_i<DIR>(u[2 + 8]);
  u[2 + 12] = cmul(u[2 + 12], w6);
  u[3 + 4] = cmul(u[3 + 4], w3);
  u[3 + 8] = cmul(u[3 + 8], w6);
  u[3 + 12] = cmul(u[3 + 12], w9);
  // DFT over n1 (stride 1) for each k2
#pragma unroll
  for (int k2 = 0; k2 < 4; ++k2) dft4s<DIR, 16>(u, 4 * k2, 1);
  // output index k = k2 + 4 k1 is at u[k1 + 4 k2]: transpose the 4 x 4 block
  cplx t;
  t = u[1]; u[1] = u[4]; u[4] = t;
  t = u[2]; u[2] = u[8]; u[8] = t;
  t = u[3]; u[3] = u[12]; u[12] = t;
  t = u[6]; u[6] = u[9]; u[9] = t;
  t = u[7]; u[7] = u[13]; u[13] = t;
  t = u[11]; u[11] = u[14]; u[14] = t;
}

template <int R, int DIR>
AZ_D void dftR(cplx (&u)[R]) {
  if constexpr (R == 16) dft16<DIR>(u);
  else if constexpr (R == 8) dft8<DIR>(u);
  else if constexpr (R == 4) dft4<DIR>(u);
  else dft2<DIR>(u);
}

// shared-memory padding: one complex slot per E keeps the stride-E writes of a first stage
// conflict-free.  A 128-bit shared access is served per quarter warp (8 lanes x 16 B = one 128-byte
// wavefront), so 8 consecutive butterflies must land in 8 distinct 16-byte bank groups: with E
// values per thread the stride-E write index E j + r becomes (E + 1) j + r -> bank group j + r.
// (A stride-8 transform padded every 16 would put lanes j, j + 1 in the same group: 2-way.)
template <int E>
AZ_HD constexpr int padE(int i) { return i + (i >> (E >= 16 ? 4 : 3)); }
template <int E>
AZ_HD constexpr int padded_lenE(int L) { return L + (L >> (E >= 16 ? 4 : 3)) + 1; }
AZ_HD constexpr int padded_len(int L) { return padded_lenE<16>(L); }

// radix of the stage whose span is NS
template <int L, int E, int NS>
struct StageRadix {
  static constexpr int value = (L / NS) >= E ? E : (L / NS);
};

// twiddle operands of the stage whose span is NS: per butterfly b, w^(2^q) (q < NQ) with
// w = e^{DIR 2 pi i k / (NS R)}, k = (j + b T) mod NS, read from the table (conjugated for DIR > 0)
template <int L, int E, int NS>
struct StageTw {
  static constexpr int R = StageRadix<L, E, NS>::value;
  static constexpr int NB = E / R;
  static constexpr int NQ = R >= 16 ? 4 : (R >= 8 ? 3 : (R >= 4 ? 2 : 1));
};

template <int L, int E, int DIR, int NS>
AZ_D void load_tw(cplx (&wp)[StageTw<L, E, NS>::NB][4], int j, const cplx* __restrict__ tw, int twn) {
  using S = StageTw<L, E, NS>;
  constexpr int T = L / E;
#pragma unroll
  for (int b = 0; b < S::NB; ++b) {
    const int k = (j + b * T) & (NS - 1);
    const int tstep = k * (twn / (NS * S::R));
#pragma unroll
    for (int q = 0; q < S::NQ; ++q) {
      wp[b][q] = tw[tstep << q];
      if (DIR > 0) wp[b][q].y = -wp[b][q].y;
    }
  }
}

// One stage and, recursively, the rest.  PRE: this stage's twiddle operands wpre were loaded by the
// previous stage, so the table reads overlap its butterflies and exchange instead of stalling this
// stage's multiplies; a stage prefetches the next one's when they are at most PF complex values per
// thread (the register budget: PF = 8 for the 2048-point row transforms, 4 for the column passes).
template <int L, int E, int DIR, int NS, int PF, bool PRE>
AZ_D void stages(cplx (&v)[E], int j, cplx* buf, const cplx* __restrict__ tw, int twn,
                 const cplx (&wpre)[StageTw<L, E, NS>::NB][4]) {
  constexpr int R = StageRadix<L, E, NS>::value;
  constexpr int T = L / E;
  constexpr int NB = E / R;            // butterflies per thread
  constexpr bool last = NS * R == L;
  constexpr int NSN = last ? NS : NS * R;   // next stage's span
  constexpr bool pre_next = !last && StageTw<L, E, NSN>::NB * StageTw<L, E, NSN>::NQ <= PF;
  cplx wn[StageTw<L, E, NSN>::NB][4];
  if constexpr (pre_next) load_tw<L, E, DIR, NSN>(wn, j, tw, twn);
  cplx wp[NB][4];
  if constexpr (NS > 1) {
    if constexpr (PRE) {
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int q = 0; q < 4; ++q) wp[b][q] = wpre[b][q];
    } else {
      load_tw<L, E, DIR, NS>(wp, j, tw, twn);
    }
  }
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    cplx u[R];
#pragma unroll
    for (int r = 0; r < R; ++r) u[r] = v[b + r * NB];
    if constexpr (NS > 1) {
      // w^r from w, w^2, w^4, w^8 (at most 3 extra products per power: a few ulps)
#pragma unroll
      for (int r = 1; r < R; ++r) {
        cplx w = make_double2(1.0, 0.0);
        bool first = true;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (r & (1 << q)) {
            w = first ? wp[b][q] : cmul(w, wp[b][q]);
            first = false;
          }
        u[r] = cmul(u[r], w);
      }
    }
    dftR<R, DIR>(u);
#pragma unroll
    for (int r = 0; r < R; ++r) v[b + r * NB] = u[r];
  }
  if constexpr (!last) {
    constexpr int R2 = StageRadix<L, E, NS * R>::value;
    constexpr int NB2 = E / R2;
    __syncthreads();   // previous readers of buf are done
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int jj = j + b * T;
      const int k = jj & (NS - 1);
      const int o = (jj / NS) * NS * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) buf[padE<E>(o + r * NS)] = v[b + r * NB];
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < NB2; ++b) {
      const int jj = j + b * T;
#pragma unroll
      for (int r = 0; r < R2; ++r) v[b + r * NB2] = buf[padE<E>(jj + r * (L / R2))];
    }
    stages<L, E, DIR, NS * R, PF, pre_next>(v, j, buf, tw, twn, wn);
  }
}

// All threads of the CTA must call this (it contains __syncthreads).  buf: padded_lenE<E>(L) complex
// values private to this FFT.  tw[t] = e^{-2 pi i t / twn}, twn >= L a power of two.
template <int L, int E, int DIR, int PF = 8>
AZ_D void fft(cplx (&v)[E], int j, cplx* buf, const cplx* __restrict__ tw, int twn) {
  static_assert((L & (L - 1)) == 0 && (E & (E - 1)) == 0 && E <= 16 && E >= 2, "power-of-two sizes");
  static_assert(L % E == 0, "E must divide L");
  const cplx none[StageTw<L, E, 1>::NB][4] = {};   // the first stage has no twiddles
  stages<L, E, DIR, 1, PF, false>(v, j, buf, tw, twn, none);
}

}  // namespace fftr
