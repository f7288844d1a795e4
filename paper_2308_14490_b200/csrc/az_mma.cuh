// FP64 tensor-core (DMMA) warp tiles for the dense part of the path:
// the blocked Householder QR trailing updates and the block one-sided Jacobi SVD.
//
// tcgen05/UMMA has no FP64 kind on sm_100a, so the FP64 tensor path is the warp-level
// mma.sync.aligned.m8n8k4.row.col.f64 (SASS DMMA.8x8x4).  Fragment ownership (lane l):
//   A (8 x 4, row):  a    = A[l / 4][l % 4]
//   B (4 x 8, col):  b    = B[l % 4][l / 4]
//   C (8 x 8):       c[0] = C[l / 4][2 (l % 4)],  c[1] = C[l / 4][2 (l % 4) + 1]
// Shared-memory operand tiles use a row stride S with S % 16 == 4 (in doubles): the 16 lanes of a
// half-warp then read 16 distinct 8-byte bank pairs for both fragment shapes below.
#pragma once
#include "az_common.cuh"

AZ_D void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Operand layouts in shared memory.
//   KMAJ: element (i, k) at s[k * S + i]   (i = m for A, n for B)
//   IMAJ: element (i, k) at s[i * S + k]
enum { KMAJ = 0, IMAJ = 1 };

template <int LAYOUT>
AZ_D double frag_ld(const double* s, int S, int i, int k) {
  return LAYOUT == KMAJ ? s[k * S + i] : s[i * S + k];
}

// acc[mi][ni] (8x8 tiles) += A[m0 + 8 mi .., k0..k0+KD) * B[k0.., n0 + 8 ni ..)
// A element (m, k) and B element (k, n) are read with frag_ld<LA>(As, SA, m, k) and
// frag_ld<LB>(Bs, SB, n, k).  KU: k-steps unrolled together (fragment loads hoisted over them).
template <int MI, int NI, int LA, int LB, int KU = 2>
AZ_D void warp_mma(double (&acc)[MI][NI][2], const double* As, int SA, const double* Bs, int SB, int m0, int n0,
                   int k0, int KD, int lane) {
  const int r = lane >> 2, q = lane & 3;
#pragma unroll KU
  for (int kk = k0; kk < k0 + KD; kk += 4) {
    double a[MI], b[NI];
#pragma unroll
    for (int i = 0; i < MI; ++i) a[i] = frag_ld<LA>(As, SA, m0 + 8 * i + r, kk + q);
#pragma unroll
    for (int j = 0; j < NI; ++j) b[j] = frag_ld<LB>(Bs, SB, n0 + 8 * j + r, kk + q);
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) dmma(acc[i][j], a[i], b[j]);
  }
}

template <int MI, int NI>
AZ_D void acc_zero(double (&acc)[MI][NI][2]) {
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// Row / column of the C element held in acc[i][j][e] by `lane` (tile origin m0, n0).
AZ_D int acc_row(int m0, int i, int lane) { return m0 + 8 * i + (lane >> 2); }
AZ_D int acc_col(int n0, int j, int e, int lane) { return n0 + 8 * j + 2 * (lane & 3) + e; }
