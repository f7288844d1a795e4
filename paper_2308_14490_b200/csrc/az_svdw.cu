// Truncated SVD solve for wide sketches (r > 128, "followed by
// the SVD"): block one-sided Jacobi on B = R_S^T with DMMA Gram matrices.
//
// As in az_svd.cu, one-sided Jacobi orthogonalises the columns of B = R_S^T:  B W = U' Sigma, so
// R_S = W Sigma U'^T, W holds the left singular vectors of R_S and is applied to c = Q^T b' on the
// fly (c <- W^T c); finally y = sum_{sigma_i > theta sigma_1} (B W)_i (W^T c)_i / sigma_i^2.
// Block version (columns in blocks of BW = 32, pairs of blocks -> X = [B_i B_j], r x 64):
//   G = X^T X                      (DMMA, fixed-order reduction)
//   G = V diag V^T                 (cyclic two-sided Jacobi on G in shared memory)
//   X <- X V,   c_pair <- V^T c_pair
// All block pairs of a round-robin round are disjoint and run as one launch (one CTA per pair);
// a sweep is nblk - 1 rounds.  Convergence: max over pairs of |G_pq| / sqrt(G_pp G_qq) below
// tol = 4 u sqrt(r) (the rounding level of a length-r dot product of orthogonal columns), ignoring
// columns whose norm is far below the truncation level (1e-3 theta sigma_1), which cannot change
// the kept part of the solution (same skip rule as az_svd.cu).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "az_internal.h"
#include "az_mma.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

constexpr int BW = 32;        // columns per block
constexpr int PW = 2 * BW;    // pair width
constexpr int GS = PW + 1;    // G stride (conflict-free row and column access)
constexpr int VS = PW + 4;    // V stride (B operand, KMAJ)
constexpr int XS = PW + 4;    // X tile stride
constexpr int GK = 32, GKS = GK + 4;   // Gram staging: [col][k], stride 36

struct BJArgs {
  double* B;        // r x r, column-major, ld = r
  int64_t r;
  double* C;        // r x nrhs, ld = r
  int nrhs;
  int nblk;         // column blocks (padded to even in the schedule)
  const double* smax2;    // max squared column norm at the start of the sweep
  double theta;
  unsigned long long* off;  // max relative off-diagonal seen this sweep (double bits, >= 0)
  double tol;               // rotate while |G_pq| > tol sqrt(G_pp G_qq)
  int inner_sweeps;
  long long* dbg;           // optional phase timestamps (cluster 0, rank 0): 8 x clock64
};

AZ_D void pair_of(int round, int pi, int n, int& p, int& q) {
  if (pi == 0) {
    p = round;
    q = n - 1;
  } else {
    p = (round + pi) % (n - 1);
    q = (round - pi + (n - 1)) % (n - 1);
  }
  if (p > q) {
    const int t = p;
    p = q;
    q = t;
  }
}

// One CTA cluster per block pair: the CS CTAs of the cluster split the r rows; their partial
// Gram matrices are reduced in a fixed order through distributed shared memory into the leader
// (cluster rank 0), which runs the eigensolver; every CTA then reads V from the leader's shared
// memory and rotates its own rows.
__global__ void __launch_bounds__(256, 1) k_bjac_round(BJArgs a, int round) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ double sm[];
  double* G = sm;                     // PW x GS
  double* V = G + PW * GS;            // PW x VS  (V[t][p] at t * VS + p)
  double* X = V + PW * VS;            // staging: Gram [col][k] (PW x GKS) / update [col][row] (PW x XS)
  double* Cs = X + PW * XS;           // 64 x XS: a 64-column tile of the pair's C rows ([col][k])
  __shared__ double rc[PW / 2], rs[PW / 2];
  __shared__ int rp[PW / 2], rq[PW / 2];
  __shared__ int any_rot;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int CS = (int)cluster.num_blocks(), crank = (int)cluster.block_rank();
  const int n = a.nblk + (a.nblk & 1);
  int bi, bj;
  pair_of(round, blockIdx.x / CS, n, bi, bj);
  if (bj >= a.nblk) return;           // whole cluster returns together (same pair)
  const int64_t r = a.r;
  const int64_t slice = ((r + CS - 1) / CS + 63) / 64 * 64;
  const int64_t rb = (int64_t)crank * slice, re = min(r, rb + slice);
  // column of X -> column of B (or -1 past the end)
  auto bcol = [&](int c) -> int64_t {
    const int64_t col = (c < BW) ? (int64_t)bi * BW + c : (int64_t)bj * BW + (c - BW);
    return col < r ? col : -1;
  };
  const bool dbg = a.dbg && blockIdx.x == 0 && threadIdx.x == 0;
  if (dbg) a.dbg[0] = clock64();
  // ---------------- partial Gram G = X^T X over rows [rb, re) ----------------
  {
    // G is symmetric: only the blocks II, IJ and JJ are formed (JI is mirrored by the leader after the
    // cluster reduction).  Warps 0-3 take II / IJ over one k half of the staged tile each, warps 4-7
    // take JJ over one k quarter each: 3 of the 4 block products, the same DMMA count on each SM
    // sub-partition (warps s and s + 4).
    const int blk = (w < 4) ? (w & 1) : 2;            // 0: II, 1: IJ, 2: JJ
    const int gm0 = (blk == 2) ? BW : 0, gn0 = (blk == 0) ? 0 : BW;
    double acc[4][4][2];
    acc_zero(acc);
    const int lk = tid & 31, li = tid >> 5;
    int64_t colp[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) colp[t] = bcol(li + 8 * t);
    double v[8];
    auto load = [&](int64_t k0) {
      const int64_t k = k0 + lk;
#pragma unroll
      for (int t = 0; t < 8; ++t) v[t] = (k < re && colp[t] >= 0) ? a.B[colp[t] * r + k] : 0.0;
    };
    load(rb);
    // two staging buffers in X and the C tile buffer behind it (free until the c rows at the end), one
    // barrier per tile: a warp stores tile t + 2 into the buffer of tile t only after the barrier of
    // tile t + 1, which every warp reaches after its MMAs of tile t
    static_assert(2 * GKS <= 2 * XS, "Gram double buffer must fit X + Cs");
    int par = 0;
    for (int64_t k0 = rb; k0 < re; k0 += GK, par ^= 1) {
      double* Xt = X + par * (PW * GKS);
#pragma unroll
      for (int t = 0; t < 8; ++t) Xt[(li + 8 * t) * GKS + lk] = v[t];
      __syncthreads();
      if (k0 + GK < re) load(k0 + GK);     // next tile in flight during the MMAs
      if (w < 4)
        warp_mma<4, 4, IMAJ, IMAJ>(acc, Xt, GKS, Xt, GKS, gm0, gn0, (w >> 1) * 16, 16, lane);
      else
        warp_mma<4, 4, IMAJ, IMAJ>(acc, Xt, GKS, Xt, GKS, gm0, gn0, (w - 4) * 8, 8, lane);
    }
    // fixed-order sums of the k parts into G: step 0 warps 0, 1, 4 store; step 1 warps 2, 3, 5 add;
    // step 2 warp 6; step 3 warp 7
    const int step = (w < 4) ? (w >> 1) : (w - 4);
#pragma unroll 1
    for (int sidx = 0; sidx < 4; ++sidx) {
      if (step == sidx) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              double* g = &G[acc_row(gm0, i, lane) * GS + acc_col(gn0, j, e, lane)];
              *g = sidx == 0 ? acc[i][j][e] : *g + acc[i][j][e];
            }
      }
      if (sidx < 3) __syncthreads();
    }
  }
  if (dbg) a.dbg[1] = clock64();
  cluster.sync();                     // partial Grams complete
  if (dbg) a.dbg[2] = clock64();
  const double negl = (1e-3 * a.theta) * (1e-3 * a.theta) * (*a.smax2);
  if (CS > 1) {
    // distributed fixed-order reduction: CTA c sums its slice of the entries over ranks 0..CS-1
    // and writes the sums into the leader's staging buffer X (free at this point)
    double* Xl = cluster.map_shared_rank(X, 0);
    const int per = (PW * GS + CS - 1) / CS;
    const int e0 = crank * per, e1 = min(PW * GS, e0 + per);
    for (int e = e0 + tid; e < e1; e += 256) {
      double t = 0.0;
      for (int c = 0; c < CS; ++c) t += cluster.map_shared_rank(G, c)[e];
      Xl[e] = t;
    }
    cluster.sync();
    if (crank == 0) {
      for (int e = tid; e < PW * GS; e += 256) G[e] = X[e];
      __syncthreads();
    }
  }
  if (crank == 0) {
    // the block JI of the symmetric G (not formed above)
    for (int e = tid; e < BW * BW; e += 256) {
      const int p = e / BW, q = BW + e % BW;
      G[q * GS + p] = G[p * GS + q];
    }
    __syncthreads();
    // ---------------- convergence measure ----------------
    double mx = 0.0;
    for (int e = tid; e < PW * PW; e += 256) {
      const int p = e / PW, q = e % PW;
      if (p < q) {
        const double gp = G[p * GS + p], gq = G[q * GS + q];
        if (fmin(gp, gq) >= negl && gp > 0.0 && gq > 0.0) mx = fmax(mx, fabs(G[p * GS + q]) / sqrt(gp * gq));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0 && mx > 0.0) atomicMax(a.off, (unsigned long long)__double_as_longlong(mx));
    if (tid == 0) any_rot = 0;
    __syncthreads();
    if (lane == 0 && mx > a.tol) atomicOr(&any_rot, 1);
    __syncthreads();
    if (any_rot) {
      // ---------------- eigen-decomposition of G by cyclic Jacobi ----------------
      // A half warp per rotation pair, each thread two pairs (pk0 and pk0 + 16; 32 disjoint pairs per
      // round): each thread recomputes its pairs' (c, s) itself (no broadcast), then rotates 4 of the
      // 64 entries of rows p, q (phase A) and of columns p, q of G and V (phase B): two barriers per
      // round.  Entry t = sub + 16 i: a half warp's 16 accesses fall in 16 distinct bank pairs for
      // rows (stride 1) and columns (stride GS = 65); V is rotated in the free staging buffer X at the
      // same stride and copied to its DMMA layout (stride VS) at the end -- the rounds are bound by
      // shared-memory wavefronts, which the former 8-threads-per-pair layout (two pairs per half warp)
      // and V's stride 68 multiplied by bank conflicts.  Same operations per entry, same results.
      double* Ve = X;   // PW x GS
      for (int e = tid; e < PW * PW; e += 256) Ve[(e / PW) * GS + (e % PW)] = (e / PW == e % PW) ? 1.0 : 0.0;
      __shared__ int rot_any;
      const int pk0 = tid >> 4, sub = tid & 15;
      constexpr int NE = PW / 16;
      const double tol2 = a.tol * a.tol;
      for (int sw = 0; sw < a.inner_sweeps; ++sw) {
        if (tid == 0) rot_any = 0;
        __syncthreads();
        for (int rd = 0; rd < PW - 1; ++rd) {
          int pp[2], qq[2];
          double cc[2], ss[2];
          bool rr[2];
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            int p, q;
            pair_of(rd, pk0 + 16 * h2, PW, p, q);
            pp[h2] = p;
            qq[h2] = q;
            const double gp = G[p * GS + p], gq = G[q * GS + q], g = G[p * GS + q];
            double c = 1.0, sn = 0.0;
            const double g2 = g * g;
            const bool rot_pq = g != 0.0 && g2 > tol2 * gp * gq && fmin(gp, gq) >= negl;
            if (rot_pq) {
              // t = tan = 2 g sign(d) / (|d| + sqrt(d^2 + 4 g^2)), d = G_qq - G_pp
              // (MUFU-seeded reciprocal / rsqrt with Newton steps, as in az_svd.cu: the IEEE division and
              // square root dominated this latency-bound chain -- one inner sweep cost ~0.2 ms per round)
              const double d = gq - gp;
              const double h = fma(d, d, 4.0 * g2);
              const double t = (d >= 0.0 ? 2.0 * g : -2.0 * g) * fast_rcp(fabs(d) + h * fast_rsqrt(h));
              c = fast_rsqrt(fma(t, t, 1.0));
              sn = c * t;
              if (sub == 0) rot_any = 1;
            }
            cc[h2] = c;
            ss[h2] = sn;
            rr[h2] = rot_pq;
          }
          if (dbg && rd == 5 && sw == 0) a.dbg[6] = clock64();
          __syncthreads();   // every pair has read its 2 x 2 block before any row is rotated
          if (dbg && rd == 5 && sw == 0) a.dbg[7] = clock64();
          // all loads of a phase are issued before its first store (no load waits on a store)
          {
            double xp[2][NE], xq[2][NE];
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2)
              if (rr[h2])
#pragma unroll
                for (int i = 0; i < NE; ++i) {
                  const int t = sub + 16 * i;
                  xp[h2][i] = G[pp[h2] * GS + t];
                  xq[h2][i] = G[qq[h2] * GS + t];
                }
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2)
              if (rr[h2])
#pragma unroll
                for (int i = 0; i < NE; ++i) {
                  const int t = sub + 16 * i;
                  G[pp[h2] * GS + t] = cc[h2] * xp[h2][i] - ss[h2] * xq[h2][i];
                  G[qq[h2] * GS + t] = ss[h2] * xp[h2][i] + cc[h2] * xq[h2][i];
                }
          }
          __syncthreads();
          {
            double xp[2][NE], xq[2][NE], vp[2][NE], vq[2][NE];
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2)
              if (rr[h2])
#pragma unroll
                for (int i = 0; i < NE; ++i) {
                  const int t = sub + 16 * i;
                  xp[h2][i] = G[t * GS + pp[h2]];
                  xq[h2][i] = G[t * GS + qq[h2]];
                  vp[h2][i] = Ve[t * GS + pp[h2]];
                  vq[h2][i] = Ve[t * GS + qq[h2]];
                }
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2)
              if (rr[h2])
#pragma unroll
                for (int i = 0; i < NE; ++i) {
                  const int t = sub + 16 * i;
                  G[t * GS + pp[h2]] = cc[h2] * xp[h2][i] - ss[h2] * xq[h2][i];
                  G[t * GS + qq[h2]] = ss[h2] * xp[h2][i] + cc[h2] * xq[h2][i];
                  Ve[t * GS + pp[h2]] = cc[h2] * vp[h2][i] - ss[h2] * vq[h2][i];
                  Ve[t * GS + qq[h2]] = ss[h2] * vp[h2][i] + cc[h2] * vq[h2][i];
                }
          }
          __syncthreads();
        }
        if (!rot_any) break;
      }
      for (int e = tid; e < PW * PW; e += 256) V[(e / PW) * VS + (e % PW)] = Ve[(e / PW) * GS + (e % PW)];
    }
  }
  if (dbg) a.dbg[3] = clock64();
  cluster.sync();                     // leader's V and flag ready
  const int rot = *cluster.map_shared_rank(&any_rot, 0);
  if (rot && crank != 0) {
    const double* Vr = cluster.map_shared_rank(V, 0);
    for (int e = tid; e < PW * VS; e += 256) V[e] = Vr[e];
  }
  cluster.sync();                     // leader's shared memory no longer read remotely
  if (dbg) a.dbg[4] = clock64();
  if (!rot) return;
  // ---------------- X <- X V over this CTA's row slice, tiles of 64 rows ----------------
  {
    const int wm = w & 1, wn = w >> 1;       // warp tile 32 rows x 16 cols
    const int lr = tid & 63, lc = tid >> 6;  // load: element (row lr, col lc + 4 t)
    int64_t colp[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) colp[t] = bcol(lc + 4 * t);
    double v[16];
    auto load = [&](int64_t r0) {
      const int64_t row = r0 + lr;
#pragma unroll
      for (int t = 0; t < 16; ++t) v[t] = (colp[t] >= 0 && row < re) ? a.B[colp[t] * r + row] : 0.0;
    };
    load(rb);
    // two staging buffers (X and the C tile buffer behind it, free until the c rows below), one
    // barrier per tile (as in the Gram phase)
    int par = 0;
    __syncthreads();
    for (int64_t r0 = rb; r0 < re; r0 += 64, par ^= 1) {
      double* Xt = X + par * (PW * XS);
#pragma unroll
      for (int t = 0; t < 16; ++t) Xt[(lc + 4 * t) * XS + lr] = v[t];
      __syncthreads();
      if (r0 + 64 < re) load(r0 + 64);
      double acc[4][2][2];
      acc_zero(acc);
      warp_mma<4, 2, KMAJ, KMAJ>(acc, Xt, XS, V, VS, wm * 32, wn * 16, 0, PW, lane);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t row = r0 + acc_row(wm * 32, i, lane);
            const int64_t col = bcol(acc_col(wn * 16, j, e, lane));
            if (col >= 0 && row < re) a.B[col * r + row] = acc[i][j][e];
          }
    }
  }
  if (dbg) a.dbg[5] = clock64();
  // ---------------- c rows of the pair <- V^T c ----------------
  // the cluster's CTAs split the right-hand-side columns; 64-column tiles on DMMA
  // (A = V^T: m = new index, k = old index; B = the pair's rows of C, [col][k])
  if (a.nrhs > 0) {
    const int ntl = (a.nrhs + 63) / 64;
    const int wm = w & 1, wn = w >> 1;       // warp tile 32 x 16
    for (int tl = crank; tl < ntl; tl += CS) {
      const int c0 = tl * 64;
      __syncthreads();
      for (int e = tid; e < 64 * PW; e += 256) {
        const int kk = e % PW, cc = e / PW;
        const int64_t row = bcol(kk);
        Cs[cc * XS + kk] = (row >= 0 && c0 + cc < a.nrhs) ? a.C[(int64_t)(c0 + cc) * r + row] : 0.0;
      }
      __syncthreads();
      double acc[4][2][2];
      acc_zero(acc);
      warp_mma<4, 2, KMAJ, IMAJ>(acc, V, VS, Cs, XS, wm * 32, wn * 16, 0, PW, lane);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int nn = acc_row(wm * 32, i, lane);
            const int cc = acc_col(wn * 16, j, e, lane);
            const int64_t row = bcol(nn);
            if (row >= 0 && c0 + cc < a.nrhs) a.C[(int64_t)(c0 + cc) * r + row] = acc[i][j][e];
          }
    }
  }
}

// squared column norms of B and their max
__global__ void __launch_bounds__(256) k_bjac_colnorms(const double* B, int64_t r, double* nrm2) {
  const int64_t col = blockIdx.x;
  double s = 0.0;
  for (int64_t t = threadIdx.x; t < r; t += 256) s = fma(B[col * r + t], B[col * r + t], s);
  __shared__ double red[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t += red[i];
    nrm2[col] = t;
  }
}

__global__ void k_bjac_max(const double* nrm2, int64_t r, double* smax2, unsigned long long* off) {
  __shared__ double red[32];
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < r; i += blockDim.x) m = fmax(m, nrm2[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = fmax(t, red[i]);
    *smax2 = t;
    *off = 0ull;
  }
}

// y[t][c] = sum_{kept i} B[t][i] C[i][c] / nrm2[i]   (kept: nrm2 > theta^2 smax2); 32 rhs per CTA
__global__ void __launch_bounds__(256) k_bjac_solve(const double* B, const double* C, const double* nrm2,
                                                    const double* smax2, int64_t r, int nrhs, double theta,
                                                    double* y, int64_t ldy) {
  __shared__ double Ds[64][33];   // D[i][c] for 64 i
  const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int c0 = blockIdx.y * 32;
  const int nc = min(32, nrhs - c0);
  const double thr2 = theta * theta * (*smax2);
  double acc[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) acc[c] = 0.0;
  for (int64_t i0 = 0; i0 < r; i0 += 64) {
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * 32; e += 256) {
      const int ii = e % 64, c = e / 64;
      const int64_t i = i0 + ii;
      double d = 0.0;
      if (i < r && c < nc) {
        const double s2 = nrm2[i];
        if (s2 > thr2 && s2 > 0.0) d = C[(int64_t)(c0 + c) * r + i] / s2;
      }
      Ds[ii][c] = d;
    }
    __syncthreads();
    if (t < r)
      for (int ii = 0; ii < 64 && i0 + ii < r; ++ii) {
        const double b = B[(i0 + ii) * r + t];
#pragma unroll
        for (int c = 0; c < 32; ++c) acc[c] = fma(b, Ds[ii][c], acc[c]);
      }
  }
  if (t < r)
#pragma unroll
    for (int c = 0; c < 32; ++c)
      if (c < nc) y[(int64_t)(c0 + c) * ldy + t] = acc[c];
}

// sorted singular values (rank by counting) and the kept count
__global__ void k_bjac_sigma(const double* nrm2, const double* smax2, int64_t r, double theta, double* sig_out,
                             int64_t* rank_dev) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double thr2 = theta * theta * (*smax2);
  if (i < r) {
    const double v = nrm2[i];
    int64_t pos = 0;
    for (int64_t t = 0; t < r; ++t) {
      const double u = nrm2[t];
      pos += (u > v || (u == v && t < i));
    }
    if (sig_out) sig_out[pos] = sqrt(v);
    if (v > thr2 && v > 0.0) atomicAdd((unsigned long long*)rank_dev, 1ull);
  }
}

// B = R_S^T, C = c
__global__ void k_bjac_load(const double* Rf, int64_t ldr, int64_t r, int nrhs, double* B, double* C) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < r * r) {
    const int64_t i = e % r, t = e / r;   // B[t][i] = R_S[i][t] -> B(col i, row t) at i * r + t
    B[i * r + t] = (i <= t) ? Rf[t * ldr + i] : 0.0;
  }
  if (e < r * nrhs) {
    const int64_t p = e % r, c = e / r;
    C[c * r + p] = Rf[(r + c) * ldr + p];
  }
}

static size_t a256(size_t v) { return (v + 255) & ~(size_t)255; }

// dst[:, j] = src[:, perm[j]] (r x r, ld r)
__global__ void k_bjac_permute(const double* src, double* dst, const int* perm, int64_t r) {
  const int64_t j = blockIdx.x;
  const int64_t pj = perm[j];
  for (int64_t t = threadIdx.x; t < r; t += blockDim.x) dst[j * r + t] = src[pj * r + t];
}

// Cd[j][c] = Cs[perm[j]][c] (r x nrhs, ld r)
__global__ void k_bjac_permute_rows(const double* Cs, double* Cd, const int* perm, int64_t r, int64_t nrhs) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= r * nrhs) return;
  const int64_t j = e % r, c = e / r;
  Cd[c * r + j] = Cs[c * r + perm[j]];
}

// At the start of every sweep the columns of B (and the rows of C) are permuted into decreasing norm
// (de Rijk-style ordering at sweep level, a dynamic stand-in for Drmac & Veselic's column pivoting):
// one outer sweep fewer on c3 / c4 (10 -> 9, 9 -> 8), c5 rounds 14.6 -> 13.2 s.  AZ_BJAC_SORT=0
// keeps the fixed column order.
// (experiment modes: 2 = increasing norm, 3 = decreasing norm dealt round-robin over the blocks)
static int bjac_sort_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("AZ_BJAC_SORT");
    v = e ? atoi(e) : 1;
    if (v < 0 || v > 3) v = 1;
  }
  return v;
}
static bool bjac_sort() { return bjac_sort_mode() != 0; }

// AZ_BJAC_QRCP=1: the first preconditioning QR with panel-level column pivoting (before each 64-column
// panel the 64 trailing columns of largest remaining norm are moved into it, in decreasing norm):
// R_S^T P = Q2 R2, so pinv(R_S) c = Q2 pinv(R3) Q3^T (P^T c)  (Drmac & Veselic's pivoted
// preconditioner, with the pivot search per panel instead of per column)
static bool bjac_qrcp() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("AZ_BJAC_QRCP");
    v = (e && *e == '1') ? 1 : 0;
  }
  return v == 1;
}

// nrm[c - j0] = || A[j0:r, c] ||^2 for the trailing columns c in [j0, r)  (A: r x r, ld r)
__global__ void __launch_bounds__(256) k_tail_norms(const double* A, int64_t r, int64_t j0, double* nrm) {
  const int64_t col = j0 + blockIdx.x;
  double s = 0.0;
  for (int64_t t = j0 + threadIdx.x; t < r; t += 256) s = fma(A[col * r + t], A[col * r + t], s);
  __shared__ double red[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t += red[i];
    nrm[blockIdx.x] = t;
  }
}

// column moves: scratch[:, i] = A[:, from[i]] (phase 0); A[:, to[i]] = scratch[:, i] (phase 1)
__global__ void k_move_cols(double* A, double* scratch, const int* from, const int* to, int64_t r, int phase) {
  const int i = blockIdx.x;
  if (phase == 0)
    for (int64_t t = threadIdx.x; t < r; t += blockDim.x) scratch[(int64_t)i * r + t] = A[(int64_t)from[i] * r + t];
  else
    for (int64_t t = threadIdx.x; t < r; t += blockDim.x) A[(int64_t)to[i] * r + t] = scratch[(int64_t)i * r + t];
}

static int g_last_sweeps = 0;
// inner cyclic sweeps of the pair's 64 x 64 Gram eigensolver per round (AZ_BJAC_INNER, default 1)
static int inner_sweeps() {
  static int v = 0;
  if (!v) {
    const char* e = getenv("AZ_BJAC_INNER");
    v = e ? atoi(e) : 1;
    if (v < 1 || v > 16) v = 1;
  }
  return v;
}
int az_bjac_sweeps_last() { return g_last_sweeps; }   // outer sweeps of the last block-Jacobi SVD

// QR preconditioning (Drmac & Veselic): R_S^T = Q2 R2, R2^T = Q3 R3, so R_S = Q3 R3 Q2^T and
// pinv(R_S) c = Q2 pinv(R3) (Q3^T c).  One-sided Jacobi on R3^T needs markedly fewer sweeps than on
// R_S^T; the two extra QRs cost ~2.7 r^3 flops against 8 r^3 per sweep.  AZ_BJAC_PRECOND=0 disables.
static bool bjac_precond() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("AZ_BJAC_PRECOND");
    v = (e && *e == '0') ? 0 : 1;
  }
  return v == 1;
}

static int64_t precond_min() {
  static int64_t v = -1;
  if (v < 0) {
    const char* e = getenv("AZ_BJAC_PRECOND_MIN");
    v = e ? atoll(e) : 2500;   // measured: c4 876 -> 829 ms, c3 4.03 -> 3.97 s against 0 (always)
  }
  return v;
}

static size_t tsvdw_pre_bytes(int64_t r, int64_t nrhs) {
  if (!bjac_precond()) return 0;
  const int64_t QBw = az_qrw_panel_width();
  const int64_t np = (r + QBw - 1) / QBw;
  return 2 * a256(sizeof(double) * r * r) + 2 * a256(sizeof(double) * np * QBw * QBw) +
         a256(sizeof(double) * r * std::max<int64_t>(nrhs, 1)) + a256(az_qrw_ws_bytes(r, std::max<int64_t>(r, nrhs)));
}

size_t az_tsvdw_ws_bytes(int64_t r, int64_t nrhs) {
  return a256(sizeof(double) * r * r) + a256(sizeof(double) * r * nrhs) + a256(sizeof(double) * r) + 1024 +
         tsvdw_pre_bytes(r, nrhs);
}

// dst (r x r, ld r) = upper triangle of src (ld lds) transposed: dst[i][j] = src[j][i] for j <= i
__global__ void k_upper_T(const double* src, int64_t lds, int64_t r, double* dst) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= r * r) return;
  const int64_t i = e % r, j = e / r;   // dst column j, row i
  dst[j * r + i] = (j <= i) ? src[i * lds + j] : 0.0;
}

__global__ void k_copy_block(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int64_t cols) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const int64_t i = e % rows, c = e / rows;
  dst[c * ldd + i] = src[c * lds + i];
}

az_status_t az_tsvdw_impl(const double* Rf, int64_t ldr, int64_t r, int64_t nrhs, double theta, double* y,
                          int64_t ldy, double* sigma_out, int64_t* rank_out, void* ws, size_t ws_bytes,
                          cudaStream_t st, int max_sweeps, int* sweeps_out, const int64_t** rank_dev) {
  if (ws_bytes < az_tsvdw_ws_bytes(r, nrhs)) {
    az_set_error("az_tsvd_solve (block Jacobi): workspace too small");
    return AZ_ERR_WORKSPACE;
  }
  char* p = (char*)ws;
  double* B = (double*)p;
  p += a256(sizeof(double) * r * r);
  double* C = (double*)p;
  p += a256(sizeof(double) * r * nrhs);
  double* nrm2 = (double*)p;
  p += a256(sizeof(double) * r);
  double* smax2 = (double*)p;
  unsigned long long* off = (unsigned long long*)(p + 64);
  int64_t* d_rank = (int64_t*)(p + 128);
  if (rank_dev) *rank_dev = d_rank;
  // ---- optional QR preconditioning ----
  // (small sketches -- the R22 pre-tests of the probe blocks -- converge in a few more cheap sweeps
  // than the two preconditioning QRs cost: AZ_BJAC_PRECOND_MIN, the smallest r preconditioned)
  const bool pre = bjac_precond() && r >= precond_min();
  double *M2 = nullptr, *M3 = nullptr, *T2 = nullptr, *T3 = nullptr, *Z = nullptr;
  void* qws = nullptr;
  size_t qbytes = 0;
  std::vector<int64_t> pj2, pj3;
  std::vector<int> pn2, pn3;
  int64_t np2 = 0, np3 = 0;
  std::vector<int> perm;   // AZ_BJAC_QRCP: column j of R_S^T P is column perm[j] of R_S^T
  if (bjac_precond()) {   // the workspace holds these buffers whenever preconditioning is enabled
    const int64_t QBw = az_qrw_panel_width();
    const int64_t npm = (r + QBw - 1) / QBw;
    char* q = p + 1024;
    auto take = [&](size_t bytes) {
      char* ptr = q;
      q += a256(bytes);
      return ptr;
    };
    M2 = (double*)take(sizeof(double) * r * r);
    M3 = (double*)take(sizeof(double) * r * r);
    T2 = (double*)take(sizeof(double) * npm * QBw * QBw);
    T3 = (double*)take(sizeof(double) * npm * QBw * QBw);
    Z = (double*)take(sizeof(double) * r * std::max<int64_t>(nrhs, 1));
    qbytes = az_qrw_ws_bytes(r, std::max<int64_t>(r, nrhs));
    qws = take(qbytes);
    pj2.resize(npm);
    pj3.resize(npm);
    pn2.resize(npm);
    pn3.resize(npm);
  }
  if (pre) {
    AzTrace tr("bjac_precond", st, 2 * r * r * r);
    k_upper_T<<<az_div_up(r * r, 256), 256, 0, st>>>(Rf, ldr, r, M2);                 // R_S^T
    AZ_LAUNCH_CHECK();
    if (!bjac_qrcp()) {
      AZ_TRY(az_qrw_factor(M2, r, r, 0, r, T2, pj2.data(), pn2.data(), &np2, qws, qbytes, st));   // = Q2 R2
    } else {
      // R_S^T P = Q2 R2 panel by panel; B (not loaded yet) is the column-move scratch, Z holds the
      // trailing norms and T3 (not used yet) the move lists
      const int64_t QBw = az_qrw_panel_width();
      perm.resize(r);
      for (int64_t i = 0; i < r; ++i) perm[i] = (int)i;
      std::vector<double> hn(r);
      std::vector<int> idx, from, to;
      int* d_mv = (int*)T3;
      double* d_nrm = Z;
      for (int64_t j0 = 0; j0 < r; j0 += QBw) {
        const int64_t nbp = std::min<int64_t>(QBw, r - j0), nt = r - j0;
        k_tail_norms<<<(unsigned)nt, 256, 0, st>>>(M2, r, j0, d_nrm);
        AZ_LAUNCH_CHECK();
        AZ_CUDA_CHECK(cudaMemcpyAsync(hn.data(), d_nrm, sizeof(double) * nt, cudaMemcpyDeviceToHost, st));
        AZ_CUDA_CHECK(cudaStreamSynchronize(st));
        idx.resize(nt);
        for (int64_t i = 0; i < nt; ++i) idx[i] = (int)i;
        std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return hn[x] > hn[y]; });
        // position j0 + i takes the i-th largest column; the panel columns not chosen fill the
        // vacated positions of the chosen ones from outside the panel
        std::vector<int> dest(nt, -1);   // dest[old offset] = new offset (affected columns only)
        std::vector<char> chosen(nt, 0);
        for (int64_t i = 0; i < nbp; ++i) chosen[idx[i]] = 1;
        std::vector<int> vac;            // offsets >= nbp vacated by chosen columns
        for (int64_t i = 0; i < nbp; ++i) {
          dest[idx[i]] = (int)i;
          if (idx[i] >= nbp) vac.push_back(idx[i]);
        }
        std::sort(vac.begin(), vac.end());
        size_t v = 0;
        for (int64_t i = 0; i < nbp; ++i)
          if (!chosen[i]) dest[i] = vac[v++];
        from.clear();
        to.clear();
        for (int64_t i = 0; i < nt; ++i)
          if (dest[i] >= 0 && dest[i] != i) {
            from.push_back((int)(j0 + i));
            to.push_back((int)(j0 + dest[i]));
          }
        if (!from.empty()) {
          const int nm = (int)from.size();
          std::vector<int> hv(from);
          hv.insert(hv.end(), to.begin(), to.end());
          AZ_CUDA_CHECK(cudaMemcpyAsync(d_mv, hv.data(), sizeof(int) * 2 * nm, cudaMemcpyHostToDevice, st));
          k_move_cols<<<nm, 256, 0, st>>>(M2, B, d_mv, d_mv + nm, r, 0);
          AZ_LAUNCH_CHECK();
          k_move_cols<<<nm, 256, 0, st>>>(M2, B, d_mv, d_mv + nm, r, 1);
          AZ_LAUNCH_CHECK();
          std::vector<int> old(perm.begin() + j0, perm.end());
          for (int i = 0; i < nm; ++i) perm[to[i]] = old[from[i] - j0];
          AZ_CUDA_CHECK(cudaStreamSynchronize(st));   // hv is reused next panel
        }
        AZ_TRY(az_qrw_factor(M2, r, r, j0, j0 + nbp, T2, pj2.data(), pn2.data(), &np2, qws, qbytes, st));
        if (j0 + nbp < r)
          AZ_TRY(az_qrw_apply(M2, r, r, pj2.data(), pn2.data(), T2, np2 - 1, np2, M2 + (j0 + nbp) * r, r,
                              r - j0 - nbp, qws, qbytes, st));
      }
    }
    k_upper_T<<<az_div_up(r * r, 256), 256, 0, st>>>(M2, r, r, M3);                    // R2^T
    AZ_LAUNCH_CHECK();
    AZ_TRY(az_qrw_factor(M3, r, r, 0, r, T3, pj3.data(), pn3.data(), &np3, qws, qbytes, st));   // = Q3 R3
    if (nrhs > 0) {
      k_copy_block<<<az_div_up(r * nrhs, 256), 256, 0, st>>>(Rf + r * ldr, ldr, C, r, r, nrhs);
      AZ_LAUNCH_CHECK();
      if (!perm.empty()) {   // P^T c: row j of the permuted c is row perm[j] of c (nrm2 is free here)
        int* d_permc = (int*)nrm2;
        AZ_CUDA_CHECK(cudaMemcpyAsync(d_permc, perm.data(), sizeof(int) * r, cudaMemcpyHostToDevice, st));
        k_bjac_permute_rows<<<az_div_up(r * nrhs, 256), 256, 0, st>>>(C, Z, d_permc, r, nrhs);
        AZ_LAUNCH_CHECK();
        k_copy_block<<<az_div_up(r * nrhs, 256), 256, 0, st>>>(Z, r, C, r, r, nrhs);
        AZ_LAUNCH_CHECK();
        AZ_CUDA_CHECK(cudaStreamSynchronize(st));   // perm (host) outlives the copy
      }
      AZ_TRY(az_qrw_apply(M3, r, r, pj3.data(), pn3.data(), T3, 0, np3, C, r, nrhs, qws, qbytes, st));   // Q3^T c
    }
  }
  {
    AzTrace tr("bjac_load", st);
    if (pre)   // B = R3^T; C already holds Q3^T c
      k_bjac_load<<<az_div_up(r * r, 256), 256, 0, st>>>(M3, r, r, 0, B, C);
    else
      k_bjac_load<<<az_div_up(r * std::max<int64_t>(r, nrhs), 256), 256, 0, st>>>(Rf, ldr, r, (int)nrhs, B, C);
    AZ_LAUNCH_CHECK();
  }
  const int nblk = (int)((r + BW - 1) / BW);
  const int n = nblk + (nblk & 1);
  const size_t smem = (size_t)(PW * GS + PW * VS + PW * XS + 64 * XS) * sizeof(double);
  AZ_CUDA_CHECK(az_smem_attr(k_bjac_round, smem));
  // cluster size: the largest power of two with all CTAs of a round in ONE wave (every wave pays
  // the leader's eigensolver latency once), each slice >= 256 rows.  AZ_BJAC_CS overrides.
  int CS = 1;
  {
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    while (CS < 8 && (int64_t)(n / 2) * CS * 2 <= sms && r / (2 * CS) >= 256) CS *= 2;
    // more pairs than SMs: a round takes two waves at CS = 1 whose second is partly empty; pairs of
    // CTAs split each pair's rows instead (c5, 240 pairs: rounds 16.2 -> 14.8 s, CS = 4 16.6 s)
    if (CS == 1 && (int64_t)(n / 2) > sms && r / 4 >= 256) CS = 2;
    if (const char* e = getenv("AZ_BJAC_CS"))
      if (*e) CS = std::max(1, std::min(8, atoi(e)));
  }
  BJArgs a;
  a.B = B;
  a.r = r;
  a.C = C;
  a.nrhs = (int)nrhs;
  a.nblk = nblk;
  a.smax2 = smax2;
  a.theta = theta;
  a.off = off;
  a.tol = 4.0 * 1.1102230246251565e-16 * std::sqrt((double)r);
  a.inner_sweeps = inner_sweeps();
  a.dbg = nullptr;
  static long long* d_dbg = nullptr;
  const bool want_dbg = getenv("AZ_DEBUG_JACOBI") != nullptr;
  if (want_dbg) {
    if (!d_dbg) cudaMalloc(&d_dbg, 8 * sizeof(long long));
    a.dbg = d_dbg;
  }
  int sw = 0;
  // sweep-level norm ordering: the permuted copies go to second buffers, the two of each pair swapping
  // roles each sweep -- B's to M3 (free once B is loaded), C's to Z (unused without preconditioning)
  // or to the preconditioning QR's workspace (free until the closing Q2 product, which follows the
  // solve's last read of C); stream-ordered allocations only where the workspace has no such room
  const bool sort_cols = bjac_sort() && r > PW;
  const size_t cbytes = sizeof(double) * r * std::max<int64_t>(nrhs, 1);
  double* Bsp = M3;
  double* Bmal = nullptr;
  double* Csp = pre ? (qbytes >= cbytes ? (double*)qws : nullptr) : Z;
  double* Cmal = nullptr;
  int* d_perm = (int*)T3;   // T3 (>= r QBw doubles) is read only by the Q3^T c product before the sweeps
  int* pmal = nullptr;
  std::vector<double> h_n2;
  std::vector<int> h_perm;
  if (sort_cols) {
    if (!Bsp) {
      AZ_CUDA_CHECK(cudaMallocAsync((void**)&Bmal, sizeof(double) * r * r, st));
      Bsp = Bmal;
    }
    if (!Csp) {
      AZ_CUDA_CHECK(cudaMallocAsync((void**)&Cmal, cbytes, st));
      Csp = Cmal;
    }
    if (!d_perm) {
      AZ_CUDA_CHECK(cudaMallocAsync((void**)&pmal, sizeof(int) * r, st));
      d_perm = pmal;
    }
    h_n2.resize(r);
    h_perm.resize(r);
  }
  for (; sw < max_sweeps; ++sw) {
    {
      AzTrace tr("bjac_norms", st);
      k_bjac_colnorms<<<(unsigned)r, 256, 0, st>>>(B, r, nrm2);
      AZ_LAUNCH_CHECK();
      k_bjac_max<<<1, 1024, 0, st>>>(nrm2, r, smax2, off);
      AZ_LAUNCH_CHECK();
    }
    if (sort_cols) {
      AzTrace tr("bjac_sort", st);
      AZ_CUDA_CHECK(cudaMemcpyAsync(h_n2.data(), nrm2, sizeof(double) * r, cudaMemcpyDeviceToHost, st));
      AZ_CUDA_CHECK(cudaStreamSynchronize(st));
      for (int64_t i = 0; i < r; ++i) h_perm[i] = (int)i;
      const int mode = bjac_sort_mode();
      if (mode == 2)
        std::stable_sort(h_perm.begin(), h_perm.end(), [&](int x, int y) { return h_n2[x] < h_n2[y]; });
      else
        std::stable_sort(h_perm.begin(), h_perm.end(), [&](int x, int y) { return h_n2[x] > h_n2[y]; });
      if (mode == 3) {   // sorted column t -> block t % nblk, slot t / nblk
        std::vector<int> dealt(r, -1);
        int64_t t = 0;
        for (int64_t slot = 0; slot < BW; ++slot)
          for (int64_t blk = 0; blk < nblk; ++blk) {
            const int64_t pos = blk * BW + slot;
            if (pos < r && t < r) dealt[pos] = h_perm[t++];
          }
        for (int64_t i = 0; i < r; ++i)
          if (dealt[i] < 0) dealt[i] = h_perm[t++];
        h_perm.swap(dealt);
      }
      AZ_CUDA_CHECK(cudaMemcpyAsync(d_perm, h_perm.data(), sizeof(int) * r, cudaMemcpyHostToDevice, st));
      k_bjac_permute<<<(unsigned)r, 256, 0, st>>>(B, Bsp, d_perm, r);
      AZ_LAUNCH_CHECK();
      if (nrhs > 0) {
        k_bjac_permute_rows<<<az_div_up(r * nrhs, 256), 256, 0, st>>>(C, Csp, d_perm, r, nrhs);
        AZ_LAUNCH_CHECK();
      }
      std::swap(B, Bsp);
      std::swap(C, Csp);
      a.B = B;
      a.C = C;
      AZ_CUDA_CHECK(cudaStreamSynchronize(st));   // h_perm is reused next sweep
    }
    for (int rd = 0; rd < n - 1; ++rd) {
      AzTrace tr("bjac_round", st, 16 * r * BW * BW * (n / 2));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(n / 2 * CS));
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = CS;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      AZ_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_bjac_round, a, rd));
      AZ_LAUNCH_CHECK();
    }
    unsigned long long h_off = 0;
    AZ_CUDA_CHECK(cudaMemcpyAsync(&h_off, off, sizeof(h_off), cudaMemcpyDeviceToHost, st));
    AZ_CUDA_CHECK(cudaStreamSynchronize(st));
    double offd;
    memcpy(&offd, &h_off, sizeof(offd));
    if (want_dbg) {
      long long h[8];
      cudaMemcpy(h, d_dbg, sizeof(h), cudaMemcpyDeviceToHost);
      fprintf(stderr, "bjac r=%lld CS=%d sweep %d off %.3e tol %.3e | last round clocks (cluster 0 leader): gram %lld "
              "csync %lld eig %lld vsync %lld update %lld | inner round sync1 %lld\n",
              (long long)r, CS, sw, offd, a.tol, h[1] - h[0], h[2] - h[1], h[3] - h[2], h[4] - h[3], h[5] - h[4],
              h[7] - h[6]);
    }
    if (offd <= 4.0 * a.tol) {   // rounding level of the measured off-diagonals
      ++sw;
      break;
    }
  }
  if (sweeps_out) *sweeps_out = sw;
  g_last_sweeps = sw;
  {
    AzTrace tr("bjac_norms", st);
    k_bjac_colnorms<<<(unsigned)r, 256, 0, st>>>(B, r, nrm2);
    AZ_LAUNCH_CHECK();
    k_bjac_max<<<1, 1024, 0, st>>>(nrm2, r, smax2, off);
    AZ_LAUNCH_CHECK();
  }
  if (nrhs > 0) {
    AzTrace tr("bjac_solve", st, 2 * r * r * nrhs);
    // preconditioned: z = pinv(R3) (Q3^T c), then y = Q2 z
    k_bjac_solve<<<dim3(az_div_up(r, 256), az_div_up(nrhs, 32)), 256, 0, st>>>(B, C, nrm2, smax2, r, (int)nrhs,
                                                                               theta, pre ? Z : y, pre ? r : ldy);
    AZ_LAUNCH_CHECK();
    if (pre) {
      k_copy_block<<<az_div_up(r * nrhs, 256), 256, 0, st>>>(Z, r, y, ldy, r, nrhs);
      AZ_LAUNCH_CHECK();
      AZ_TRY(az_qrw_apply_q(M2, r, r, pj2.data(), pn2.data(), T2, 0, np2, y, ldy, nrhs, qws, qbytes, st));
    }
  }
  if (sort_cols) {
    if (Cmal) AZ_CUDA_CHECK(cudaFreeAsync(Cmal, st));
    if (Bmal) AZ_CUDA_CHECK(cudaFreeAsync(Bmal, st));
    if (pmal) AZ_CUDA_CHECK(cudaFreeAsync(pmal, st));
  }
  AZ_CUDA_CHECK(cudaMemsetAsync(d_rank, 0, sizeof(int64_t), st));
  k_bjac_sigma<<<az_div_up(r, 256), 256, 0, st>>>(nrm2, smax2, r, theta, sigma_out, d_rank);
  AZ_LAUNCH_CHECK();
  if (rank_out) {
    AZ_CUDA_CHECK(cudaMemcpyAsync(rank_out, d_rank, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    AZ_CUDA_CHECK(cudaStreamSynchronize(st));
  }
  return AZ_OK;
}
