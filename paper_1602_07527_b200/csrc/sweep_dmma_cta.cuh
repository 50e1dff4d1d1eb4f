// sweep_dmma_cta.cuh -- on-chip kernels for one matrix / diagonal block with n <= 128,
// one CTA (8 warps) each, built on 8x8 DMMA tiles (mma.sync.m8n8k4.f64) held in shared
// memory.  Arithmetic is fp64 for both fp64 and fp32 inputs (fp32 is converted on load /
// store; the fp64 tensor cores make this cheaper than a SIMT fp32 sweep).
//
//  k_rev_dmma_cta   reverse sweep: the blocked reverse of PAPER.md:689-701 with N_b = 8,
//                   diagonal 8x8 tiles by Eq. 10 (the paper's own choice
//                   for diagonal blocks):
//                     s1 Cbar <- Cbar D^{-1};  s2 Bbar <- Bbar - Cbar R;
//                     s3 Dbar <- Dbar - tril(Cbar^T C);
//                     s4 Dbar <- Phi(D^{-T}(P+P^T)D^{-1}), P = Phi(D^T Dbar), S = D^{-T}(P+P^T)D^{-1};
//                     s5 Rbar <- Rbar - Cbar^T B - S R
//  k_fwd_dmma_cta   forward sweep: the blocked forward of PAPER.md:655-666 with N_b = 8,
//                   diagonal 8x8 tiles by Eq. 8:
//                     f1 Ddot <- Ddot - tril(Rdot R^T + R Rdot^T)
//                     f2 Ddot <- D Phi(D^{-1} Ddot D^{-T})              (Ddot read as symmetric)
//                     f3 Cdot <- Cdot - Bdot R^T - B Rdot^T
//                     f4 Cdot <- (Cdot - C Ddot^T) D^{-T}
//  k_trinv_dmma     inverse of a lower-triangular block (the panel solves of the blocked
//                   sweeps, run as GEMMs against it):
//                     X(J,J) = D_J^{-1};  X(I,J) = -D_I^{-1} sum_{K=J}^{I-1} D(I,K) X(K,J)
//
// Tiles of every update are distributed over the warps.  Shared memory holds the lower
// 8x8 tiles, tile-packed, with an XOR swizzle that makes every A / B fragment load
// bank-conflict free (139 KB for two 128 x 128 triangles).
#pragma once
#include "common.cuh"
#include "gemm.cuh"  // dmma884

namespace cd {

// offset of element (r, c) inside a swizzled 8x8 tile: (r, c) at c*8 + (r ^ 4*((c>>1)&1))
__device__ __forceinline__ int t8(int r, int c) { return c * 8 + (r ^ ((c & 2) << 1)); }

// lower tile (bi >= bj) of an NBLK x NBLK tiling, column-major tile order
__device__ __forceinline__ int tile_base(int NBLK, int bi, int bj) {
  return (bj * NBLK - (bj * (bj - 1)) / 2 + (bi - bj)) * 64;
}
__device__ __forceinline__ int tat(int NBLK, int i, int m) {
  return tile_base(NBLK, i >> 3, m >> 3) + t8(i & 7, m & 7);
}

#ifndef CD_DC_MINB
#define CD_DC_MINB 4  // 64 registers: 4 CTAs per SM at n <= 64 (batched fp32 diagonal blocks: -5 %)
#endif
// phase clocks of CTA 0 of the on-chip sweeps (measurement only: cd_debug_phase_clocks selects the
// CLK = true instantiation; stamps are taken by thread 0 of CTA 0 only).  A compile-time switch:
// a runtime flag read from global memory at kernel start held warp 0 -- and through it the whole
// staging -- for one memory latency (~1 us with a cold L2) in every production launch.
__device__ long long g_dc_clk[40];
#define dc_clk(i)                                                      \
  do {                                                                 \
    if (dc_clk_on) g_dc_clk[i] = clock64();                            \
  } while (0)
constexpr int DC_NMAX = 128;  // largest n (and diagonal block) handled on chip
constexpr int DC_WARPS = 8;
constexpr int DC_THREADS = DC_WARPS * 32;

inline size_t dmma_cta_smem(int NBLK) {
  const int ntile = NBLK * (NBLK + 1) / 2;
  return size_t(2 * ntile * 64 + NBLK * 64 + 2 * 64 + 8 * NBLK) * sizeof(double) + 16;
}

// Stage tril of an n x n column-major matrix into swizzled tiles (fp64), zero the upper
// parts of the diagonal tiles, pad beyond n with the identity (ident) or zeros.
template <typename TIO>
__device__ __forceinline__ void dc_stage(int NBLK, const TIO* __restrict__ g, int64_t ld, int n, double* s,
                                         bool ident) {
  const int NP = 8 * NBLK, NTILE = NBLK * (NBLK + 1) / 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if constexpr (sizeof(TIO) == 8) {
    if ((ld & 1) == 0 && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
      // 16-byte copies of row pairs (i, i + 1), i even: a pair lands on two consecutive swizzled
      // slots of one tile (t8 only flips bit 2 of the row).  Odd columns start with their diagonal
      // element alone, so nothing above the diagonal is fetched.
      for (int m = warp; m < n; m += DC_WARPS) {
        const double* gc = g + int64_t(m) * ld;
        if ((m & 1) && lane == 0) cp_async_zfill<8>(s + tat(NBLK, m, m), gc + m, true);
        for (int i = ((m + 1) & ~1) + 2 * lane; i < n; i += 64) {
          if (i + 1 < n) {
            const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(s + tat(NBLK, i, m)));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gc + i) : "memory");
          } else {
            cp_async_zfill<8>(s + tat(NBLK, i, m), gc + i, true);
          }
        }
      }

    } else {
      for (int m = warp; m < n; m += DC_WARPS)
        for (int i = m + lane; i < n; i += 32) cp_async_zfill<8>(s + tat(NBLK, i, m), g + i + int64_t(m) * ld, true);
    }
  } else {
    // fp32: all loads of a group of 4 columns are issued before the first convert / store
    // (one-by-one, every column cost a full memory latency: 30-40 % of the stall samples)
    for (int m0 = warp; m0 < n; m0 += 4 * DC_WARPS) {
      float v[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int m = m0 + a * DC_WARPS, i = m + lane + 32 * r;
          v[a][r] = (m < n && i < n) ? __ldg(g + i + int64_t(m) * ld) : 0.f;
        }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int m = m0 + a * DC_WARPS, i = m + lane + 32 * r;
          if (m < n && i < n) s[tat(NBLK, i, m)] = double(v[a][r]);
        }
    }
  }
  for (int e = tid; e < NBLK * 64; e += DC_THREADS) {
    const int blk = e >> 6, r = e & 7, c = (e >> 3) & 7;
    const int i = 8 * blk + r, m = 8 * blk + c;
    const int o = tile_base(NBLK, blk, blk) + t8(r, c);
    if (r < c) s[o] = 0.0;
    else if (i >= n) s[o] = (ident && i == m) ? 1.0 : 0.0;
  }
  if (n < NP) {
    for (int e = tid; e < NTILE * 64; e += DC_THREADS) {
      int tix = e >> 6, bj = 0;
      while (tix >= NBLK - bj) {
        tix -= NBLK - bj;
        ++bj;
      }
      const int bi = bj + tix;
      if (bi == bj) continue;
      const int r = e & 7, c = (e >> 3) & 7;
      if (8 * bi + r >= n || 8 * bj + c >= n) s[tile_base(NBLK, bi, bj) + t8(r, c)] = 0.0;
    }
  }
}

// 1/L_ii (sRd) and the inverse of every diagonal 8x8 tile (sDi); block-wide info.
__device__ __forceinline__ void dc_diag_inverses(int NBLK, const double* sL, double* sDi, double* sRd, int n,
                                                 int* sbad) {
  const int NP = 8 * NBLK;
  const int tid = threadIdx.x;
  for (int i = tid; i < NP; i += DC_THREADS) {
    const double d = sL[tat(NBLK, i, i)];
    if (i < n && bad_pivot(d)) atomicMin(sbad, i + 1);
    sRd[i] = 1.0 / d;
  }
  __syncthreads();
  for (int e = tid; e < NBLK * 8; e += DC_THREADS) {
    const int blk = e >> 3, c = e & 7, j0 = 8 * blk;
    const double* D = sL + tile_base(NBLK, blk, blk);
    double x[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r < c) {
        x[r] = 0.0;
      } else if (r == c) {
        x[r] = sRd[j0 + r];
      } else {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < r; ++q)
          if (q >= c) s += D[t8(r, q)] * x[q];
        x[r] = -s * sRd[j0 + r];
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) sDi[blk * 64 + t8(r, c)] = x[r];
  }
  __syncthreads();
}

// write tril (and optionally the mirror) of the tile-packed matrix to global
template <typename TIO>
__device__ __forceinline__ void dc_store(int NBLK, TIO* __restrict__ g, int64_t ld, int n, const double* s,
                                         int out_mode) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (sizeof(TIO) == 8 && out_mode == 0 && (ld & 1) == 0 && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
    // tril only, row pairs as 16-byte stores (odd columns: the diagonal element alone)
    for (int m = warp; m < n; m += DC_WARPS) {
      TIO* gc = g + int64_t(m) * ld;
      if ((m & 1) && lane == 0) gc[m] = TIO(s[tat(NBLK, m, m)]);
      for (int i = ((m + 1) & ~1) + 2 * lane; i < n; i += 64) {
        const double* sp = s + tat(NBLK, i, m);
        if (i + 1 < n) *reinterpret_cast<double2*>(gc + i) = *reinterpret_cast<const double2*>(sp);
        else gc[i] = TIO(sp[0]);
      }
    }
    return;
  }
  for (int m = warp; m < n; m += DC_WARPS)
    for (int i = m + lane; i < n; i += 32) {
      double v = s[tat(NBLK, i, m)];
      if (out_mode == 2 && i != m) v *= 0.5;
      g[i + int64_t(m) * ld] = TIO(v);
    }
  if (out_mode != 0) {
    for (int i = warp; i < n; i += DC_WARPS)
      for (int m = lane; m < i; m += 32) {
        double v = s[tat(NBLK, i, m)];
        if (out_mode == 2) v *= 0.5;
        g[m + int64_t(i) * ld] = TIO(v);
      }
  }
}

// ============================================================================ reverse
// NB_ > 0: the block count is a compile-time constant (n = 8 NB_ - 7 .. 8 NB_), so the tile
// indexing and the per-step work lists fold away (single small matrices: the launch latency is
// the whole cost)
template <typename TIO, int NB_ = 0, bool CLK = false>
__global__ void __launch_bounds__(DC_THREADS, CD_DC_MINB)
    k_rev_dmma_cta(int n, Opnd Ld, Opnd Ad, int out_mode, Opnd Sd, int* __restrict__ info) {
  const int NBLK = NB_ ? NB_ : (n + 7) >> 3;
  const int NP = 8 * NBLK;
  const int NTILE = NBLK * (NBLK + 1) / 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sL = reinterpret_cast<double*>(smem_raw);
  double* sA = sL + NTILE * 64;
  double* sDi = sA + NTILE * 64;
  double* sX = sDi + NBLK * 64;
  double* sS = sX + 64;
  double* sRd = sS + 64;
  int* sbad = reinterpret_cast<int*>(sRd + NP);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t b = blockIdx.x;
  const TIO* L = optr<TIO>(Ld, b);
  TIO* A = optr_w<TIO>(Ad, b);

  const bool dc_clk_on = CLK && blockIdx.x == 0 && tid == 0;
  dc_clk(0);
  if (tid == 0) *sbad = 0x7fffffff;
  dc_stage<TIO>(NBLK, L, Ld.ld, n, sL, true);
  dc_clk(37);
  dc_stage<TIO>(NBLK, A, Ad.ld, n, sA, false);
  dc_clk(38);
  cp_async_wait_all();
  dc_clk(39);
  __syncthreads();
  dc_clk(1);
  dc_diag_inverses(NBLK, sL, sDi, sRd, n, sbad);
  if (tid == 0 && info) info[b] = (*sbad == 0x7fffffff) ? 0 : *sbad;
  dc_clk(2);

  for (int J = NBLK - 1; J >= 0; --J) {
    const int PT = NBLK - 1 - J, QT = J;
    const double* Di = sDi + J * 64;
    double* Dt = sA + tile_base(NBLK, J, J);
    const double* Lt = sL + tile_base(NBLK, J, J);
    dc_clk(3 + 4 * (NBLK - 1 - J));

    // s1: Cbar <- Cbar D^{-1}
    for (int rt = warp; rt < PT; rt += DC_WARPS) {
      double* Ct = sA + tile_base(NBLK, J + 1 + rt, J);
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(c0, c1, Ct[t8(g, 4 * kk + t)], Di[t8(4 * kk + t, g)]);
      __syncwarp();
      Ct[t8(g, 2 * t)] = c0;
      Ct[t8(g, 2 * t + 1)] = c1;
    }
    __syncthreads();
    dc_clk(4 + 4 * (NBLK - 1 - J));

    // s3 (last warp): Dbar <- Dbar - tril(Cbar^T C);   s2 (all warps): Bbar <- Bbar - Cbar R
    if (warp == DC_WARPS - 1 && PT > 0) {
      double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
      for (int rt = 0; rt < PT; ++rt) {
        const double* Ct = sA + tile_base(NBLK, J + 1 + rt, J);
        const double* Lc = sL + tile_base(NBLK, J + 1 + rt, J);
        dmma884(a0, a1, Ct[t8(t, g)], Lc[t8(t, g)]);
        dmma884(b0, b1, Ct[t8(4 + t, g)], Lc[t8(4 + t, g)]);
      }
      a0 += b0;
      a1 += b1;
      if (g >= 2 * t) Dt[t8(g, 2 * t)] -= a0;
      if (g >= 2 * t + 1) Dt[t8(g, 2 * t + 1)] -= a1;
    }
    // s5a (warps from the top, one per column tile): Rbar <- Rbar - Cbar^T B -- independent of the
    // diagonal block, so only S R is left after s4 (the R column tile J-1 is the next step's
    // critical path).  Warps below take the s2 tiles.
    for (int ct = DC_WARPS - 2 - warp; warp < DC_WARPS - 1 && PT > 0 && ct < QT; ct += DC_WARPS - 1) {
      double* Rb = sA + tile_base(NBLK, J, ct);
      double c0 = Rb[t8(g, 2 * t)], c1 = Rb[t8(g, 2 * t + 1)];
      double d0 = 0.0, d1 = 0.0;
      for (int rt = 0; rt < PT; ++rt) {
        const double* Ct = sA + tile_base(NBLK, J + 1 + rt, J);
        const double* Bt = sL + tile_base(NBLK, J + 1 + rt, ct);
        dmma884(c0, c1, Ct[t8(t, g)], -Bt[t8(t, g)]);
        dmma884(d0, d1, Ct[t8(4 + t, g)], -Bt[t8(4 + t, g)]);
      }
      Rb[t8(g, 2 * t)] = c0 + d0;
      Rb[t8(g, 2 * t + 1)] = c1 + d1;
    }
    for (int idx = warp; idx < PT * QT; idx += DC_WARPS) {
      const int rt = idx / QT, ct = idx - rt * QT;
      const double* Ct = sA + tile_base(NBLK, J + 1 + rt, J);
      double* Bt = sA + tile_base(NBLK, J + 1 + rt, ct);
      const double* Rt = sL + tile_base(NBLK, J, ct);
      double c0 = Bt[t8(g, 2 * t)], c1 = Bt[t8(g, 2 * t + 1)];
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(c0, c1, Ct[t8(g, 4 * kk + t)], -Rt[t8(4 * kk + t, g)]);
      Bt[t8(g, 2 * t)] = c0;
      Bt[t8(g, 2 * t + 1)] = c1;
    }
    __syncthreads();
    dc_clk(5 + 4 * (NBLK - 1 - J));

    // s4 (warp 0): Y = D^{-T}(P + P^T)D^{-1}, P = Phi(D^T Dbar); S = Y; tril(Dbar) = Phi(Y)
    if (warp == 0) {
      double p0 = 0.0, p1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(p0, p1, Lt[t8(4 * kk + t, g)], Dt[t8(4 * kk + t, g)]);
      const int c0i = 2 * t, c1i = 2 * t + 1;
      p0 = (g > c0i) ? p0 : (g == c0i ? 0.5 * p0 : 0.0);
      p1 = (g > c1i) ? p1 : (g == c1i ? 0.5 * p1 : 0.0);
      sX[t8(g, c0i)] = p0;
      sX[t8(g, c1i)] = p1;
      __syncwarp();
      const double x0 = p0 + sX[t8(c0i, g)];
      const double x1 = p1 + sX[t8(c1i, g)];
      __syncwarp();
      sX[t8(g, c0i)] = x0;
      sX[t8(g, c1i)] = x1;
      __syncwarp();
      double z0 = 0.0, z1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(z0, z1, sX[t8(g, 4 * kk + t)], Di[t8(4 * kk + t, g)]);
      __syncwarp();
      sX[t8(g, c0i)] = z0;
      sX[t8(g, c1i)] = z1;
      __syncwarp();
      double y0 = 0.0, y1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(y0, y1, Di[t8(4 * kk + t, g)], sX[t8(4 * kk + t, g)]);
      sS[t8(g, c0i)] = y0;
      sS[t8(g, c1i)] = y1;
      if (g >= c0i) Dt[t8(g, c0i)] = (g == c0i) ? 0.5 * y0 : y0;
      if (g >= c1i) Dt[t8(g, c1i)] = (g == c1i) ? 0.5 * y1 : y1;
    }
    __syncthreads();
    dc_clk(6 + 4 * (NBLK - 1 - J));

    // s5b: Rbar <- Rbar - S R   (the Cbar^T B part ran in s5a)
    for (int ct = warp; ct < QT; ct += DC_WARPS) {
      double* Rb = sA + tile_base(NBLK, J, ct);
      const double* Rt = sL + tile_base(NBLK, J, ct);
      double c0 = Rb[t8(g, 2 * t)], c1 = Rb[t8(g, 2 * t + 1)];
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(c0, c1, sS[t8(g, 4 * kk + t)], -Rt[t8(4 * kk + t, g)]);
      Rb[t8(g, 2 * t)] = c0;
      Rb[t8(g, 2 * t + 1)] = c1;
    }
    __syncthreads();
  }

  dc_clk(35);
  dc_store<TIO>(NBLK, A, Ad.ld, n, sA, out_mode);
  dc_clk(36);
  if (Sd.base || Sd.arr) {  // S = Dbar + Dbar^T (diagonal doubled), dense
    TIO* S = optr_w<TIO>(Sd, b);
    for (int c = warp; c < n; c += DC_WARPS)
      for (int i = lane; i < n; i += 32) {
        const double v = (i >= c) ? sA[tat(NBLK, i, c)] : sA[tat(NBLK, c, i)];
        S[i + int64_t(c) * Sd.ld] = TIO((i == c) ? 2.0 * v : v);
      }
  }
}

// ============================================================================ forward
// Optionally writes a clean dense copy of tril(Ldot) (upper zero) to Dd, the operand of
// Cdot <- (Cdot - C Ddot^T) D^{-T} in the blocked driver.
template <typename TIO>
__global__ void __launch_bounds__(DC_THREADS, CD_DC_MINB)
    k_fwd_dmma_cta(int n, Opnd Ld, Opnd Ad, Opnd Dd, int* __restrict__ info) {
  const int NBLK = (n + 7) >> 3;
  const int NP = 8 * NBLK;
  const int NTILE = NBLK * (NBLK + 1) / 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sL = reinterpret_cast<double*>(smem_raw);
  double* sA = sL + NTILE * 64;
  double* sDi = sA + NTILE * 64;
  double* sX = sDi + NBLK * 64;
  double* sY = sX + 64;
  double* sRd = sY + 64;
  int* sbad = reinterpret_cast<int*>(sRd + NP);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t b = blockIdx.x;
  const TIO* L = optr<TIO>(Ld, b);
  TIO* A = optr_w<TIO>(Ad, b);

  if (tid == 0) *sbad = 0x7fffffff;
  dc_stage<TIO>(NBLK, L, Ld.ld, n, sL, true);
  dc_stage<TIO>(NBLK, A, Ad.ld, n, sA, false);
  cp_async_wait_all();
  __syncthreads();
  dc_diag_inverses(NBLK, sL, sDi, sRd, n, sbad);
  if (tid == 0 && info) info[b] = (*sbad == 0x7fffffff) ? 0 : *sbad;

  for (int J = 0; J < NBLK; ++J) {
    const int PT = NBLK - 1 - J, QT = J;
    const double* Di = sDi + J * 64;
    double* Dt = sA + tile_base(NBLK, J, J);
    const double* Lt = sL + tile_base(NBLK, J, J);

    if (warp == 0) {
      // f1: Ddot <- Ddot - tril(Rdot R^T + R Rdot^T)
      double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
      for (int ct = 0; ct < QT; ++ct) {
        const double* Rd = sA + tile_base(NBLK, J, ct);
        const double* Rt = sL + tile_base(NBLK, J, ct);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          dmma884(c0, c1, Rd[t8(g, 4 * kk + t)], Rt[t8(g, 4 * kk + t)]);  // Rdot R^T
          dmma884(d0, d1, Rt[t8(g, 4 * kk + t)], Rd[t8(g, 4 * kk + t)]);  // R Rdot^T
        }
      }
      const int c0i = 2 * t, c1i = 2 * t + 1;
      if (g >= c0i) Dt[t8(g, c0i)] -= c0 + d0;
      if (g >= c1i) Dt[t8(g, c1i)] -= c1 + d1;
      __syncwarp();
      // f2: Ddot <- D Phi(D^{-1} Ddot D^{-T}), Ddot read as the symmetric matrix of its lower
      //     triangle (Eq. 8 on the block)
      double x0 = 0.0, x1 = 0.0;  // X = D^{-1} S
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const int k = 4 * kk + t;
        const double sv = (k >= g) ? Dt[t8(k, g)] : Dt[t8(g, k)];  // S(k, g)
        dmma884(x0, x1, Di[t8(g, k)], sv);
      }
      sX[t8(g, c0i)] = x0;
      sX[t8(g, c1i)] = x1;
      __syncwarp();
      double y0 = 0.0, y1 = 0.0;  // Y = X D^{-T}
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(y0, y1, sX[t8(g, 4 * kk + t)], Di[t8(g, 4 * kk + t)]);
      y0 = (g > c0i) ? y0 : (g == c0i ? 0.5 * y0 : 0.0);  // Phi
      y1 = (g > c1i) ? y1 : (g == c1i ? 0.5 * y1 : 0.0);
      sY[t8(g, c0i)] = y0;
      sY[t8(g, c1i)] = y1;
      __syncwarp();
      double l0 = 0.0, l1 = 0.0;  // Ldot = D Phi(Y)
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(l0, l1, Lt[t8(g, 4 * kk + t)], sY[t8(4 * kk + t, g)]);
      Dt[t8(g, c0i)] = (g >= c0i) ? l0 : 0.0;
      Dt[t8(g, c1i)] = (g >= c1i) ? l1 : 0.0;
    }
    __syncthreads();

    // f3 + f4 per row tile below the block
    for (int rt = warp; rt < PT; rt += DC_WARPS) {
      const int I = J + 1 + rt;
      double* Ct = sA + tile_base(NBLK, I, J);
      const double* Cl = sL + tile_base(NBLK, I, J);
      double c0 = Ct[t8(g, 2 * t)], c1 = Ct[t8(g, 2 * t + 1)];
      double d0 = 0.0, d1 = 0.0;
      for (int ct = 0; ct < QT; ++ct) {
        const double* Bd = sA + tile_base(NBLK, I, ct);
        const double* Bl = sL + tile_base(NBLK, I, ct);
        const double* Rd = sA + tile_base(NBLK, J, ct);
        const double* Rt = sL + tile_base(NBLK, J, ct);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          dmma884(c0, c1, Bd[t8(g, 4 * kk + t)], -Rt[t8(g, 4 * kk + t)]);  // - Bdot R^T
          dmma884(d0, d1, Bl[t8(g, 4 * kk + t)], -Rd[t8(g, 4 * kk + t)]);  // - B Rdot^T
        }
      }
#pragma unroll
      for (int kk = 0; kk < 2; ++kk)
        dmma884(d0, d1, Cl[t8(g, 4 * kk + t)], -Dt[t8(g, 4 * kk + t)]);   // - C Ddot^T
      c0 += d0;
      c1 += d1;
      Ct[t8(g, 2 * t)] = c0;
      Ct[t8(g, 2 * t + 1)] = c1;
      __syncwarp();
      double e0 = 0.0, e1 = 0.0;  // Cdot <- Cdot D^{-T}
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(e0, e1, Ct[t8(g, 4 * kk + t)], Di[t8(g, 4 * kk + t)]);
      __syncwarp();
      Ct[t8(g, 2 * t)] = e0;
      Ct[t8(g, 2 * t + 1)] = e1;
    }
    __syncthreads();
  }

  dc_store<TIO>(NBLK, A, Ad.ld, n, sA, 0);
  if (Dd.base || Dd.arr) {  // clean dense tril(Ldot)
    TIO* Dc = optr_w<TIO>(Dd, b);
    for (int c = warp; c < n; c += DC_WARPS)
      for (int i = lane; i < n; i += 32) Dc[i + int64_t(c) * Dd.ld] = TIO((i >= c) ? sA[tat(NBLK, i, c)] : 0.0);
  }
}

// ============================================================================ inverse
// Dinv[b][q] = tril(L[j0:j0+w, j0:j0+w])^{-1}, dense w x w (ld = ldi), upper zero, at
// Dinv + (b * blocks + q) * stride_blk + (q odd ? odd_off : 0); grid = (blocks, batch); block ranges
// as block_range (misc.cuh).  (odd_off = 64 with stride_blk = 64 ldi and ldi = 128 puts the
// 64-wide inverses on the diagonal of 128-wide blocks: rf32_inv128 fills in the rest.)
template <typename TIO>
__global__ void __launch_bounds__(DC_THREADS, CD_DC_MINB)
    k_trinv_dmma(int n, int nb, int reverse, Opnd Ld, TIO* __restrict__ Dinv, int64_t ldi, int64_t stride_blk,
                 int64_t odd_off) {
  const int NBLK = (nb + 7) >> 3;  // tiling of the widest block; shorter blocks are padded
  const int NP = 8 * NBLK;
  const int NTILE = NBLK * (NBLK + 1) / 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sL = reinterpret_cast<double*>(smem_raw);
  double* sX = sL + NTILE * 64;
  double* sDi = sX + NTILE * 64;
  double* sRd = sDi + NBLK * 64 + 128;
  int* sbad = reinterpret_cast<int*>(sRd + NP);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int q = blockIdx.x;
  const int64_t b = blockIdx.y;
  int j0, w;
  {
    const int r = n % nb;
    if (!reverse || r == 0) {
      j0 = q * nb;
      w = min(nb, n - j0);
    } else if (q == 0) {
      j0 = 0;
      w = r;
    } else {
      j0 = r + (q - 1) * nb;
      w = nb;
    }
  }
  const TIO* L = optr<TIO>(Ld, b) + j0 + int64_t(j0) * Ld.ld;
  if (tid == 0) *sbad = 0x7fffffff;
  dc_stage<TIO>(NBLK, L, Ld.ld, w, sL, true);
  cp_async_wait_all();
  __syncthreads();
  dc_diag_inverses(NBLK, sL, sDi, sRd, w, sbad);
  // column blocks of the inverse over warps: X(J,J) = Dinv_J, then down the column
  for (int J = warp; J < NBLK; J += DC_WARPS) {
    double* XJJ = sX + tile_base(NBLK, J, J);
    for (int e = lane; e < 64; e += 32) XJJ[e] = sDi[J * 64 + e];
    __syncwarp();
    for (int I = J + 1; I < NBLK; ++I) {
      double a0 = 0.0, a1 = 0.0, c0 = 0.0, c1 = 0.0;
      for (int K = J; K < I; ++K) {
        const double* DIK = sL + tile_base(NBLK, I, K);
        const double* XKJ = sX + tile_base(NBLK, K, J);
        dmma884(a0, a1, DIK[t8(g, t)], XKJ[t8(t, g)]);
        dmma884(c0, c1, DIK[t8(g, 4 + t)], XKJ[t8(4 + t, g)]);
      }
      double* XIJ = sX + tile_base(NBLK, I, J);
      XIJ[t8(g, 2 * t)] = a0 + c0;  // temporary: sum D(I,K) X(K,J)
      XIJ[t8(g, 2 * t + 1)] = a1 + c1;
      __syncwarp();
      double x0 = 0.0, x1 = 0.0;  // X(I,J) = -D_I^{-1} sum
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(x0, x1, sDi[I * 64 + t8(g, 4 * kk + t)], -XIJ[t8(4 * kk + t, g)]);
      __syncwarp();
      XIJ[t8(g, 2 * t)] = x0;
      XIJ[t8(g, 2 * t + 1)] = x1;
      __syncwarp();
    }
  }
  __syncthreads();
  TIO* X = Dinv + (int64_t(b) * gridDim.x + q) * stride_blk + ((q & 1) ? odd_off : 0);
  for (int c = warp; c < w; c += DC_WARPS)
    for (int i = lane; i < w; i += 32) X[i + int64_t(c) * ldi] = TIO((i >= c) ? sX[tat(NBLK, i, c)] : 0.0);
}

}  // namespace cd
