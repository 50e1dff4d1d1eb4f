// sweep_dmma_cta.cuh -- fp64 reverse mode for one matrix / diagonal block with n <= 128,
// one CTA (8 warps) per matrix: the blocked reverse sweep of PAPER.md:689-701 with
// N_b = 8 on DMMA tiles (mma.sync.m8n8k4.f64), the 8x8 diagonal blocks by Eq. 10
// (as the paper's own implementation does).
// Same tile arithmetic as sweep_dmma32.cuh (see there), with the tiles of each
// update distributed over the warps of the CTA:
//
//   for J = NBLK-1 .. 0:   s1  Cbar <- Cbar D^{-1}            tiles over warps
//                          s2  Bbar <- Bbar - Cbar R          tiles over warps
//                          s3  Dbar <- Dbar - tril(Cbar^T C)  one warp (two accumulators)
//                          s4  Dbar <- Phi(D^{-T}(P+P^T)D^{-1}), S = D^{-T}(P+P^T)D^{-1}
//                          s5  Rbar <- Rbar - Cbar^T B - S R  tiles over warps
//
// This is the diagonal-block kernel of the blocked driver (N_b = 128 -> 16 tiles) and
// the single / batched kernel for 32 < n <= 128.  Shared memory: the lower 8x8 tiles
// of L and Abar, tile-packed and swizzled (bank-conflict-free fragments), 139 KB at
// n = 128.
#pragma once
#include "common.cuh"
#include "gemm.cuh"          // dmma884

namespace cd {

// offset of element (r, c) inside a swizzled 8x8 tile: (r, c) at c*8 + (r ^ 4*((c>>1)&1)),
// which makes every A / B fragment load of mma.m8n8k4 bank-conflict free
__device__ __forceinline__ int t8(int r, int c) { return c * 8 + (r ^ ((c & 2) << 1)); }

template <int NBLK>
__device__ __forceinline__ int tile_base(int bi, int bj) {  // lower tile (bi >= bj), column-major tile order
  return (bj * NBLK - (bj * (bj - 1)) / 2 + (bi - bj)) * 64;
}

constexpr int DC_WARPS = 8;
constexpr int DC_THREADS = DC_WARPS * 32;

template <int NBLK>
inline size_t dmma_cta_smem() {
  constexpr int ntile = NBLK * (NBLK + 1) / 2;
  return size_t(2 * ntile * 64 + NBLK * 64 + 2 * 64 + 8 * NBLK) * sizeof(double) + 16;
}

template <int NBLK>
__global__ void __launch_bounds__(DC_THREADS, 1)
    k_rev_dmma_cta(int n, Opnd Ld, Opnd Ad, int out_mode, Opnd Sd, int* __restrict__ info) {
  constexpr int NP = 8 * NBLK;
  constexpr int NTILE = NBLK * (NBLK + 1) / 2;
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
  const double* L = optr<double>(Ld, b);
  double* A = optr_w<double>(Ad, b);
  auto at = [](int i, int m) { return tile_base<NBLK>(i >> 3, m >> 3) + t8(i & 7, m & 7); };

  if (tid == 0) *sbad = 0x7fffffff;
  // ---- stage the lower triangles (one column per warp pass, lanes over rows)
  for (int m = warp; m < n; m += DC_WARPS)
    for (int i = m + lane; i < n; i += 32) {
      const int o = at(i, m);
      cp_async_zfill<8>(sL + o, L + i + int64_t(m) * Ld.ld, true);
      cp_async_zfill<8>(sA + o, A + i + int64_t(m) * Ad.ld, true);
    }
  // upper triangles of the diagonal tiles -> 0; padding beyond n -> blockdiag(I) / 0
  for (int e = tid; e < NBLK * 64; e += DC_THREADS) {
    const int blk = e >> 6, r = e & 7, c = (e >> 3) & 7;
    const int i = 8 * blk + r, m = 8 * blk + c;
    const int o = tile_base<NBLK>(blk, blk) + t8(r, c);
    if (r < c) {
      sL[o] = 0.0;
      sA[o] = 0.0;
    } else if (i >= n) {
      sL[o] = (i == m) ? 1.0 : 0.0;
      sA[o] = 0.0;
    }
  }
  if (n < NP) {
    for (int e = tid; e < NTILE * 64; e += DC_THREADS) {
      // decode tile index -> (bi, bj), column-major tile order
      int tix = e >> 6, bj = 0;
      while (tix >= NBLK - bj) {
        tix -= NBLK - bj;
        ++bj;
      }
      const int bi = bj + tix;
      if (bi == bj) continue;
      const int r = e & 7, c = (e >> 3) & 7;  // note: element order inside the tile is irrelevant here
      if (8 * bi + r >= n || 8 * bj + c >= n) {
        sL[tile_base<NBLK>(bi, bj) + t8(r, c)] = 0.0;
        sA[tile_base<NBLK>(bi, bj) + t8(r, c)] = 0.0;
      }
    }
  }
  cp_async_wait_all();
  __syncthreads();
  for (int i = tid; i < NP; i += DC_THREADS) {
    const double d = sL[at(i, i)];
    if (i < n && bad_pivot(d)) atomicMin(sbad, i + 1);
    sRd[i] = 1.0 / d;
  }
  __syncthreads();
  if (tid == 0 && info) info[b] = (*sbad == 0x7fffffff) ? 0 : *sbad;

  // ---- D^{-1} of every diagonal 8x8 block: thread -> (block, column)
  for (int e = tid; e < NBLK * 8; e += DC_THREADS) {
    const int blk = e >> 3, c = e & 7, j0 = 8 * blk;
    const double* D = sL + tile_base<NBLK>(blk, blk);
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

  for (int J = NBLK - 1; J >= 0; --J) {
    const int PT = NBLK - 1 - J, QT = J;
    const double* Di = sDi + J * 64;
    double* Dt = sA + tile_base<NBLK>(J, J);
    const double* Lt = sL + tile_base<NBLK>(J, J);

    // s1: Cbar <- Cbar D^{-1}
    for (int rt = warp; rt < PT; rt += DC_WARPS) {
      double* Ct = sA + tile_base<NBLK>(J + 1 + rt, J);
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(c0, c1, Ct[t8(g, 4 * kk + t)], Di[t8(4 * kk + t, g)]);
      __syncwarp();
      Ct[t8(g, 2 * t)] = c0;
      Ct[t8(g, 2 * t + 1)] = c1;
    }
    __syncthreads();

    // s3 (last warp): Dbar <- Dbar - tril(Cbar^T C);   s2 (all warps): Bbar <- Bbar - Cbar R
    if (warp == DC_WARPS - 1 && PT > 0) {
      double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
      for (int rt = 0; rt < PT; ++rt) {
        const double* Ct = sA + tile_base<NBLK>(J + 1 + rt, J);
        const double* Lc = sL + tile_base<NBLK>(J + 1 + rt, J);
        dmma884(a0, a1, Ct[t8(t, g)], Lc[t8(t, g)]);
        dmma884(b0, b1, Ct[t8(4 + t, g)], Lc[t8(4 + t, g)]);
      }
      a0 += b0;
      a1 += b1;
      if (g >= 2 * t) Dt[t8(g, 2 * t)] -= a0;
      if (g >= 2 * t + 1) Dt[t8(g, 2 * t + 1)] -= a1;
    }
    for (int idx = warp; idx < PT * QT; idx += DC_WARPS) {
      const int rt = idx / QT, ct = idx - rt * QT;
      const double* Ct = sA + tile_base<NBLK>(J + 1 + rt, J);
      double* Bt = sA + tile_base<NBLK>(J + 1 + rt, ct);
      const double* Rt = sL + tile_base<NBLK>(J, ct);
      double c0 = Bt[t8(g, 2 * t)], c1 = Bt[t8(g, 2 * t + 1)];
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(c0, c1, Ct[t8(g, 4 * kk + t)], -Rt[t8(4 * kk + t, g)]);
      Bt[t8(g, 2 * t)] = c0;
      Bt[t8(g, 2 * t + 1)] = c1;
    }
    __syncthreads();

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

    // s5: Rbar <- Rbar - Cbar^T B - S R
    for (int ct = warp; ct < QT; ct += DC_WARPS) {
      double* Rb = sA + tile_base<NBLK>(J, ct);
      const double* Rt = sL + tile_base<NBLK>(J, ct);
      double c0 = Rb[t8(g, 2 * t)], c1 = Rb[t8(g, 2 * t + 1)];
      double d0 = 0.0, d1 = 0.0;
      for (int rt = 0; rt < PT; ++rt) {
        const double* Ct = sA + tile_base<NBLK>(J + 1 + rt, J);
        const double* Bt = sL + tile_base<NBLK>(J + 1 + rt, ct);
        dmma884(c0, c1, Ct[t8(t, g)], -Bt[t8(t, g)]);
        dmma884(d0, d1, Ct[t8(4 + t, g)], -Bt[t8(4 + t, g)]);
      }
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(d0, d1, sS[t8(g, 4 * kk + t)], -Rt[t8(4 * kk + t, g)]);
      Rb[t8(g, 2 * t)] = c0 + d0;
      Rb[t8(g, 2 * t + 1)] = c1 + d1;
    }
    __syncthreads();
  }

  // ---- write back tril (and the requested mirror); optional dense S = Dbar + Dbar^T
  for (int m = warp; m < n; m += DC_WARPS)
    for (int i = m + lane; i < n; i += 32) {
      double v = sA[at(i, m)];
      if (out_mode == 2 && i != m) v *= 0.5;
      A[i + int64_t(m) * Ad.ld] = v;
    }
  if (out_mode != 0) {
    for (int i = warp; i < n; i += DC_WARPS)
      for (int m = lane; m < i; m += 32) {
        double v = sA[at(i, m)];
        if (out_mode == 2) v *= 0.5;
        A[m + int64_t(i) * Ad.ld] = v;
      }
  }
  if (Sd.base || Sd.arr) {
    double* S = optr_w<double>(Sd, b);
    for (int e = tid; e < n * n; e += DC_THREADS) {
      const int i = e % n, c = e / n;
      const double v = (i >= c) ? sA[at(i, c)] : sA[at(c, i)];
      S[i + int64_t(c) * Sd.ld] = (i == c) ? 2.0 * v : v;
    }
  }
}

}  // namespace cd
