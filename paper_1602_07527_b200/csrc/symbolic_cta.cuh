// symbolic_cta.cuh -- the SYMBOLIC route for small matrices (n <= 64, one CTA per matrix,
// batched): the closed forms of PAPER.md §3 instead of the algorithmic sweeps, as the paper
// suggests for small matrices (north star (d)):
//
//   reverse (Eq. 10):  tril(Sigmabar) = Phi(L^{-T} (P + P^T) L^{-1}),
//                                        P = Phi(L^T Lbar)
//   forward (Eq. 8,  PAPER.md:219-221):  Ldot = L Phi(L^{-1} Sigmadot L^{-T})
//
// All in fp64 on 8x8 DMMA tiles held in shared memory (the swizzled tile-packed layout of
// sweep_dmma_cta.cuh): stage tril(L) and the input triangle, invert L (diagonal 8x8
// inverses, then X(I,J) = -D_I^{-1} sum_K L(I,K) X(K,J) by column blocks), then three tile
// products with Phi applied where Eqs. 8 / 10 put it.  Every product is a sum over 8x8
// tiles distributed over the 8 warps; phases are separated by block barriers.  Output
// conventions (TRIL / SYM / GRAD) as the algorithmic kernels.  The symbolic route issues
// more flops than the sweep (about 4x for reverse at n = 64) but has no sequential column
// chain: its latency is four product phases.
#pragma once
#include "common.cuh"
#include "gemm.cuh"
#include "sweep_dmma_cta.cuh"

namespace cd {

constexpr int SYM_NMAX = 64;

inline size_t symbolic_smem(int NBLK) {
  const int nt = NBLK * (NBLK + 1) / 2, nf = NBLK * NBLK;
  // sL, sA, sLi, sP (lower tiles) + sZ (full) + diagonal inverses / reciprocals
  return size_t(4 * nt * 64 + nf * 64 + NBLK * 64 + 8 * NBLK) * sizeof(double) + 16;
}

__device__ __forceinline__ int ftile(int NBLK, int I, int J) { return (J * NBLK + I) * 64; }  // full tiling

template <typename TIO>
__global__ void __launch_bounds__(DC_THREADS, 1)
    k_symbolic_cta(int n, int rev, Opnd Ld, Opnd Ad, int out_mode, int* __restrict__ info) {
  const int NBLK = (n + 7) >> 3;
  const int NT = NBLK * (NBLK + 1) / 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sL = reinterpret_cast<double*>(smem_raw);
  double* sA = sL + NT * 64;
  double* sLi = sA + NT * 64;
  double* sP = sLi + NT * 64;
  double* sZ = sP + NT * 64;
  double* sDi = sZ + NBLK * NBLK * 64;
  double* sRd = sDi + NBLK * 64;
  int* sbad = reinterpret_cast<int*>(sRd + 8 * NBLK);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t b = blockIdx.x;
  const TIO* L = optr<TIO>(Ld, b);
  TIO* A = optr_w<TIO>(Ad, b);
  auto LT = [&](const double* base, int I, int J) { return base + tile_base(NBLK, I, J); };  // lower tile

  if (tid == 0) *sbad = 0x7fffffff;
  dc_stage<TIO>(NBLK, L, Ld.ld, n, sL, true);
  dc_stage<TIO>(NBLK, A, Ad.ld, n, sA, false);
  cp_async_wait_all();
  __syncthreads();
  dc_diag_inverses(NBLK, sL, sDi, sRd, n, sbad);
  if (tid == 0 && info) info[b] = (*sbad == 0x7fffffff) ? 0 : *sbad;

  // ---- L^{-1} by column blocks (lower tiles of sLi)
  for (int J = warp; J < NBLK; J += DC_WARPS) {
    double* XJJ = sLi + tile_base(NBLK, J, J);
    for (int e = lane; e < 64; e += 32) XJJ[e] = sDi[J * 64 + e];
    __syncwarp();
    for (int I = J + 1; I < NBLK; ++I) {
      double a0 = 0.0, a1 = 0.0;
      for (int K = J; K < I; ++K) {
        const double* DIK = LT(sL, I, K);
        const double* XKJ = LT(sLi, K, J);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) dmma884(a0, a1, DIK[t8(g, 4 * kk + t)], XKJ[t8(4 * kk + t, g)]);
      }
      double* XIJ = sLi + tile_base(NBLK, I, J);
      XIJ[t8(g, 2 * t)] = a0;  // temporary: sum_K D(I,K) X(K,J)
      XIJ[t8(g, 2 * t + 1)] = a1;
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

  const int c0 = 2 * t, c1 = 2 * t + 1;
  if (rev) {
    // ---- P = Phi(L^T Lbar)   (lower tiles):  P(I,J) = sum_{R >= I} L(R,I)^T Lbar(R,J)
    for (int task = warp; task < NT; task += DC_WARPS) {
      int I = 0, J = 0, r = task;  // column-major lower tile order
      while (r >= NBLK - J) r -= NBLK - J, ++J;
      I = J + r;
      double p0 = 0.0, p1 = 0.0;
      for (int R = I; R < NBLK; ++R) {
        const double* LRI = LT(sL, R, I);
        const double* ARJ = LT(sA, R, J);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) dmma884(p0, p1, LRI[t8(4 * kk + t, g)], ARJ[t8(4 * kk + t, g)]);
      }
      if (I == J) {
        p0 = g > c0 ? p0 : (g == c0 ? 0.5 * p0 : 0.0);
        p1 = g > c1 ? p1 : (g == c1 ? 0.5 * p1 : 0.0);
      }
      double* PIJ = sP + tile_base(NBLK, I, J);
      PIJ[t8(g, c0)] = p0;
      PIJ[t8(g, c1)] = p1;
    }
    __syncthreads();
    // ---- Z = (P + P^T) L^{-1}   (full):  Z(I,J) = sum_{K >= J} X(I,K) Linv(K,J)
    for (int task = warp; task < NBLK * NBLK; task += DC_WARPS) {
      const int I = task % NBLK, J = task / NBLK;
      double z0 = 0.0, z1 = 0.0;
      for (int K = J; K < NBLK; ++K) {
        const double* LiKJ = LT(sLi, K, J);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int k = 4 * kk + t;
          double x;  // X(I,K)(g, k)
          if (I > K) x = LT(sP, I, K)[t8(g, k)];
          else if (I < K) x = LT(sP, K, I)[t8(k, g)];
          else x = LT(sP, I, I)[t8(g, k)] + LT(sP, I, I)[t8(k, g)];
          dmma884(z0, z1, x, LiKJ[t8(k, g)]);
        }
      }
      double* ZIJ = sZ + ftile(NBLK, I, J);
      ZIJ[t8(g, c0)] = z0;
      ZIJ[t8(g, c1)] = z1;
    }
    __syncthreads();
    // ---- tril(Sigmabar) = Phi(L^{-T} Z)   (lower):  Y(I,J) = sum_{K >= I} Linv(K,I)^T Z(K,J)
    for (int task = warp; task < NT; task += DC_WARPS) {
      int I = 0, J = 0, r = task;
      while (r >= NBLK - J) r -= NBLK - J, ++J;
      I = J + r;
      double y0 = 0.0, y1 = 0.0;
      for (int K = I; K < NBLK; ++K) {
        const double* LiKI = LT(sLi, K, I);
        const double* ZKJ = sZ + ftile(NBLK, K, J);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) dmma884(y0, y1, LiKI[t8(4 * kk + t, g)], ZKJ[t8(4 * kk + t, g)]);
      }
      if (I == J) {
        y0 = g > c0 ? y0 : (g == c0 ? 0.5 * y0 : 0.0);
        y1 = g > c1 ? y1 : (g == c1 ? 0.5 * y1 : 0.0);
      }
      double* OIJ = sA + tile_base(NBLK, I, J);
      OIJ[t8(g, c0)] = y0;
      OIJ[t8(g, c1)] = y1;
    }
  } else {
    // ---- Y = L^{-1} X  (full), X = Sigmadot read symmetric from its lower triangle:
    //      Y(I,J) = sum_{K <= I} Linv(I,K) X(K,J)
    for (int task = warp; task < NBLK * NBLK; task += DC_WARPS) {
      const int I = task % NBLK, J = task / NBLK;
      double y0 = 0.0, y1 = 0.0;
      for (int K = 0; K <= I; ++K) {
        const double* LiIK = LT(sLi, I, K);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int k = 4 * kk + t;
          double x;  // X(K,J)(k, g)
          if (K > J) x = LT(sA, K, J)[t8(k, g)];
          else if (K < J) x = LT(sA, J, K)[t8(g, k)];
          else x = k >= g ? LT(sA, K, K)[t8(k, g)] : LT(sA, K, K)[t8(g, k)];
          dmma884(y0, y1, LiIK[t8(g, k)], x);
        }
      }
      double* YIJ = sZ + ftile(NBLK, I, J);
      YIJ[t8(g, c0)] = y0;
      YIJ[t8(g, c1)] = y1;
    }
    __syncthreads();
    // ---- F = Phi(Y L^{-T})  (lower):  F(I,J) = sum_{K <= J} Y(I,K) Linv(J,K)^T
    for (int task = warp; task < NT; task += DC_WARPS) {
      int I = 0, J = 0, r = task;
      while (r >= NBLK - J) r -= NBLK - J, ++J;
      I = J + r;
      double f0 = 0.0, f1 = 0.0;
      for (int K = 0; K <= J; ++K) {
        const double* YIK = sZ + ftile(NBLK, I, K);
        const double* LiJK = LT(sLi, J, K);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) dmma884(f0, f1, YIK[t8(g, 4 * kk + t)], LiJK[t8(g, 4 * kk + t)]);
      }
      if (I == J) {
        f0 = g > c0 ? f0 : (g == c0 ? 0.5 * f0 : 0.0);
        f1 = g > c1 ? f1 : (g == c1 ? 0.5 * f1 : 0.0);
      }
      double* FIJ = sP + tile_base(NBLK, I, J);
      FIJ[t8(g, c0)] = f0;
      FIJ[t8(g, c1)] = f1;
    }
    __syncthreads();
    // ---- Ldot = L F  (lower):  Ldot(I,J) = sum_{J <= K <= I} L(I,K) F(K,J)
    for (int task = warp; task < NT; task += DC_WARPS) {
      int I = 0, J = 0, r = task;
      while (r >= NBLK - J) r -= NBLK - J, ++J;
      I = J + r;
      double d0 = 0.0, d1 = 0.0;
      for (int K = J; K <= I; ++K) {
        const double* LIK = LT(sL, I, K);
        const double* FKJ = LT(sP, K, J);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) dmma884(d0, d1, LIK[t8(g, 4 * kk + t)], FKJ[t8(4 * kk + t, g)]);
      }
      double* OIJ = sA + tile_base(NBLK, I, J);
      OIJ[t8(g, c0)] = d0;
      OIJ[t8(g, c1)] = d1;
    }
  }
  __syncthreads();
  dc_store<TIO>(NBLK, A, Ad.ld, n, sA, rev ? out_mode : 0);
}

}  // namespace cd
