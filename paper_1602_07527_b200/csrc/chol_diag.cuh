// chol_diag.cuh -- on-chip Cholesky factorisation of a diagonal block (n <= 128, one CTA per
// block / matrix) and its inverse, for the fused factorisation + forward sweep
// (chol_blocked: "D <- chol_unblocked(D)"; the forward
// sensitivities can be accumulated in the same loop).
//
// Right-looking blocked Cholesky on 8x8 DMMA tiles in shared memory (layout of
// sweep_dmma_cta.cuh), for J = 0 .. NBLK-1:
//   warp 0:    D_JJ <- chol_unblocked(D_JJ) (PAPER.md:437-445 on the 8x8 tile), and D_JJ^{-1}
//   all warps: L_IJ <- A_IJ D_JJ^{-T}                       (I > J)
//              A_IK <- A_IK - L_IJ L_KJ^T                   (I >= K > J, lower tiles)
// then tril(D) is written back and D^{-1} (dense, upper zero) goes to `Dinv` for the panel
// solve and the forward Eq. 8.  A non-positive or non-finite pivot sets info (1-based).
#pragma once
#include "common.cuh"
#include "gemm.cuh"
#include "sweep_dmma_cta.cuh"

namespace cd {

// factor block `blk` (0-based) of the matrix whose block partition is (j0 = blk*nb forward);
// grid = (1, batch) per call site; the block view is D = A[j0:j0+w, j0:j0+w]
template <typename TIO>
__global__ void __launch_bounds__(DC_THREADS, 1)
    k_chol_diag(int w, Opnd Ad, TIO* __restrict__ Dinv, int64_t ldi, int64_t stride_i, int j0, int* __restrict__ info) {
  const int NBLK = (w + 7) >> 3;
  const int NTILE = NBLK * (NBLK + 1) / 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sL = reinterpret_cast<double*>(smem_raw);
  double* sX = sL + NTILE * 64;
  double* sDi = sX + NTILE * 64;   // inverses of the factored 8x8 diagonal tiles
  double* sRd = sDi + NBLK * 64 + 128;
  int* sbad = reinterpret_cast<int*>(sRd + 8 * NBLK);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t b = blockIdx.y;
  TIO* A = optr_w<TIO>(Ad, b);

  if (tid == 0) *sbad = 0x7fffffff;
  dc_stage<TIO>(NBLK, A, Ad.ld, w, sL, true);  // padding: identity (chol of blockdiag(D, I))
  cp_async_wait_all();
  __syncthreads();

  for (int J = 0; J < NBLK; ++J) {
    double* T = sL + tile_base(NBLK, J, J);
    if (warp == 0) {
      // unblocked Cholesky of the 8x8 tile, column by column
      for (int c = 0; c < 8; ++c) {
        if (lane == 0) {
          const double v = T[t8(c, c)];
          if (!(v > 0.0) && 8 * J + c < w) atomicMin(sbad, 8 * J + c + 1);
          T[t8(c, c)] = sqrt(v);
        }
        __syncwarp();
        const double d = T[t8(c, c)];
        if (lane > c && lane < 8) T[t8(lane, c)] /= d;
        __syncwarp();
        // trailing update of the tile: (r, m) with c < m <= r  (at most 28 pairs)
        for (int e = lane; e < 64; e += 32) {
          const int r = e >> 3, m = e & 7;
          if (m > c && r >= m) T[t8(r, m)] -= T[t8(r, c)] * T[t8(m, c)];
        }
        __syncwarp();
      }
      // D_JJ^{-1}: lane c < 8 computes column c by forward substitution
      if (lane < 8) {
        const int c = lane;
        double x[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          if (r < c) {
            x[r] = 0.0;
          } else {
            double s = (r == c) ? 1.0 : 0.0;
#pragma unroll
            for (int q = 0; q < r; ++q)
              if (q >= c) s -= T[t8(r, q)] * x[q];
            x[r] = s / T[t8(r, r)];
          }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) sDi[J * 64 + t8(r, c)] = x[r];
      }
    }
    __syncthreads();
    // panel: L_IJ = A_IJ D_JJ^{-T}
    const double* Di = sDi + J * 64;
    for (int I = J + 1 + warp; I < NBLK; I += DC_WARPS) {
      double* AIJ = sL + tile_base(NBLK, I, J);
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(c0, c1, AIJ[t8(g, 4 * kk + t)], Di[t8(g, 4 * kk + t)]);
      __syncwarp();
      AIJ[t8(g, 2 * t)] = c0;
      AIJ[t8(g, 2 * t + 1)] = c1;
    }
    __syncthreads();
    // trailing: A_IK -= L_IJ L_KJ^T  (I >= K > J)
    const int R = NBLK - 1 - J;
    for (int idx = warp; idx < R * (R + 1) / 2; idx += DC_WARPS) {
      int K = 0, r = idx;  // column-major lower order over the trailing (R x R) tiles
      while (r >= R - K) r -= R - K, ++K;
      const int I = J + 1 + K + r, Kt = J + 1 + K;
      const double* LIJ = sL + tile_base(NBLK, I, J);
      const double* LKJ = sL + tile_base(NBLK, Kt, J);
      double* AIK = sL + tile_base(NBLK, I, Kt);
      double c0 = AIK[t8(g, 2 * t)], c1 = AIK[t8(g, 2 * t + 1)];
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(c0, c1, LIJ[t8(g, 4 * kk + t)], -LKJ[t8(g, 4 * kk + t)]);
      if (I == Kt) {  // diagonal tile: keep the upper part zero
        if (g < 2 * t) c0 = 0.0;
        if (g < 2 * t + 1) c1 = 0.0;
      }
      AIK[t8(g, 2 * t)] = c0;
      AIK[t8(g, 2 * t + 1)] = c1;
    }
    __syncthreads();
  }
  if (tid == 0 && info) {
    const int v = (*sbad == 0x7fffffff) ? 0 : j0 + *sbad;
    if (v && (info[b] == 0 || v < info[b])) info[b] = v;
  }
  dc_store<TIO>(NBLK, A, Ad.ld, w, sL, 0);
  // D^{-1}: diagonal-tile inverses are in sDi; off-diagonal tiles by column blocks
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
      XIJ[t8(g, 2 * t)] = a0 + c0;
      XIJ[t8(g, 2 * t + 1)] = a1 + c1;
      __syncwarp();
      double x0 = 0.0, x1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(x0, x1, sDi[I * 64 + t8(g, 4 * kk + t)], -XIJ[t8(4 * kk + t, g)]);
      __syncwarp();
      XIJ[t8(g, 2 * t)] = x0;
      XIJ[t8(g, 2 * t + 1)] = x1;
      __syncwarp();
    }
  }
  __syncthreads();
  TIO* X = Dinv + b * stride_i;
  for (int c = warp; c < w; c += DC_WARPS)
    for (int i = lane; i < w; i += 32) X[i + int64_t(c) * ldi] = TIO((i >= c) ? sX[tat(NBLK, i, c)] : 0.0);
}

}  // namespace cd
