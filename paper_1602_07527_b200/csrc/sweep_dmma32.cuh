// sweep_dmma32.cuh -- batched fp64 reverse mode for n <= 32 on the fp64 tensor cores:
// one WARP per matrix, the paper's blocked reverse sweep with
// N_b = 8, so that every Level-3 update is a handful of 8x8x4 DMMA tiles
// (mma.sync.m8n8k4.f64), and the 8x8 diagonal-block update done with the symbolic
// Eq. 10 -- the replacement the paper itself uses for the
// diagonal block:
//
//   for each 8-block J (bottom-right first), R, D, B, C = level3partition(L, J):
//     Cbar <- Cbar D^{-1}                 (PT x 2 DMMA;  D^{-1} precomputed per block)
//     Bbar <- Bbar - Cbar R               (PT x QT x 2 DMMA)
//     Dbar <- Dbar - tril(Cbar^T C)       (PT x 2 DMMA)
//     Dbar <- Phi(D^{-T} (P + P^T) D^{-1}),  P = Phi(D^T Dbar)      (6 DMMA, Eq. 10)
//            and S = Dbar + Dbar^T = D^{-T}(P + P^T)D^{-1} exactly (pre-Phi value)
//     Rbar <- Rbar - Cbar^T B - S R       (QT x (2 PT + 2) DMMA)
//   52 DMMA + 24 (diagonal blocks) per 32 x 32 matrix.
//
// Shared memory holds only the 10 lower 8x8 tiles of L and Abar (tile-packed,
// 5 KB each) with an XOR swizzle inside each tile -- element (r, c) at
// c*8 + (r ^ 4*((c>>1)&1)) -- that makes every A / B fragment load of
// mma.m8n8k4 bank-conflict free.  Only the lower triangles move through HBM (one
// contiguous run per column, cp.async) and only tril(Sigma_bar) is written back.
// n < 32 is embedded as blockdiag(L, I), (Abar, 0): exact.
#pragma once
#include "common.cuh"
#include "gemm.cuh"  // dmma884

namespace cd {

constexpr int D32_WPB = 2;                                      // warps (matrices) per CTA
constexpr int D32_TILES = 10;                                   // lower 8x8 tiles of 32 x 32
constexpr int D32_PER_WARP = 2 * D32_TILES * 64 + 4 * 64 + 2 * 64 + 32;  // doubles
constexpr int D32_MIN_CTAS = 6;                                 // target residency per SM

inline size_t dmma32_smem() { return size_t(D32_WPB) * D32_PER_WARP * sizeof(double); }

// offset of element (r, c) inside a swizzled 8x8 tile
__device__ __forceinline__ int t8(int r, int c) { return c * 8 + (r ^ ((c & 2) << 1)); }

template <int NBLK>
__device__ __forceinline__ int tile_base(int bi, int bj) {  // lower tile (bi >= bj), column-major tile order
  return (bj * NBLK - (bj * (bj - 1)) / 2 + (bi - bj)) * 64;
}

template <int NBLK>
__global__ void __launch_bounds__(D32_WPB * 32, D32_MIN_CTAS)
    k_rev_dmma32(int n, int64_t batch, Opnd Ld, Opnd Ad, int out_mode, int* __restrict__ info) {
  constexpr int NP = 8 * NBLK;  // padded size
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* sL = reinterpret_cast<double*>(smem_raw) + w * D32_PER_WARP;
  double* sA = sL + D32_TILES * 64;
  double* sDi = sA + D32_TILES * 64;  // NBLK tiles: D^{-1}
  double* sX = sDi + 4 * 64;          // scratch tile
  double* sS = sX + 64;               // S = Dbar + Dbar^T of the current block
  double* sRd = sS + 64;              // 1 / L_jj
  const int g = lane >> 2, t = lane & 3;
  auto at = [](int i, int m) { return tile_base<NBLK>(i >> 3, m >> 3) + t8(i & 7, m & 7); };

  // this lane's share of the packed lower triangle, column by column: element
  // e = lane + 32k -> (row i, column m) and its swizzled smem offset
  const int tri = n * (n + 1) / 2;
  int ent[17];
  {
    int m = 0, cs = 0;
#pragma unroll
    for (int k = 0; k < 17; ++k) {
      const int e = lane + 32 * k;
      while (m < n && e >= cs + (n - m)) {
        cs += n - m;
        ++m;
      }
      const int i = m + (e - cs);
      ent[k] = (e < tri) ? (at(i, m) | (i << 10) | (m << 16)) : -1;
    }
  }

  for (int64_t b = int64_t(blockIdx.x) * D32_WPB + w; b < batch; b += int64_t(gridDim.x) * D32_WPB) {
    const double* L = optr<double>(Ld, b);
    double* A = optr_w<double>(Ad, b);

    // ---- stage lower triangles (coalesced: consecutive lanes read consecutive rows)
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 17; ++k) {
      if (ent[k] >= 0) {
        const int so = ent[k] & 1023, i = (ent[k] >> 10) & 63, m = ent[k] >> 16;
        cp_async_zfill<8>(sL + so, L + i + m * Ld.ld, true);
        cp_async_zfill<8>(sA + so, A + i + m * Ad.ld, true);
      }
    }
    // zero the upper triangles of the diagonal tiles (Eq. 10 step reads full tiles);
    // pad n < NP to blockdiag(L, I) / (A, 0)
    for (int e = lane; e < NBLK * 64; e += 32) {
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
      for (int bj = 0; bj < NBLK; ++bj)
        for (int bi = bj + 1; bi < NBLK; ++bi)
          for (int e = lane; e < 64; e += 32) {
            const int r = e & 7, c = e >> 3;
            if (8 * bi + r >= n || 8 * bj + c >= n) {
              sL[tile_base<NBLK>(bi, bj) + t8(r, c)] = 0.0;
              sA[tile_base<NBLK>(bi, bj) + t8(r, c)] = 0.0;
            }
          }
    }
    cp_async_wait_all();
    __syncwarp();
    {
      const bool bad = lane < n && bad_pivot(sL[at(lane, lane)]);
      const unsigned msk = __ballot_sync(0xffffffffu, bad);
      if (info && lane == 0) info[b] = msk ? __ffs(msk) : 0;
      if (lane < NP) sRd[lane] = 1.0 / sL[at(lane, lane)];
    }
    __syncwarp();

    // ---- D^{-1} of every diagonal block: lane -> (block, column c), forward substitution
    {
      const int blk = lane >> 3, c = lane & 7, j0 = 8 * blk;
      if (blk < NBLK) {
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
    }
    __syncwarp();

#pragma unroll
    for (int J = NBLK - 1; J >= 0; --J) {
      const int PT = NBLK - 1 - J;  // 8-row tiles below the block
      const int QT = J;             // 8-col tiles left of the block
      const double* Di = sDi + J * 64;
      double* Dt = sA + tile_base<NBLK>(J, J);        // Dbar tile
      const double* Lt = sL + tile_base<NBLK>(J, J);  // D tile

      // s1: Cbar <- Cbar D^{-1}   (in place, tile by tile)
#pragma unroll
      for (int rt = 0; rt < 3; ++rt) {
        if (rt < PT) {
          double* Ct = sA + tile_base<NBLK>(J + 1 + rt, J);
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) dmma884(c0, c1, Ct[t8(g, 4 * kk + t)], Di[t8(4 * kk + t, g)]);
          __syncwarp();
          Ct[t8(g, 2 * t)] = c0;
          Ct[t8(g, 2 * t + 1)] = c1;
        }
      }
      __syncwarp();

      // s2: Bbar <- Bbar - Cbar R
#pragma unroll
      for (int rt = 0; rt < 3; ++rt) {
        if (rt < PT) {
          const double* Ct = sA + tile_base<NBLK>(J + 1 + rt, J);
#pragma unroll
          for (int ct = 0; ct < 3; ++ct) {
            if (ct < QT) {
              double* Bt = sA + tile_base<NBLK>(J + 1 + rt, ct);
              const double* Rt = sL + tile_base<NBLK>(J, ct);
              double c0 = Bt[t8(g, 2 * t)], c1 = Bt[t8(g, 2 * t + 1)];
#pragma unroll
              for (int kk = 0; kk < 2; ++kk) dmma884(c0, c1, Ct[t8(g, 4 * kk + t)], -Rt[t8(4 * kk + t, g)]);
              Bt[t8(g, 2 * t)] = c0;
              Bt[t8(g, 2 * t + 1)] = c1;
            }
          }
        }
      }
      // s3: Dbar <- Dbar - tril(Cbar^T C)
      if (PT > 0) {
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int rt = 0; rt < 3; ++rt) {
          if (rt < PT) {
            const double* Ct = sA + tile_base<NBLK>(J + 1 + rt, J);
            const double* Lc = sL + tile_base<NBLK>(J + 1 + rt, J);
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) dmma884(c0, c1, Ct[t8(4 * kk + t, g)], Lc[t8(4 * kk + t, g)]);
          }
        }
        if (g >= 2 * t) Dt[t8(g, 2 * t)] -= c0;
        if (g >= 2 * t + 1) Dt[t8(g, 2 * t + 1)] -= c1;
      }
      __syncwarp();

      // s4: diagonal block by Eq. 10:  Y = D^{-T}(P + P^T)D^{-1},  P = Phi(D^T Dbar)
      {
        double p0 = 0.0, p1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) dmma884(p0, p1, Lt[t8(4 * kk + t, g)], Dt[t8(4 * kk + t, g)]);
        const int c0i = 2 * t, c1i = 2 * t + 1;
        p0 = (g > c0i) ? p0 : (g == c0i ? 0.5 * p0 : 0.0);  // Phi
        p1 = (g > c1i) ? p1 : (g == c1i ? 0.5 * p1 : 0.0);
        sX[t8(g, c0i)] = p0;
        sX[t8(g, c1i)] = p1;
        __syncwarp();
        const double x0 = p0 + sX[t8(c0i, g)];  // X = P + P^T
        const double x1 = p1 + sX[t8(c1i, g)];
        __syncwarp();
        sX[t8(g, c0i)] = x0;
        sX[t8(g, c1i)] = x1;
        __syncwarp();
        double z0 = 0.0, z1 = 0.0;  // Z = X D^{-1}
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) dmma884(z0, z1, sX[t8(g, 4 * kk + t)], Di[t8(4 * kk + t, g)]);
        __syncwarp();
        sX[t8(g, c0i)] = z0;
        sX[t8(g, c1i)] = z1;
        __syncwarp();
        double y0 = 0.0, y1 = 0.0;  // Y = D^{-T} Z
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) dmma884(y0, y1, Di[t8(4 * kk + t, g)], sX[t8(4 * kk + t, g)]);
        sS[t8(g, c0i)] = y0;  // S = Y
        sS[t8(g, c1i)] = y1;
        if (g >= c0i) Dt[t8(g, c0i)] = (g == c0i) ? 0.5 * y0 : y0;  // tril(Dbar) = Phi(Y)
        if (g >= c1i) Dt[t8(g, c1i)] = (g == c1i) ? 0.5 * y1 : y1;
      }
      __syncwarp();

      // s5: Rbar <- Rbar - Cbar^T B - S R
#pragma unroll
      for (int ct = 0; ct < 3; ++ct) {
        if (ct < QT) {
          double* Rb = sA + tile_base<NBLK>(J, ct);
          const double* Rt = sL + tile_base<NBLK>(J, ct);
          double c0 = Rb[t8(g, 2 * t)], c1 = Rb[t8(g, 2 * t + 1)];
#pragma unroll
          for (int rt = 0; rt < 3; ++rt) {
            if (rt < PT) {
              const double* Ct = sA + tile_base<NBLK>(J + 1 + rt, J);
              const double* Bt = sL + tile_base<NBLK>(J + 1 + rt, ct);
#pragma unroll
              for (int kk = 0; kk < 2; ++kk) dmma884(c0, c1, Ct[t8(4 * kk + t, g)], -Bt[t8(4 * kk + t, g)]);
            }
          }
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) dmma884(c0, c1, sS[t8(g, 4 * kk + t)], -Rt[t8(4 * kk + t, g)]);
          Rb[t8(g, 2 * t)] = c0;
          Rb[t8(g, 2 * t + 1)] = c1;
        }
      }
      __syncwarp();
    }

    // ---- write back tril(Sigma_bar) (and the requested mirror)
#pragma unroll
    for (int k = 0; k < 17; ++k) {
      if (ent[k] >= 0) {
        const int so = ent[k] & 1023, i = (ent[k] >> 10) & 63, m = ent[k] >> 16;
        double v = sA[so];
        if (out_mode == 2 && i != m) v *= 0.5;
        A[i + m * Ad.ld] = v;
      }
    }
    if (out_mode != 0) {
      for (int i = 1; i < n; ++i) {
        if (lane < i) {
          double v = sA[at(i, lane)];
          if (out_mode == 2) v *= 0.5;
          A[lane + i * Ad.ld] = v;
        }
      }
    }
  }
}

}  // namespace cd
