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
// Shared memory per warp: L and Abar column-major with pitch 36 (= 4 mod 16
// doubles: every A/B fragment load is bank-conflict free), D^{-1} of the 4 blocks
// and two 8x8 scratch tiles (pitch 12).  Only the lower triangles are read from
// HBM (one contiguous run per column, cp.async) and only tril(Sigma_bar) is
// written back.  n < 32 is embedded as blockdiag(L, I), (Abar, 0): exact.
#pragma once
#include "common.cuh"
#include "gemm.cuh"  // dmma884

namespace cd {

constexpr int D32_P = 36;    // column pitch of the 32 x 32 tiles
constexpr int D32_TP = 12;   // column pitch of 8 x 8 scratch tiles
constexpr int D32_WPB = 2;   // warps (matrices) per CTA
constexpr int D32_PER_WARP = 2 * 32 * D32_P + 4 * 8 * D32_TP + 2 * 8 * D32_TP + 32;  // doubles

inline size_t dmma32_smem() { return size_t(D32_WPB) * D32_PER_WARP * sizeof(double); }

template <int NBLK>
__global__ void __launch_bounds__(D32_WPB * 32)
    k_rev_dmma32(int n, int64_t batch, Opnd Ld, Opnd Ad, int out_mode, int* __restrict__ info) {
  constexpr int NP = 8 * NBLK;  // padded size
  constexpr int P = D32_P, TP = D32_TP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* sL = reinterpret_cast<double*>(smem_raw) + w * D32_PER_WARP;
  double* sA = sL + 32 * P;
  double* sDi = sA + 32 * P;      // 4 blocks x (8 x TP)
  double* sX = sDi + 4 * 8 * TP;  // scratch 8 x 8
  double* sS = sX + 8 * TP;       // S = Dbar + Dbar^T of the current block
  double* sRd = sS + 8 * TP;      // 1 / L_jj
  const int g = lane >> 2, t = lane & 3;
  // this lane's share of the packed lower triangle (column-major order): element
  // e = lane + 32k -> (row i, column m), packed as i | m << 8; -1 when e >= n(n+1)/2
  const int tri = n * (n + 1) / 2;
  int ent[17];
  {
    int m = 0, cs = 0;  // start of column m in the packed order
#pragma unroll
    for (int k = 0; k < 17; ++k) {
      const int e = lane + 32 * k;
      while (m < n && e >= cs + (n - m)) {
        cs += n - m;
        ++m;
      }
      ent[k] = (e < tri) ? ((m + (e - cs)) | (m << 8)) : -1;
    }
  }

  for (int64_t b = int64_t(blockIdx.x) * D32_WPB + w; b < batch; b += int64_t(gridDim.x) * D32_WPB) {
  const double* L = optr<double>(Ld, b);
  double* A = optr_w<double>(Ad, b);

  // ---- stage lower triangles (coalesced: consecutive lanes, consecutive rows)
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 17; ++k) {
    if (ent[k] >= 0) {
      const int i = ent[k] & 255, m = ent[k] >> 8;
      cp_async_zfill<8>(sL + m * P + i, L + i + m * Ld.ld, true);
      cp_async_zfill<8>(sA + m * P + i, A + i + m * Ad.ld, true);
    }
  }
  if (n < NP) {  // pad to blockdiag(L, I) / (A, 0)
    for (int m = 0; m < NP; ++m) {
      if (lane < NP && lane >= m && (lane >= n || m >= n)) {
        sL[m * P + lane] = (lane == m) ? 1.0 : 0.0;
        sA[m * P + lane] = 0.0;
      }
    }
  }
  cp_async_wait_all();
  // zero the upper triangles of the diagonal 8x8 tiles (the symbolic step reads full tiles)
  for (int e = lane; e < NBLK * 64; e += 32) {
    const int blk = e >> 6, r = e & 7, c = (e >> 3) & 7;
    if (r < c) {
      sL[(8 * blk + c) * P + 8 * blk + r] = 0.0;
      sA[(8 * blk + c) * P + 8 * blk + r] = 0.0;
    }
  }
  __syncwarp();
  {
    const bool bad = lane < n && bad_pivot(sL[lane * P + lane]);
    const unsigned msk = __ballot_sync(0xffffffffu, bad);
    if (info && lane == 0) info[b] = msk ? __ffs(msk) : 0;
    if (lane < NP) sRd[lane] = 1.0 / sL[lane * P + lane];
  }
  __syncwarp();

  // ---- D^{-1} of every diagonal block: lane -> (block, column c), forward substitution
  {
    const int blk = lane >> 3, c = lane & 7, j0 = 8 * blk;
    if (blk < NBLK) {
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
            if (q >= c) s += sL[(j0 + q) * P + j0 + r] * x[q];
          x[r] = -s * sRd[j0 + r];
        }
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) sDi[blk * 8 * TP + c * TP + r] = x[r];
    }
  }
  __syncwarp();

#pragma unroll
  for (int J = NBLK - 1; J >= 0; --J) {
    const int j = 8 * J;
    constexpr int dummy = 0;
    (void)dummy;
    const int PT = NBLK - 1 - J;  // 8-row tiles below the block
    const int QT = J;             // 8-col tiles left of the block
    const double* Di = sDi + J * 8 * TP;

    // s1: Cbar <- Cbar D^{-1}   (in place, tile by tile)
#pragma unroll
    for (int rt = 0; rt < 3; ++rt) {
      if (rt < PT) {
        const int r0 = j + 8 + 8 * rt;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)
          dmma884(c0, c1, sA[(j + 4 * kk + t) * P + r0 + g], Di[g * TP + 4 * kk + t]);
        __syncwarp();
        sA[(j + 2 * t) * P + r0 + g] = c0;
        sA[(j + 2 * t + 1) * P + r0 + g] = c1;
      }
    }
    __syncwarp();

    // s2: Bbar <- Bbar - Cbar R ;  s3: Dbar <- Dbar - tril(Cbar^T C)
#pragma unroll
    for (int rt = 0; rt < 3; ++rt) {
      if (rt < PT) {
        const int r0 = j + 8 + 8 * rt;
#pragma unroll
        for (int ct = 0; ct < 3; ++ct) {
          if (ct < QT) {
            const int cc = 8 * ct;
            double c0 = sA[(cc + 2 * t) * P + r0 + g], c1 = sA[(cc + 2 * t + 1) * P + r0 + g];
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
              dmma884(c0, c1, sA[(j + 4 * kk + t) * P + r0 + g], -sL[(cc + g) * P + j + 4 * kk + t]);
            sA[(cc + 2 * t) * P + r0 + g] = c0;
            sA[(cc + 2 * t + 1) * P + r0 + g] = c1;
          }
        }
      }
    }
    if (PT > 0) {
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int rt = 0; rt < 3; ++rt) {
        if (rt < PT) {
          const int r0 = j + 8 + 8 * rt;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
            dmma884(c0, c1, sA[(j + g) * P + r0 + 4 * kk + t], sL[(j + g) * P + r0 + 4 * kk + t]);
        }
      }
      // Dbar(g, 2t+e) -= acc for the lower triangle
      if (g >= 2 * t) sA[(j + 2 * t) * P + j + g] -= c0;
      if (g >= 2 * t + 1) sA[(j + 2 * t + 1) * P + j + g] -= c1;
    }
    __syncwarp();

    // s4: diagonal block by Eq. 10:  Y = D^{-T}(P + P^T)D^{-1},  P = Phi(D^T Dbar)
    {
      double p0 = 0.0, p1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk)
        dmma884(p0, p1, sL[(j + g) * P + j + 4 * kk + t], sA[(j + g) * P + j + 4 * kk + t]);
      // Phi
      const int c0i = 2 * t, c1i = 2 * t + 1;
      p0 = (g > c0i) ? p0 : (g == c0i ? 0.5 * p0 : 0.0);
      p1 = (g > c1i) ? p1 : (g == c1i ? 0.5 * p1 : 0.0);
      sX[c0i * TP + g] = p0;
      sX[c1i * TP + g] = p1;
      __syncwarp();
      const double x0 = p0 + sX[g * TP + c0i];  // X = P + P^T
      const double x1 = p1 + sX[g * TP + c1i];
      __syncwarp();
      sX[c0i * TP + g] = x0;
      sX[c1i * TP + g] = x1;
      __syncwarp();
      double z0 = 0.0, z1 = 0.0;  // Z = X D^{-1}
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(z0, z1, sX[(4 * kk + t) * TP + g], Di[g * TP + 4 * kk + t]);
      __syncwarp();
      sX[c0i * TP + g] = z0;
      sX[c1i * TP + g] = z1;
      __syncwarp();
      double y0 = 0.0, y1 = 0.0;  // Y = D^{-T} Z
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) dmma884(y0, y1, Di[g * TP + 4 * kk + t], sX[g * TP + 4 * kk + t]);
      // S = Y (full);  tril(Dbar) = Phi(Y)
      sS[c0i * TP + g] = y0;
      sS[c1i * TP + g] = y1;
      if (g >= c0i) sA[(j + c0i) * P + j + g] = (g == c0i) ? 0.5 * y0 : y0;
      if (g >= c1i) sA[(j + c1i) * P + j + g] = (g == c1i) ? 0.5 * y1 : y1;
    }
    __syncwarp();

    // s5: Rbar <- Rbar - Cbar^T B - S R
#pragma unroll
    for (int ct = 0; ct < 3; ++ct) {
      if (ct < QT) {
        const int cc = 8 * ct;
        double c0 = sA[(cc + 2 * t) * P + j + g], c1 = sA[(cc + 2 * t + 1) * P + j + g];
#pragma unroll
        for (int rt = 0; rt < 3; ++rt) {
          if (rt < PT) {
            const int r0 = j + 8 + 8 * rt;
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
              dmma884(c0, c1, sA[(j + g) * P + r0 + 4 * kk + t], -sL[(cc + g) * P + r0 + 4 * kk + t]);
          }
        }
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)
          dmma884(c0, c1, sS[(4 * kk + t) * TP + g], -sL[(cc + g) * P + j + 4 * kk + t]);
        sA[(cc + 2 * t) * P + j + g] = c0;
        sA[(cc + 2 * t + 1) * P + j + g] = c1;
      }
    }
    __syncwarp();
  }

  // ---- write back tril(Sigma_bar) (and the requested mirror)
#pragma unroll
  for (int k = 0; k < 17; ++k) {
    if (ent[k] >= 0) {
      const int i = ent[k] & 255, m = ent[k] >> 8;
      double v = sA[m * P + i];
      if (out_mode == 2 && i != m) v *= 0.5;
      A[i + m * Ad.ld] = v;
    }
  }
  if (out_mode != 0) {
    for (int i = 1; i < n; ++i) {
      if (lane < i) {
        double v = sA[lane * P + i];
        if (out_mode == 2) v *= 0.5;
        A[lane + i * Ad.ld] = v;
      }
    }
  }
  }  // matrices of this warp
}

}  // namespace cd
