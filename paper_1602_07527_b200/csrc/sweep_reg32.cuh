// sweep_reg32.cuh -- batched fp64 reverse mode for n <= 32, register-resident:
// one WARP per matrix, the blocked reverse sweep of PAPER.md:689-701 with N_b = 8 on
// DMMA tiles (mma.sync.m8n8k4.f64) and the 8x8 diagonal blocks by Eq. 10
// (the paper's own choice for diagonal blocks) --
// the same tile arithmetic as sweep_dmma_cta.cuh, but with both matrices held in
// REGISTERS in the fragment layouts the tensor-core instructions consume:
//
//   lane (g, t) = (lane >> 2, lane & 3) holds, for every lower 8x8 tile (bi, bj):
//     L    in "T-pattern":  L(8bi + 4kk + t, 8bj + g),   kk = 0, 1   (the B operand /
//                            transposed-A operand of every update in the sweep)
//     Abar in "C-pattern":  Abar(8bi + g, 8bj + 2t + e), e = 0, 1    (the accumulator)
//
// so every update is DMMA on registers; the few operands needed in another layout are
// rebuilt with warp shuffles.  Loads go straight from HBM into these layouts (each warp
// load touches whole 32-byte sectors of the lower triangle only), results go straight
// back; shared memory holds only the four 8x8 diagonal blocks of L and their inverses.
// With no large shared-memory footprint, occupancy is set by registers, which keeps
// enough matrices in flight per SM to stream HBM.  n < 32 is embedded as
// blockdiag(L, I), (Abar, 0): exact.
#pragma once
#include "common.cuh"
#include "gemm.cuh"  // dmma884

namespace cd {

constexpr int R32_WPB = 4;                  // warps (independent matrices) per CTA
constexpr int R32_SMEM_PER_WARP = 2 * 4 * 64;  // doubles: diagonal L tiles + their inverses

inline size_t reg32_smem() { return size_t(R32_WPB) * R32_SMEM_PER_WARP * sizeof(double); }

// C-pattern (g, 2t+e) -> A-pattern (g, 4kk+t), kk = 0, 1
__device__ __forceinline__ void r32_to_A(double c0, double c1, int g, int t, double& a0, double& a1) {
  const int s0 = g * 4 + (t >> 1), s1 = g * 4 + 2 + (t >> 1);
  const double x0 = __shfl_sync(0xffffffffu, c0, s0), y0 = __shfl_sync(0xffffffffu, c1, s0);
  const double x1 = __shfl_sync(0xffffffffu, c0, s1), y1 = __shfl_sync(0xffffffffu, c1, s1);
  a0 = (t & 1) ? y0 : x0;
  a1 = (t & 1) ? y1 : x1;
}
// C-pattern (g, 2t+e) -> T-pattern (4kk+t, g), kk = 0, 1
__device__ __forceinline__ void r32_to_T(double c0, double c1, int g, int t, double& b0, double& b1) {
  const int s0 = t * 4 + (g >> 1), s1 = (4 + t) * 4 + (g >> 1);
  const double x0 = __shfl_sync(0xffffffffu, c0, s0), y0 = __shfl_sync(0xffffffffu, c1, s0);
  const double x1 = __shfl_sync(0xffffffffu, c0, s1), y1 = __shfl_sync(0xffffffffu, c1, s1);
  b0 = (g & 1) ? y0 : x0;
  b1 = (g & 1) ? y1 : x1;
}
// C-pattern of M -> C-pattern of M^T:  (g, c) of M^T = M(c, g), c = 2t + e
__device__ __forceinline__ void r32_transpose(double c0, double c1, int g, int t, double& d0, double& d1) {
  const int s0 = (2 * t) * 4 + (g >> 1), s1 = (2 * t + 1) * 4 + (g >> 1);
  const double x0 = __shfl_sync(0xffffffffu, c0, s0), y0 = __shfl_sync(0xffffffffu, c1, s0);
  const double x1 = __shfl_sync(0xffffffffu, c0, s1), y1 = __shfl_sync(0xffffffffu, c1, s1);
  d0 = (g & 1) ? y0 : x0;
  d1 = (g & 1) ? y1 : x1;
}

// The register-resident sweep proper (shared by the kernels that stage the operands
// differently): diagonal-block inverses (+ info), then the N_b = 8 blocked reverse sweep
// on the fragments.  dat(blk, q, r) = L(8 blk + r, 8 blk + q) (diagonal tile, column q, row r).
template <int NBLK, class DAt>
__device__ __forceinline__ void r32_core(double (&Lt)[NBLK * (NBLK + 1) / 2][2], double (&Ac)[NBLK * (NBLK + 1) / 2][2],
                                         DAt dat, double* sDi, int n, int* __restrict__ info, int64_t b, int lane) {
  const int g = lane >> 2, t = lane & 3;
  auto TI = [](int bi, int bj) { return bj * NBLK - (bj * (bj - 1)) / 2 + (bi - bj); };
    {
      const int blk = lane >> 3, c = lane & 7;
      bool bad = false;
      {  // all lanes take part (shuffles); lanes of blocks >= NBLK work on tile 0 and discard
        const int dblk = blk < NBLK ? blk : 0;
        bad = blk < NBLK && (8 * blk + c < n) && bad_pivot(dat(dblk, c, c));
        // 1/D(r,r), r = 0..7: each lane computes its own column's, the rest by shuffle
        const double rdc = 1.0 / dat(dblk, c, c);
        double x[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const double rdr = __shfl_sync(0xffffffffu, rdc, (lane & ~7) | r);
          if (r < c) {
            x[r] = 0.0;
          } else {
            double s = (r == c) ? 1.0 : 0.0;
#pragma unroll
            for (int q = 0; q < r; ++q)
              if (q >= c) s -= dat(dblk, q, r) * x[q];
            x[r] = s * rdr;
          }
        }
        if (blk < NBLK) {
#pragma unroll
          for (int r = 0; r < 8; ++r) sDi[blk * 64 + c * 8 + r] = x[r];  // Dinv(r, c), col-major
        }
      }
      const unsigned msk = __ballot_sync(0xffffffffu, bad);
      if (info && lane == 0) {
        int first = 0;
        if (msk) {
          // lane = blk*8 + c  ->  diagonal index 8*blk + c
          first = __ffs(msk);
        }
        info[b] = first;
      }
    }
    __syncwarp();

#pragma unroll
    for (int J = NBLK - 1; J >= 0; --J) {
      constexpr int dummy = 0;
      (void)dummy;
      const int PT = NBLK - 1 - J, QT = J;
      double di0 = sDi[J * 64 + g * 8 + t], di1 = sDi[J * 64 + g * 8 + 4 + t];  // Dinv(4kk+t, g)
      double cA[3][2], cT[3][2];
      // s1: Cbar <- Cbar D^{-1}
#pragma unroll
      for (int rt = 0; rt < 3; ++rt) {
        if (rt < PT) {
          double* C = Ac[TI(J + 1 + rt, J)];
          double a0, a1;
          r32_to_A(C[0], C[1], g, t, a0, a1);
          double x0 = 0.0, x1 = 0.0;
          dmma884(x0, x1, a0, di0);
          dmma884(x0, x1, a1, di1);
          C[0] = x0;
          C[1] = x1;
          r32_to_A(x0, x1, g, t, cA[rt][0], cA[rt][1]);
          r32_to_T(x0, x1, g, t, cT[rt][0], cT[rt][1]);
        }
      }
      // s2: Bbar <- Bbar - Cbar R
#pragma unroll
      for (int rt = 0; rt < 3; ++rt)
#pragma unroll
        for (int ct = 0; ct < 3; ++ct)
          if (rt < PT && ct < QT) {
            double* B = Ac[TI(J + 1 + rt, ct)];
            const double* R = Lt[TI(J, ct)];
            dmma884(B[0], B[1], cA[rt][0], -R[0]);
            dmma884(B[0], B[1], cA[rt][1], -R[1]);
          }
      // s3: Dbar <- Dbar - tril(Cbar^T C)
      double* Dbar = Ac[TI(J, J)];
      if (PT > 0) {
        double p0 = 0.0, p1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll
        for (int rt = 0; rt < 3; ++rt)
          if (rt < PT) {
            const double* Cl = Lt[TI(J + 1 + rt, J)];
            dmma884(p0, p1, cT[rt][0], Cl[0]);
            dmma884(q0, q1, cT[rt][1], Cl[1]);
          }
        if (g >= 2 * t) Dbar[0] -= p0 + q0;
        if (g >= 2 * t + 1) Dbar[1] -= p1 + q1;
      }
      // s4: Dbar <- Phi(D^{-T}(P + P^T)D^{-1}), P = Phi(D^T Dbar); S = D^{-T}(P+P^T)D^{-1}  (Eq. 10)
      double s0, s1;
      {
        double b0, b1;
        r32_to_T(Dbar[0], Dbar[1], g, t, b0, b1);
        const double* D = Lt[TI(J, J)];
        double p0 = 0.0, p1 = 0.0;
        dmma884(p0, p1, D[0], b0);  // D^T Dbar : A = D^T (T-pattern of D)
        dmma884(p0, p1, D[1], b1);
        const int c0 = 2 * t, c1 = 2 * t + 1;
        p0 = (g > c0) ? p0 : (g == c0 ? 0.5 * p0 : 0.0);
        p1 = (g > c1) ? p1 : (g == c1 ? 0.5 * p1 : 0.0);
        double pt0, pt1;
        r32_transpose(p0, p1, g, t, pt0, pt1);
        const double x0 = p0 + pt0, x1 = p1 + pt1;  // X = P + P^T
        double xa0, xa1;
        r32_to_A(x0, x1, g, t, xa0, xa1);
        double z0 = 0.0, z1 = 0.0;  // Z = X D^{-1}
        dmma884(z0, z1, xa0, di0);
        dmma884(z0, z1, xa1, di1);
        double zb0, zb1;
        r32_to_T(z0, z1, g, t, zb0, zb1);
        double y0 = 0.0, y1 = 0.0;  // Y = D^{-T} Z
        dmma884(y0, y1, di0, zb0);
        dmma884(y0, y1, di1, zb1);
        r32_to_A(y0, y1, g, t, s0, s1);  // S = Y, as the A operand of s5
        Dbar[0] = (g > c0) ? y0 : (g == c0 ? 0.5 * y0 : 0.0);
        Dbar[1] = (g > c1) ? y1 : (g == c1 ? 0.5 * y1 : 0.0);
      }
      // s5: Rbar <- Rbar - Cbar^T B - (Dbar + Dbar^T) R
#pragma unroll
      for (int ct = 0; ct < 3; ++ct)
        if (ct < QT) {
          double* Rb = Ac[TI(J, ct)];
          double e0 = 0.0, e1 = 0.0;
#pragma unroll
          for (int rt = 0; rt < 3; ++rt)
            if (rt < PT) {
              const double* Bl = Lt[TI(J + 1 + rt, ct)];
              dmma884(Rb[0], Rb[1], cT[rt][0], -Bl[0]);
              dmma884(e0, e1, cT[rt][1], -Bl[1]);
            }
          const double* R = Lt[TI(J, ct)];
          dmma884(Rb[0], Rb[1], s0, -R[0]);
          dmma884(e0, e1, s1, -R[1]);
          Rb[0] += e0;
          Rb[1] += e1;
        }
    }

}

template <int NBLK>
__global__ void __launch_bounds__(R32_WPB * 32, 3)
    k_rev_reg32(int n, int64_t batch, Opnd Ld, Opnd Ad, int out_mode, int* __restrict__ info) {
  constexpr int NT = NBLK * (NBLK + 1) / 2;  // lower tiles
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  double* sD = reinterpret_cast<double*>(smem_raw) + w * R32_SMEM_PER_WARP;  // 4 diag tiles of L, col-major 8x8
  double* sDi = sD + 4 * 64;                                                 // their inverses
  // tile index of (bi, bj), bi >= bj, column-major tile order
  auto TI = [](int bi, int bj) { return bj * NBLK - (bj * (bj - 1)) / 2 + (bi - bj); };

  for (int64_t b = int64_t(blockIdx.x) * R32_WPB + w; b < batch; b += int64_t(gridDim.x) * R32_WPB) {
    const double* Lg = optr<double>(Ld, b);
    double* Ag = optr_w<double>(Ad, b);
    double Lt[NT][2], Ac[NT][2];
    // ---- loads (lower triangles only; padding -> blockdiag(I) / 0)
    if (n == 8 * NBLK) {  // no padding: only the diagonal tiles are masked
#pragma unroll
      for (int bj = 0; bj < NBLK; ++bj)
#pragma unroll
        for (int bi = bj; bi < NBLK; ++bi) {
          const int ti = TI(bi, bj);
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int r = 8 * bi + 4 * kk + t, c = 8 * bj + g;
            Lt[ti][kk] = (bi > bj || r >= c) ? __ldg(Lg + r + int64_t(c) * Ld.ld) : 0.0;
          }
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = 8 * bi + g, c = 8 * bj + 2 * t + e;
            Ac[ti][e] = (bi > bj || r >= c) ? Ag[r + int64_t(c) * Ad.ld] : 0.0;
          }
        }
    } else {
#pragma unroll
      for (int bj = 0; bj < NBLK; ++bj)
#pragma unroll
        for (int bi = bj; bi < NBLK; ++bi) {
          const int ti = TI(bi, bj);
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int r = 8 * bi + 4 * kk + t, c = 8 * bj + g;
            double v = 0.0;
            if (r < n && c < n) {
              if (r >= c) v = Lg[r + int64_t(c) * Ld.ld];
            } else if (r == c) {
              v = 1.0;
            }
            Lt[ti][kk] = v;
          }
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = 8 * bi + g, c = 8 * bj + 2 * t + e;
            Ac[ti][e] = (r < n && c < n && r >= c) ? Ag[r + int64_t(c) * Ad.ld] : 0.0;
          }
        }
    }
    // ---- diagonal blocks of L -> smem (for their inverses), info
    __syncwarp();
#pragma unroll
    for (int J = 0; J < NBLK; ++J)
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) sD[J * 64 + g * 8 + 4 * kk + t] = Lt[TI(J, J)][kk];  // (row 4kk+t, col g)
    __syncwarp();
    r32_core<NBLK>(Lt, Ac, [&](int blk, int q, int r) { return sD[blk * 64 + q * 8 + r]; }, sDi, n, info, b, lane);
    // ---- store tril(Sigma_bar) (and the requested mirror)
    if (out_mode == 0 && n == 8 * NBLK) {
#pragma unroll
      for (int bj = 0; bj < NBLK; ++bj)
#pragma unroll
        for (int bi = bj; bi < NBLK; ++bi)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = 8 * bi + g, c = 8 * bj + 2 * t + e;
            if (bi > bj || r >= c) Ag[r + int64_t(c) * Ad.ld] = Ac[TI(bi, bj)][e];
          }
    } else {
#pragma unroll
      for (int bj = 0; bj < NBLK; ++bj)
#pragma unroll
        for (int bi = bj; bi < NBLK; ++bi)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = 8 * bi + g, c = 8 * bj + 2 * t + e;
            if (r < n && c < n && r >= c) {
              double v = Ac[TI(bi, bj)][e];
              if (out_mode == 2 && r != c) v *= 0.5;
              Ag[r + int64_t(c) * Ad.ld] = v;
              if (out_mode != 0 && r != c) Ag[c + int64_t(r) * Ad.ld] = v;
            }
          }
    }
  }
}

}  // namespace cd
