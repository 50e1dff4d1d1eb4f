// sweep_bulk32.cuh -- batched fp64 reverse mode for n = 8, 16, 24, 32 (config 3: 65536 x
// N=32): the register-resident N_b = 8 blocked sweep of sweep_reg32.cuh (r32_core, same
// arithmetic: PAPER.md:689-701 with the 8x8 diagonal blocks by Eq. 10), fed by the TMA
// engine instead of per-lane global loads.
//
// Why: per-lane 8-byte fragment loads touch 4-8 cache lines per warp instruction, so the
// L1/TEX pipeline (not HBM) saturated first (ncu: L1 83 %, DRAM 45 % for k_rev_reg32),
// and the warp-shuffle layout changes cost ~16 instructions each.  Here
//   * the lower part of each column, rows (c & ~1) .. n-1, is copied HBM -> shared memory
//     by 16-byte cp.async (a half-warp per column: coalesced, no registers; per-lane
//     cp.async.bulk was tried and serialised into a 32-iteration issue loop per copy);
//     the column placement (base offsets b(c) = 4((c >> 1) & 3) + 8(c & 1) mod 16
//     doubles) makes both fragment patterns bank-conflict free;
//   * the two K=4 halves of every 8x8x8 tile product take k = 2t + kk (kk = 0, 1) instead
//     of 4kk + t, so a lane's A operand is exactly its accumulator pair (no layout change
//     for A operands at all) and a B operand is a row pair -- one 16-byte load;
//   * L's buffer is refilled with the next matrix as soon as its fragments are in
//     registers, Abar has two buffers: the next matrix streams in during the compute;
//   * the column bases come from constant memory (compile-time indices fold into the copy
//     addresses), the columns are packed with minimal padding (B32Layout: 580 doubles per
//     buffer instead of 756) and the diagonal-block inverses stay in registers after one
//     in-place pass through the scratch tiles: 45 % fewer shared-memory loads per matrix
//     (0.228 -> 0.206 ms for 65536 x N=32 on one box).  Four CTAs per SM (55.7 KB of shared
//     memory each now fits) need <= 128 registers and measured slower than three at 166;
//   * the remaining layout changes (transposes) go through an 8x8 shared-memory scratch
//     tile of pitch 10 (one 16-byte store + two loads, conflict free) instead of shuffles;
//   * results are stored straight from the accumulator layout (each warp store covers 4
//     columns x 64 contiguous bytes), lower triangle only; the one row above the diagonal
//     that an odd column's copy fetched is never used and never written.
#pragma once
#include "common.cuh"
#include "sweep_reg32.cuh"

namespace cd {

// Column placement: column c's lower rows (c & ~1) .. N-1 live at buf[base[c] + r]; base[c] = want(c)
// (mod 16 doubles) = 4((c >> 1) & 3) + 8(c & 1) makes both fragment patterns bank-conflict free.
// The columns are packed greedily (at each step the unplaced column that needs the least padding
// at the current end, lowest index first): 580 doubles per buffer for N = 32 against 756 when
// placed in index order -- the difference is what lets four CTAs share an SM.
template <int N>
struct B32Layout {
  int base[N];
  int total;  // doubles per operand buffer (multiple of 2)
  __host__ __device__ constexpr B32Layout() : base(), total(0) {
    bool used[N] = {};
    int cur = 0;
    for (int it = 0; it < N; ++it) {
      int bc = 0, bp = 99;
      for (int c = 0; c < N; ++c) {
        if (used[c]) continue;
        const int lo = c & ~1, want = (4 * ((c >> 1) & 3) + 8 * (c & 1)) % 16;
        const int pad = (((want + lo - cur) % 16) + 16) % 16;
        if (pad < bp) bp = pad, bc = c;
      }
      used[bc] = true;
      base[bc] = cur + bp - (bc & ~1);
      cur += bp + N - (bc & ~1);
    }
    total = (cur + 1) & ~1;
  }
};

// 8x8 scratch tile (row-major, pitch SC_P = 10: conflict free for both accesses) for the
// transposes: put the C layout M(g, 2t + e), read the B layout M(2t + kk, g).
constexpr int SC_P = 10, SC_TILE = 8 * SC_P + 4;  // tile stride 84 = 4 (mod 16): the four
                                                  // diagonal blocks read in parallel hit different banks

// the layouts, in constant memory (compile-time indices fold to constant-bank operands; the
// per-lane bases are read once per kernel)
__constant__ B32Layout<8> c_b32_8 = B32Layout<8>();
__constant__ B32Layout<16> c_b32_16 = B32Layout<16>();
__constant__ B32Layout<24> c_b32_24 = B32Layout<24>();
__constant__ B32Layout<32> c_b32_32 = B32Layout<32>();
template <int N>
__device__ __forceinline__ const B32Layout<N>& b32_lay() {
  if constexpr (N == 8) return c_b32_8;
  else if constexpr (N == 16) return c_b32_16;
  else if constexpr (N == 24) return c_b32_24;
  else return c_b32_32;
}

template <int NBLK>
__host__ __device__ constexpr int b32_total() {  // doubles per operand buffer (>= the NBLK scratch tiles)
  return B32Layout<8 * NBLK>().total > NBLK * SC_TILE ? B32Layout<8 * NBLK>().total : NBLK * SC_TILE;
}
template <int NBLK>
__host__ __device__ constexpr int b32_warp_doubles() {
  return 3 * b32_total<NBLK>();  // L buffer, two Abar buffers (the free one doubles as scratch)
}

constexpr int B32_WPB = 4;  // warps (one matrix each) per CTA
template <int NBLK>
inline size_t b32_smem() {
  return size_t(B32_WPB) * b32_warp_doubles<NBLK>() * sizeof(double);
}

__device__ __forceinline__ void sc_put(double* S, int g, int t, double c0, double c1) {
  *reinterpret_cast<double2*>(S + g * SC_P + 2 * t) = make_double2(c0, c1);
}
__device__ __forceinline__ void sc_getT(const double* S, int g, int t, double& b0, double& b1) {
  b0 = S[(2 * t) * SC_P + g];
  b1 = S[(2 * t + 1) * SC_P + g];
}

template <int NBLK, int MINB = 3>
__global__ void __launch_bounds__(B32_WPB * 32, MINB)
    k_rev_bulk32(int64_t batch, Opnd Ld, Opnd Ad, int* __restrict__ info) {
  constexpr int N = 8 * NBLK, NT = NBLK * (NBLK + 1) / 2;
  constexpr int TOT = b32_total<NBLK>();
  constexpr int WD = b32_warp_doubles<NBLK>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  double* ws = reinterpret_cast<double*>(smem_raw) + w * WD;
  static_assert(TOT >= NBLK * SC_TILE, "Abar buffer too small for the scratch tiles");
  double* sLb = ws;                                        // L buffer
  auto sAb = [&](int k) { return ws + (1 + k) * TOT; };  // Abar buffers
  // column bases (constant memory; a static shared table's 1 KB allocation would cost the fourth CTA per SM)
  const B32Layout<N>& lay = b32_lay<N>();
  auto TI = [](int bi, int bj) { return bj * NBLK - (bj * (bj - 1)) / 2 + (bi - bj); };

  // per-lane column bases: B layout (column 8bj + g), C layout (columns 8bj + 2t + e)
  int bT[NBLK], bC[NBLK][2];
#pragma unroll
  for (int bj = 0; bj < NBLK; ++bj) {
    bT[bj] = lay.base[8 * bj + g];
    bC[bj][0] = lay.base[8 * bj + 2 * t];
    bC[bj][1] = lay.base[8 * bj + 2 * t + 1];
  }

  // operand copies: 16-byte cp.async of the lower row pairs (r, r+1), r >= (c & ~1), a
  // half-warp per column (coalesced 256-byte column segments, no register staging)
  auto copy_in = [&](double* dstbuf, const Opnd& O, int64_t b) {
    const double* src = optr<double>(O, b);
#pragma unroll
    for (int c0 = 0; c0 < N; c0 += 2) {
      const int c = c0 + (lane >> 4), r = 2 * (lane & 15);
      const int bc = (lane >> 4) ? lay.base[c0 + 1 < N ? c0 + 1 : c0] : lay.base[c0];  // compile-time pair
      if (r < N && r >= (c & ~1)) {
        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dstbuf + bc + r));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src + r + int64_t(c) * O.ld) : "memory");
      }
    }
  };

  // L: one buffer, refilled with the next matrix as soon as this one's fragments are in
  // registers; Abar: two buffers, the next matrix's copy issued before waiting on this one's
  const int64_t stride = int64_t(gridDim.x) * B32_WPB;
  int64_t b = int64_t(blockIdx.x) * B32_WPB + w;
  if (b < batch) {
    copy_in(sAb(0), Ad, b);
    cp_async_commit();
    copy_in(sLb, Ld, b);
    cp_async_commit();
  }
  for (int it = 0; b < batch; b += stride, ++it) {
    const int k = it & 1;
    const bool more = b + stride < batch;
    if (more) {  // buffer k^1's last use ended with the previous matrix
      copy_in(sAb(k ^ 1), Ad, b + stride);
      cp_async_commit();
      cp_async_wait<1>();  // all but the group just issued
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    double* sA = sAb(k);
    // Lt: B layout L(8bi + 2t + kk, 8bj + g) (one 16-byte load);  Ac: C layout Abar(8bi + g, 8bj + 2t + e)
    double Lt[NT][2], Ac[NT][2];
#pragma unroll
    for (int bj = 0; bj < NBLK; ++bj)
#pragma unroll
      for (int bi = bj; bi < NBLK; ++bi) {
        const int ti = TI(bi, bj);
        const double2 v = *reinterpret_cast<const double2*>(sLb + bT[bj] + 8 * bi + 2 * t);
        const int r = 8 * bi + 2 * t, c = 8 * bj + g;
        Lt[ti][0] = (bi > bj || r >= c) ? v.x : 0.0;
        Lt[ti][1] = (bi > bj || r + 1 >= c) ? v.y : 0.0;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int ra = 8 * bi + g, ca = 8 * bj + 2 * t + e;
          Ac[ti][e] = (bi > bj || ra >= ca) ? sA[bC[bj][e] + ra] : 0.0;
        }
      }
    __syncwarp();
    if (more) {  // L's buffer is free: the next L streams in during the compute
      copy_in(sLb, Ld, b + stride);
      cp_async_commit();
    }
    double* sD = sA;  // Abar buffer k is free now: NBLK scratch tiles (8 x 8, pitch SC_P)
    // scratch: the diagonal tiles of L, 8 x 8 column-major with pitch SC_P
#pragma unroll
    for (int J = 0; J < NBLK; ++J)  // D(2t + kk, g) -> column g, rows 2t, 2t+1
      *reinterpret_cast<double2*>(sD + J * SC_TILE + g * SC_P + 2 * t) = make_double2(Lt[TI(J, J)][0], Lt[TI(J, J)][1]);
    __syncwarp();
    // ---- diagonal-block inverses (lane = (block, column)) and info; each inverse overwrites its
    //      diagonal tile, then every lane keeps its B-layout fragments Dinv(2t + kk, g) in registers
    double dinv[NBLK][2];
    {
      const int blk = lane >> 3, c = lane & 7;
      const int dblk = blk < NBLK ? blk : 0;
      double* D = sD + dblk * SC_TILE;  // D(r, q) = D[q * SC_P + r]
      const bool bad = blk < NBLK && bad_pivot(D[c * SC_P + c]);
      const double rdc = 1.0 / D[c * SC_P + c];
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
            if (q >= c) s -= D[q * SC_P + r] * x[q];
          x[r] = s * rdr;
        }
      }
      __syncwarp();  // every lane's reads of D done before the in-place store
      if (blk < NBLK) {
#pragma unroll
        for (int r = 0; r < 8; r += 2)  // Dinv(r, c), column-major, pitch SC_P
          *reinterpret_cast<double2*>(D + c * SC_P + r) = make_double2(x[r], x[r + 1]);
      }
      const unsigned msk = __ballot_sync(0xffffffffu, bad);
      if (info && lane == 0) info[b] = msk ? __ffs(msk) : 0;
    }
    __syncwarp();
#pragma unroll
    for (int J = 0; J < NBLK; ++J) {
      const double2 dv = *reinterpret_cast<const double2*>(sD + J * SC_TILE + g * SC_P + 2 * t);
      dinv[J][0] = dv.x;
      dinv[J][1] = dv.y;
    }
    __syncwarp();  // the scratch tiles are reused below
    double* S = sD;  // NBLK scratch tiles (the diagonal tiles of L are dead now)

#pragma unroll
    for (int J = NBLK - 1; J >= 0; --J) {
      const int PT = NBLK - 1 - J, QT = J;
      // Dinv in B layout Dinv(2t + kk, g); also the A operand of D^{-T}
      const double di0 = dinv[J][0], di1 = dinv[J][1];
      double cT[3][2];
      // s1: Cbar <- Cbar D^{-1}
      if (PT > 0) {
#pragma unroll
        for (int rt = 0; rt < 3; ++rt)
          if (rt < PT) {
            double* C = Ac[TI(J + 1 + rt, J)];
            double x0 = 0.0, x1 = 0.0;
            dmma884(x0, x1, C[0], di0);
            dmma884(x0, x1, C[1], di1);
            C[0] = x0;
            C[1] = x1;
            sc_put(S + rt * SC_TILE, g, t, x0, x1);
          }
        __syncwarp();
#pragma unroll
        for (int rt = 0; rt < 3; ++rt)
          if (rt < PT) sc_getT(S + rt * SC_TILE, g, t, cT[rt][0], cT[rt][1]);
      }
      // s2: Bbar <- Bbar - Cbar R
#pragma unroll
      for (int rt = 0; rt < 3; ++rt)
#pragma unroll
        for (int ct = 0; ct < 3; ++ct)
          if (rt < PT && ct < QT) {
            double* B = Ac[TI(J + 1 + rt, ct)];
            const double* C = Ac[TI(J + 1 + rt, J)];
            const double* R = Lt[TI(J, ct)];
            dmma884(B[0], B[1], C[0], -R[0]);
            dmma884(B[0], B[1], C[1], -R[1]);
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
      // s4: Dbar <- Phi(D^{-T} X D^{-1}), X = P + P^T, P = Phi(M), M = D^T Dbar;  S = D^{-T} X D^{-1}
      //     (Eq. 10).  One transpose (Dbar's B layout) serves both M = D^T Dbar and
      //     M^T = Dbar^T D, so X = P + P^T is formed in the C layout without another; X is
      //     symmetric, so its B layout equals its C layout and W = D^{-T} X, Y = W D^{-1}
      //     need no layout change either.
      double s0, s1;
      {
        double* T0 = S + (NBLK - 1) * SC_TILE;  // s1 uses at most tiles 0 .. NBLK-2
        sc_put(T0, g, t, Dbar[0], Dbar[1]);
        __syncwarp();
        double b0, b1;
        sc_getT(T0, g, t, b0, b1);  // Dbar(2t + kk, g)
        const double* D = Lt[TI(J, J)];
        double m0 = 0.0, m1 = 0.0, n0 = 0.0, n1 = 0.0;
        dmma884(m0, m1, D[0], b0);  // M = D^T Dbar
        dmma884(m0, m1, D[1], b1);
        dmma884(n0, n1, b0, D[0]);  // M^T = Dbar^T D
        dmma884(n0, n1, b1, D[1]);
        const int c0 = 2 * t, c1 = 2 * t + 1;
        const double x0 = g >= c0 ? m0 : n0, x1 = g >= c1 ? m1 : n1;  // X = Phi(M) + Phi(M)^T
        double w0 = 0.0, w1 = 0.0;  // W = D^{-T} X
        dmma884(w0, w1, di0, x0);
        dmma884(w0, w1, di1, x1);
        double y0 = 0.0, y1 = 0.0;  // Y = W D^{-1}
        dmma884(y0, y1, w0, di0);
        dmma884(y0, y1, w1, di1);
        s0 = y0;  // S = Y in A (= C) layout, for s5
        s1 = y1;
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
      __syncwarp();  // scratch reads of this step done before the next step's stores
    }

    // ---- tril(Sigma_bar) straight from the C-layout registers: per tile two warp stores,
    //      each 4 columns x 64 contiguous bytes; the upper triangle is never written
    {
      double* Ag = optr_w<double>(Ad, b);
#pragma unroll
      for (int bj = 0; bj < NBLK; ++bj)
#pragma unroll
        for (int bi = bj; bi < NBLK; ++bi)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = 8 * bi + g, c = 8 * bj + 2 * t + e;
            if (bi > bj || r >= c) Ag[r + int64_t(c) * Ad.ld] = Ac[TI(bi, bj)][e];
          }
    }
    __syncwarp();
  }
}

}  // namespace cd
