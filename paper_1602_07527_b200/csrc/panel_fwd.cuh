// panel_fwd.cuh -- the per-panel steps of the blocked FORWARD sweep as ONE cooperative
// kernel (fp64, DMMA), the forward counterpart of panel_rev.cuh.  For panel J = [j, k)
// (q = j columns to its left):
//
//   phase 0  the previous panel's  Cdot <- W D^{-T}   (W is left in place by
//            k_fwd_sk), 32 x 32 output tiles staged and copied back after a grid sync;
//   phase 1  Ddot <- Ddot - tril(Rdot R^T + R Rdot^T): one CTA per (128-wide
//            K chunk, lower 32 x 32 tile) computes a partial (both products);
//   phase 2  deterministic grid reduction of the partials into Ddot;
//   phase 3  the diagonal block by Eq. 8 (the paper names Eqs. 8/10 as
//            the natural diagonal-block updates):
//              Y = D^{-1} Ddot_sym,  F = Phi(Y D^{-T}),  Ldot_D = D F,
//            Ldot_D written over tril(Ddot) and as the clean dense copy Dc (upper zero)
//            that the next k_fwd_sk consumes (segment C Ddot^T).
// Grid syncs separate the phases.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "gemm.cuh"
#include "panel_rev.cuh"  // PR_* constants, cp_async8, pr_tile32

namespace cd {

struct PanelFwdParams {
  Opnd A, L;             // Adot and L (whole matrices)
  const double* Dinv;    // this panel's D^{-1} (w x w, ld dld; batch stride dstride)
  const double* Dinv_prev;  // the previous panel's (phase 0), or nullptr
  int64_t dstride;
  int dld;
  int n, j, w;
  int j_prev, k_prev, tiles_prev;  // phase 0: rows [k_prev, n) in ceil(.) 128-row tiles, cols [j_prev, j_prev+128)
  int kchunks;           // phase 1: q / 128
  int64_t batch;
  double* part;          // [batch * kchunks][128 * 128] (phase 1); phase 0 staging [units][32 * 32]
  double* Yws;           // dense 128 x 128 per batch entry
  double* Fws;           // dense 128 x 128 per batch entry
  double* Dc;            // dense, ld 132, batch stride 132 * 128
  // generalisations for the fused factorisation + forward sweep (chol_fwd_fused):
  Opnd T0;               // phase-0 target matrix (W <- W D^{-T} in place); the forward sweep: A
  int single;            // phase 1: one product R R^T (K = 128 per chunk) instead of both
  int skip3;             // skip phase 3 (Eq. 8)
  int dbg_skip;          // measurement only (CD_DEBUG_PANEL_SKIP): bit i skips phase i; results wrong
  int kslot_cap;         // phase 1 partial slots available per batch entry (balanced K split, batch 1)
  int split_max;         // phase 0: 128-row tiles cut into up to this many sub-tiles (1, 2, 4)
};

// acc (64 x 32 warp tiles of a 128 x 128 tile) += sum over K of A(m, kk) B(kk, c), K in
// chunks of 16 (3-stage cp.async pipeline); fa / fb return the source pointer or nullptr
// (zero).  skip(kc) (warp-uniform) drops a chunk for this warp.  Stage layout As[k][m],
// Bs[k][c], pitch 132 (conflict-free fragments).  Used when a phase has enough 128-wide
// units to fill the GPU (fewer operand re-reads than 32 x 32 tiles).
// RT < 8: only the first ROWS = 16 RT rows of A (the warp tiles shrink to ROWS / 2 x 32; acc rows
// i < RT are used)
template <int RT = 8, class FA, class FB, class SK>
__device__ __forceinline__ void pf_prod128(double* sm, int K, FA fa, FB fb, SK skip, double (&acc)[8][4][2]) {
  constexpr int P = 132, STG = 2 * 16 * P, ROWS = 16 * RT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3, g = lane >> 2, t = lane & 3;
  const int nkc = (K + 15) / 16;
  auto load = [&](int st, int kc) {
    double* as = sm + st * STG;
    double* bs = as + 16 * P;
    for (int e = tid; e < 16 * 128; e += PR_THREADS) {
      const int m = e & 127, kx = e >> 7;
      const int kk = kc * 16 + kx;
      const double* pa = (kk < K && m < ROWS) ? fa(m, kk) : nullptr;
      const double* pb = kk < K ? fb(kk, m) : nullptr;
      // no source -> a zero by a plain shared store (never a zero-size copy from a dummy address)
      if (pa) cp_async8(as + kx * P + m, pa, true);
      else if (m < ROWS) as[kx * P + m] = 0.0;
      if (pb) cp_async8(bs + kx * P + m, pb, true);
      else bs[kx * P + m] = 0.0;
    }
  };
  __syncthreads();  // previous users of the stage buffers are done
#pragma unroll 1
  for (int s = 0; s < 2; ++s) {
    if (s < nkc) load(s, s);
    cp_async_commit();
  }
#pragma unroll 1
  for (int kc = 0; kc < nkc; ++kc) {
    cp_async_wait<1>();
    __syncthreads();
    if (kc + 2 < nkc) load((kc + 2) % 3, kc + 2);
    cp_async_commit();
    if (!skip(kc)) {
      const double* as = sm + (kc % 3) * STG;
      const double* bs = as + 16 * P;
#pragma unroll
      for (int kq = 0; kq < 4; ++kq) {
        const int kx = kq * 4 + t;
        double a[RT], bb[4];
#pragma unroll
        for (int i = 0; i < RT; ++i) a[i] = as[kx * P + wm * (ROWS / 2) + i * 8 + g];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) bb[jj] = bs[kx * P + wn * 32 + jj * 8 + g];
#pragma unroll
        for (int i = 0; i < RT; ++i)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) dmma884(acc[i][jj][0], acc[i][jj][1], a[i], bb[jj]);
      }
    }
  }
  cp_async_wait_all();
}

// Phase 0 on sub-tiles of ROWS = 16 RT rows (RT = 8: whole 128-row tiles), s = 128 / ROWS per tile:
// Cdot_rows <- W_rows D_prev^{-T} in place (a CTA reads all 128 columns of its rows before writing)
template <int RT>
__device__ __forceinline__ void pf_phase0_units(const PanelFwdParams& p, double* sm, int64_t nunits, int s) {
  constexpr int ROWS = 16 * RT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3, g = lane >> 2, t = lane & 3;
  const int64_t nsub = int64_t(p.tiles_prev) * s;
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t b = u / nsub;
    const int st_ = int(u - b * nsub), tl = st_ / s, h = st_ - tl * s;
    const int r0 = p.k_prev + 128 * tl + ROWS * h;
    double* Wt = optr_w<double>(p.T0, b) + r0 + int64_t(p.j_prev) * p.T0.ld;
    const double* Di = p.Dinv_prev + b * p.dstride;
    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) acc[i][jj][0] = acc[i][jj][1] = 0.0;
    pf_prod128<RT>(
        sm, 128,
        [&](int m, int kk) -> const double* { return r0 + m < p.n ? Wt + m + int64_t(kk) * p.T0.ld : nullptr; },
        [&](int kk, int c) -> const double* { return c >= kk ? Di + c + int64_t(kk) * p.dld : nullptr; },
        [&](int kc) { return kc * 16 > wn * 32 + 31; },  // D^{-T}(kk, c) = 0 for kk > c
        acc);
    __syncthreads();  // every warp has read its W rows before any is overwritten
#pragma unroll
    for (int i = 0; i < RT; ++i)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = wm * (ROWS / 2) + i * 8 + g, c = wn * 32 + jj * 8 + 2 * t + e;
          if (r0 + r < p.n) Wt[r + int64_t(c) * p.T0.ld] = acc[i][jj][e];
        }
  }
}

__global__ void __launch_bounds__(PR_THREADS, 1) k_panel_fwd(const PanelFwdParams p) {
  extern __shared__ __align__(16) unsigned char smem_pf[];
  double* sm = reinterpret_cast<double*>(smem_pf);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int w = p.w;
  namespace cg = cooperative_groups;

  // ---------------- phase 0: previous panel  Cdot <- W D_prev^{-T} ----------------
  // whole 128-row tiles when there are enough of them; otherwise 64- / 32-row sub-tiles
  // (p.split_max), or 32 x 32 output tiles staged through global memory (p.split_max < 2 or
  // fewer than 16 tiles)
  const int64_t units0 = p.batch * p.tiles_prev;
  const int s0 = p.split_max >= 4 && units0 * 4 <= int64_t(gridDim.x)   ? 4
                 : p.split_max >= 2 && units0 * 2 <= int64_t(gridDim.x) ? 2
                                                                        : 1;
  // (below 16 tiles the 32 x 32 staged tiles win: a sub-tile loads all of D^{-T} for few rows --
  // N = 1024 forward 680 vs 722 us)
  const bool big0 = (s0 > 1 && units0 >= 16) || units0 >= int64_t(gridDim.x) / 2;
  const bool ph0 = p.Dinv_prev && !(p.dbg_skip & 1);
  if (ph0 && big0) {
    if (s0 == 4) pf_phase0_units<2>(p, sm, units0 * 4, 4);
    else if (s0 == 2) pf_phase0_units<4>(p, sm, units0 * 2, 2);
    else pf_phase0_units<8>(p, sm, units0, 1);
    __threadfence();
    cg::this_grid().sync();
  } else if (ph0) {
    const int64_t units = p.batch * p.tiles_prev * 16;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      const int64_t bt = u >> 4;
      const int64_t b = bt / p.tiles_prev;
      const int tl = int(bt - b * p.tiles_prev);
      const int ti = int(u & 15) >> 2, tj = int(u & 3);
      const int r0 = p.k_prev + 128 * tl + 32 * ti, c0 = 32 * tj;
      const double* Wt = optr<double>(p.T0, b) + r0 + int64_t(p.j_prev) * p.T0.ld;  // rows r0.., panel cols
      const double* Di = p.Dinv_prev + b * p.dstride;
      // write target: column-group tj of the same rows; the 4 column groups of a row group
      // read all of W's columns, so results go to the Yws-like staging slot first
      double* st = p.part + u * int64_t(32 * 32);
      pr_tile32kx(
          sm, 128, [&](int m, int kk) -> const double* { return r0 + m < p.n ? Wt + m + int64_t(kk) * p.T0.ld : nullptr; },
          [&](int kk, int n) -> const double* {
            const int cc = c0 + n;
            return cc >= kk ? Di + cc + int64_t(kk) * p.dld : nullptr;  // D^{-T}(kk, cc) = Dinv(cc, kk)
          },
          [&](int m, int n, double v) { __stcg(st + m + n * 32, v); }, [](int) { return true; }, [](int) { return true; });
    }
    __threadfence();
    cg::this_grid().sync();
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {  // copy the staged tiles back
      const int64_t bt = u >> 4;
      const int64_t b = bt / p.tiles_prev;
      const int tl = int(bt - b * p.tiles_prev);
      const int ti = int(u & 15) >> 2, tj = int(u & 3);
      const int r0 = p.k_prev + 128 * tl + 32 * ti, c0 = 32 * tj;
      double* Wt = optr_w<double>(p.T0, b) + r0 + int64_t(p.j_prev + c0) * p.T0.ld;
      const double* st = p.part + u * int64_t(32 * 32);
      for (int e = tid; e < 32 * 32; e += PR_THREADS) {
        const int m = e & 31, n = e >> 5;
        if (r0 + m < p.n) Wt[m + int64_t(n) * p.T0.ld] = __ldcg(st + e);
      }
    }
    __threadfence();
    cg::this_grid().sync();
  }

  // ---------------- phase 1: partials of Rdot R^T + R Rdot^T ----------------
  const int kch1 = (p.dbg_skip & 2) ? 0 : p.kchunks;
  // unit = (128-wide K chunk, lower 32 x 32 tile of the w x w block): K = 256 (both
  // products); with enough K chunks, one CTA per chunk computes the whole 128 x 128 block
  const bool big1 = p.batch * kch1 >= int64_t(gridDim.x) / 2;
  // single matrix with many K chunks: every CTA takes one balanced K range (a multiple of 16
  // columns) of the whole 128 x 128 block instead of one 128-wide chunk, so all SMs share the
  // work (kchunks < #SMs left the rest idle); its partial goes to slot blockIdx.x
  const int gk = min(int(gridDim.x), p.kslot_cap);
  const bool bal1 = big1 && p.batch == 1 && gk >= kch1;
  const int nslot1 = bal1 ? gk : kch1;  // phase 1 partial slots per batch entry (phase 2 sums them)
  if (bal1) {
    const int lane_ = threadIdx.x & 31, wm = warp >> 2, wn = warp & 3, g = lane_ >> 2, t = lane_ & 3;
    const int q16 = (128 * kch1) / 16;  // K in 16-column groups
    for (int u = blockIdx.x; u < gk; u += gridDim.x) {
      const int k_lo = 16 * int(int64_t(q16) * u / gk), k_hi = 16 * int(int64_t(q16) * (u + 1) / gk);
      const int kw = k_hi - k_lo;
      double acc[8][4][2];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[i][jj][0] = acc[i][jj][1] = 0.0;
      if (kw > 0) {
        const double* Ad = optr<double>(p.A, 0) + p.j + int64_t(k_lo) * p.A.ld;
        const double* Lr = optr<double>(p.L, 0) + p.j + int64_t(k_lo) * p.L.ld;
        pf_prod128(
            sm, p.single ? kw : 2 * kw,
            [&](int m, int kk) -> const double* {
              if (m >= w) return nullptr;
              return kk < kw ? Ad + m + int64_t(kk) * p.A.ld : Lr + m + int64_t(kk - kw) * p.L.ld;
            },
            [&](int kk, int c) -> const double* {
              if (c >= w) return nullptr;
              return kk < kw ? Lr + c + int64_t(kk) * p.L.ld : Ad + c + int64_t(kk - kw) * p.A.ld;
            },
            [&](int) { return wm * 64 + 63 < wn * 32; },  // warp tile entirely above the diagonal
            acc);
      }
      double* slot = p.part + int64_t(u) * (128 * 128);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = wm * 64 + i * 8 + g, c = wn * 32 + jj * 8 + 2 * t + e;
            if (r >= c) __stcg(slot + r + c * 128, acc[i][jj][e]);
          }
    }
  } else if (big1) {
    const int lane_ = threadIdx.x & 31, wm = warp >> 2, wn = warp & 3, g = lane_ >> 2, t = lane_ & 3;
    const int64_t units = p.batch * kch1;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      const int64_t b = u / kch1;
      const int kc0 = 128 * int(u - b * kch1);
      const double* Ad = optr<double>(p.A, b) + p.j + int64_t(kc0) * p.A.ld;
      const double* Lr = optr<double>(p.L, b) + p.j + int64_t(kc0) * p.L.ld;
      double acc[8][4][2];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[i][jj][0] = acc[i][jj][1] = 0.0;
      pf_prod128(
          sm, p.single ? 128 : 256,
          [&](int m, int kk) -> const double* {
            if (m >= w) return nullptr;
            return kk < 128 ? Ad + m + int64_t(kk) * p.A.ld : Lr + m + int64_t(kk - 128) * p.L.ld;
          },
          [&](int kk, int c) -> const double* {
            if (c >= w) return nullptr;
            return kk < 128 ? Lr + c + int64_t(kk) * p.L.ld : Ad + c + int64_t(kk - 128) * p.A.ld;
          },
          [&](int) { return wm * 64 + 63 < wn * 32; },  // warp tile entirely above the diagonal
          acc);
      double* slot = p.part + u * int64_t(128 * 128);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = wm * 64 + i * 8 + g, c = wn * 32 + jj * 8 + 2 * t + e;
            if (r >= c) __stcg(slot + r + c * 128, acc[i][jj][e]);
          }
    }
  } else {
    const int64_t units = p.batch * kch1 * 10;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      const int64_t bk = u / 10;
      const int lt = int(u - bk * 10);
      int ti = 0, tj = 0;  // lower tile lt -> (ti >= tj)
      {
        int r = lt;
        while (r > ti) r -= ++ti;
        tj = r;
      }
      const int64_t b = bk / kch1;
      const int kc0 = 128 * int(bk - b * kch1);
      const double* Ad = optr<double>(p.A, b) + p.j + int64_t(kc0) * p.A.ld;  // Rdot chunk, rows j..
      const double* Lr = optr<double>(p.L, b) + p.j + int64_t(kc0) * p.L.ld;  // R chunk
      const int a0 = 32 * ti, c0 = 32 * tj;
      double* slot = p.part + bk * int64_t(128 * 128);
      // kk < 128 -> Rdot(a, kk) R(c, kk); kk >= 128 -> R(a, kk') Rdot(c, kk')
      pr_tile32kx(
          sm, p.single ? 128 : 256,
          [&](int m, int kk) -> const double* {
            const int a = a0 + m;
            if (a >= w) return nullptr;
            return kk < 128 ? Ad + a + int64_t(kk) * p.A.ld : Lr + a + int64_t(kk - 128) * p.L.ld;
          },
          [&](int kk, int n) -> const double* {
            const int cc = c0 + n;
            if (cc >= w) return nullptr;
            return kk < 128 ? Lr + cc + int64_t(kk) * p.L.ld : Ad + cc + int64_t(kk - 128) * p.A.ld;
          },
          [&](int m, int n, double v) {
            const int a = a0 + m, cc = c0 + n;
            if (a >= cc) __stcg(slot + a + cc * 128, v);
          },
          [](int) { return true; }, [](int) { return true; });  // rows of Rdot / R (A) and of R / Rdot (B): contiguous along m / n
    }
  }
  __threadfence();
  cg::this_grid().sync();

  // ---------------- phase 2: Ddot -= sum of the partials (lower triangle) ----------------
  if (p.kchunks > 0 && !(p.dbg_skip & 4)) {
    const int64_t nwarps = int64_t(gridDim.x) * (PR_THREADS / 32);
    const int64_t gw = int64_t(blockIdx.x) * (PR_THREADS / 32) + warp;
    const int64_t ntri = int64_t(w) * (w + 1) / 2;
    const int64_t nel = ntri * p.batch;
    const int q = lane & 7;
    for (int64_t wb = gw * 4; wb < nel; wb += nwarps * 4) {
      const int64_t el = wb + (lane >> 3);
      const bool on = el < nel;
      int64_t b = 0;
      int a = 0, c = 0;
      if (on) {
        b = el / ntri;
        const int rem = int(el - b * ntri);
        const double tw = 2.0 * w + 1.0;
        c = int((tw - sqrt(tw * tw - 8.0 * rem)) * 0.5);
        c = max(0, min(c, w - 1));
        while (c > 0 && c * w - c * (c - 1) / 2 > rem) --c;
        while (c + 1 < w && (c + 1) * w - (c + 1) * c / 2 <= rem) ++c;
        a = c + (rem - (c * w - c * (c - 1) / 2));
      }
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      if (on) {
        const double* pb = p.part + b * nslot1 * int64_t(128 * 128) + a + c * 128;
        constexpr int64_t TS = 128 * 128;
        int tl = q;
        for (; tl + 24 < nslot1; tl += 32) {
          const double x0 = __ldcg(pb + tl * TS), x1 = __ldcg(pb + (tl + 8) * TS);
          const double x2 = __ldcg(pb + (tl + 16) * TS), x3 = __ldcg(pb + (tl + 24) * TS);
          s0 += x0, s1 += x1, s2 += x2, s3 += x3;
        }
        if (tl < nslot1) s0 += __ldcg(pb + tl * TS);
        if (tl + 8 < nslot1) s1 += __ldcg(pb + (tl + 8) * TS);
        if (tl + 16 < nslot1) s2 += __ldcg(pb + (tl + 16) * TS);
      }
      double s = (s0 + s1) + (s2 + s3);
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      s += __shfl_xor_sync(0xffffffffu, s, 4);
      if (q == 0 && on) {
        double* D = optr_w<double>(p.A, b) + (p.j + a) + int64_t(p.j + c) * p.A.ld;
        *D -= s;
      }
    }
    __threadfence();
    cg::this_grid().sync();
  }

  // ---------------- phase 3: Ldot_D = D Phi(D^{-1} Ddot_sym D^{-T})  (Eq. 8) ----------------
  const int64_t u3 = (p.skip3 || (p.dbg_skip & 8)) ? 0 : p.batch * 16;
  // 3a: Y = D^{-1} X,  X(r, c) = Ddot(max, min)
  for (int64_t u = blockIdx.x; u < u3; u += gridDim.x) {
    const int64_t b = u >> 4;
    const int ti = int(u & 15) >> 2, tj = int(u & 3);
    const double* Di = p.Dinv + b * p.dstride;
    const double* Ab = optr<double>(p.A, b) + p.j + int64_t(p.j) * p.A.ld;
    double* Yb = p.Yws + b * 128 * 128;
    const int a0 = 32 * ti, c0 = 32 * tj;
    pr_tile32kx(
        sm, 128,
        [&](int m, int k) -> const double* {  // A(m, k) = Dinv(a0 + m, k)
          const int a = a0 + m;
          return (k < w && a < w && k <= a) ? Di + a + int64_t(k) * p.dld : nullptr;
        },
        [&](int k, int n) -> const double* {  // B(k, n) = X(k, c0 + n)
          const int cc = c0 + n;
          if (k >= w || cc >= w) return nullptr;
          return k >= cc ? Ab + k + int64_t(cc) * p.A.ld : Ab + cc + int64_t(k) * p.A.ld;
        },
        [&](int m, int n, double v) { Yb[(a0 + m) + (c0 + n) * 128] = v; }, [](int) { return true; }, [](int) { return false; });
  }
  __threadfence();
  cg::this_grid().sync();
  // 3b (lower tiles): F = Phi(Y D^{-T})
  for (int64_t u = blockIdx.x; u < u3; u += gridDim.x) {
    const int64_t b = u >> 4;
    const int ti = int(u & 15) >> 2, tj = int(u & 3);
    if (ti < tj) continue;
    const double* Di = p.Dinv + b * p.dstride;
    const double* Yb = p.Yws + b * 128 * 128;
    double* Fb = p.Fws + b * 128 * 128;
    const int a0 = 32 * ti, c0 = 32 * tj;
    pr_tile32kx(
        sm, 128,
        [&](int m, int k) -> const double* { return (k < w && a0 + m < w) ? Yb + (a0 + m) + k * 128 : nullptr; },
        [&](int k, int n) -> const double* {  // B(k, n) = Dinv(c0 + n, k)
          const int cc = c0 + n;
          return (k < w && cc < w && k <= cc) ? Di + cc + int64_t(k) * p.dld : nullptr;
        },
        [&](int m, int n, double v) {
          const int a = a0 + m, cc = c0 + n;
          Fb[a + cc * 128] = a > cc ? v : (a == cc ? 0.5 * v : 0.0);
        },
        [](int) { return true; }, [](int) { return true; });
  }
  __threadfence();
  cg::this_grid().sync();
  // 3c (lower tiles): Ldot_D = D F  -> tril(Ddot) and Dc
  for (int64_t u = blockIdx.x; u < u3; u += gridDim.x) {
    const int64_t b = u >> 4;
    const int ti = int(u & 15) >> 2, tj = int(u & 3);
    const double* Lb = optr<double>(p.L, b) + p.j + int64_t(p.j) * p.L.ld;
    const double* Fb = p.Fws + b * 128 * 128;
    double* Ab = optr_w<double>(p.A, b) + p.j + int64_t(p.j) * p.A.ld;
    double* Dcb = p.Dc + b * int64_t(132 * 128);
    const int a0 = 32 * ti, c0 = 32 * tj;
    if (ti < tj) {  // upper tile of Dc: zero
      for (int e = tid; e < 32 * 32; e += PR_THREADS) Dcb[(a0 + (e & 31)) + (c0 + (e >> 5)) * 132] = 0.0;
      continue;
    }
    pr_tile32kx(
        sm, 128,
        [&](int m, int k) -> const double* {  // A(m, k) = D(a0 + m, k)
          const int a = a0 + m;
          return (k < w && a < w && k <= a) ? Lb + a + int64_t(k) * p.L.ld : nullptr;
        },
        [&](int k, int n) -> const double* {  // B(k, n) = F(k, c0 + n), lower
          const int cc = c0 + n;
          return (k < w && cc < w && k >= cc) ? Fb + k + cc * 128 : nullptr;
        },
        [&](int m, int n, double v) {
          const int a = a0 + m, cc = c0 + n;
          const bool low = a >= cc && a < w && cc < w;
          if (low) Ab[a + int64_t(cc) * p.A.ld] = v;
          Dcb[a + cc * 132] = low ? v : 0.0;
        },
        [](int) { return true; }, [](int) { return false; });
  }
}

}  // namespace cd
