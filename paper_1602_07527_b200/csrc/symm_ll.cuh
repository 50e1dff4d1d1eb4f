// symm_ll.cuh -- left-looking trailing update of the blocked reverse sweep (fp64, DMMA).
//
// PAPER.md:704-707 ("the partitioning into columns is arbitrary") lets the updates that
// chol_blocked_rev applies to the left part of the matrix,
//     Bbar <- Bbar - Cbar R,      Rbar <- Rbar - Cbar^T B - (Dbar + Dbar^T) R,
// be delayed until the column block they land in is next.  Summed over all blocks J to
// the right of the panel J' = [j, k), the delayed updates of Abar[k:n, j:k] are
//
//     Cbar_J' <- Cbar_J' - M L[k:n, j:k],      M = T + T^T  (diagonal doubled),
//
// with T = tril(Sigmabar)[k:n, k:n] the FINISHED trailing part of the result (the
// sweep never touches a column block again once it is done).  Rows j:k of the panel
// receive nothing from the right (they sit above every J).  So one step of the sweep
// becomes: this update (a SYMM with K = p = n - k), then the panel solve, the Dbar
// correction and the diagonal-block sweep exactly as in PAPER.md:695-698.  The update
// reads tril(T) in place and never read-modify-writes the big trailing region (the
// right-looking B̄ update re-reads and re-writes p x q elements per step); its output is
// the narrow p x w panel.
//
// Tile structure (nb = 128 = BM, every block right of the panel is a full 128-block, so
// output row tiles and K blocks coincide with diagonal blocks):
//   output tile i (rows k+128i ..), K block s (cols k+128s ..) of M:
//     s <  i : T[i, s]            read in place, column-major   (A tile "KM": As[k][m])
//     s == i : S_i = D̄_i + D̄_iᵀ   dense copy kept by the sweep  (workspace, "KM")
//     s >  i : T[s, i]ᵀ           read in place, transposed     (A tile "MK": As[m][k])
//   B tile = L[k+128s+kk .., j:j+128] (Bs[n][k]).
//
// Work split: stream-K.  The batch * m tiles * (128/BK)m k-tiles are cut into G equal
// contiguous ranges, one per CTA (G <= #SMs, one CTA per SM).  A tile covered by one
// CTA is written directly (Cin prefetched into the accumulators); a tile split across
// CTAs has each piece stored to a partial slot, and the LAST arriving CTA (atomic
// counter) sums Cin + all pieces in fixed CTA order -- bitwise deterministic -- and
// resets the counter.  No separate reduction kernel.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "gemm.cuh"
#include "gemm_tma.cuh"

namespace cd {

// K step 32 x 3 stages (221 KB): half the per-stage barrier traffic of 16 x 5 at the same
// bytes in flight (N=16384 reverse 94.3 -> 93.2 ms)
#ifndef CD_LL_BK
#define CD_LL_BK 32
#endif
#ifndef CD_LL_STAGES
#define CD_LL_STAGES 3
#endif
constexpr int LL_BM = 128, LL_BN = 128, LL_BK = CD_LL_BK;
constexpr int LL_KT_PER_BLK = 128 / LL_BK;  // k-tiles per 128-wide K block
constexpr int LL_STAGES = CD_LL_STAGES;
constexpr int LL_CONSUMERS = 8;                    // warps 0..7 (two warpgroups)
constexpr int LL_THREADS = (LL_CONSUMERS + 4) * 32;  // + one producer warpgroup (warps 8..11)
constexpr int LL_A_KM_PITCH = LL_BM + 4, LL_A_MK_PITCH = LL_BK + 4, LL_B_PITCH = LL_BK + 4;
constexpr int LL_A_SIZE = LL_BM * (LL_BK + 4) > LL_BK * (LL_BM + 4) ? LL_BM * (LL_BK + 4) : LL_BK * (LL_BM + 4);
constexpr int LL_B_SIZE = LL_BN * (LL_BK + 4);  // 2560
constexpr uint32_t LL_BYTES_KM = uint32_t(LL_BK * (LL_BM + 4)) * 8u;  // 16896
constexpr uint32_t LL_BYTES_MK = uint32_t(LL_BM * (LL_BK + 4)) * 8u;  // 20480
constexpr uint32_t LL_BYTES_B = uint32_t(LL_BN * (LL_BK + 4)) * 8u;   // 20480
constexpr size_t LL_SMEM = size_t(LL_STAGES) * (LL_A_SIZE + LL_B_SIZE) * 8 + 2 * LL_STAGES * 8 + 16 + 1024;
constexpr int LL_TILE = LL_BM * LL_BN;  // doubles per partial slot

struct LLMaps {
  CUtensorMap aN;  // Abar, box {132 rows, BK cols}
  CUtensorMap aT;  // Abar, box {BK+4 rows, 128 cols}
  CUtensorMap s;   // S workspace (132 x 128*nblk per batch), box {132, BK}
  CUtensorMap l;   // L, box {BK+4, 128}
  int batched;
};

struct LLParams {
  Opnd A;          // Abar, whole matrix (Cin and D of the output panel)
  int n, k, j, w;  // trailing region starts at row/col k; panel columns [j, j+w)
  int m;           // output row tiles = (n - k) / 128
  int nblk;        // blocks of the reverse partition (S slot of the block at row r0: nblk - (n - r0)/128)
  int G;           // CTAs
  int64_t total;   // batch * m * (128/BK)m k-tiles (< 2^31, checked by the host)
  double* part;    // [G][2][128*128] partial slots
  int* cnt;        // [batch * m] arrival counters (zero on entry, reset by the last CTA)
  int defer;       // split tiles: pieces only; k_symm_ll_reduce (next launch) sums them
};

__device__ __forceinline__ int64_t ll_start(int64_t c, int64_t total, int G) { return (c * total) / G; }
__device__ __forceinline__ int ll_cta_of(int64_t x, int64_t total, int G) {
  int c = int((x * G) / total);
  while (c + 1 < G && ll_start(c + 1, total, G) <= x) ++c;
  while (c > 0 && ll_start(c, total, G) > x) --c;
  return c;
}

__global__ void __launch_bounds__(LL_THREADS, 1) k_symm_ll(const LLParams p, const __grid_constant__ LLMaps tm) {
  extern __shared__ __align__(1024) unsigned char smem_ll[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_ll) + 1023) & ~uintptr_t(1023));
  double* As = reinterpret_cast<double*>(base);
  double* Bs = As + LL_STAGES * LL_A_SIZE;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + LL_STAGES * LL_B_SIZE);
  uint64_t* empty = full + LL_STAGES;
  int* s_flag = reinterpret_cast<int*>(empty + LL_STAGES);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cta = blockIdx.x;
  const int a0 = int(ll_start(cta, p.total, p.G)), a1 = int(ll_start(cta + 1, p.total, p.G));
  const int per_tile = LL_KT_PER_BLK * p.m;  // k-tiles per output tile

  if (tid == 0) {
    for (int s = 0; s < LL_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], LL_CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // launched with programmatic stream serialization (PDL) after the previous panel kernel: the
  // prologue above overlaps its tail; every global access below waits for it to complete
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  __syncthreads();

  if (warp >= LL_CONSUMERS) {
    // ---------------- producer warpgroup: registers handed to the consumers; one lane issues TMA ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == LL_CONSUMERS && lane == 0) {
      int it = 0;
      for (int x = a0; x < a1; ++x, ++it) {
        const int s = it % LL_STAGES;
        if (it >= LL_STAGES) mbar_wait(&empty[s], ((it / LL_STAGES) - 1) & 1);
        const int tg = x / per_tile;
        const int kt = x - tg * per_tile;
        const int b = tg / p.m, i = tg - b * p.m;
        const int sb = kt / LL_KT_PER_BLK, kk = (kt % LL_KT_PER_BLK) * LL_BK;
        const int r0 = p.k + LL_BM * i, c0 = p.k + LL_BM * sb + kk;
        double* as = As + s * LL_A_SIZE;
        double* bs = Bs + s * LL_B_SIZE;
        mbar_expect_tx(&full[s], (sb <= i ? LL_BYTES_KM : LL_BYTES_MK) + LL_BYTES_B);
        const CUtensorMap* am;
        int ac0, ac1;
        if (sb < i) {
          am = &tm.aN, ac0 = r0, ac1 = c0;
        } else if (sb == i) {
          am = &tm.s, ac0 = 0, ac1 = (p.nblk - (p.n - r0) / LL_BM) * LL_BM + kk;
        } else {
          am = &tm.aT, ac0 = c0, ac1 = r0;
        }
        if (tm.batched) {
          tma_load_3d(as, am, ac0, ac1, b, &full[s]);
          tma_load_3d(bs, &tm.l, c0, p.j, b, &full[s]);
        } else {
          tma_load_2d(as, am, ac0, ac1, &full[s]);
          tma_load_2d(bs, &tm.l, c0, p.j, &full[s]);
        }
      }
    }
    return;
  }

  // ---------------- consumers: 8 warps, 64 x 32 warp tiles ----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
  const int wm = warp >> 2, wn = warp & 3, g = lane >> 2, t = lane & 3;
  double acc[8][4][2];
  int it = 0;
  int x = a0;
  while (x < a1) {
    const int tg = x / per_tile;
    const int ts = tg * per_tile, te = ts + per_tile;
    const int xe = te < a1 ? te : a1;
    const bool whole = (x == ts && xe == te);
    const int b = tg / p.m, i = tg - b * p.m;
    const int r0 = p.k + LL_BM * i;
    double* Dp = optr_w<double>(p.A, b) + r0 + int64_t(p.j) * p.A.ld;
    // accumulators start as Cin (whole tile) or 0 (a piece); the sum enters with sign -1
#pragma unroll
    for (int ii = 0; ii < 8; ++ii)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = wm * 64 + ii * 8 + g;
          const int c = wn * 32 + jj * 8 + 2 * t + e;
          acc[ii][jj][e] = (whole && c < p.w && r0 + r < p.n) ? __ldcg(Dp + r + int64_t(c) * p.A.ld) : 0.0;
        }
    for (; x < xe; ++x, ++it) {
      const int s = it % LL_STAGES;
      mbar_wait(&full[s], (it / LL_STAGES) & 1);
      const int kt = x - ts;
      const bool km = kt / LL_KT_PER_BLK <= i;
      const double* as = As + s * LL_A_SIZE;
      const double* bs = Bs + s * LL_B_SIZE;
      if (km) {
#pragma unroll
        for (int kq = 0; kq < LL_BK / 4; ++kq) {
          const int kx = kq * 4 + t;
          double a[8], bb[4];
#pragma unroll
          for (int ii = 0; ii < 8; ++ii) a[ii] = as[kx * LL_A_KM_PITCH + wm * 64 + ii * 8 + g];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) bb[jj] = -bs[(wn * 32 + jj * 8 + g) * LL_B_PITCH + kx];
#pragma unroll
          for (int ii = 0; ii < 8; ++ii)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) dmma884(acc[ii][jj][0], acc[ii][jj][1], a[ii], bb[jj]);
        }
      } else {
#pragma unroll
        for (int kq = 0; kq < LL_BK / 4; ++kq) {
          const int kx = kq * 4 + t;
          double a[8], bb[4];
#pragma unroll
          for (int ii = 0; ii < 8; ++ii) a[ii] = as[(wm * 64 + ii * 8 + g) * LL_A_MK_PITCH + kx];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) bb[jj] = -bs[(wn * 32 + jj * 8 + g) * LL_B_PITCH + kx];
#pragma unroll
          for (int ii = 0; ii < 8; ++ii)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) dmma884(acc[ii][jj][0], acc[ii][jj][1], a[ii], bb[jj]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    if (whole) {
#pragma unroll
      for (int ii = 0; ii < 8; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = wm * 64 + ii * 8 + g;
            const int c = wn * 32 + jj * 8 + 2 * t + e;
            if (c < p.w && r0 + r < p.n) __stcg(Dp + r + int64_t(c) * p.A.ld, acc[ii][jj][e]);
          }
      continue;
    }
    // ---- a piece of a split tile: store to this CTA's slot, last arrival finishes ----
    {
      const int slot = 2 * cta + (ts <= a0 ? 0 : 1);
      double* mine = p.part + int64_t(slot) * LL_TILE;
#pragma unroll
      for (int ii = 0; ii < 8; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = wm * 64 + ii * 8 + g;
            const int c = wn * 32 + jj * 8 + 2 * t + e;
            __stcg(mine + r + c * LL_BM, acc[ii][jj][e]);
          }
    }
    if (p.defer) continue;  // the pieces are summed by k_symm_ll_reduce
    __threadfence();
    asm volatile("bar.sync 1, %0;\n" ::"n"(LL_CONSUMERS * 32) : "memory");
    const int c_lo = ll_cta_of(ts, p.total, p.G), c_hi = ll_cta_of(te - 1, p.total, p.G);
    if (tid == 0) {
      const int old = atomicAdd(&p.cnt[tg], 1);
      *s_flag = (old == c_hi - c_lo) ? 1 : 0;
    }
    asm volatile("bar.sync 1, %0;\n" ::"n"(LL_CONSUMERS * 32) : "memory");
    if (*s_flag) {
      __threadfence();
      // D = Cin + sum of the pieces in CTA order (each piece already carries the -1), in
      // the accumulator layout so that every load of a piece is independent
#pragma unroll
      for (int ii = 0; ii < 8; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = wm * 64 + ii * 8 + g;
            const int c = wn * 32 + jj * 8 + 2 * t + e;
            acc[ii][jj][e] = (c < p.w && r0 + r < p.n) ? __ldcg(Dp + r + int64_t(c) * p.A.ld) : 0.0;
          }
      for (int cc = c_lo; cc <= c_hi; ++cc) {
        const int slot = 2 * cc + (ll_start(cc, p.total, p.G) >= ts ? 0 : 1);
        const double* pp = p.part + int64_t(slot) * LL_TILE;
#pragma unroll
        for (int ii = 0; ii < 8; ++ii)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int r = wm * 64 + ii * 8 + g;
              const int c = wn * 32 + jj * 8 + 2 * t + e;
              acc[ii][jj][e] += __ldcg(pp + r + c * LL_BM);
            }
      }
#pragma unroll
      for (int ii = 0; ii < 8; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = wm * 64 + ii * 8 + g;
            const int c = wn * 32 + jj * 8 + 2 * t + e;
            if (c < p.w && r0 + r < p.n) __stcg(Dp + r + int64_t(c) * p.A.ld, acc[ii][jj][e]);
          }
      if (tid == 0) p.cnt[tg] = 0;
    }
    // s_flag is rewritten only after the next piece's first barrier
  }
}

// The deferred stream-K fixup (p.defer of k_symm_ll / k_fwd_sk): for every output tile split across
// CTAs, D = Cin + the pieces in CTA order -- the sum the last-arriving CTA forms otherwise -- spread
// over the whole grid, one element per thread, instead of one CTA reading every piece of its tile.
// With few output tiles (mid N) the stream-K kernel then runs ~one k-tile per CTA on every SM
// instead of >= 4 k-tiles on a few of them.  Tiles covered by one CTA were written by it: skipped.
// Tiles: batch x m of 128 rows (from row k) x w columns (from column j), KT k-tiles each.
__device__ __forceinline__ void ll_sk_reduce(const Opnd& A, int n, int k, int j, int w, int m, int KT, int G,
                                             int64_t total, const double* __restrict__ part) {
  const int64_t per = int64_t(LL_BM) * w;  // elements per output tile
  const int64_t tot = (total / KT) * per;  // batch * m tiles
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
    const int tg = int(e / per);
    const int rc = int(e - int64_t(tg) * per), c = rc / LL_BM, r = rc - c * LL_BM;
    const int ts = tg * KT, te = ts + KT;
    const int c_lo = ll_cta_of(ts, total, G), c_hi = ll_cta_of(te - 1, total, G);
    const int b = tg / m, i = tg - b * m;
    const int r0 = k + LL_BM * i;
    if (c_lo == c_hi || r0 + r >= n) continue;
    double* Dp = optr_w<double>(A, b) + (r0 + r) + int64_t(j + c) * A.ld;
    double acc = __ldcg(Dp);
    for (int cc = c_lo; cc <= c_hi; ++cc) {
      const int slot = 2 * cc + (ll_start(cc, total, G) >= ts ? 0 : 1);
      acc += __ldcg(part + int64_t(slot) * LL_TILE + r + c * LL_BM);
    }
    __stcg(Dp, acc);
  }
}

__global__ void __launch_bounds__(256) k_symm_ll_reduce(const LLParams p) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");  // PDL: k_symm_ll's pieces are complete
  ll_sk_reduce(p.A, p.n, p.k, p.j, p.w, p.m, LL_KT_PER_BLK * p.m, p.G, p.total, p.part);
}

}  // namespace cd
