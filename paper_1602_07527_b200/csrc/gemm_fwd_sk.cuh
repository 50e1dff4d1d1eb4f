// gemm_fwd_sk.cuh -- the Level-3 update of the blocked forward sweep (fp64, DMMA):
//
//     W = Cdot - Bdot R^T - B Rdot^T - C Ddot^T          (before the D^{-T})
//
// for the panel J = [j, k) (w = 128 columns), rows [k, n), q = j columns to the left:
//   segment 0: A = Adot[k:n, 0:q]  (Bdot),  B(kk, c) = L[j + c, kk]      (R^T),     K = q
//   segment 1: A = L[k:n, 0:q]     (B),     B(kk, c) = Adot[j + c, kk]   (Rdot^T),  K = q
//   segment 2: A = L[k:n, j:k]     (C),     B(kk, c) = Dc[c, kk]         (Ddot^T),  K = w
// written in place over Cdot.  With `chol` set it is the factorisation's C <- C - B R^T
// (chol_blocked) instead: segment 0 only, both operands from L.
// The output is a narrow p x 128 panel with K = 2q + w, the
// same shape as the left-looking reverse update, so it uses the same machinery as
// k_symm_ll: TMA-fed DMMA with one producer and two consumer warpgroups (setmaxnreg), and
// stream-K over batch x m x KT k-tiles with the deterministic last-arrival fixup instead
// of split-K partials + a reduction launch.  Every operand tile is one TMA box of 132 x BK
// (the 4-row pad makes the shared-memory pitch 4 mod 16 doubles: conflict-free fragments):
// A as As[k][m], B as Bs[k][c].
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "gemm.cuh"
#include "gemm_tma.cuh"
#include "symm_ll.cuh"  // ll_start / ll_cta_of, LL_* tile constants

namespace cd {

constexpr int FS_PITCH = LL_BM + 4;                       // 132
constexpr int FS_TILE = LL_BK * FS_PITCH;                 // 2112 doubles per operand stage
constexpr uint32_t FS_BYTES = uint32_t(FS_TILE) * 8u;     // 16896
constexpr size_t FS_SMEM = size_t(LL_STAGES) * 2 * FS_TILE * 8 + 2 * LL_STAGES * 8 + 16 + 1024;

struct FSMaps {
  CUtensorMap adot;  // Adot, box {132 rows, 16 cols}
  CUtensorMap l;     // L, same box
  CUtensorMap dc;    // Dc workspace (132 x 128 per batch entry), same box
  int batched;
};

struct FSParams {
  Opnd A;            // Adot, whole matrix (Cin and D of the output panel)
  int n, k, j, w, q;
  int m;             // output row tiles = ceil((n - k) / 128)
  int KT;            // k-tiles per output tile = (2q + w) / BK
  int G;
  int64_t total;     // batch * m * KT (< 2^31)
  double* part;      // [G][2][128*128]
  int* cnt;          // [batch * m], zero on entry, reset by the last CTA
  int chol;          // factorisation mode (chol_blocked): W = C - B R^T, one
                     // segment with A and B both from the `l` map (KT = q / 16)
  int defer;         // split tiles: pieces only; k_fwd_sk_reduce (next launch) sums them
};

__global__ void __launch_bounds__(LL_THREADS, 1) k_fwd_sk(const FSParams p, const __grid_constant__ FSMaps tm) {
  extern __shared__ __align__(1024) unsigned char smem_fs[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_fs) + 1023) & ~uintptr_t(1023));
  double* As = reinterpret_cast<double*>(base);
  double* Bs = As + LL_STAGES * FS_TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + LL_STAGES * FS_TILE);
  uint64_t* empty = full + LL_STAGES;
  int* s_flag = reinterpret_cast<int*>(empty + LL_STAGES);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cta = blockIdx.x;
  const int a0 = int(ll_start(cta, p.total, p.G)), a1 = int(ll_start(cta + 1, p.total, p.G));
  const int per_tile = p.KT;
  const int kq = p.q / LL_BK;  // k-tiles of segment 0 (and of segment 1)

  if (tid == 0) {
    for (int s = 0; s < LL_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], LL_CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // launched with programmatic stream serialization (PDL) after the panel kernel: the prologue
  // above overlaps its tail; every global access below waits for it to complete
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  __syncthreads();

  if (warp >= LL_CONSUMERS) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == LL_CONSUMERS && lane == 0) {
      int it = 0;
      for (int x = a0; x < a1; ++x, ++it) {
        const int s = it % LL_STAGES;
        if (it >= LL_STAGES) mbar_wait(&empty[s], ((it / LL_STAGES) - 1) & 1);
        const int tg = x / per_tile;
        const int kt = x - tg * per_tile;
        const int b = tg / p.m, i = tg - b * p.m;
        const int r0 = p.k + LL_BM * i;
        const CUtensorMap *am, *bm;
        int ac0, ac1, bc0, bc1;
        if (kt < kq) {  // Bdot R^T  (factorisation mode: B R^T)
          const int kk = kt * LL_BK;
          am = p.chol ? &tm.l : &tm.adot, ac0 = r0, ac1 = kk;
          bm = &tm.l, bc0 = p.j, bc1 = kk;
        } else if (kt < 2 * kq) {  // B Rdot^T
          const int kk = (kt - kq) * LL_BK;
          am = &tm.l, ac0 = r0, ac1 = kk;
          bm = &tm.adot, bc0 = p.j, bc1 = kk;
        } else {  // C Ddot^T
          const int kk = (kt - 2 * kq) * LL_BK;
          am = &tm.l, ac0 = r0, ac1 = p.j + kk;
          bm = &tm.dc, bc0 = 0, bc1 = kk;
        }
        double* as = As + s * FS_TILE;
        double* bs = Bs + s * FS_TILE;
        mbar_expect_tx(&full[s], 2 * FS_BYTES);
        if (tm.batched) {
          tma_load_3d(as, am, ac0, ac1, b, &full[s]);
          tma_load_3d(bs, bm, bc0, bc1, b, &full[s]);
        } else {
          tma_load_2d(as, am, ac0, ac1, &full[s]);
          tma_load_2d(bs, bm, bc0, bc1, &full[s]);
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
      const double* as = As + s * FS_TILE;
      const double* bs = Bs + s * FS_TILE;
#pragma unroll
      for (int kq4 = 0; kq4 < LL_BK / 4; ++kq4) {
        const int kx = kq4 * 4 + t;
        double a[8], bb[4];
#pragma unroll
        for (int ii = 0; ii < 8; ++ii) a[ii] = as[kx * FS_PITCH + wm * 64 + ii * 8 + g];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) bb[jj] = -bs[kx * FS_PITCH + wn * 32 + jj * 8 + g];
#pragma unroll
        for (int ii = 0; ii < 8; ++ii)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) dmma884(acc[ii][jj][0], acc[ii][jj][1], a[ii], bb[jj]);
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
    if (p.defer) continue;  // the pieces are summed by k_fwd_sk_reduce
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
  }
}

// The deferred fixup of k_fwd_sk (p.defer): ll_sk_reduce (symm_ll.cuh) over its tiles.
__global__ void __launch_bounds__(256) k_fwd_sk_reduce(const FSParams p) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");  // PDL: k_fwd_sk's pieces are complete
  ll_sk_reduce(p.A, p.n, p.k, p.j, p.w, p.m, p.KT, p.G, p.total, p.part);
}

}  // namespace cd
