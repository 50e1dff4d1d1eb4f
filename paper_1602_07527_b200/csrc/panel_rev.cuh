// panel_rev.cuh -- the panel step of the blocked reverse sweep as ONE cooperative kernel
// (fp64, DMMA):
//
//     Cbar <- Cbar D^{-1}                  ("solving a triangular system")
//     Dbar <- Dbar - tril(Cbar^T C)        (only the triangle is needed,
//                                           PAPER.md:717-723)
//
// for the p x w panel Cbar = Abar[k:n, j:k], C = L[k:n, j:k], D^{-1} precomputed by
// k_trinv.  One CTA per 128-row tile of the panel (looping if there are more tiles than
// SMs):
//   phase 1  W = Cbar_t D^{-1} (lower-triangular D^{-1}: K chunks that cannot reach a
//            warp's columns are skipped), stored in place and kept in shared memory;
//            P_t = tril(W^T C_t) (warps above the diagonal skip), stored to slot t;
//   grid sync (cooperative launch: all CTAs co-resident);
//   phase 2  Dbar -= sum_t P_t over the lower triangle, eight lanes per element with a
//            fixed summation tree (bitwise deterministic);
//   phase 3  the diagonal block Dbar <- chol_unblocked_rev(D, Dbar) by Eq. 10, three
//            32x32-tiled products over the grid (see below), also emitting S = Dbar + Dbar^T.
// Replaces two split-K GEMM launches, their reduction launches and the one-CTA diagonal
// sweep on the critical path.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "gemm.cuh"

namespace cd {

constexpr int PR_THREADS = 256;
constexpr int PR_BK = 16;
constexpr int PR_STAGES = 3;
constexpr int PR_KM_PITCH = 128 + 4;  // As[k][m]
constexpr int PR_NK_PITCH = PR_BK + 4;  // Bs[n][k]
constexpr int PR_A_SIZE = PR_BK * PR_KM_PITCH;  // 2112
constexpr int PR_B_SIZE = 128 * PR_NK_PITCH;    // 2560
constexpr int PR_W_PITCH = 132;
constexpr size_t PR_SMEM_A = size_t(PR_STAGES) * (PR_A_SIZE + PR_B_SIZE) * 8;              // step A stages
constexpr size_t PR_SMEM_C = size_t(128) * PR_W_PITCH * 8 + size_t(PR_STAGES) * PR_B_SIZE * 8;  // W + step C stages
constexpr size_t PR_SMEM_AC = PR_SMEM_A > PR_SMEM_C ? PR_SMEM_A : PR_SMEM_C;

struct PanelParams {
  Opnd A, L;         // Abar and L (whole matrices)
  const double* Dinv;  // w x w (ld dld) inverse of the diagonal block (per batch: + b * dstride)
  int64_t dstride;
  int dld;
  int n, j, w, k;    // panel rows [k, n), columns [j, j + w)
  int tiles;         // (n - k) / 128 per matrix
  int64_t batch;
  double* part;      // [batch * tiles][128 * 128] slots
  // phase 3 (diagonal block by Eq. 10): scratch P, Z (dense 128 x 128 per batch entry) and
  // the S output (dense, ld s_ld, batch stride s_stride; nullptr = not needed)
  double* Pws;
  double* Zws;
  double* S;
  int s_ld;
  int64_t s_stride;
  int dbg_skip;  // measurement only (CD_DEBUG_PANEL_SKIP): bit i skips phase i+1; results wrong
  double* Wst;   // small-panel phase 1 staging of W: [batch * tiles][128 * 128]
  // phase 0 (small panels, instead of a k_symm_ll launch): Cbar -= (T + T^T) L[k:n, j:k]
  int symm;              // 1: run phase 0
  const double* Sall;    // S blocks (ld s_ld, block stride s_blk, batch stride s_stride) = diagonal tiles of M
  int64_t s_blk;
  int nblk;              // S slot of the block at row r0: nblk - (n - r0) / 128
  int split_max;         // phase 1: 128-row tiles split into up to this many sub-tiles (1, 2, 4)
};

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc, bool valid) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gsrc), "r"(valid ? 8 : 0));
}

__device__ __forceinline__ void cp_async_wait_n(int n) {  // all but the n most recent groups
  switch (n) {
    case 0: cp_async_wait<0>(); break;
    case 1: cp_async_wait<1>(); break;
    case 2: cp_async_wait<2>(); break;
    case 3: cp_async_wait<3>(); break;
    case 4: cp_async_wait<4>(); break;
    case 5: cp_async_wait<5>(); break;
    case 6: cp_async_wait<6>(); break;
    case 7: cp_async_wait<7>(); break;
    case 8: cp_async_wait<8>(); break;
    case 9: cp_async_wait<9>(); break;
    case 10: cp_async_wait<10>(); break;
    default: cp_async_wait<11>(); break;
  }
}

// One 32 x 32 output tile of C = A B (K any multiple of 128, zero-padded) on a CTA.  The source
// functors return a global pointer to A(m, k) / B(k, n), or nullptr for a zero; every element is
// staged by an 8-byte cp.async into shared memory.  K advances in 128-wide chunks, two in flight
// (double buffer), each chunk in four commit groups of 32 k, so the DMMA work on one group
// overlaps the landing of the next.  am(kb) tells whether A is contiguous along m in the chunk
// starting at k = kb (a column-major block): its copies then walk m (coalesced) and the chunk is
// stored [k][m] (pitch 36); otherwise they walk k and it is stored [m][k] (pitch 132).  bn(kb)
// likewise for B along n (stored [k][n], else [n][k]).  Each warp owns two 8 x 8 sub-tiles; the
// epilogue functor gets (row m, column n, value).
constexpr int PT_P = 132, PT_PKM = 36;
constexpr int PT_A = 128 * PT_PKM > 32 * PT_P ? 128 * PT_PKM : 32 * PT_P;  // 4608 doubles
constexpr int PT_SLOT = 2 * PT_A;                                          // A and B, 9216 doubles
// K chunks in flight: PT_NSLOT buffers (a third one, 221 KB of shared memory, measured no faster:
// N = 1024 reverse 468.6 vs 466 us, N = 16384 92.44 vs 92.36 ms -- the tiles are not waiting on L2)
#ifndef CD_PT_NSLOT
#define CD_PT_NSLOT 2
#endif
constexpr int PT_NSLOT = CD_PT_NSLOT;
constexpr size_t PR_SMEM = size_t(PT_NSLOT) * PT_SLOT * 8 > PR_SMEM_AC ? size_t(PT_NSLOT) * PT_SLOT * 8 : PR_SMEM_AC;
static_assert(PR_SMEM <= 232448, "panel kernels' shared memory exceeds the per-CTA limit");

template <class FA, class FB, class EP, class AM, class BN>
__device__ __forceinline__ void pr_tile32kx(double* sm, int K, FA fa, FB fb, EP ep, AM am, BN bn) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int mt = warp >> 1, nt0 = (warp & 1) * 2;  // sub-tiles (mt, nt0) and (mt, nt0 + 1)
  double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  const int nch = (K + 127) / 128;
  auto load = [&](int ch) {
    double* As = sm + (ch % PT_NSLOT) * PT_SLOT;
    double* Bs = As + PT_A;
    const int kb = 128 * ch;
    const bool mf = am(kb), nf = bn(kb);
#pragma unroll 1
    for (int q = 0; q < 4; ++q) {
      for (int e = tid; e < 32 * 32; e += PR_THREADS) {
        // an element with no source (nullptr) is a zero: a plain shared store (a zero-size
        // cp.async would still need a valid global source address)
        {
          const int k = nf ? 32 * q + (e >> 5) : 32 * q + (e & 31), nn = nf ? (e & 31) : (e >> 5);
          const double* pb = fb(kb + k, nn);
          double* db = Bs + (nf ? k * PT_PKM + nn : nn * PT_P + k);
          if (pb) cp_async8(db, pb, true);
          else *db = 0.0;
        }
        {
          const int k = mf ? 32 * q + (e >> 5) : 32 * q + (e & 31), m = mf ? (e & 31) : (e >> 5);
          const double* pa = fa(m, kb + k);
          double* da = As + (mf ? k * PT_PKM + m : m * PT_P + k);
          if (pa) cp_async8(da, pa, true);
          else *da = 0.0;
        }
      }
      cp_async_commit();
    }
  };
  __syncthreads();  // shared memory reuse
#pragma unroll 1
  for (int c = 0; c < PT_NSLOT - 1 && c < nch; ++c) load(c);
#pragma unroll 1
  for (int ch = 0; ch < nch; ++ch) {
    // chunk ch + NSLOT - 1 goes into the buffer chunk ch - 1 used (freed by the barrier after it)
    if (ch + PT_NSLOT - 1 < nch) load(ch + PT_NSLOT - 1);
    const int ahead = min(PT_NSLOT - 1, nch - 1 - ch);  // chunks issued after this one
    const double* As = sm + (ch % PT_NSLOT) * PT_SLOT;
    const double* Bs = As + PT_A;
    const bool mf = am(128 * ch), nf = bn(128 * ch);
#pragma unroll 1
    for (int q = 0; q < 4; ++q) {
      cp_async_wait_n(3 - q + 4 * ahead);
      __syncthreads();
#pragma unroll
      for (int kq = 8 * q; kq < 8 * q + 8; ++kq) {
        const double a = mf ? As[(4 * kq + t) * PT_PKM + 8 * mt + g] : As[(8 * mt + g) * PT_P + 4 * kq + t];
#pragma unroll
        for (int u = 0; u < 2; ++u)
          dmma884(c[u][0], c[u][1], a,
                  nf ? Bs[(4 * kq + t) * PT_PKM + 8 * (nt0 + u) + g] : Bs[(8 * (nt0 + u) + g) * PT_P + 4 * kq + t]);
      }
    }
    __syncthreads();  // this buffer is refilled by chunk ch + NSLOT
  }
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int e = 0; e < 2; ++e) ep(8 * mt + g, 8 * (nt0 + u) + 2 * t + e, c[u][e]);
}

template <class FA, class FB, class EP>
__device__ __forceinline__ void pr_tile32k(double* sm, int K, FA fa, FB fb, EP ep) {
  pr_tile32kx(sm, K, fa, fb, ep, [](int) { return false; }, [](int) { return false; });
}

template <class FA, class FB, class EP>
__device__ __forceinline__ void pr_tile32(double* sm, FA fa, FB fb, EP ep) {
  pr_tile32k(sm, 128, fa, fb, ep);
}

// Phase 1 of k_panel_rev on sub-tiles of ROWS = 16 RT rows (RT = 8: whole 128-row tiles; 4 / 2:
// halves / quarters, s = 128 / ROWS of them per tile, when the panel has few tiles):
//   step A  W = Cbar_sub D^{-1}  (stored in place and kept in shared memory)
//   step C  P_sub = tril(W^T C_sub)  (K = ROWS), stored to its own partial slot (s per tile)
template <int RT>
__device__ __forceinline__ void pr_phase1_units(const PanelParams& p, double* sm, int64_t nunits, int s) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // warp -> (wm, wn): the SM sub-partition (warp & 3) gets one column group from each
  // end, so the triangular work of step A is balanced across sub-partitions
  const int wm = warp >> 2, wn = wm == 0 ? (warp & 3) : 3 - (warp & 3), g = lane >> 2, t = lane & 3;
  const int w = p.w;
  constexpr int ROWS = 16 * RT;  // rows of a sub-tile; each warp owns ROWS / 2 of them in step A
  const int64_t nsl = int64_t(p.tiles) * s;
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t b = u / nsl;
    const int st_ = int(u - b * nsl), tl = st_ / s, h = st_ - tl * s;
    const int r0 = p.k + 128 * tl + ROWS * h;
    double* Cb = optr_w<double>(p.A, b) + r0 + int64_t(p.j) * p.A.ld;     // Cbar sub-tile (ROWS x w)
    const double* Ct = optr<double>(p.L, b) + r0 + int64_t(p.j) * p.L.ld;  // C tile
    const double* Di = p.Dinv + b * p.dstride;

    // ---------------- step A: W = Cbar_t D^{-1} ----------------
    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) acc[i][jj][0] = acc[i][jj][1] = 0.0;
    const int nkc = (w + PR_BK - 1) / PR_BK;
    auto load_a = [&](int st, int kc) {
      double* as = sm + st * (PR_A_SIZE + PR_B_SIZE);
      double* bs = as + PR_A_SIZE;
      for (int e = tid; e < PR_BK * ROWS; e += PR_THREADS) {
        const int m = e % ROWS, kx = e / ROWS;  // A: Cbar[m, kc + kx]
        const int kk = kc * PR_BK + kx;
        cp_async8(as + kx * PR_KM_PITCH + m, Cb + m + int64_t(min(kk, w - 1)) * p.A.ld, kk < w);
      }
      for (int e = tid; e < PR_BK * 128; e += PR_THREADS) {
        const int kx = e % PR_BK, nn = e / PR_BK;  // B: Dinv[kc + kx, nn]
        const int kk = kc * PR_BK + kx;
        const bool ok = kk < w && nn < w;
        cp_async8(bs + nn * PR_NK_PITCH + kx, Di + (ok ? kk + int64_t(nn) * p.dld : 0), ok);
      }
    };
#pragma unroll 1
    for (int q = 0; q < PR_STAGES - 1; ++q) {
      if (q < nkc) load_a(q, q);
      cp_async_commit();
    }
#pragma unroll 1
    for (int kc = 0; kc < nkc; ++kc) {
      cp_async_wait<PR_STAGES - 2>();
      __syncthreads();
      if (kc + PR_STAGES - 1 < nkc) load_a((kc + PR_STAGES - 1) % PR_STAGES, kc + PR_STAGES - 1);
      cp_async_commit();
      // D^{-1}[kk, c] = 0 for kk < c: this chunk reaches columns c <= kc*16 + 15 only
      if (kc * PR_BK + PR_BK - 1 >= wn * 32) {
        const double* as = sm + (kc % PR_STAGES) * (PR_A_SIZE + PR_B_SIZE);
        const double* bs = as + PR_A_SIZE;
#pragma unroll
        for (int kq = 0; kq < PR_BK / 4; ++kq) {
          const int kx = kq * 4 + t;
          double a[RT], bb[4];
#pragma unroll
          for (int i = 0; i < RT; ++i) a[i] = as[kx * PR_KM_PITCH + wm * (ROWS / 2) + i * 8 + g];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) bb[jj] = bs[(wn * 32 + jj * 8 + g) * PR_NK_PITCH + kx];
#pragma unroll
          for (int i = 0; i < RT; ++i)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) dmma884(acc[i][jj][0], acc[i][jj][1], a[i], bb[jj]);
        }
      }
    }
    cp_async_wait_all();
    __syncthreads();  // stage buffers dead: W and the step C stages alias them
    double* Ws = sm;
    double* Cs = sm + 128 * PR_W_PITCH;
#pragma unroll
    for (int i = 0; i < RT; ++i)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = wm * (ROWS / 2) + i * 8 + g;
          const int c = wn * 32 + jj * 8 + 2 * t + e;
          Ws[r + c * PR_W_PITCH] = acc[i][jj][e];  // columns >= w are exactly 0
          if (c < w) Cb[r + int64_t(c) * p.A.ld] = acc[i][jj][e];
        }

    // ---------------- step C: P_t = tril(W^T C_t) ----------------
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) acc[i][jj][0] = acc[i][jj][1] = 0.0;
    auto load_c = [&](int st, int rc) {
      double* bs = Cs + st * PR_B_SIZE;
      for (int e = tid; e < PR_BK * 128; e += PR_THREADS) {
        const int kx = e % PR_BK, nn = e / PR_BK;  // B: C[rc*16 + kx, nn]
        const bool ok = nn < w;
        cp_async8(bs + nn * PR_NK_PITCH + kx, Ct + (rc * PR_BK + kx) + int64_t(ok ? nn : 0) * p.L.ld, ok);
      }
    };
    constexpr int NRC = ROWS / PR_BK;  // K of step C = the sub-tile's rows
#pragma unroll 1
    for (int q = 0; q < PR_STAGES - 1; ++q) {
      if (q < NRC) load_c(q, q);
      cp_async_commit();
    }
    const bool active = wm * 64 + 63 >= wn * 32;  // some a >= b in this warp's tile
#pragma unroll 1
    for (int rc = 0; rc < NRC; ++rc) {
      cp_async_wait<PR_STAGES - 2>();
      __syncthreads();
      if (rc + PR_STAGES - 1 < NRC) load_c((rc + PR_STAGES - 1) % PR_STAGES, rc + PR_STAGES - 1);
      cp_async_commit();
      if (active) {
        const double* bs = Cs + (rc % PR_STAGES) * PR_B_SIZE;
#pragma unroll
        for (int kq = 0; kq < PR_BK / 4; ++kq) {
          const int kx = kq * 4 + t;
          double a[8], bb[4];
#pragma unroll
          for (int i = 0; i < 8; ++i) a[i] = Ws[(wm * 64 + i * 8 + g) * PR_W_PITCH + rc * PR_BK + kx];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) bb[jj] = bs[(wn * 32 + jj * 8 + g) * PR_NK_PITCH + kx];
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) dmma884(acc[i][jj][0], acc[i][jj][1], a[i], bb[jj]);
        }
      }
    }
    cp_async_wait_all();
    double* slot = p.part + u * int64_t(128 * 128);
    if (active) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = wm * 64 + i * 8 + g;
            const int c = wn * 32 + jj * 8 + 2 * t + e;
            if (r >= c) __stcg(slot + r + c * 128, acc[i][jj][e]);
          }
    }
    __syncthreads();  // before the next tile reuses the shared memory
  }

}

__global__ void __launch_bounds__(PR_THREADS, 1) k_panel_rev(const PanelParams p) {
  extern __shared__ __align__(16) unsigned char smem_pr[];
  double* sm = reinterpret_cast<double*>(smem_pr);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int w = p.w;
  const int64_t units = p.batch * p.tiles;

  // ---------------- phase 0 (small panels): Cbar -= M L[k:n, j:k], M = T + T^T ----------------
  // The left-looking trailing update of symm_ll.cuh for panels with few row tiles, done here
  // in 32 x 32 output tiles over the grid (K = p) instead of a separate stream-K launch:
  // M(r, c) = T(r, c) below the diagonal blocks, T(c, r) above them, S on them.
  if (p.symm && !(p.dbg_skip & 8)) {
    const int64_t u0 = units * 16;
    const int pk = p.n - p.k;
    for (int64_t u = blockIdx.x; u < u0; u += gridDim.x) {
      const int64_t bt = u >> 4;
      const int64_t b = bt / p.tiles;
      const int tl = int(bt - b * p.tiles);
      const int ti = int(u & 15) >> 2, tj = int(u & 3);
      const int r0 = p.k + 128 * tl + 32 * ti, c0 = 32 * tj;
      const int rb = 128 * tl;  // row block (relative to k) of this output tile
      const double* Ab = optr<double>(p.A, b);
      const double* Lb = optr<double>(p.L, b) + p.k + int64_t(p.j) * p.L.ld;
      const double* Sb = p.Sall + b * p.s_stride + int64_t(p.nblk - (p.n - (p.k + rb)) / 128) * p.s_blk;
      double* Cb = optr_w<double>(p.A, b) + r0 + int64_t(p.j) * p.A.ld;
      pr_tile32kx(
          sm, pk,
          [&](int m, int kk) -> const double* {  // M(r0 + m, k + kk)
            const int r = r0 + m - p.k, cblk = kk & ~127;
            if (cblk < rb) return Ab + (r0 + m) + int64_t(p.k + kk) * p.A.ld;        // T(r, c)
            if (cblk > rb) return Ab + (p.k + kk) + int64_t(r0 + m) * p.A.ld;        // T(c, r)
            return Sb + (r - rb) + int64_t(kk - rb) * p.s_ld;                         // S block
          },
          [&](int kk, int n) -> const double* { return c0 + n < w ? Lb + kk + int64_t(c0 + n) * p.L.ld : nullptr; },
          [&](int m, int n, double v) {
            if (c0 + n < w) Cb[m + int64_t(c0 + n) * p.A.ld] -= v;
          },
          [&](int kb) { return kb <= rb; },  // T(r, c) / S columns: contiguous along m
          [](int) { return false; });
    }
    __threadfence();
    cooperative_groups::this_grid().sync();
  }

  // few tiles (early steps): split every tile's work into 32 x 32 tiles over the grid --
  // 1a: W = Cbar D^{-1} (16 tiles per 128-row tile, staged), grid sync, 1b: the lower
  // 32 x 32 tiles of P_t = W^T C (K = the tile's 128 rows) and W copied back in place
  // phase 1 split: with few tiles the 128-row tiles are cut into 64- or 32-row sub-tiles so that
  // more SMs share the work (p.split_max); the 32 x 32-tile path below is the alternative for the
  // fewest tiles (p.split_max < 4)
  const bool small = p.split_max < 4 && units * 4 <= int64_t(gridDim.x);
  const int split = small                                                 ? 1
                    : p.split_max >= 4 && units * 4 <= int64_t(gridDim.x) ? 4
                    : p.split_max >= 2 && units * 2 <= int64_t(gridDim.x) ? 2
                                                                          : 1;
  if (small && !(p.dbg_skip & 1)) {
    const int64_t ua = units * 16;
    for (int64_t u = blockIdx.x; u < ua; u += gridDim.x) {
      const int64_t bt = u >> 4;
      const int64_t b = bt / p.tiles;
      const int tl = int(bt - b * p.tiles);
      const int ti = int(u & 15) >> 2, tj = int(u & 3);
      const int r0 = p.k + 128 * tl + 32 * ti, c0 = 32 * tj;
      const double* Cb = optr<double>(p.A, b) + r0 + int64_t(p.j) * p.A.ld;
      const double* Di = p.Dinv + b * p.dstride;
      double* st = p.Wst + bt * (128 * 128) + 32 * ti;  // staging, ld 128
      pr_tile32kx(
          sm, 128, [&](int m, int k) -> const double* { return k < w ? Cb + m + int64_t(k) * p.A.ld : nullptr; },
          [&](int k, int n) -> const double* {  // D^{-1}(k, c0 + n), zero above the diagonal
            const int cc = c0 + n;
            return (k < w && cc < w && k >= cc) ? Di + k + int64_t(cc) * p.dld : nullptr;
          },
          [&](int m, int n, double v) { __stcg(st + m + (c0 + n) * 128, v); }, [](int) { return true; },
          [](int) { return false; });
    }
    __threadfence();
    cooperative_groups::this_grid().sync();
    const int64_t ub = units * 11;  // 10 lower P_t tiles + 1 copy-back unit per 128-row tile
    for (int64_t u = blockIdx.x; u < ub; u += gridDim.x) {
      const int64_t bt = u / 11;
      const int lt = int(u - bt * 11);
      const int64_t b = bt / p.tiles;
      const int tl = int(bt - b * p.tiles);
      const int r0 = p.k + 128 * tl;
      const double* Wb = p.Wst + bt * (128 * 128);
      if (lt == 10) {  // W -> Abar (in place of Cbar)
        double* Cb = optr_w<double>(p.A, b) + r0 + int64_t(p.j) * p.A.ld;
        for (int e = tid; e < 128 * w; e += PR_THREADS) {
          const int r = e & 127, c = e >> 7;
          Cb[r + int64_t(c) * p.A.ld] = __ldcg(Wb + e);
        }
        continue;
      }
      int ti = 0, tj = 0;  // lower tile lt -> (ti >= tj)
      {
        int r = lt;
        while (r > ti) r -= ++ti;
        tj = r;
      }
      const double* Ct = optr<double>(p.L, b) + r0 + int64_t(p.j) * p.L.ld;
      double* slot = p.part + bt * int64_t(128 * 128);
      const int a0 = 32 * ti, c0 = 32 * tj;
      pr_tile32(
          sm, [&](int m, int k) -> const double* { return (a0 + m < w) ? Wb + k + (a0 + m) * 128 : nullptr; },
          [&](int k, int n) -> const double* { return (c0 + n < w) ? Ct + k + int64_t(c0 + n) * p.L.ld : nullptr; },
          [&](int m, int n, double v) {
            const int a = a0 + m, cc = c0 + n;
            if (a >= cc) __stcg(slot + a + cc * 128, v);
          });
    }
  }

  if (!small && !(p.dbg_skip & 1)) {
    if (split == 4) pr_phase1_units<2>(p, sm, units * 4, 4);
    else if (split == 2) pr_phase1_units<4>(p, sm, units * 2, 2);
    else pr_phase1_units<8>(p, sm, units, 1);
  }

  // ---------------- phase 2: Dbar -= sum_t P_t (lower triangle) ----------------
  __threadfence();
  cooperative_groups::this_grid().sync();
  // 8 lanes per element (a warp takes 4 elements per round), each lane two independent
  // chains over the tiles; fixed combination tree -> bitwise deterministic.  The grid is
  // always every co-resident CTA (CTAs without a tile join here), so few tiles still
  // spread over the whole GPU.
  const int64_t nwarps = int64_t(gridDim.x) * (PR_THREADS / 32);
  const int64_t gw = int64_t(blockIdx.x) * (PR_THREADS / 32) + warp;
  const int64_t ntri = int64_t(w) * (w + 1) / 2;
  const int64_t nel = ntri * p.batch;  // lower-triangle entries (a >= c), column-packed
  const int nsl = p.tiles * split;     // P partial slots per matrix
  const int q = lane & 7;
  for (int64_t wb = gw * 4; wb < nel && !(p.dbg_skip & 2); wb += nwarps * 4) {
    const int64_t el = wb + (lane >> 3);
    const bool on = el < nel;
    int64_t b = 0;
    int a = 0, c = 0;
    if (on) {
      b = el / ntri;
      const int rem = int(el - b * ntri);
      // column-packed: column c starts at off(c) = c*w - c*(c-1)/2 and holds w - c entries
      const double tw = 2.0 * w + 1.0;
      c = int((tw - sqrt(tw * tw - 8.0 * rem)) * 0.5);
      c = max(0, min(c, w - 1));
      while (c > 0 && c * w - c * (c - 1) / 2 > rem) --c;
      while (c + 1 < w && (c + 1) * w - (c + 1) * c / 2 <= rem) ++c;
      a = c + (rem - (c * w - c * (c - 1) / 2));
    }
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    if (on) {
      const double* pb = p.part + b * nsl * int64_t(128 * 128) + a + c * 128;
      constexpr int64_t TS = 128 * 128;
      int tl = q;
      for (; tl + 24 < nsl; tl += 32) {  // four independent loads in flight per lane
        const double x0 = __ldcg(pb + tl * TS), x1 = __ldcg(pb + (tl + 8) * TS);
        const double x2 = __ldcg(pb + (tl + 16) * TS), x3 = __ldcg(pb + (tl + 24) * TS);
        s0 += x0, s1 += x1, s2 += x2, s3 += x3;
      }
      if (tl < nsl) s0 += __ldcg(pb + tl * TS);
      if (tl + 8 < nsl) s1 += __ldcg(pb + (tl + 8) * TS);
      if (tl + 16 < nsl) s2 += __ldcg(pb + (tl + 16) * TS);
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

  // ---------------- phase 3: Dbar <- chol_unblocked_rev(D, Dbar) by Eq. 10 ----------------
  // The paper's own blocked implementation updates diagonal blocks with Eq. 10
  // (Eq. 10 = PAPER.md:248-256):
  //   P = Phi(D^T Dbar),  Y = D^{-T} (P + P^T) D^{-1},  tril(Dbar) = Phi(Y),  S = Y (= Dbar + Dbar^T)
  // as three 128 x 128 products in 32 x 32 tiles over the grid (grid syncs between them).
  // D^{-1} is the block inverse k_trinv already made for the panel solve.
  __threadfence();
  cooperative_groups::this_grid().sync();
  const int64_t u3 = (p.dbg_skip & 4) ? 0 : p.batch * 16;
  // 3a (lower tiles): X = P + P^T, P = Phi(D^T Dbar), written symmetric (D, Dbar read as
  // lower triangles; X(a, a) = (D^T Dbar)(a, a), X(a, c) = X(c, a) = P(a, c) for a > c)
  for (int64_t u = blockIdx.x; u < u3; u += gridDim.x) {
    const int64_t b = u >> 4;
    const int ti = int(u & 15) >> 2, tj = int(u & 3);
    if (ti < tj) continue;  // uniform per CTA
    const double* Lb = optr<double>(p.L, b) + p.j + int64_t(p.j) * p.L.ld;
    const double* Ab = optr<double>(p.A, b) + p.j + int64_t(p.j) * p.A.ld;
    double* Xb = p.Pws + b * 128 * 128;
    const int a0 = 32 * ti, c0 = 32 * tj;
    pr_tile32(
        sm,
        [&](int m, int k) -> const double* {  // A(m, k) = D(k, a0 + m)
          const int a = a0 + m;
          return (k < w && a < w && k >= a) ? Lb + k + int64_t(a) * p.L.ld : nullptr;
        },
        [&](int k, int n) -> const double* {  // B(k, n) = Dbar(k, c0 + n)
          const int cc = c0 + n;
          return (k < w && cc < w && k >= cc) ? Ab + k + int64_t(cc) * p.A.ld : nullptr;
        },
        [&](int m, int n, double v) {
          const int a = a0 + m, cc = c0 + n;
          if (a > cc) {
            Xb[a + cc * 128] = v;
            Xb[cc + a * 128] = v;
          } else if (a == cc) {
            Xb[a + cc * 128] = v;
          }
        });
  }
  __threadfence();
  cooperative_groups::this_grid().sync();
  // 3b: Z = X D^{-1}   (A(m, k) = X(a0 + m, k) = X(k, a0 + m): a contiguous column)
  for (int64_t u = blockIdx.x; u < u3; u += gridDim.x) {
    const int64_t b = u >> 4;
    const int ti = int(u & 15) >> 2, tj = int(u & 3);
    const double* Xb = p.Pws + b * 128 * 128;
    const double* Di = p.Dinv + b * p.dstride;
    double* Zb = p.Zws + b * 128 * 128;
    const int a0 = 32 * ti, c0 = 32 * tj;
    pr_tile32(
        sm,
        [&](int m, int k) -> const double* {
          return (k < w && a0 + m < w) ? Xb + k + (a0 + m) * 128 : nullptr;
        },
        [&](int k, int n) -> const double* {
          const int cc = c0 + n;
          return (k < w && cc < w) ? Di + k + int64_t(cc) * p.dld : nullptr;
        },
        [&](int m, int n, double v) { Zb[(a0 + m) + (c0 + n) * 128] = v; });
  }
  __threadfence();
  cooperative_groups::this_grid().sync();
  // 3c: Y = D^{-T} Z (lower tiles);  tril(Dbar) = Phi(Y);  S = Y mirrored from its lower triangle
  for (int64_t u = blockIdx.x; u < u3; u += gridDim.x) {
    const int64_t b = u >> 4;
    const int ti = int(u & 15) >> 2, tj = int(u & 3);
    if (ti < tj) continue;  // uniform per CTA
    const double* Di = p.Dinv + b * p.dstride;
    const double* Zb = p.Zws + b * 128 * 128;
    double* Ab = optr_w<double>(p.A, b) + p.j + int64_t(p.j) * p.A.ld;
    double* Sb = p.S ? p.S + b * p.s_stride : nullptr;
    const int a0 = 32 * ti, c0 = 32 * tj;
    pr_tile32(
        sm,
        [&](int m, int k) -> const double* {  // A(m, k) = Dinv(k, a0 + m)
          const int a = a0 + m;
          return (k < w && a < w) ? Di + k + int64_t(a) * p.dld : nullptr;
        },
        [&](int k, int n) -> const double* { return (k < w && c0 + n < w) ? Zb + k + (c0 + n) * 128 : nullptr; },
        [&](int m, int n, double v) {
          const int a = a0 + m, cc = c0 + n;
          if (a < w && cc < w && a >= cc) {
            Ab[a + int64_t(cc) * p.A.ld] = a == cc ? 0.5 * v : v;
            if (Sb) {
              Sb[a + int64_t(cc) * p.s_ld] = v;
              Sb[cc + int64_t(a) * p.s_ld] = v;
            }
          }
        });
  }
}

}  // namespace cd
