// sweep_warp.cuh -- one WARP per matrix, n <= 32: the unblocked reverse / forward
// sweeps of the paper for batches of small matrices (north star (d)).
//
//   reverse: chol_unblocked_rev, PAPER.md:566-578  (j = N..1, five in-place updates)
//   forward: chol_unblocked_fwd, PAPER.md:489-498  (j = 1..N, two in-place updates)
//
// Data path per matrix: lower triangles of L and A stream HBM -> shared memory with
// cp.async (column m read by lanes m..n-1: contiguous, coalesced; the upper triangle
// is never read), then into registers:
//   reverse: lane m holds COLUMN m of L and Abar (the rank-1 update Bbar -= cbar r
//            and the GEMV rbar -= [dbar cbar^T][r;B] are then lane-local; cbar is
//            broadcast through shared memory),
//   forward: lane i holds ROW i of L and Adot (the GEMVs Bdot r^T, B rdot^T are then
//            lane-local; row j is broadcast through shared memory).
// A matrix with n < 32 is embedded as blockdiag(L, I) / (A, 0): the padding adds
// exact zeros only, so results equal the n x n computation.
#pragma once
#include "common.cuh"

namespace cd {

constexpr int SW_PITCH = 33;                 // smem column pitch (odd: conflict-free row & column access)
constexpr int SW_MAT = 32 * SW_PITCH;        // elements per staged matrix
constexpr int SW_WPB = 4;                    // warps (matrices in flight) per CTA

template <typename T>
constexpr size_t sweep_warp_smem() {
  return size_t(SW_WPB) * (2 * SW_MAT + 32) * sizeof(T);
}

// Stage tril of a column-major n x n matrix into smem s[m*33 + i] (i >= m only).
template <typename T>
__device__ __forceinline__ void sw_stage(const T* __restrict__ g, int64_t ld, int n, T* s, int lane) {
  for (int m = 0; m < n; ++m) {
    if (lane >= m && lane < n) cp_async_zfill<sizeof(T)>(s + m * SW_PITCH + lane, g + lane + m * ld, true);
  }
}

// Write lower triangle (and the requested upper triangle) from smem s[m*33+i] to global.
// mode: 0 TRIL, 1 SYM (mirror), 2 GRAD (off-diagonal halved, mirrored).
template <typename T>
__device__ __forceinline__ void sw_store(T* __restrict__ g, int64_t ld, int n, const T* s, int lane, int mode) {
  for (int m = 0; m < n; ++m) {
    if (lane >= m && lane < n) {
      T v = s[m * SW_PITCH + lane];
      if (mode == 2 && lane != m) v *= T(0.5);
      g[lane + m * ld] = v;
    }
  }
  if (mode != 0) {
    // upper element (m, i), m < i, equals lower (i, m): column i of the upper part, lanes = rows m
    for (int i = 1; i < n; ++i) {
      if (lane < i) {
        T v = s[lane * SW_PITCH + i];
        if (mode == 2) v *= T(0.5);
        g[lane + i * ld] = v;
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(SW_WPB * 32, 3)
    k_sweep_warp_rev(int n, int64_t batch, Opnd Ld, Opnd Ad, int out_mode, int* __restrict__ info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T* sL = sm + w * (2 * SW_MAT + 32);
  T* sA = sL + SW_MAT;
  T* sc = sA + SW_MAT;  // broadcast slot: [dbar, cbar_{j+1..}] of the current column
  const int64_t b = int64_t(blockIdx.x) * SW_WPB + w;
  if (b >= batch) return;
  const T* L = optr<T>(Ld, b);
  T* A = optr_w<T>(Ad, b);

  sw_stage<T>(L, Ld.ld, n, sL, lane);
  sw_stage<T>(A, Ad.ld, n, sA, lane);
  cp_async_wait_all();
  __syncwarp();

  // numerical status: first (1-based) zero / non-finite diagonal entry of L
  {
    bool bad = lane < n && bad_pivot(sL[lane * SW_PITCH + lane]);
    unsigned m = __ballot_sync(0xffffffffu, bad);
    if (info && lane == 0) info[b] = m ? __ffs(m) : 0;
  }

  // lane m <- column m (rows >= m); padding: identity for L, zero for A
  T Lc[32], Ac[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const bool in = (i >= lane) && (i < n) && (lane < n);
    Lc[i] = in ? sL[lane * SW_PITCH + i] : (i == lane ? T(1) : T(0));
    Ac[i] = in ? sA[lane * SW_PITCH + i] : T(0);
  }

#pragma unroll
  for (int j = 31; j >= 0; --j) {
    if (lane == j) {
      // dbar <- dbar - c^T cbar / d ;  [dbar; cbar] <- [dbar; cbar] / d
      T s = T(0);
#pragma unroll
      for (int i = j + 1; i < 32; ++i) s += Lc[i] * Ac[i];
      const T rd = T(1) / Lc[j];
      const T dbar = (Ac[j] - s * rd) * rd;
      Ac[j] = dbar;
      sc[j] = dbar;
#pragma unroll
      for (int i = j + 1; i < 32; ++i) {
        Ac[i] *= rd;
        sc[i] = Ac[i];
      }
    }
    __syncwarp();
    if (lane < j) {
      // rbar <- rbar - [dbar cbar^T][r; B] ;  Bbar <- Bbar - cbar r
      const T r_m = Lc[j];  // L(j, m)
      T s = sc[j] * r_m;
#pragma unroll
      for (int i = j + 1; i < 32; ++i) {
        const T cb = sc[i];
        s += cb * Lc[i];
        Ac[i] -= cb * r_m;
      }
      Ac[j] -= s;
    }
    if (lane == j) Ac[j] *= T(0.5);  // dbar <- dbar / 2
    __syncwarp();
  }

  // registers -> smem (column lane) -> global (coalesced columns)
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i >= lane && lane < n && i < n) sA[lane * SW_PITCH + i] = Ac[i];
  __syncwarp();
  sw_store<T>(A, Ad.ld, n, sA, lane, out_mode);
}

template <typename T>
__global__ void __launch_bounds__(SW_WPB * 32, 3)
    k_sweep_warp_fwd(int n, int64_t batch, Opnd Ld, Opnd Ad, int* __restrict__ info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T* sL = sm + w * (2 * SW_MAT + 32);
  T* sA = sL + SW_MAT;
  T* sc = sA + SW_MAT;  // row j of Adot (rdot, ddot) broadcast slot
  const int64_t b = int64_t(blockIdx.x) * SW_WPB + w;
  if (b >= batch) return;
  const T* L = optr<T>(Ld, b);
  T* A = optr_w<T>(Ad, b);

  sw_stage<T>(L, Ld.ld, n, sL, lane);
  sw_stage<T>(A, Ad.ld, n, sA, lane);
  cp_async_wait_all();
  __syncwarp();
  {
    bool bad = lane < n && bad_pivot(sL[lane * SW_PITCH + lane]);
    unsigned m = __ballot_sync(0xffffffffu, bad);
    if (info && lane == 0) info[b] = m ? __ffs(m) : 0;
  }
  // pad L with identity rows/cols beyond n (in smem, so row j broadcasts see them)
  for (int m = 0; m < 32; ++m) {
    if (lane >= m && (lane >= n || m >= n)) sL[m * SW_PITCH + lane] = (lane == m) ? T(1) : T(0);
  }
  __syncwarp();

  // lane i <- row i (cols <= i)
  T Lr[32], Ar[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    const bool in = (m <= lane) && (lane < n);
    Lr[m] = (m <= lane) ? sL[m * SW_PITCH + lane] : T(0);
    Ar[m] = in ? sA[m * SW_PITCH + lane] : T(0);
  }

#pragma unroll
  for (int j = 0; j < 32; ++j) {
    if (lane == j) {
      // ddot <- (ddot/2 - r rdot^T) / d
      T s = T(0);
#pragma unroll
      for (int m = 0; m < j; ++m) s += Lr[m] * Ar[m];
      const T ddot = (Ar[j] * T(0.5) - s) / Lr[j];
      Ar[j] = ddot;
#pragma unroll
      for (int m = 0; m <= j; ++m) sc[m] = Ar[m];
    }
    __syncwarp();
    if (lane > j) {
      // cdot <- (cdot - Bdot r^T - B rdot^T - c ddot) / d
      T t1 = T(0), t2 = T(0);
#pragma unroll
      for (int m = 0; m < j; ++m) {
        t1 += Ar[m] * sL[m * SW_PITCH + j];  // Bdot r^T : r = L(j, 0:j) (smem broadcast)
        t2 += Lr[m] * sc[m];                 // B rdot^T
      }
      Ar[j] = (Ar[j] - t1 - t2 - Lr[j] * sc[j]) / sL[j * SW_PITCH + j];
    }
    __syncwarp();
  }

#pragma unroll
  for (int m = 0; m < 32; ++m)
    if (m <= lane && lane < n) sA[m * SW_PITCH + lane] = Ar[m];
  __syncwarp();
  sw_store<T>(A, Ad.ld, n, sA, lane, 0);
}

}  // namespace cd
