// sweep_cta.cuh -- one CTA per matrix / diagonal block, n <= CTA_NMAX: the unblocked
// sweeps with both lower triangles resident in shared memory (north star (a):
// "shared-memory-resident diagonal-block kernel ... with warp-shuffle reductions").
//
// Used (i) for single / batched matrices with 32 < n <= CTA_NMAX and (ii) as the
// diagonal-block routine of the blocked sweeps (PAPER.md:698 `chol_unblocked_rev(D,
// Dbar)`, PAPER.md:662 `chol_unblocked_fwd(D, Ddot)`).
//
// Reverse: for each column j = n-1..1 one __syncthreads():
//   all warps apply  rbar <- rbar - [dbar cbar^T][r;B]  and  Bbar <- Bbar - cbar r
//   column-by-column (warp per column m < j, lanes over rows i > j, warp-shuffle
//   reduction for rbar_m); the warp that owns column j-1 does it first and then
//   immediately performs the next column's  dbar <- dbar - c^T cbar/d,
//   [dbar; cbar] <- [dbar; cbar]/d,  dbar <- dbar/2  (lines 572-573, 576).
// Forward, right-looking form: after column j is
//   final, its contribution  Bdot r^T + B rdot^T  to every later column is
//   subtracted at once (a rank-2 update of the trailing triangle), so each column
//   needs one barrier and no reductions; the sums are those of line 496 reordered.
#pragma once
#include "common.cuh"

namespace cd {

constexpr int CTA_NMAX = 128;
constexpr int CTA_THREADS = 512;

template <typename T>
inline size_t sweep_cta_smem(int n) {
  const size_t tri = size_t(n) * (n + 1) / 2;
  return 2 * tri * sizeof(T) + 4 * sizeof(T) + 16;
}

template <typename T>
__device__ __forceinline__ void cta_stage(const T* __restrict__ g, int64_t ld, int n, T* s, int warp, int lane,
                                          int nw) {
  for (int m = warp; m < n; m += nw) {
    const int cs = tri_col(n, m);
    for (int i = m + lane; i < n; i += 32) cp_async_zfill<sizeof(T)>(s + cs + i - m, g + i + int64_t(m) * ld, true);
  }
}

// Diagonal check -> smallest bad 1-based index (0 if none), block-wide.
template <typename T>
__device__ __forceinline__ void cta_info(const T* sL, int n, int* sbad, int* info, int64_t b) {
  for (int t = threadIdx.x; t < n; t += blockDim.x)
    if (bad_pivot(sL[tri_col(n, t)])) atomicMin(sbad, t + 1);
  __syncthreads();
  if (threadIdx.x == 0 && info) info[b] = (*sbad == 0x7fffffff) ? 0 : *sbad;
}

// S = Dbar + Dbar^T of the final tril(Dbar) (diagonal doubled), dense, for the
// blocked reverse's  Rbar -= (Dbar + Dbar^T) R  (reading R2).
template <typename T>
__device__ __forceinline__ void cta_write_sym2(T* S, int64_t lds, int n, const T* sA) {
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e % n, m = e / n;
    T v;
    if (i > m) v = sA[tri_col(n, m) + i - m];
    else if (i < m) v = sA[tri_col(n, i) + m - i];
    else v = T(2) * sA[tri_col(n, m)];
    S[i + int64_t(m) * lds] = v;
  }
}

template <typename T>
__global__ void __launch_bounds__(CTA_THREADS)
    k_sweep_cta_rev(int n, Opnd Ld, Opnd Ad, int out_mode, Opnd Sd, int* __restrict__ info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tri = n * (n + 1) / 2;
  T* sL = reinterpret_cast<T*>(smem_raw);
  T* sA = sL + tri;
  T* sdb = sA + tri;  // [2] dbar (before halving) of the current / next column
  int* sbad = reinterpret_cast<int*>(sdb + 4);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t b = blockIdx.x;
  const T* L = optr<T>(Ld, b);
  T* A = optr_w<T>(Ad, b);

  if (threadIdx.x == 0) *sbad = 0x7fffffff;
  cta_stage<T>(L, Ld.ld, n, sL, warp, lane, nw);
  cta_stage<T>(A, Ad.ld, n, sA, warp, lane, nw);
  cp_async_wait_all();
  __syncthreads();
  cta_info<T>(sL, n, sbad, info, b);

  // column n-1: no cbar; dbar <- dbar/d, then /2
  if (threadIdx.x == 0) {
    const int cs = tri_col(n, n - 1);
    const T db = sA[cs] / sL[cs];
    sA[cs] = db * T(0.5);
    sdb[(n - 1) & 1] = db;
  }
  __syncthreads();

  for (int j = n - 1; j >= 1; --j) {
    const int csj = tri_col(n, j);
    const T dbar = sdb[j & 1];
    T cb[CTA_NMAX / 32];
#pragma unroll
    for (int u = 0; u < CTA_NMAX / 32; ++u) {
      const int i = j + 1 + lane + 32 * u;
      cb[u] = (i < n) ? sA[csj + i - j] : T(0);
    }
    // largest m <= j-1 owned by this warp (owner of m is m % nw)
    const int jm1 = j - 1;
    const int mtop = jm1 - (((jm1 - warp) % nw) + nw) % nw;
    for (int m = mtop; m >= 0; m -= nw) {
      const int csm = tri_col(n, m);
      const T r_m = sL[csm + j - m];  // L(j, m)
      T acc = T(0);
#pragma unroll
      for (int u = 0; u < CTA_NMAX / 32; ++u) {
        const int i = j + 1 + lane + 32 * u;
        if (i < n) {
          acc += cb[u] * sL[csm + i - m];           // [cbar^T] B
          sA[csm + i - m] -= cb[u] * r_m;          // Bbar <- Bbar - cbar r
        }
      }
      acc = warp_sum(acc);
      if (lane == 0) sA[csm + j - m] -= dbar * r_m + acc;  // rbar <- rbar - [dbar cbar^T][r;B] (574)
      if (m == jm1) {
        // next column (j-1): dbar <- dbar - c^T cbar/d; [dbar;cbar] /= d; dbar/2 (572-573, 576)
        __syncwarp();
        const int jj = jm1;
        T s = T(0);
        for (int i = jj + 1 + lane; i < n; i += 32) s += sL[csm + i - jj] * sA[csm + i - jj];
        s = warp_sum(s);
        const T rd = T(1) / sL[csm];
        const T db = (sA[csm] - s * rd) * rd;
        for (int i = jj + 1 + lane; i < n; i += 32) sA[csm + i - jj] *= rd;
        if (lane == 0) {
          sA[csm] = db * T(0.5);
          sdb[jj & 1] = db;
        }
      }
    }
    __syncthreads();
  }

  // write back tril (and the requested mirror) ; optional S for the blocked driver
  for (int m = warp; m < n; m += nw) {
    const int cs = tri_col(n, m);
    for (int i = m + lane; i < n; i += 32) {
      T v = sA[cs + i - m];
      if (out_mode == 2 && i != m) v *= T(0.5);
      A[i + int64_t(m) * Ad.ld] = v;
    }
  }
  if (out_mode != 0) {
    for (int i = warp; i < n; i += nw)      // global column i, upper rows m < i
      for (int m = lane; m < i; m += 32) {
        T v = sA[tri_col(n, m) + i - m];
        if (out_mode == 2) v *= T(0.5);
        A[m + int64_t(i) * Ad.ld] = v;
      }
  }
  if (Sd.base || Sd.arr) cta_write_sym2<T>(optr_w<T>(Sd, b), Sd.ld, n, sA);
}

// Forward. Optionally writes a clean dense copy of tril(Ldot) (upper zero) to Dd,
// the operand of  Cdot <- (Cdot - C Ddot^T) D^{-T}.
template <typename T>
__global__ void __launch_bounds__(CTA_THREADS)
    k_sweep_cta_fwd(int n, Opnd Ld, Opnd Ad, Opnd Dd, int* __restrict__ info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tri = n * (n + 1) / 2;
  T* sL = reinterpret_cast<T*>(smem_raw);
  T* sA = sL + tri;
  int* sbad = reinterpret_cast<int*>(sA + tri + 4);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t b = blockIdx.x;
  const T* L = optr<T>(Ld, b);
  T* A = optr_w<T>(Ad, b);
  T* Dc = (Dd.base || Dd.arr) ? optr_w<T>(Dd, b) : nullptr;

  if (threadIdx.x == 0) *sbad = 0x7fffffff;
  cta_stage<T>(L, Ld.ld, n, sL, warp, lane, nw);
  cta_stage<T>(A, Ad.ld, n, sA, warp, lane, nw);
  cp_async_wait_all();
  __syncthreads();
  cta_info<T>(sL, n, sbad, info, b);

  for (int j = 0; j < n; ++j) {
    const int csj = tri_col(n, j);
    const T d = sL[csj];
    const T rd = T(1) / d;
    const T ddot = sA[csj] * T(0.5) * rd;  // (pending ddot)/2 / d
    // final column j: cdot_i = (pending_i - c_i ddot) / d
    for (int i = j + threadIdx.x; i < n; i += blockDim.x) {
      const T v = (i == j) ? ddot : (sA[csj + i - j] - sL[csj + i - j] * ddot) * rd;
      A[i + int64_t(j) * Ad.ld] = v;
      if (Dc) Dc[i + int64_t(j) * Dd.ld] = v;
    }
    if (Dc)
      for (int i = threadIdx.x; i < j; i += blockDim.x) Dc[i + int64_t(j) * Dd.ld] = T(0);
    // trailing rank-2 update: pending(i, jj) -= cdot_i L(jj, j) + L(i, j) cdot_jj, i >= jj > j
    for (int jj = j + 1 + warp; jj < n; jj += nw) {
      const int csjj = tri_col(n, jj);
      const T Ljj = sL[csj + jj - j];
      const T cjj = (sA[csj + jj - j] - Ljj * ddot) * rd;
      for (int i = jj + lane; i < n; i += 32) {
        const T Lij = sL[csj + i - j];
        const T ci = (sA[csj + i - j] - Lij * ddot) * rd;
        sA[csjj + i - jj] -= ci * Ljj + Lij * cjj;
      }
    }
    __syncthreads();
  }
}

}  // namespace cd
