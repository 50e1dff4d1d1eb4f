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
constexpr int CTA_THREADS = 512;      // forward sweep
constexpr int CTA_REV_THREADS = 1024; // reverse sweep: 8 threads per column m

template <typename T>
inline size_t sweep_cta_smem(int n) {
  const size_t tri = size_t(n) * (n + 1) / 2;
  return 2 * tri * sizeof(T) + (CTA_NMAX + 8) * sizeof(T) + 16;
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

// Row-major packed lower triangle: row i holds (i, 0..i) at i(i+1)/2.
__device__ __forceinline__ int tri_row(int i) { return (i * (i + 1)) >> 1; }

template <typename T>
__device__ __forceinline__ void cta_stage_rows(const T* __restrict__ g, int64_t ld, int n, T* s, int warp, int lane,
                                               int nw) {
  for (int m = warp; m < n; m += nw)
    for (int i = m + lane; i < n; i += 32) cp_async_zfill<sizeof(T)>(s + tri_row(i) + m, g + i + int64_t(m) * ld, true);
}

// Reverse sweep, one CTA (8 threads per column m of the rank-1 / GEMV updates).
// Column j's values are kept UNSCALED (u = Abar[j+1:n, j]) while in use; with rd = 1/d:
//   dbar   = (dbar - (c^T u) rd) rd
//   rbar_m -= dbar L(j,m) + rd * sum_i u_i L(i,m)                     (574)
//   Bbar(i,m) -= u_i * (rd L(j,m))                                    (575)
//   Abar(j,j) = dbar / 2                                              (576)
// and cbar = u * rd is applied to every column once, at the end.  The threads
// (8) that own column m = j-1 fold the NEXT column's dot product c^T u into their
// update loop, so each column costs a single __syncthreads().
template <typename T>
__global__ void __launch_bounds__(CTA_REV_THREADS)
    k_sweep_cta_rev(int n, Opnd Ld, Opnd Ad, int out_mode, Opnd Sd, int* __restrict__ info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tri = n * (n + 1) / 2;
  T* sL = reinterpret_cast<T*>(smem_raw);
  T* sA = sL + tri;
  T* sRd = sA + tri;                 // [n] 1 / L_jj
  T* sdb = sRd + CTA_NMAX;           // [2] dbar (before halving)
  int* sbad = reinterpret_cast<int*>(sdb + 4);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int64_t b = blockIdx.x;
  const T* L = optr<T>(Ld, b);
  T* A = optr_w<T>(Ad, b);

  if (tid == 0) *sbad = 0x7fffffff;
  cta_stage_rows<T>(L, Ld.ld, n, sL, warp, lane, nw);
  cta_stage_rows<T>(A, Ad.ld, n, sA, warp, lane, nw);
  cp_async_wait_all();
  __syncthreads();
  for (int t = tid; t < n; t += blockDim.x) {
    const T d = sL[tri_row(t) + t];
    if (bad_pivot(d)) atomicMin(sbad, t + 1);
    sRd[t] = T(1) / d;
  }
  __syncthreads();
  if (tid == 0) {
    if (info) info[b] = (*sbad == 0x7fffffff) ? 0 : *sbad;
    const int c = tri_row(n - 1) + n - 1;  // column n-1: no cbar
    const T db = sA[c] * sRd[n - 1];
    sA[c] = db * T(0.5);
    sdb[(n - 1) & 1] = db;
  }
  __syncthreads();

  const int m = tid >> 3, q = tid & 7;
  for (int j = n - 1; j >= 1; --j) {
    if ((warp << 2) < j) {  // warp owns columns m = 4*warp .. 4*warp+3
      const bool act = m < j;
      const T dbar = sdb[j & 1];
      const T rdj = sRd[j];
      const T Ljm = act ? sL[tri_row(j) + m] : T(0);
      const T wgt = rdj * Ljm;
      const bool nxt = (m == j - 1);
      T acc = T(0), sj = T(0);
      if (act) {
        // rows i = j+1+q, +8, ...; batches of 4 rows with all loads issued first
        for (int i0 = j + 1 + q; i0 < n; i0 += 32) {
          T u[4], Lm[4], a[4];
          int ro[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int i = i0 + 8 * k;
            ro[k] = tri_row(i);
            const bool ok = i < n;
            u[k] = ok ? sA[ro[k] + j] : T(0);
            Lm[k] = ok ? sL[ro[k] + m] : T(0);
            a[k] = ok ? sA[ro[k] + m] : T(0);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            acc += u[k] * Lm[k];
            a[k] -= u[k] * wgt;                  // Bbar <- Bbar - cbar r
            if (nxt) sj += Lm[k] * a[k];
          }
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (i0 + 8 * k < n) sA[ro[k] + m] = a[k];
        }
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      T r = T(0);
      if (act && q == 0) {                       // rbar <- rbar - [dbar cbar^T][r;B]
        r = sA[tri_row(j) + m] - (dbar * Ljm + rdj * acc);
        sA[tri_row(j) + m] = r;
      }
      sj += __shfl_xor_sync(0xffffffffu, sj, 1);
      sj += __shfl_xor_sync(0xffffffffu, sj, 2);
      sj += __shfl_xor_sync(0xffffffffu, sj, 4);
      r = __shfl_sync(0xffffffffu, r, lane & ~7);
      if (nxt && q == 0) {
        // next column j-1:  s = c^T u over rows j..n-1 (row j is the new rbar)
        const T s = sj + Ljm * r;
        const T rdm = sRd[m];
        const int dg = tri_row(m) + m;
        const T db = (sA[dg] - s * rdm) * rdm;
        sA[dg] = db * T(0.5);
        sdb[m & 1] = db;
      }
    }
    __syncthreads();
  }
  // cbar = u * rd for every column (strict lower part)
  for (int e = tid; e < tri; e += blockDim.x) {
    // row i = floor((sqrt(8e+1)-1)/2), col = e - i(i+1)/2
    int i = int((sqrtf(8.f * e + 1.f) - 1.f) * 0.5f);
    while (tri_row(i + 1) <= e) ++i;
    while (tri_row(i) > e) --i;
    const int c = e - tri_row(i);
    if (i > c) sA[e] *= sRd[c];
  }
  __syncthreads();

  for (int mm = warp; mm < n; mm += nw)
    for (int i = mm + lane; i < n; i += 32) {
      T v = sA[tri_row(i) + mm];
      if (out_mode == 2 && i != mm) v *= T(0.5);
      A[i + int64_t(mm) * Ad.ld] = v;
    }
  if (out_mode != 0) {
    for (int i = warp; i < n; i += nw)  // global column i, upper rows mm < i
      for (int mm = lane; mm < i; mm += 32) {
        T v = sA[tri_row(i) + mm];
        if (out_mode == 2) v *= T(0.5);
        A[mm + int64_t(i) * Ad.ld] = v;
      }
  }
  if (Sd.base || Sd.arr) {  // S = Dbar + Dbar^T (diagonal doubled), dense
    T* S = optr_w<T>(Sd, b);
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int i = e % n, c = e / n;
      const T v = (i >= c) ? sA[tri_row(i) + c] : sA[tri_row(c) + i];
      S[i + int64_t(c) * Sd.ld] = (i == c) ? T(2) * v : v;
    }
  }
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
