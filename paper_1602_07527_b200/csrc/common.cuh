// common.cuh -- shared device helpers of libcholdiff (product path; no oracle code).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cd {

// Operand descriptor: a (possibly batched) column-major matrix view.
//   matrix b base = (arr ? arr[b] : base + b*stride) + off      (all in elements)
//   element (i, j) of the view = base_b[i + j*ld]
struct Opnd {
  const void* base;
  const void* const* arr;
  int64_t stride;
  int64_t ld;
  int64_t off;
};

template <typename T>
__device__ __forceinline__ const T* optr(const Opnd& o, int64_t b) {
  const T* p = o.arr ? reinterpret_cast<const T*>(o.arr[b]) : reinterpret_cast<const T*>(o.base) + b * o.stride;
  return p + o.off;
}
template <typename T>
__device__ __forceinline__ T* optr_w(const Opnd& o, int64_t b) {
  return const_cast<T*>(optr<T>(o, b));
}

inline Opnd make_opnd(const void* base, const void* const* arr, int64_t stride, int64_t ld, int64_t row0,
                      int64_t col0) {
  Opnd o;
  o.base = base;
  o.arr = arr;
  o.stride = stride;
  o.ld = ld;
  o.off = row0 + col0 * ld;
  return o;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ bool bad_pivot(T d) {
  return d == T(0) || !isfinite(d);
}

// cp.async with zero-fill (src_bytes = 0 -> destination zero-filled, nothing read)
template <int BYTES>
__device__ __forceinline__ void cp_async_zfill(void* smem_dst, const void* gsrc, bool valid) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  int src_bytes = valid ? BYTES : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(saddr), "l"(gsrc), "n"(BYTES),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// packed column-major lower triangle of an n x n matrix: column m starts at
// m*n - m*(m-1)/2; element (i, m), i >= m, at colstart(m) + (i - m).
__device__ __forceinline__ int tri_col(int n, int m) { return m * n - (m * (m - 1)) / 2; }

}  // namespace cd
