// misc.cuh -- small kernels of the blocked sweeps: block partition, copies, output-
// convention epilogues (Eq. 9 mirror / GRAD) and status.
#pragma once
#include "common.cuh"

namespace cd {

// Partition of [0, n) into diagonal blocks of width nb.
//   reverse: the short block (n mod nb) is the FIRST one
//   forward: the short block is the LAST one
__host__ __device__ inline int nblocks(int n, int nb) { return (n + nb - 1) / nb; }
__host__ __device__ inline void block_range(int n, int nb, bool reverse, int q, int& j0, int& w) {
  const int r = n % nb;
  if (!reverse || r == 0) {
    j0 = q * nb;
    w = min(nb, n - j0);
  } else if (q == 0) {
    j0 = 0;
    w = r;
  } else {
    j0 = r + (q - 1) * nb;
    w = nb;
  }
}

// D(i, j) = S(i, j), M x N per batch entry.
template <typename T>
__global__ void k_copy(int M, int N, int64_t batch, Opnd S, Opnd D) {
  const int64_t MN = int64_t(M) * N, total = MN * batch;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(idx % M), c = int((idx / M) % N);
    const int64_t b = idx / MN;
    optr_w<T>(D, b)[r + int64_t(c) * D.ld] = optr<T>(S, b)[r + int64_t(c) * S.ld];
  }
}

// D(r, c) -= S(r, c) over an M x N view (tril: only r >= c), one matrix -- the distributed
// forward sweep's application of the reduced partial products (include/choldiff.h).
template <typename T>
__global__ void k_sub(int M, int N, Opnd S, Opnd D, int tril) {
  const int64_t total = int64_t(M) * N;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(idx % M), c = int(idx / M);
    if (tril && r < c) continue;
    optr_w<T>(D, 0)[r + int64_t(c) * D.ld] -= optr<T>(S, 0)[r + int64_t(c) * S.ld];
  }
}

// D(i, j) = S(i, j) for i >= j (lower triangles only), n x n per batch entry.
template <typename T>
__global__ void k_copy_tril(int n, int64_t batch, Opnd S, Opnd D) {
  const int64_t nn = int64_t(n) * n, total = nn * batch;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(idx % n), c = int((idx / n) % n);
    if (r < c) continue;
    const int64_t b = idx / nn;
    optr_w<T>(D, b)[r + int64_t(c) * D.ld] = optr<T>(S, b)[r + int64_t(c) * S.ld];
  }
}

// S = tril(A) + tril(A)^T (diagonal doubled), dense n x n; or (clean=1) S = tril(A), upper 0.
template <typename T>
__global__ void k_sym2(int n, int64_t batch, Opnd A, Opnd S, int clean) {
  const int64_t nn = int64_t(n) * n, total = nn * batch;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(idx % n), m = int((idx / n) % n);
    const int64_t b = idx / nn;
    const T* a = optr<T>(A, b);
    T v;
    if (clean) v = (i >= m) ? a[i + int64_t(m) * A.ld] : T(0);
    else if (i > m) v = a[i + int64_t(m) * A.ld];
    else if (i < m) v = a[m + int64_t(i) * A.ld];
    else v = T(2) * a[i + int64_t(i) * A.ld];
    optr_w<T>(S, b)[i + int64_t(m) * S.ld] = v;
  }
}

// Output convention epilogue on the full n x n matrix (mode 1 SYM: mirror lower to
// upper; mode 2 GRAD: halve lower off-diagonals, then mirror).
template <typename T>
__global__ void k_out_mode(int n, int64_t batch, Opnd A, int mode) {
  const int64_t nn = int64_t(n) * n, total = nn * batch;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(idx % n), m = int((idx / n) % n);
    if (i <= m) continue;
    const int64_t b = idx / nn;
    T* a = optr_w<T>(A, b);
    T v = a[i + int64_t(m) * A.ld];
    if (mode == 2) {
      v *= T(0.5);
      a[i + int64_t(m) * A.ld] = v;
    }
    a[m + int64_t(i) * A.ld] = v;
  }
}

// Elementwise steps of the large-n symbolic route (dense n x n per batch entry):
//   mode 0: D = tril(S), upper zero                       (clean triangular operand)
//   mode 1: D = Phi(S) + Phi(S)^T, from tril(S)            (X = P + P^T; D != S)
//   mode 2: D = symmetric from tril(S)                      (Sigma_dot read as symmetric)
//   mode 3: D = Phi(S) (lower, diagonal halved, upper zero)
//   mode 4: tril(D) = Phi(S) (lower only, D's upper untouched)
template <typename T>
__global__ void k_sym_elem(int n, int64_t batch, Opnd S, Opnd D, int mode) {
  const int64_t nn = int64_t(n) * n, total = nn * batch;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(idx % n), c = int((idx / n) % n);
    const int64_t b = idx / nn;
    const T* s = optr<T>(S, b);
    T* d = optr_w<T>(D, b);
    const T lo = r >= c ? s[r + int64_t(c) * S.ld] : s[c + int64_t(r) * S.ld];  // tril(S)(max, min)
    T v;
    switch (mode) {
      case 0: v = r >= c ? lo : T(0); break;
      case 1: case 2: v = lo; break;                 // Phi(S)+Phi(S)^T has the diagonal of S
      case 3: v = r > c ? lo : (r == c ? T(0.5) * lo : T(0)); break;
      default:
        if (r < c) continue;
        v = r > c ? lo : T(0.5) * lo;
    }
    d[r + int64_t(c) * D.ld] = v;
  }
}

// tril(D) = tril(S) converted between element types (n x n per batch entry)
template <typename TS, typename TD>
__global__ void k_convert_tril(int n, int64_t batch, Opnd S, Opnd D) {
  const int64_t nn = int64_t(n) * n, total = nn * batch;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(idx % n), c = int((idx / n) % n);
    if (r < c) continue;
    const int64_t b = idx / nn;
    optr_w<TD>(D, b)[r + int64_t(c) * D.ld] = TD(optr<TS>(S, b)[r + int64_t(c) * S.ld]);
  }
}

// info[b] = first 1-based j with L[j-1, j-1] zero or non-finite, else 0.  One CTA per matrix.
template <typename T>
__global__ void k_diag_info(int n, Opnd Ld, int* __restrict__ info) {
  __shared__ int sbad;
  if (threadIdx.x == 0) sbad = 0x7fffffff;
  __syncthreads();
  const int64_t b = blockIdx.x;
  const T* L = optr<T>(Ld, b);
  for (int j = threadIdx.x; j < n; j += blockDim.x)
    if (bad_pivot(L[j + int64_t(j) * Ld.ld])) atomicMin(&sbad, j + 1);
  __syncthreads();
  if (threadIdx.x == 0) info[b] = (sbad == 0x7fffffff) ? 0 : sbad;
}

}  // namespace cd
