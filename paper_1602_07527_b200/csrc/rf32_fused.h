// rf32_fused.h -- internal interface (between choldiff.cu and rf32_fused.cu) of the fused
// per-matrix fp32 batched sweeps (SURVEY §8 row a15, configs[3]).  Not part of the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace cd {

// mode bit 0: reverse sweep (tril(Abar) = Lbar -> tril(Sigma_bar)), bit 1: forward sweep
// (tril(Adot) = tril(Sigma_dot) -> L_dot), both in place, column-major, fp32.
struct RF32Call {
  int mode;
  int n;
  int64_t batch;
  const float* L;
  int64_t ldl, sL;
  float* Ab;
  int64_t lda, sA;
  float* Ad;
  int64_t ldd, sD;
};

// true when the fused kernel handles this call: 128 < n <= 512, n % 64 == 0, 16-byte aligned
// bases, leading dimensions and batch strides multiples of 4 elements
bool rf32_fused_supported(const RF32Call& c);
// device workspace (bytes): the diagonal-block inverses, the symmetric diagonal blocks
// S_J = Dbar_J + Dbar_J^T and the tf32-rounded shadows L_r, T_r, Ldot_r
size_t rf32_fused_ws(int n, int64_t batch);
// enqueue on `st`: the block inverses (k_rf_trinv) then the fused sweeps (k_rf32).  Returns
// cudaSuccess or the launch error; *launches += kernels enqueued.
cudaError_t rf32_fused_launch(const RF32Call& c, void* ws, cudaStream_t st, int sms, int64_t* launches);

// The layered fp32 schedule's diagonal-block update of one 64-wide panel for every matrix of a batch
// (rev: Eq. 10 -> tril(Dbar), S = Dbar + Dbar^T dense; fwd: Eq. 8 -> tril(Ddot), S = tril(Ddot) with
// zeros above; S may be null), given the block inverses (64 x 64, ld 64, batch stride dstride).
// A / L / S point at the diagonal block of matrix 0.
cudaError_t rf32_diag64(bool rev, int64_t batch, const float* L, int64_t ldl, int64_t sL, float* A, int64_t lda,
                        int64_t sA, const float* Dinv, int64_t dstride, float* S, int64_t lds, int64_t sS,
                        cudaStream_t st);

// The same for 128-wide panels (the block's own sweep as two 64-wide steps, k_rf_diag128): Dinv
// points at the 128 x 128 inverse of the block (ld ldi); S (optional) receives Dbar + Dbar^T (rev) /
// tril(Ddot) with zeros above (fwd), 128 x 128.
cudaError_t rf32_diag128(bool rev, int64_t batch, const float* L, int64_t ldl, int64_t sL, float* A, int64_t lda,
                         int64_t sA, const float* Dinv, int64_t ldi, int64_t dstride, float* S, int64_t lds,
                         int64_t sS, cudaStream_t st);
// Complete the 128-wide block inverses (128 x 128 each, ld 128, n / 128 per matrix, consecutive)
// whose 64-wide diagonal blocks are in place: lower-left block from L, upper-right zero.
cudaError_t rf32_inv128(int n, int64_t batch, const float* L, int64_t ldl, int64_t sL, float* Dinv, cudaStream_t st);
// all 128-wide inverses of the layered fp32 route in one launch (recursive doubling, 3xTF32 products)
cudaError_t rf32_trinv128(int n, int64_t batch, const float* L, int64_t ldl, int64_t sL, float* Dinv, cudaStream_t st);

}  // namespace cd
