// gemm_tma.cuh -- TMA-fed, warp-specialised fp64 DMMA GEMM (the Level-3 updates of the
// blocked sweeps) for B200 / sm_100a.
//
//   warp 8        : producer -- one elected lane issues cp.async.bulk.tensor (TMA) loads
//                   of the A and B tiles of every K step into a STAGES-deep ring, each
//                   stage guarded by a full / empty mbarrier pair;
//   warps 0..7    : consumers -- mma.sync.m8n8k4.f64 (DMMA) on 64 x 32 warp tiles of the
//                   128 x 128 CTA tile, operands read from shared memory with
//                   bank-conflict-free pitches (the TMA box is 4 elements wider than the
//                   tile, 132 / 20 doubles, so the shared-memory pitch is 4 mod 16).
//
// beta*Cin is loaded into the accumulators before the main loop (alpha = +-1), so the
// read-modify-write of the trailing updates costs no exposed epilogue latency.  OOB
// rows / columns / K-tails are zero-filled by TMA (the tensor maps are clipped to each
// operand's view).  Same GemmParams semantics as k_gemm (gemm.cuh); split-K partials
// are reduced by k_splitk_reduce.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "gemm.cuh"

namespace cd {

constexpr int TG_STAGES = 4;
constexpr int TG_CONSUMERS = 8;
constexpr int TG_THREADS = (TG_CONSUMERS + 1) * 32;

struct TmaMaps {
  CUtensorMap a[3];
  CUtensorMap b[3];
  int a_shift[3], b_shift[3];  // element shift that made each map's base 16-byte aligned
  int batched;                 // maps are 3-D (rows, cols, batch)
};

template <int TA, int TB>
struct TmaLayout {
  static constexpr int BM = 128, BN = 128, BK = 16;
  static constexpr bool A_KM = TA == 0;  // As[k][m] pitch 132, else As[m][k] pitch 20
  static constexpr int A_PITCH = A_KM ? BM + 4 : BK + 4;
  static constexpr int A_SIZE = A_KM ? BK * (BM + 4) : BM * (BK + 4);
  static constexpr bool B_KN = TB == 1;  // Bs[k][n] pitch 132, else Bs[n][k] pitch 20
  static constexpr int B_PITCH = B_KN ? BN + 4 : BK + 4;
  static constexpr int B_SIZE = B_KN ? BK * (BN + 4) : BN * (BK + 4);
  static constexpr uint32_t STAGE_BYTES = uint32_t(A_SIZE + B_SIZE) * 8u;
  static constexpr size_t SMEM = size_t(TG_STAGES) * (A_SIZE + B_SIZE) * 8 + 2 * TG_STAGES * 8 + 1024;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

template <int TA, int TB>
__global__ void __launch_bounds__(TG_THREADS, 1) k_gemm_tma(const GemmParams p, const __grid_constant__ TmaMaps tm) {
  using Lay = TmaLayout<TA, TB>;
  constexpr int BM = Lay::BM, BN = Lay::BN, BK = Lay::BK;
  extern __shared__ __align__(1024) unsigned char smem_tma[];
  // 1024-byte aligned carve-up: [A stages][B stages][full bars][empty bars]
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_tma) + 1023) & ~uintptr_t(1023));
  double* As = reinterpret_cast<double*>(base);
  double* Bs = As + TG_STAGES * Lay::A_SIZE;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + TG_STAGES * Lay::B_SIZE);
  uint64_t* empty = full + TG_STAGES;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t zb = blockIdx.z;
  const int split = int(zb % p.splits);
  const int64_t b = zb / p.splits;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kt0 = split * p.kt_per_split;
  const int kt1 = min(p.KT, kt0 + p.kt_per_split);
  const int nkt = kt1 - kt0;

  if (tid == 0) {
    for (int s = 0; s < TG_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TG_CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == TG_CONSUMERS) {
    // ---------------- producer ----------------
    if (lane == 0) {
      for (int it = 0; it < nkt; ++it) {
        const int s = it % TG_STAGES;
        if (it >= TG_STAGES) mbar_wait(&empty[s], ((it / TG_STAGES) - 1) & 1);
        const int kt = kt0 + it;
        int sg = 0;
        if (p.nseg > 1 && kt * BK >= p.seg[1].kv0) sg = 1;
        if (p.nseg > 2 && kt * BK >= p.seg[2].kv0) sg = 2;
        const int kl = kt * BK - p.seg[sg].kv0;
        mbar_expect_tx(&full[s], Lay::STAGE_BYTES);
        double* as = As + s * Lay::A_SIZE;
        double* bs = Bs + s * Lay::B_SIZE;
        // A: TA=0 map dims (rows=M, cols=K): coords {m, k}; TA=1 map dims (rows=K, cols=M): {k, m}
        const int ac0 = TA == 0 ? m0 + tm.a_shift[sg] : kl + tm.a_shift[sg];
        const int ac1 = TA == 0 ? kl : m0;
        // B: TB=0 map dims (rows=K, cols=N): {k, n}; TB=1 map dims (rows=N, cols=K): {n, k}
        const int bc0 = TB == 0 ? kl + tm.b_shift[sg] : n0 + tm.b_shift[sg];
        const int bc1 = TB == 0 ? n0 : kl;
        if (tm.batched) {
          tma_load_3d(as, &tm.a[sg], ac0, ac1, int(b), &full[s]);
          tma_load_3d(bs, &tm.b[sg], bc0, bc1, int(b), &full[s]);
        } else {
          tma_load_2d(as, &tm.a[sg], ac0, ac1, &full[s]);
          tma_load_2d(bs, &tm.b[sg], bc0, bc1, &full[s]);
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int wm = warp >> 2, wn = warp & 3, g = lane >> 2, t = lane & 3;
  double acc[8][4][2];
  // D = Cin - sum (alpha = -1, beta = 1) or Cin + sum (alpha = 1, beta = 1): the
  // accumulators start as Cin (raw global loads straight into the accumulator
  // registers, all independent, overlapping the TMA prologue) and the sign of the
  // sum is carried by the B fragments; the epilogue is then pure stores.
  const bool pre = p.splits == 1 && p.beta == 1.0 && (p.alpha == 1.0 || p.alpha == -1.0);
  const double bsign = pre ? p.alpha : 1.0;
  {
    const double* Cp = pre ? optr<double>(p.Cin, b) : nullptr;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = m0 + wm * 64 + i * 8 + g;
          const int c = n0 + wn * 32 + j * 8 + 2 * t + e;
          acc[i][j][e] = (pre && r < p.M && c < p.N) ? __ldcg(Cp + r + int64_t(c) * p.Cin.ld) : 0.0;
        }
  }

  for (int it = 0; it < nkt; ++it) {
    const int s = it % TG_STAGES;
    mbar_wait(&full[s], (it / TG_STAGES) & 1);
    const double* as = As + s * Lay::A_SIZE;
    const double* bs = Bs + s * Lay::B_SIZE;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      const int k = kk * 4 + t;
      double a[8], bb[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int m = wm * 64 + i * 8 + g;
        a[i] = Lay::A_KM ? as[k * Lay::A_PITCH + m] : as[m * Lay::A_PITCH + k];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = wn * 32 + j * 8 + g;
        bb[j] = bsign * (Lay::B_KN ? bs[k * Lay::B_PITCH + n] : bs[n * Lay::B_PITCH + k]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  const double alpha = p.alpha, beta = p.beta;
  double* D = optr_w<double>(p.D, b);
  const double* Cin = (beta != 0.0 && !pre) ? optr<double>(p.Cin, b) : nullptr;
  double* part = p.splits > 1 ? reinterpret_cast<double*>(p.part) + (int64_t(split) * p.batch + b) * int64_t(p.M) * p.N
                              : nullptr;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = m0 + wm * 64 + i * 8 + g;
        const int c = n0 + wn * 32 + j * 8 + 2 * t + e;
        if (r < p.M && c < p.N && (!p.tril || r + p.tril - 1 >= c)) {
          if (part) {
            __stcg(part + r + int64_t(c) * p.M, acc[i][j][e]);
          } else if (pre) {
            __stcg(D + r + int64_t(c) * p.D.ld, acc[i][j][e]);
          } else {
            double v = alpha * acc[i][j][e];
            if (Cin) v += beta * __ldcg(Cin + r + int64_t(c) * p.Cin.ld);
            __stcg(D + r + int64_t(c) * p.D.ld, v);
          }
        }
      }
}

}  // namespace cd
