// gemm.cuh -- the Level-3 updates of the blocked sweeps (PAPER.md:634-636, 655-666,
// 689-701) as one tiled GEMM kernel family:
//
//     D = alpha * sum_s op(A_s) op(B_s) + beta * Cin      (up to 3 K-segments s)
//
// with optional lower-triangle output mask (the paper's "only the triangular part
// ... is required"), optional split-K with a
// deterministic fixed-order reduction, batch over grid.z, column-major operands of
// any leading dimension (cp.async zero-fill handles every ragged edge).
//
// fp64: tensor cores via mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4; sm_100 has no
//       tcgen05 fp64 kind).  CTA tile 128x128x16, 8 warps of 64x32, 3-stage
//       cp.async pipeline; shared-memory pitches = 4 (mod 16) doubles so every
//       fragment load is bank-conflict free.
// fp32: FFMA SIMT, 8x8 register micro-tiles, CTA 128x128x32.
#pragma once
#include "common.cuh"

namespace cd {

constexpr int G_BM = 128, G_BN = 128, G_THREADS = 256, G_STAGES = 3;
template <typename T>
struct GBK {
  static constexpr int v = sizeof(T) == 8 ? 16 : 32;
};

struct GemmSeg {
  Opnd A, B;
  int K;    // true K extent of this segment
  int kv0;  // virtual K offset (multiple of BK)
};

struct GemmParams {
  int M, N, nseg, KT, splits, kt_per_split;
  int64_t batch;
  GemmSeg seg[3];
  Opnd Cin;  // beta * Cin (ignored if beta == 0)
  Opnd D;    // output
  double alpha, beta;
  int tril;   // 0: full output; t > 0: write only rows r, cols c with r + (t - 1) >= c
  void* part; // split-K partials: [split][batch][N][M]
  int dtrans; // 1: D and Cin hold the TRANSPOSED result (N x M, ld as given); fp32 TMA epilogue only
};

template <typename T, int TA, int TB>
struct GemmLayout {
  static constexpr bool F64 = sizeof(T) == 8;
  static constexpr int BM = G_BM, BN = G_BN, BK = GBK<T>::v;
  static constexpr bool A_KM = !F64 || TA == 0;  // As[k][m] (else As[m][k])
  static constexpr int A_PITCH = A_KM ? BM + 4 : BK + 4;
  static constexpr int A_SIZE = A_KM ? BK * (BM + 4) : BM * (BK + 4);
  static constexpr bool B_KN = !F64 || TB == 1;  // Bs[k][n] (else Bs[n][k])
  static constexpr int B_PITCH = B_KN ? BN + 4 : BK + 4;
  static constexpr int B_SIZE = B_KN ? BK * (BN + 4) : BN * (BK + 4);
  static constexpr size_t SMEM = size_t(G_STAGES) * (A_SIZE + B_SIZE) * sizeof(T);
};

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <typename T, int TA, int TB>
__global__ void __launch_bounds__(G_THREADS, 1) k_gemm(GemmParams p) {
  using Lay = GemmLayout<T, TA, TB>;
  constexpr int BM = Lay::BM, BN = Lay::BN, BK = Lay::BK;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* As = reinterpret_cast<T*>(smem_raw);
  T* Bs = As + G_STAGES * Lay::A_SIZE;

  const int64_t zb = blockIdx.z;
  const int split = int(zb % p.splits);
  const int64_t b = zb / p.splits;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kt0 = split * p.kt_per_split;
  const int kt1 = min(p.KT, kt0 + p.kt_per_split);
  const int nkt = kt1 - kt0;
  const int tid = threadIdx.x;

  const T* Ab[3];
  const T* Bb[3];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    Ab[s] = s < p.nseg ? optr<T>(p.seg[s].A, b) : nullptr;
    Bb[s] = s < p.nseg ? optr<T>(p.seg[s].B, b) : nullptr;
  }

  auto load_tile = [&](int stage, int kt) {
    int s = 0;
    if (p.nseg > 1 && kt * BK >= p.seg[1].kv0) s = 1;
    if (p.nseg > 2 && kt * BK >= p.seg[2].kv0) s = 2;
    const int kl = kt * BK - p.seg[s].kv0;
    const int K = p.seg[s].K;
    const T* A = Ab[s];
    const T* B = Bb[s];
    const int64_t lda = p.seg[s].A.ld, ldb = p.seg[s].B.ld;
    T* as = As + stage * Lay::A_SIZE;
    T* bs = Bs + stage * Lay::B_SIZE;
#pragma unroll 4
    for (int e = tid; e < BM * BK; e += G_THREADS) {
      int m, k;
      if (TA == 0) { m = e % BM; k = e / BM; } else { k = e % BK; m = e / BK; }
      const bool v = (m0 + m < p.M) && (kl + k < K);
      const T* src = v ? (TA == 0 ? A + (m0 + m) + int64_t(kl + k) * lda : A + (kl + k) + int64_t(m0 + m) * lda) : A;
      T* dst = Lay::A_KM ? as + k * Lay::A_PITCH + m : as + m * Lay::A_PITCH + k;
      cp_async_zfill<sizeof(T)>(dst, src, v);
    }
#pragma unroll 4
    for (int e = tid; e < BK * BN; e += G_THREADS) {
      int n, k;
      if (TB == 0) { k = e % BK; n = e / BK; } else { n = e % BN; k = e / BN; }
      const bool v = (n0 + n < p.N) && (kl + k < K);
      const T* src = v ? (TB == 0 ? B + (kl + k) + int64_t(n0 + n) * ldb : B + (n0 + n) + int64_t(kl + k) * ldb) : B;
      T* dst = Lay::B_KN ? bs + k * Lay::B_PITCH + n : bs + n * Lay::B_PITCH + k;
      cp_async_zfill<sizeof(T)>(dst, src, v);
    }
  };

#pragma unroll
  for (int s = 0; s < G_STAGES - 1; ++s) {
    if (s < nkt) load_tile(s, kt0 + s);
    cp_async_commit();
  }

  const int lane = tid & 31, warp = tid >> 5;

  if constexpr (Lay::F64) {
    // ---------------- fp64: DMMA m8n8k4, warp tile 64 x 32 ----------------
    const int wm = warp >> 2, wn = warp & 3, g = lane >> 2, t = lane & 3;
    double acc[8][4][2];
    // beta * Cin is folded into the accumulators up front (alpha = +-1): the Cin
    // loads are all independent and overlap the pipeline prologue, and the
    // epilogue becomes pure stores (no load-after-store chains on aliased C/D).
    const bool pre = p.splits == 1 && p.beta != 0.0 && (p.alpha == 1.0 || p.alpha == -1.0);
    {
      const double sc = pre ? p.beta / p.alpha : 0.0;
      const T* Cp = pre ? optr<T>(p.Cin, b) : nullptr;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = m0 + wm * 64 + i * 8 + g;
            const int c = n0 + wn * 32 + j * 8 + 2 * t + e;
            acc[i][j][e] = (pre && r < p.M && c < p.N) ? sc * double(Cp[r + int64_t(c) * p.Cin.ld]) : 0.0;
          }
    }

    for (int it = 0; it < nkt; ++it) {
      cp_async_wait<G_STAGES - 2>();
      __syncthreads();
      const int nxt = it + G_STAGES - 1;
      if (nxt < nkt) load_tile(nxt % G_STAGES, kt0 + nxt);
      cp_async_commit();
      const double* as = reinterpret_cast<const double*>(As) + (it % G_STAGES) * Lay::A_SIZE;
      const double* bs = reinterpret_cast<const double*>(Bs) + (it % G_STAGES) * Lay::B_SIZE;
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
          bb[j] = Lay::B_KN ? bs[k * Lay::B_PITCH + n] : bs[n * Lay::B_PITCH + k];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
      }
    }
    cp_async_wait_all();

    // epilogue: acc[i][j][e] -> (row wm*64 + i*8 + g, col wn*32 + j*8 + 2t + e)
    const double alpha = p.alpha, beta = p.beta;
    T* D = optr_w<T>(p.D, b);
    const T* Cin = (beta != 0.0 && !pre) ? optr<T>(p.Cin, b) : nullptr;
    T* part = p.splits > 1 ? reinterpret_cast<T*>(p.part) + (int64_t(split) * p.batch + b) * int64_t(p.M) * p.N
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
              part[r + int64_t(c) * p.M] = acc[i][j][e];
            } else {
              double v = alpha * acc[i][j][e];
              if (Cin) v += beta * double(Cin[r + int64_t(c) * p.Cin.ld]);
              D[r + int64_t(c) * p.D.ld] = T(v);
            }
          }
        }
  } else {
    // ---------------- fp32: FFMA SIMT, 8x8 micro-tile ----------------
    const int tr = tid >> 4, tc = tid & 15;
    float acc[8][8];
    const bool pre = p.splits == 1 && p.beta != 0.0 && (p.alpha == 1.0 || p.alpha == -1.0);
    {
      const float sc = pre ? float(p.beta / p.alpha) : 0.f;
      const T* Cp = pre ? optr<T>(p.Cin, b) : nullptr;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int r = m0 + (i < 4 ? tr * 4 + i : 64 + tr * 4 + i - 4);
          const int c = n0 + (j < 4 ? tc * 4 + j : 64 + tc * 4 + j - 4);
          acc[i][j] = (pre && r < p.M && c < p.N) ? sc * float(Cp[r + int64_t(c) * p.Cin.ld]) : 0.f;
        }
    }
    for (int it = 0; it < nkt; ++it) {
      cp_async_wait<G_STAGES - 2>();
      __syncthreads();
      const int nxt = it + G_STAGES - 1;
      if (nxt < nkt) load_tile(nxt % G_STAGES, kt0 + nxt);
      cp_async_commit();
      const float* as = reinterpret_cast<const float*>(As) + (it % G_STAGES) * Lay::A_SIZE;
      const float* bs = reinterpret_cast<const float*>(Bs) + (it % G_STAGES) * Lay::B_SIZE;
#pragma unroll 8
      for (int k = 0; k < BK; ++k) {
        const float4 a0 = *reinterpret_cast<const float4*>(as + k * Lay::A_PITCH + tr * 4);
        const float4 a1 = *reinterpret_cast<const float4*>(as + k * Lay::A_PITCH + 64 + tr * 4);
        const float4 b0 = *reinterpret_cast<const float4*>(bs + k * Lay::B_PITCH + tc * 4);
        const float4 b1 = *reinterpret_cast<const float4*>(bs + k * Lay::B_PITCH + 64 + tc * 4);
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
      }
    }
    cp_async_wait_all();
    const float alpha = float(p.alpha), beta = float(p.beta);
    T* D = optr_w<T>(p.D, b);
    const T* Cin = (beta != 0.f && !pre) ? optr<T>(p.Cin, b) : nullptr;
    T* part = p.splits > 1 ? reinterpret_cast<T*>(p.part) + (int64_t(split) * p.batch + b) * int64_t(p.M) * p.N
                           : nullptr;
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = m0 + (i < 4 ? tr * 4 + i : 64 + tr * 4 + i - 4);
        const int c = n0 + (j < 4 ? tc * 4 + j : 64 + tc * 4 + j - 4);
        if (r < p.M && c < p.N && (!p.tril || r + p.tril - 1 >= c)) {
          if (part) {
            part[r + int64_t(c) * p.M] = acc[i][j];
          } else {
            float v = alpha * acc[i][j];
            if (Cin) v += beta * float(Cin[r + int64_t(c) * p.Cin.ld]);
            D[r + int64_t(c) * p.D.ld] = T(v);
          }
        }
      }
  }
}

// Deterministic split-K reduction: D = alpha * sum_{s=0..S-1} part[s] + beta * Cin.
// The fixed summation order ((s0 + s1) + (s2 + s3)) + ... keeps results bitwise
// reproducible; four independent partial sums keep the loads in flight.
template <typename T>
__global__ void k_splitk_reduce(int M, int N, int64_t batch, int splits, const T* __restrict__ part, Opnd Cin,
                                Opnd D, double alpha, double beta, int tril) {
  const int64_t MN = int64_t(M) * N, total = MN * batch;
  const int64_t sstride = MN * batch;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(idx % M);
    const int c = int((idx / M) % N);
    const int64_t b = idx / MN;
    if (tril && r + tril - 1 < c) continue;
    const T* pp = part + b * MN + r + int64_t(c) * M;
    T s0 = T(0), s1 = T(0), s2 = T(0), s3 = T(0);
    int q = 0;
    for (; q + 4 <= splits; q += 4) {
      s0 += __ldcg(pp + int64_t(q) * sstride);
      s1 += __ldcg(pp + int64_t(q + 1) * sstride);
      s2 += __ldcg(pp + int64_t(q + 2) * sstride);
      s3 += __ldcg(pp + int64_t(q + 3) * sstride);
    }
    for (; q < splits; ++q) s0 += __ldcg(pp + int64_t(q) * sstride);
    const T s = (s0 + s1) + (s2 + s3);
    T v = T(alpha) * s;
    if (beta != 0.0) v += T(beta) * optr<T>(Cin, b)[r + int64_t(c) * Cin.ld];
    optr_w<T>(D, b)[r + int64_t(c) * D.ld] = v;
  }
}

}  // namespace cd
