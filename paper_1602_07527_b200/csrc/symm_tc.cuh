// symm_tc.cuh -- the left-looking trailing update of the reverse sweep (symm_ll.cuh) for
// fp32 data on the 5th-generation tensor cores: tcgen05.mma kind::tf32, accumulators in
// TMEM, operands by TMA, stream-K over the k-chunks of all output tiles:
//
//     Cbar_J <- Cbar_J - M L[k:n, j:k],   M = T + T^T  (T = the finished tril(Sigmabar))
//
// A tiles by K block s of output tile i: s < i  T(i, s)       MN-major (4 SW128-32B-atom boxes)
//                                        s == i S_i (fp32)     MN-major, from the workspace
//                                        s > i  T(s, i)^T      K-major (one SW128 box)
// the operand major is chosen per K chunk in the instruction descriptor.  B = L[k:n, j:k]
// (K-major).  Roles as k_gemm_tc32: warp 0 TMA producer, warp 1 MMA issuer (one TMEM buffer
// per tile piece, two alternating), warps 2..5 epilogue (thread = accumulator row): a whole
// tile is written as Cin - acc, a piece of a split tile is stored to the CTA's slot and the
// last-arriving CTA sums Cin + the pieces in fixed CTA order (bitwise deterministic).  Warps
// 6..13 round each landed stage to tf32 in place (cvt.rna) before the MMA reads it.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "gemm_tc32.cuh"
#include "symm_ll.cuh"  // ll_start / ll_cta_of

namespace cd {

constexpr int STC_STAGES = 4;
constexpr int STC_CONVW = 8;
constexpr int STC_THREADS = (6 + STC_CONVW) * 32;
constexpr int STC_KC = 32;                       // K per chunk (128-byte rows of fp32)
constexpr int STC_CHUNKS_PER_BLK = 128 / STC_KC;  // 4
constexpr uint32_t STC_STAGE_BYTES = 2u * 128 * STC_KC * 4;  // A + B, 32 KB
constexpr size_t STC_SMEM = size_t(STC_STAGES) * STC_STAGE_BYTES + 1024 + 256;
constexpr int STC_TILE = 128 * 128;  // floats per partial slot

struct STCMaps {
  CUtensorMap aMN;  // Abar (fp32), box {32 rows, 32 cols}, SW128 with 32-byte atoms
  CUtensorMap aK;   // Abar (fp32), box {32 rows, 128 cols}, SW128
  CUtensorMap sMN;  // S workspace (128 x 128*nblk per batch entry), box {32, 32}, 32-byte atoms
  CUtensorMap lK;   // L (fp32), box {32, 128}, SW128
  int batched;
};

struct STCParams {
  Opnd A;            // Abar (Cin / D of the output panel)
  int n, k, j, w;
  int m;             // output row tiles (n - k) / 128
  int nblk;
  int G;
  int64_t total;     // batch * m * KC
  float* part;       // [G][2][128*128]
  int* cnt;          // [batch * m], zero on entry
};

__global__ void __launch_bounds__(STC_THREADS, 1) k_symm_tc(const STCParams p, const __grid_constant__ STCMaps tm) {
  extern __shared__ __align__(1024) unsigned char smem_stc[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_stc) + 1023) & ~uintptr_t(1023));
  unsigned char* As = base;
  unsigned char* Bs = base + STC_STAGES * (128 * STC_KC * 4);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STC_STAGES * STC_STAGE_BYTES);
  uint64_t* empty = full + STC_STAGES;
  uint64_t* accf = empty + STC_STAGES;
  uint64_t* acce = accf + 2;
  uint64_t* conv = acce + 2;  // [STC_STAGES] stage rounded (STC_CONVW warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(conv + STC_STAGES);
  int* s_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cta = blockIdx.x;
  const int KC = STC_CHUNKS_PER_BLK * p.m;  // chunks per output tile
  const int a0 = int(ll_start(cta, p.total, p.G)), a1 = int(ll_start(cta + 1, p.total, p.G));

  if (tid == 0) {
    for (int s = 0; s < STC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&conv[s], STC_CONVW);
    }
    mbar_init(&accf[0], 1);
    mbar_init(&accf[1], 1);
    mbar_init(&acce[0], 4);
    mbar_init(&acce[1], 4);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int it = 0;
      for (int x = a0; x < a1; ++x, ++it) {
        const int s = it % STC_STAGES;
        if (it >= STC_STAGES) tc_wait(&empty[s], ((it / STC_STAGES) - 1) & 1);
        const int tg = x / KC, kc = x - tg * KC;
        const int b = tg / p.m, i = tg - b * p.m;
        const int sb = kc / STC_CHUNKS_PER_BLK, kk = (kc % STC_CHUNKS_PER_BLK) * STC_KC;
        const int r0 = p.k + 128 * i, c0 = p.k + 128 * sb + kk;
        unsigned char* as = As + s * (128 * STC_KC * 4);
        unsigned char* bs = Bs + s * (128 * STC_KC * 4);
        mbar_expect_tx(&full[s], STC_STAGE_BYTES);
        if (sb < i) {  // T(i, s): MN-major, four 32(M) x 32(K) boxes
          for (int q = 0; q < 4; ++q) {
            if (tm.batched) tma_load_3d(as + q * 4096, &tm.aMN, r0 + 32 * q, c0, b, &full[s]);
            else tma_load_2d(as + q * 4096, &tm.aMN, r0 + 32 * q, c0, &full[s]);
          }
        } else if (sb == i) {  // S_i: MN-major from the workspace
          const int col = (p.nblk - (p.n - r0) / 128) * 128 + kk;
          for (int q = 0; q < 4; ++q) {
            if (tm.batched) tma_load_3d(as + q * 4096, &tm.sMN, 32 * q, col, b, &full[s]);
            else tma_load_2d(as + q * 4096, &tm.sMN, 32 * q, col, &full[s]);
          }
        } else {  // T(s, i)^T: K-major, one 32(K) x 128(M) box
          if (tm.batched) tma_load_3d(as, &tm.aK, c0, r0, b, &full[s]);
          else tma_load_2d(as, &tm.aK, c0, r0, &full[s]);
        }
        if (tm.batched) tma_load_3d(bs, &tm.lK, c0, p.j, b, &full[s]);
        else tma_load_2d(bs, &tm.lK, c0, p.j, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer: one accumulator buffer per tile piece ----------------
      int it = 0, piece = 0;
      for (int x = a0; x < a1; ++piece) {
        const int tg = x / KC;
        const int xe = min((tg + 1) * KC, a1);
        const int buf = piece & 1;
        if (piece >= 2) tc_wait(&acce[buf], ((piece >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t acc_t = tmem + uint32_t(buf * 128);
        const int i = tg % p.m;
        for (int first = 1; x < xe; ++x, ++it, first = 0) {
          const int s = it % STC_STAGES;
          tc_wait(&conv[s], (it / STC_STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const int sb = (x - tg * KC) / STC_CHUNKS_PER_BLK;
          const bool mn = sb <= i;
          const uint32_t idesc = tc_idesc(mn ? 1 : 0, 0);
          const uint32_t sa = smem_u32(As + s * (128 * STC_KC * 4));
          const uint32_t sbb = smem_u32(Bs + s * (128 * STC_KC * 4));
#pragma unroll
          for (int k8 = 0; k8 < STC_KC / 8; ++k8) {
            const uint64_t da = mn ? umma_desc(sa + k8 * 1024, 4096, 512, 1) : umma_desc(sa + k8 * 32, 16, 1024, 2);
            const uint64_t db = umma_desc(sbb + k8 * 32, 16, 1024, 2);
            const uint32_t acc = (!first || k8 > 0) ? 1u : 0u;
            asm volatile(
                "{\n.reg .pred P;\nsetp.ne.b32 P, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, P;\n}\n" ::"r"(acc_t),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                           smem_u32(&empty[s]))
                       : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         smem_u32(&accf[buf]))
                     : "memory");
      }
    }
  } else if (warp >= 6) {
    // ---------------- tf32 rounding of each landed stage ----------------
    const int ct = tid - 6 * 32;
    int it = 0;
    for (int x = a0; x < a1; ++x, ++it) {
      const int s = it % STC_STAGES;
      tc_wait(&full[s], (it / STC_STAGES) & 1);
      float4* a4 = reinterpret_cast<float4*>(As + s * (128 * STC_KC * 4));
      float4* b4 = reinterpret_cast<float4*>(Bs + s * (128 * STC_KC * 4));
#pragma unroll 4
      for (int e = ct; e < 128 * STC_KC / 4; e += STC_CONVW * 32) {
        float4 u = a4[e], v = b4[e];
        a4[e] = tf32_rna4(u);
        b4[e] = tf32_rna4(v);
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[s]);
    }
  } else {
    // ---------------- epilogue: warps 2..5, thread = accumulator row ----------------
    const int q = warp & 3;
    const int et = (warp - 2) * 32 + lane;  // 0..127 within the epilogue group
    int piece = 0;
    for (int x = a0; x < a1; ++piece) {
      const int tg = x / KC;
      const int ts = tg * KC, te = ts + KC;
      const int xe = min(te, a1);
      const bool whole = (x == ts && xe == te);
      const int b = tg / p.m, i = tg - b * p.m;
      const int buf = piece & 1;
      tc_wait(&accf[buf], (piece >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const int r = q * 32 + lane;             // row within the tile (TMEM lane)
      const int grow = p.k + 128 * i + r;      // row in the matrix
      float* Dp = optr_w<float>(p.A, b) + grow + int64_t(p.j) * p.A.ld;
      float* mine = p.part + int64_t(2 * cta + (ts <= a0 ? 0 : 1)) * STC_TILE;
#pragma unroll 1
      for (int cb = 0; cb < 128 && cb < p.w; cb += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + (uint32_t(q * 32) << 16) + uint32_t(buf * 128 + cb);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        float cin[32];
        if (whole) {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj)
            cin[jj] = (cb + jj < p.w && grow < p.n) ? __ldcg(Dp + int64_t(cb + jj) * p.A.ld) : 0.f;
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (whole) {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj)
            if (cb + jj < p.w && grow < p.n) Dp[int64_t(cb + jj) * p.A.ld] = cin[jj] - __uint_as_float(v[jj]);
        } else {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) __stcg(mine + r + (cb + jj) * 128, -__uint_as_float(v[jj]));
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[buf]);  // TMEM buffer free for the MMA issuer
      x = xe;
      if (whole) continue;
      // ---- last-arrival fixup (epilogue warps only: named barrier 1, 128 threads) ----
      __threadfence();
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      const int c_lo = ll_cta_of(ts, p.total, p.G), c_hi = ll_cta_of(te - 1, p.total, p.G);
      if (et == 0) {
        const int old = atomicAdd(&p.cnt[tg], 1);
        *s_flag = (old == c_hi - c_lo) ? 1 : 0;
      }
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (*s_flag) {
        __threadfence();
        // Cin + the pieces in CTA order (fixed order: deterministic), 8 columns at a time so
        // that 8 independent loads are in flight per piece
        for (int c0 = 0; c0 < p.w && grow < p.n; c0 += 16) {
          float v[16];
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) v[jj] = (c0 + jj < p.w) ? __ldcg(Dp + int64_t(c0 + jj) * p.A.ld) : 0.f;
          for (int cc = c_lo; cc <= c_hi; cc += 2) {  // two pieces' loads in flight at once
            const bool two = cc + 1 <= c_hi;
            const int s0 = 2 * cc + (ll_start(cc, p.total, p.G) >= ts ? 0 : 1);
            const int s1 = two ? 2 * (cc + 1) + (ll_start(cc + 1, p.total, p.G) >= ts ? 0 : 1) : s0;
            const float* p0 = p.part + int64_t(s0) * STC_TILE + r + c0 * 128;
            const float* p1 = p.part + int64_t(s1) * STC_TILE + r + c0 * 128;
            float x[16], y[16];
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              x[jj] = (c0 + jj < p.w) ? __ldcg(p0 + jj * 128) : 0.f;
              y[jj] = (two && c0 + jj < p.w) ? __ldcg(p1 + jj * 128) : 0.f;
            }
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) v[jj] = (v[jj] + x[jj]) + y[jj];
          }
#pragma unroll
          for (int jj = 0; jj < 16; ++jj)
            if (c0 + jj < p.w) Dp[int64_t(c0 + jj) * p.A.ld] = v[jj];
        }
        if (et == 0) p.cnt[tg] = 0;
      }
      asm volatile("bar.sync 1, 128;\n" ::: "memory");  // s_flag reuse
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
}

}  // namespace cd
