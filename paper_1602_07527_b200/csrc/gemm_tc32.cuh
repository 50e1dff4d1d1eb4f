// gemm_tc32.cuh -- fp32 Level-3 updates of the blocked sweeps (PAPER.md:634-636, 655-666,
// 689-701) on the 5th-generation tensor cores: tcgen05.mma kind::tf32 with the
// accumulator in TMEM, operands staged by TMA (128-byte swizzle) into a 4- or 5-stage ring.
//
//   warp 0 lane 0 : TMA producer (cp.async.bulk.tensor, mbarrier complete_tx)
//   warp 1 lane 0 : MMA issuer (tcgen05.mma.cta_group::1.kind::tf32, M=128 N=128 K=8;
//                   tcgen05.commit releases each smem stage and finally the accumulator)
//   warps 2..5    : epilogue (tcgen05.ld 32x32b: thread = accumulator row)
//   warp 6        : (EPI >= 1) the epilogue's TMA warp: prefetches Cin chunks into smem slots
//                   and stores finished chunks with cp.async.bulk.tensor (EPI = 2: transposed,
//                   through 32 x 128 boxes with the 128-byte swizzle)
//   last TC_CONVW (8) warps : round each landed operand stage to tf32 in place (cvt.rna) -- SURVEY c11:
//                   the MMA would otherwise truncate the low 13 mantissa bits (biased error;
//                   rounding cut the batched N = 512 error 4.3e-5 -> 1.1e-5 against the 1e-4 gate)
//
// Persistent grid (one CTA per SM with the TMA epilogue), two TMEM accumulator buffers so one
// unit's epilogue overlaps the next unit's loads and MMAs.
//
// Operand layouts: K-contiguous operands use the K-major SW128 canonical layout (one
// TMA box of 32 x 128, 128-byte swizzle); M/N-contiguous operands use the MN-major
// SW128-with-32-byte-atoms layout (four TMA boxes of 32 x 32, SWIZZLE_128B_ATOM_32B),
// the only MN-major layout tcgen05 accepts for tf32.  TF32 operands (10-bit mantissa, products
// accumulated in fp32): DESIGN.md §6 gives the error budget against the 1e-4 gate.  Same
// GemmParams semantics as k_gemm / k_gemm_tma.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "gemm.cuh"
#include "gemm_tma.cuh"  // mbarrier / TMA helpers, TmaMaps

namespace cd {

#ifndef CD_TC_STAGES
#define CD_TC_STAGES 3
#endif
#ifndef CD_TC_MINB
#define CD_TC_MINB 2
#endif
constexpr int TC_STAGES = CD_TC_STAGES;
constexpr int TC_THREADS = 128;
constexpr int TC_BM = 128, TC_BN = 128, TC_BK = 32;
constexpr uint32_t TC_STAGE_BYTES = (TC_BM + TC_BN) * TC_BK * 4;  // 32 KB
constexpr uint32_t TC_ECHUNK_BYTES = TC_BM * 32 * 4;              // one 128 x 32 epilogue chunk, 16 KB
#ifndef CD_TC_ESLOTS
#define CD_TC_ESLOTS 6
#endif
constexpr int TC_ESLOTS = CD_TC_ESLOTS;  // TMA epilogue chunk slots (Cin prefetch depth ESLOTS - 1)
// stages + (TMA epilogue) chunk slots + barriers / TMEM slot
__host__ __device__ constexpr size_t tc_smem(int stages, int epi, int bn = TC_BN) {
  return size_t(stages) * (TC_BM + bn) * TC_BK * 4 + (epi ? TC_ESLOTS * TC_ECHUNK_BYTES : 0) + 1024 + 256;
}
constexpr size_t TC_SMEM = tc_smem(TC_STAGES, 0);

// output / Cin maps of the TMA epilogue: fp32, box {128 rows, 32 cols}, no swizzle (so the
// staged chunk is column-major 128 x 32 and thread = row reads / writes it conflict-free)
struct TcEpiMaps {
  CUtensorMap d, cin;
};

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

// shared-memory matrix descriptor; layout 2 = SWIZZLE_128B (K-major operands),
// 1 = SWIZZLE_128B_BASE32B (MN-major tf32 operands: the only MN-major layout for tf32)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // descriptor version (Blackwell)
  d |= uint64_t(layout & 7) << 61;
  return d;
}

// instruction descriptor: D f32, A/B tf32, M=128, N=128, majors per operand
__host__ __device__ constexpr uint32_t tc_idesc(int a_mn_major, int b_mn_major, int n = 128) {
  return (1u << 4)                       // c_format = F32
         | (2u << 7) | (2u << 10)        // a_format = b_format = TF32
         | (uint32_t(a_mn_major) << 15)  // a_major (1 = MN)
         | (uint32_t(b_mn_major) << 16)  // b_major
         | ((uint32_t(n) >> 3) << 17)    // N >> 3
         | ((128u >> 4) << 24);          // M >> 4
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ float4 tf32_rna4(float4 v) {
  return make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
}

// Protocol-error watchdog of the mbarrier waits: a wait that has not completed after
// CD_WATCHDOG_NS nanoseconds of wall time (globaltimer) traps instead of hanging the GPU.  Bounded
// by elapsed time, not by a spin count, so legitimately slow runs (compute-sanitizer, debuggers,
// time slicing, concurrent streams) never trip it; -DCD_WATCHDOG_NS=0 compiles it out.
#ifndef CD_WATCHDOG_NS
#define CD_WATCHDOG_NS 20000000000ull
#endif
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
  return t;
}
__device__ __forceinline__ void tc_wait(uint64_t* bar, uint32_t parity) {
  uint32_t spins = 0;
  uint64_t t0 = 0;
  while (true) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if (CD_WATCHDOG_NS != 0 && (++spins & 0xFFFFu) == 0) {
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > uint64_t(CD_WATCHDOG_NS)) __trap();
    }
  }
}

// Persistent form: grid = a few CTAs per SM, each looping over work units u = (m tile,
// n tile, batch entry, split) with stride gridDim.x.  Roles:
//   warp 0 lane 0 : TMA producer over the (unit, K chunk) sequence (runs ahead across units)
//   warp 1 lane 0 : MMA issuer; accumulates unit i in TMEM buffer i & 1 (2 x 128 columns)
//   warps 2..5    : epilogue (warp % 4 = the TMEM lane quarter it may read); drains buffer
//                   i & 1 while the MMA issuer already fills the other one
// so TMEM allocation, barrier setup and the epilogue of one unit overlap the next unit's
// loads and MMAs (the batched updates are tens of thousands of short-K tiles).
constexpr int TCP_THREADS = 192;
// EPI = 1 adds warp 6: the epilogue's TMA warp (Cin prefetch + output stores).  The last
// TC_CONVW (8) warps round every operand stage to tf32 in place (cvt.rna) before the MMA reads it.
#ifndef CD_TC_EPI_MINB
#define CD_TC_EPI_MINB 1
#endif
#ifndef CD_TC_CONVW
#define CD_TC_CONVW 8
#endif
constexpr int TC_CONVW = CD_TC_CONVW;  // rounding warps
__host__ __device__ constexpr int tc_conv_warp0(int epi) { return epi ? 7 : 6; }
__host__ __device__ constexpr int tcp_threads(int epi) { return (tc_conv_warp0(epi) + TC_CONVW) * 32; }

// EPI = 0: registers epilogue (Cin loaded per thread-row, direct stores).
// EPI = 1: TMA epilogue -- Cin chunks (128 x 32) are prefetched by TMA into two smem slots one
//          chunks ahead (TC_ESLOTS slots), the result is written back into the slot and stored by TMA
//          (cp.async.bulk.tensor ... bulk_group), so several Cin loads and output stores are
//          in flight per CTA (a one-chunk prefetch left the batched updates latency-bound at
//          ~1.7 TB/s).  Host-side conditions: splits == 1,
//          D (and Cin) TMA-describable, and a tril mask only for the in-place update
//          (masked elements are written back unchanged).
// STG = depth of the operand ring.  BN = the N tile (128, or 64 for the nb = 64 panels: M x 64
// products would otherwise issue half-empty MMAs -- the batched forward update is tensor-bound).
template <int TA, int TB, int EPI, int STG, int BN>
__global__ void __launch_bounds__(tcp_threads(EPI), EPI ? CD_TC_EPI_MINB : CD_TC_MINB)
    k_gemm_tc32(const GemmParams p, const __grid_constant__ TmaMaps tm, const __grid_constant__ TcEpiMaps em) {
  constexpr int TC_STAGES = STG;
  constexpr int TC_BN = BN;
  constexpr uint32_t TC_STAGE_BYTES = (TC_BM + BN) * TC_BK * 4;
  extern __shared__ __align__(1024) unsigned char smem_tc[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_tc) + 1023) & ~uintptr_t(1023));
  unsigned char* As = base;                                   // stages of A (16 KB each)
  unsigned char* Bs = base + TC_STAGES * (TC_BM * TC_BK * 4);  // stages of B (BN x 32 fp32 each)
  unsigned char* Es = base + TC_STAGES * TC_STAGE_BYTES;      // EPI: 128 x 32 chunk slots
  uint64_t* full = reinterpret_cast<uint64_t*>(Es + (EPI ? TC_ESLOTS * TC_ECHUNK_BYTES : 0));
  uint64_t* empty = full + TC_STAGES;
  uint64_t* accf = empty + TC_STAGES;  // [2] accumulator ready
  uint64_t* acce = accf + 2;           // [2] accumulator drained
  uint64_t* cinf = acce + 2;           // [TC_ESLOTS] EPI: slot s ready (Cin landed / slot free)
  uint64_t* donef = cinf + TC_ESLOTS;  // [TC_ESLOTS] EPI: chunk in slot s computed (4 warps)
  uint64_t* conv = donef + TC_ESLOTS;  // [TC_STAGES] stage s rounded to tf32 (TC_CONVW warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(conv + TC_STAGES);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int mt = (p.M + TC_BM - 1) / TC_BM, ntl = (p.N + TC_BN - 1) / TC_BN;
  const int64_t units = int64_t(mt) * ntl * p.batch * p.splits;
  // (32-bit: the host guarantees units < 2^31; 64-bit division is a long subroutine)
  auto decode = [&](int64_t u, int& m0, int& n0, int64_t& b, int& split) {
    const unsigned tmn = unsigned(mt) * unsigned(ntl);
    const unsigned uu = unsigned(u);
    const unsigned zb = uu / tmn;
    const unsigned r = uu - zb * tmn;
    m0 = int(r % unsigned(mt)) * TC_BM;
    n0 = int(r / unsigned(mt)) * TC_BN;
    split = int(zb % unsigned(p.splits));
    b = int64_t(zb / unsigned(p.splits));
  };
  auto krange = [&](int split, int& kt0, int& nkt) {
    kt0 = split * p.kt_per_split;
    nkt = min(p.KT, kt0 + p.kt_per_split) - kt0;
  };

  if (tid == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&conv[s], TC_CONVW);
    }
    mbar_init(&accf[0], 1);
    mbar_init(&accf[1], 1);
    mbar_init(&acce[0], 4);
    mbar_init(&acce[1], 4);
    for (int s = 0; s < TC_ESLOTS; ++s) {
      mbar_init(&cinf[s], 1);
      mbar_init(&donef[s], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {  // TMEM: 2 x 128 columns x 128 lanes of fp32 accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // launched with programmatic stream serialization (PDL): the prologue above overlaps the previous
  // kernel's tail; every global access below waits for it to complete
  asm volatile("griddepcontrol.wait;\n" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int it = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        int m0, n0, split, kt0, nkt;
        int64_t b;
        decode(u, m0, n0, b, split);
        krange(split, kt0, nkt);
        for (int kk = 0; kk < nkt; ++kk, ++it) {
          const int s = it % TC_STAGES;
          if (it >= TC_STAGES) tc_wait(&empty[s], ((it / TC_STAGES) - 1) & 1);
          const int kt = kt0 + kk;
          int sg = 0;
          if (p.nseg > 1 && kt * TC_BK >= p.seg[1].kv0) sg = 1;
          if (p.nseg > 2 && kt * TC_BK >= p.seg[2].kv0) sg = 2;
          const int kl = kt * TC_BK - p.seg[sg].kv0;
          // MN-major A: boxes wholly below row M are not loaded (their accumulator rows are
          // never stored), so short panels (M = 64) move no zero fill
          const int na = TA == 0 ? min(4, (p.M - m0 + 31) / 32) : 4;
          mbar_expect_tx(&full[s], TC_STAGE_BYTES - uint32_t(4 - na) * 4096u);
          unsigned char* as = As + s * (TC_BM * TC_BK * 4);
          unsigned char* bs = Bs + s * (TC_BN * TC_BK * 4);
          if (TA == 0) {  // MN-major: four 32(M) x 32(K) boxes
            for (int c = 0; c < na; ++c) {
              if (tm.batched) tma_load_3d(as + c * 4096, &tm.a[sg], m0 + 32 * c, kl, int(b), &full[s]);
              else tma_load_2d(as + c * 4096, &tm.a[sg], m0 + 32 * c, kl, &full[s]);
            }
          } else {  // K-major: one 32(K) x 128(M) box
            if (tm.batched) tma_load_3d(as, &tm.a[sg], kl, m0, int(b), &full[s]);
            else tma_load_2d(as, &tm.a[sg], kl, m0, &full[s]);
          }
          if (TB == 1) {  // MN-major B
            for (int c = 0; c < BN / 32; ++c) {
              if (tm.batched) tma_load_3d(bs + c * 4096, &tm.b[sg], n0 + 32 * c, kl, int(b), &full[s]);
              else tma_load_2d(bs + c * 4096, &tm.b[sg], n0 + 32 * c, kl, &full[s]);
            }
          } else {
            if (tm.batched) tma_load_3d(bs, &tm.b[sg], kl, n0, int(b), &full[s]);
            else tma_load_2d(bs, &tm.b[sg], kl, n0, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc = tc_idesc(TA == 0 ? 1 : 0, TB == 1 ? 1 : 0, BN);
      int it = 0, i = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++i) {
        int m0, n0, split, kt0, nkt;
        int64_t b;
        decode(u, m0, n0, b, split);
        krange(split, kt0, nkt);
        const int buf = i & 1;
        if (i >= 2) tc_wait(&acce[buf], ((i >> 1) - 1) & 1);  // the epilogue drained this buffer
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t acc_t = tmem + uint32_t(buf * TC_BN);
        for (int kk = 0; kk < nkt; ++kk, ++it) {
          const int s = it % TC_STAGES;
          tc_wait(&conv[s], (it / TC_STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t sa = smem_u32(As + s * (TC_BM * TC_BK * 4));
          const uint32_t sb = smem_u32(Bs + s * (TC_BN * TC_BK * 4));
#pragma unroll
          for (int k8 = 0; k8 < TC_BK / 8; ++k8) {
            // K-major (SW128): advance 32 B along K inside the swizzle atom, 8-row groups 1 KB apart.
            // MN-major (SW128 with 32 B atoms): K rows 128 B apart, 4-row groups 512 B apart,
            // 32-element MN chunks 4 KB apart; each K = 8 step starts 8 rows (1 KB) further.
            const uint64_t da = (TA == 0) ? umma_desc(sa + k8 * 1024, 4096, 512, 1) : umma_desc(sa + k8 * 32, 16, 1024, 2);
            const uint64_t db = (TB == 1) ? umma_desc(sb + k8 * 1024, 4096, 512, 1) : umma_desc(sb + k8 * 32, 16, 1024, 2);
            const uint32_t acc = (kk > 0 || k8 > 0) ? 1u : 0u;
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
  } else if (warp >= tc_conv_warp0(EPI)) {
    // ---------------- tf32 rounding of each landed stage (round to nearest,
    // ties away -- cvt.rna -- instead of the MMA's silent truncation of the low 13 bits) --------
    const int ct = tid - tc_conv_warp0(EPI) * 32;
    int it = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      int m0, n0, split, kt0, nkt;
      int64_t b;
      decode(u, m0, n0, b, split);
      krange(split, kt0, nkt);
      for (int kk = 0; kk < nkt; ++kk, ++it) {
        const int s = it % TC_STAGES;
        tc_wait(&full[s], (it / TC_STAGES) & 1);
        float4* a4 = reinterpret_cast<float4*>(As + s * (TC_BM * TC_BK * 4));
        float4* b4 = reinterpret_cast<float4*>(Bs + s * (TC_BN * TC_BK * 4));
#ifndef CD_TC_NOROUND  // (measurement switch: the stage handshake without the rounding pass)
#pragma unroll 4
        for (int e = ct; e < TC_BM * TC_BK / 4; e += TC_CONVW * 32) {
          float4 x = a4[e];
          float4 y = e < BN * TC_BK / 4 ? b4[e] : float4{};
          x = tf32_rna4(x);
          a4[e] = x;
          if (e < BN * TC_BK / 4) b4[e] = tf32_rna4(y);
        }
#endif
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[s]);
      }
    }
  } else if (EPI >= 1 && warp == 6) {
    // ---------------- epilogue TMA warp (lane 0): Cin prefetch and output stores ----------------
    if (lane == 0) {
      const bool has_cin = p.beta != 0.0;
      auto nchunks = [&](int n0) { return (min(TC_BN, p.N - n0) + 31) / 32; };
      // ready cursor: chunk lg (chunk lc of unit lu) gets slot lg % ESLOTS -- loaded from Cin,
      // or just released when there is no Cin
      int64_t lu = blockIdx.x;
      int lc = 0, lg = 0;
      auto ready_next = [&]() {
        if (lu >= units) return;
        int m0, n0, split;
        int64_t b;
        decode(lu, m0, n0, b, split);
        const int slot = lg % TC_ESLOTS;
        if (has_cin) {
          mbar_expect_tx(&cinf[slot], TC_ECHUNK_BYTES);
          // EPI = 2: D (and Cin) are stored transposed, so the chunk is a 32-row x 128-column box
          const int x0 = EPI == 2 ? n0 + 32 * lc : m0, x1 = EPI == 2 ? m0 : n0 + 32 * lc;
          if (tm.batched) tma_load_3d(Es + slot * TC_ECHUNK_BYTES, &em.cin, x0, x1, int(b), &cinf[slot]);
          else tma_load_2d(Es + slot * TC_ECHUNK_BYTES, &em.cin, x0, x1, &cinf[slot]);
        } else {
          mbar_arrive(&cinf[slot]);
        }
        ++lg;
        if (++lc == nchunks(n0)) lc = 0, lu += gridDim.x;
      };
      for (int k = 0; k < TC_ESLOTS - 1; ++k) ready_next();
      int g = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        int m0, n0, split;
        int64_t b;
        decode(u, m0, n0, b, split);
        const int nch = nchunks(n0);
        for (int c = 0; c < nch; ++c, ++g) {
          const int slot = g % TC_ESLOTS;
          tc_wait(&donef[slot], (g / TC_ESLOTS) & 1);
          unsigned char* E = Es + slot * TC_ECHUNK_BYTES;
          const int x0 = EPI == 2 ? n0 + 32 * c : m0, x1 = EPI == 2 ? m0 : n0 + 32 * c;
          if (tm.batched) tma_store_3d(&em.d, E, x0, x1, int(b));
          else tma_store_2d(&em.d, E, x0, x1);
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
          // chunk g + ESLOTS - 1 takes the slot of chunk g - 1 once that store has read it
          asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
          ready_next();
        }
      }
      asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    }
  } else if (EPI >= 1) {
    // ---------------- TMA epilogue: warps 2..5, thread = accumulator row ----------------
    const int q = warp & 3;
    const int rr = q * 32 + lane;  // row within the tile (TMEM lane)
    const float alpha = float(p.alpha), beta = float(p.beta);
    const bool has_cin = p.beta != 0.0;
    auto nchunks = [&](int n0) { return (min(TC_BN, p.N - n0) + 31) / 32; };
    int i = 0, g = 0;  // unit counter, global chunk counter
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      int m0, n0, split, kt0, nkt;
      int64_t b;
      decode(u, m0, n0, b, split);
      krange(split, kt0, nkt);
      const int buf = i & 1;
      tc_wait(&accf[buf], (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const int nch = nchunks(n0);
      const int r = m0 + rr;
      for (int c = 0; c < nch; ++c, ++g) {
        const int slot = g % TC_ESLOTS;
        float* E = reinterpret_cast<float*>(Es + slot * TC_ECHUNK_BYTES);
        uint32_t v[32];
        const uint32_t taddr = tmem + (uint32_t(q * 32) << 16) + uint32_t(buf * TC_BN + 32 * c);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (c + 1 == nch) {  // accumulator drained: the MMA issuer may reuse the buffer
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&acce[buf]);
        }
        tc_wait(&cinf[slot], (g / TC_ESLOTS) & 1);  // Cin landed / slot released
        if constexpr (EPI == 2) {
          // transposed chunk: row rr of the box holds this thread's 32 values (128 B), its
          // 16-byte pieces permuted by the 128-byte swizzle (piece ^ (rr & 7)): conflict-free
          float4* E4 = reinterpret_cast<float4*>(E) + rr * 8;
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            const int ch = q4 ^ (rr & 7);
            const float4 ci = has_cin ? E4[ch] : make_float4(0.f, 0.f, 0.f, 0.f);
            float a[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) a[e] = nkt > 0 ? __uint_as_float(v[4 * q4 + e]) : 0.f;
            E4[ch] = make_float4(alpha * a[0] + beta * ci.x, alpha * a[1] + beta * ci.y, alpha * a[2] + beta * ci.z,
                                 alpha * a[3] + beta * ci.w);
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const int col = n0 + 32 * c + jj;
            const float acc = nkt > 0 ? __uint_as_float(v[jj]) : 0.f;
            const float ci = has_cin ? E[jj * 128 + rr] : 0.f;
            const bool keep = p.tril && !(r + p.tril - 1 >= col);
            E[jj * 128 + rr] = keep ? ci : alpha * acc + beta * ci;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&donef[slot]);
      }
    }
  } else {
    // ---------------- epilogue: warps 2..5, thread = accumulator row ----------------
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const float alpha = float(p.alpha), beta = float(p.beta);
    int i = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      int m0, n0, split, kt0, nkt;
      int64_t b;
      decode(u, m0, n0, b, split);
      krange(split, kt0, nkt);
      const int buf = i & 1;
      tc_wait(&accf[buf], (i >> 1) & 1);  // the MMA issuer commits every unit
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const int r = m0 + q * 32 + lane;
      float* D = optr_w<float>(p.D, b);
      const float* Cin = (p.beta != 0.0 && p.splits == 1) ? optr<float>(p.Cin, b) : nullptr;
      float* part = p.splits > 1
                        ? reinterpret_cast<float*>(p.part) + (int64_t(split) * p.batch + b) * int64_t(p.M) * p.N
                        : nullptr;
#pragma unroll 1
      for (int cb = 0; cb < TC_BN && n0 + cb < p.N; cb += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + (uint32_t(q * 32) << 16) + uint32_t(buf * TC_BN + cb);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        // Cin is usually D itself (in-place update): load the whole chunk first, or every
        // store would order the next load behind it (one memory latency per column)
        float cin[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int c = n0 + cb + j;
          cin[j] = (Cin && r < p.M && c < p.N) ? __ldcg(Cin + r + int64_t(c) * p.Cin.ld) : 0.f;
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (r < p.M) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int c = n0 + cb + j;
            const float acc = nkt > 0 ? __uint_as_float(v[j]) : 0.f;
            if (c < p.N && (!p.tril || r + p.tril - 1 >= c)) {
              if (part) {
                part[r + int64_t(c) * p.M] = acc;
              } else {
                D[r + int64_t(c) * p.D.ld] = alpha * acc + beta * cin[j];
              }
            }
          }
        }
      }
      // buffer drained: let the MMA issuer reuse it
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[buf]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
}

}  // namespace cd
