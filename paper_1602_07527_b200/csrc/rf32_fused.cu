// rf32_fused.cu -- batched fp32 reverse and forward sweeps, every step of a matrix's sweep inside
// one persistent kernel (SURVEY §8 row a15, configs[3]: 1024 x N = 512 fp32, reverse + forward of
// the same factors).
//
// Why fused: the layer-by-layer schedule (one launch per panel step over the whole batch)
// re-reads every matrix's trailing data from DRAM at every step and spends most of its time in
// latency-bound diagonal-block launches.  Here a CTA owns a matrix's sweep from the first panel to
// the last, so its re-reads hit L2 and the panel chain runs back to back; the reverse and forward
// sweeps of one matrix run on neighbouring CTAs at the same time, so L is fetched from DRAM once.
//
// Two matrices per CTA ("slots"), software-pipelined: while the tensor cores run the trailing
// update of one slot's panel (TMA warp + MMA warp), eight warps run the panel steps of the other
// slot (global loads, mma.sync products, stores).  Each slot alternates update -> panel ->
// update ..., handshaking through an mbarrier (acc_ready: the update's accumulators are in TMEM)
// and a shared counter (panel_cnt: the panel's results are in global memory and its TMEM rows are
// drained), so the latency of one slot's chain hides behind the other's work.
//
// Blocks of N_b = 64.  Per panel I (columns [64I, 64I+64)):
// reverse, I = nblk-1 .. 0, left-looking form of PAPER.md:689-701 (ordering freedom,
// PAPER.md:704-707; derivation in DESIGN.md §6): with T = the finished tril(Sigma_bar) right of
// the panel and S_J = Dbar_J + Dbar_J^T its diagonal blocks,
//   R1  acc = (T + T^T)[k:n, k:n] L[k:n, I]                  tcgen05 kind::tf32 (TMEM accumulators)
//   R2  Cbar = Lbar[k:n, I] - acc                            (PAPER.md:696, 699 delayed)
//   R3  Cbar <- Cbar D^{-1}
//   R4  Dbar <- Lbar[I, I] - tril(Cbar^T C)
//   R5  Dbar <- chol_unblocked_rev(D, Dbar) by Eq. 10 on the block:
//       P = Phi(D^T Dbar), X = D^{-T} (P + P^T) D^{-1}, Dbar = Phi(X), S_I = Phi(X) + Phi(X)^T
// forward, I = 0 .. nblk-1 (already left-looking):
//   F1  acc = [Ldot L][j:n, 0:j] [L Ldot][I, 0:j]^T          tcgen05 kind::tf32
//   F2  [Ddot; Cdot] = Sigma_dot[j:n, I] - acc
//   F3  Ddot <- chol_unblocked_fwd(D, Ddot) by Eq. 8: Ddot = D Phi(D^{-1} Ddot_sym D^{-T})
//
//   F4  Cdot <- (Cdot - C Ddot^T) D^{-T}
// R2-R4 and F2-F4 stream the panel through shared memory 64 rows at a time, straight out of TMEM.
//
// TF32 operands are rounded to nearest (cvt.rna), never truncated: the tensor-core
// updates read tf32-rounded shadow copies (L_r made once per call by k_rf_round; T_r, S and
// Ldot_r written by the panel steps beside the fp32 results), and mma.sync rounds its fragments.
// Block inverses D^{-1} are made once per call by k_rf_trinv (fp32 forward substitution).
//
// Warps: 0 = TMA producer, 1 = MMA issuer (+ TMEM owner), 2..9 = panel steps.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "gemm_tc32.cuh"  // tcgen05 / TMA / mbarrier helpers (umma_desc, tc_idesc, tf32_rna, tc_wait)
#include "rf32_fused.h"

namespace cd {
namespace rf {

constexpr int NBK = 64;                     // panel width N_b
constexpr int NMAX = 512;                   // 4 accumulator tiles x 64 TMEM columns per slot
constexpr int BK = 32;                      // K per pipeline stage
constexpr int STAGES = 4;
constexpr uint32_t A_BYTES = 128 * BK * 4;  // 16 KB
constexpr uint32_t B_BYTES = BK * NBK * 4;  // 8 KB
constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int PLD = 72;                     // pitch (floats) of the 64 x 64 buffers (row-major, swizzled: el())
constexpr int SCR = NBK * PLD;              // floats per 64 x 64 buffer (18 KB)
constexpr int NBUF = 7;
constexpr size_t RING_BYTES = size_t(STAGES) * STAGE_BYTES;  // 96 KB
constexpr size_t BUF_BYTES = size_t(NBUF) * SCR * 4;         // 126 KB
constexpr size_t SMEM = 1024 + RING_BYTES + BUF_BYTES + 256;  // + alignment + barriers
constexpr int THREADS = 320;
constexpr int W_P0 = 2;                     // first panel warp
constexpr int PANEL_THREADS = 256;          // warps 2..9

struct Params {
  int n, nblk, mode, nslots;
  int64_t batch;
  const float* L;
  int64_t ldl, sL;
  float* Ab;
  int64_t lda, sA;
  float* Ad;
  int64_t ldd, sD;
  const float* Dinv;  // per matrix: 64 x n column-major (ld 64), block J = columns [64J, 64J+64)
  float* S;           // same layout: S_J (reverse), tf32-rounded
  float* Tr;          // per matrix n x n (ld n): tf32-rounded copy of tril(Sigma_bar) (reverse)
  float* Ldr;         // per matrix n x n: tf32-rounded copy of L_dot (forward)
  long long* prof;    // optional: [grid][PF_N] clock64 cycles per section (CD_RF32_PROF)
};
struct Maps {
  CUtensorMap tr_mn, tr_k, ldr_mn, lr_mn, lr_k, s_mn, s_k;
};

// ---------------------------------------------------------------- shared-memory access
__device__ __forceinline__ float lds(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, float v) { asm volatile("st.shared.f32 [%0], %1;\n" ::"r"(a), "f"(v)); }
__device__ __forceinline__ float rnd(float x) { return tf32_rna(x); }

// 64 x 64 buffers: row-major, pitch 72, the low three column bits XOR-ed with sw(R) = 5 ((R >> 2) & 1):
// (R, C) at R * 72 + (C & ~7) + ((C & 7) ^ sw(R)).  Bank conflict free for every access the kernels
// make -- mma.sync fragments of either orientation (8 rows x 4 columns and 4 rows x 8 columns per
// quarter of the warp), accumulator stores (rows g, g + 4 land on opposite column parities), and 8 x 4
// element blocks (tile_rc) in either orientation -- and, the swizzle only touching bits below 8,
// additive: moving by a multiple of 8 rows or columns is a constant byte offset.  (Pitch 68 without
// a swizzle: 2-way conflicts on MN-major fragments and 4-way on column stores, half of the shared
// wavefronts of k_rf_diag128.)
__device__ __forceinline__ int sw64(int R) { return 5 * ((R >> 2) & 1); }
__device__ __forceinline__ uint32_t el(uint32_t buf, int r, int c) {
  return buf + 4u * uint32_t(r * PLD + (c & ~7) + ((c & 7) ^ sw64(r)));
}
// the element block of panel thread pt in pass q (0..15) of a 64 x 64 sweep: warp w takes rows
// 8w .. 8w+7, pass q columns 4q .. 4q+3 (a warp: 8 rows x 4 columns, conflict free both ways)
__device__ __forceinline__ void tile_rc(int pt, int q, int& r, int& c) {
  r = 8 * (pt >> 5) + (pt & 7);
  c = 4 * q + ((pt >> 3) & 3);
}
// a matrix view of a buffer: logical (r, c) is physical (R0 + r, C0 + c), or (R0 + c, C0 + r)
// when transposed (t)
struct SV {
  uint32_t buf;
  int R0, C0;
  bool t;
  __device__ __forceinline__ uint32_t at(int r, int c) const {
    return t ? el(buf, R0 + c, C0 + r) : el(buf, R0 + r, C0 + c);
  }
  __device__ __forceinline__ SV sub(int r, int c) const {
    return t ? SV{buf, R0 + c, C0 + r, t} : SV{buf, R0 + r, C0 + c, t};
  }
  __device__ __forceinline__ SV tr() const { return SV{buf, R0, C0, !t}; }  // transpose
  // byte offsets of a logical move by 8 rows / 8 columns (additive: multiples of 8)
  __device__ __forceinline__ uint32_t rstep8() const { return t ? 32u : 32u * PLD; }
  __device__ __forceinline__ uint32_t cstep8() const { return t ? 32u * PLD : 32u; }
};
__device__ __forceinline__ SV rowmajor(uint32_t base) { return SV{base, 0, 0, false}; }

// ---------------------------------------------------------------- mma.sync tf32 helpers
__device__ __forceinline__ uint32_t rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void mma8(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
// fragments of one k-step: m16n8k8 layouts a0 (g, t), a1 (g+8, t), a2 (g, t+4), a3 (g+8, t+4);
// b0 (k=t, n=g), b1 (k=t+4, n=g); accumulators c0 (g, 2t), c1 (g, 2t+1), c2 (g+8, 2t), c3 (g+8, 2t+1)
template <int NT>
struct Frag {
  float a[4];
  float b[NT][2];
};
// per-thread fragment base addresses of a view pair (k-step 0, n-tile 0); every other k-step /
// n-tile is a constant offset from these (the swizzle is additive in steps of 8)
struct FragBase {
  uint32_t a0, a2, b0, b1;  // A(g, t), A(g, t + 4), B(t, g), B(t + 4, g)
  uint32_t ar8, ak8, bk8, bn8;
};
__device__ __forceinline__ FragBase frag_base(const SV& A, const SV& B) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  return FragBase{A.at(g, t), A.at(g, t + 4), B.at(t, g), B.at(t + 4, g), A.rstep8(), A.cstep8(), B.rstep8(),
                  B.cstep8()};
}
template <int NT>
__device__ __forceinline__ void frag_load(Frag<NT>& f, const FragBase& fb, int k0) {
  const uint32_t ka = (k0 >> 3) * fb.ak8, kb = (k0 >> 3) * fb.bk8;
  f.a[0] = lds(fb.a0 + ka);
  f.a[1] = lds(fb.a0 + fb.ar8 + ka);
  f.a[2] = lds(fb.a2 + ka);
  f.a[3] = lds(fb.a2 + fb.ar8 + ka);
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    f.b[nt][0] = lds(fb.b0 + kb + nt * fb.bn8);
    f.b[nt][1] = lds(fb.b1 + kb + nt * fb.bn8);
  }
}
template <int NT>
__device__ __forceinline__ void frag_load(Frag<NT>& f, const SV& A, const SV& B, int k0) {
  frag_load(f, frag_base(A, B), k0);
}
// PRE: the operands in shared memory are already tf32-rounded (cvt.rna at store), no conversion here
template <int NT, bool PRE = false>
__device__ __forceinline__ void frag_mma(float (&acc)[NT][4], const Frag<NT>& f) {
  auto cv = [](float x) { return PRE ? __float_as_uint(x) : rna(x); };
  const uint32_t a[4] = {cv(f.a[0]), cv(f.a[1]), cv(f.a[2]), cv(f.a[3])};
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const uint32_t b[2] = {cv(f.b[nt][0]), cv(f.b[nt][1])};
    mma8(acc[nt], a, b);
  }
}
// one warp: acc[16 x 8 NT] += A[16 x K] B[K x 8 NT], both in shared memory (K a multiple of 16);
// the next k-step's fragments are loaded while the current one multiplies
template <int NT, bool PRE = false>
__device__ __forceinline__ void warp_mma(float (&acc)[NT][4], int K, const SV& A, const SV& B) {
  Frag<NT> f0, f1;
  const FragBase fb = frag_base(A, B);
  frag_load(f0, fb, 0);
#pragma unroll 1
  for (int k0 = 0; k0 < K; k0 += 16) {
    frag_load(f1, fb, k0 + 8);
    frag_mma<NT, PRE>(acc, f0);
    if (k0 + 16 < K) frag_load(f0, fb, k0 + 16);
    frag_mma<NT, PRE>(acc, f1);
  }
}
template <int NT>
__device__ __forceinline__ void zero(float (&acc)[NT][4]) {
#pragma unroll
  for (int i = 0; i < NT; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
}
// visit the accumulator elements: f(r, c, value) with r, c relative to the warp's block
template <int NT, class F>
__device__ __forceinline__ void for_acc(const float (&acc)[NT][4], F f) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    f(g, nt * 8 + 2 * t, acc[nt][0]);
    f(g, nt * 8 + 2 * t + 1, acc[nt][1]);
    f(g + 8, nt * 8 + 2 * t, acc[nt][2]);
    f(g + 8, nt * 8 + 2 * t + 1, acc[nt][3]);
  }
}

__device__ __forceinline__ void panel_sync() {  // warps 2..9
  asm volatile("bar.sync 1, %0;\n" ::"n"(PANEL_THREADS) : "memory");
}

// 64 x 64 x 64 product over the 8 panel warps: warp pw computes rows 16 (pw>>1), columns 32 (pw&1)
template <bool PRE = false, class FOUT>
__device__ __forceinline__ void gemm64(int pw, const SV& A, const SV& B, FOUT out) {
  const int r0 = 16 * (pw >> 1), c0 = 32 * (pw & 1);
  float acc[4][4];
  zero(acc);
  warp_mma<4, PRE>(acc, NBK, A.sub(r0, 0), B.sub(0, c0));
  for_acc(acc, [&](int r, int c, float v) { out(r0 + r, c0 + c, v); });
}

// ---------------------------------------------------------------- global 64 x 64 tiles
// 64 x 64 tile of a column-major matrix, 16 elements per panel thread (coalesced along columns);
// tril: elements above the diagonal are not read (zero)
struct Tile64 {
  float v[16];
  __device__ __forceinline__ void load(const float* src, int64_t ld, int pt, bool tril) {
    int i, c0;
    tile_rc(pt, 0, i, c0);
    const float* p0 = src + i + int64_t(c0) * ld;  // pass q: 4q columns further
    const int64_t step = 4 * ld;
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = (!tril || i >= c0 + 4 * q) ? __ldcg(p0 + q * step) : 0.f;
  }
  __device__ __forceinline__ void store(uint32_t buf, int pt, bool round = false) const {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      int i, c;
      tile_rc(pt, q, i, c);
      sts(el(buf, i, c), round ? rnd(v[q]) : v[q]);
    }
  }
};

// TMEM accumulator rows [r0, r0 + 64) of a slot (64 columns): the four panel warps whose lane
// quarter holds them read 32 rows x 32 columns each; f(row - r0, column, value)
template <class F>
__device__ __forceinline__ void tmem_rows64(uint32_t tacc, int r0, int warp, int pw, F f) {
  const int t = r0 >> 7, h = (r0 >> 6) & 1, q = warp & 3;
  if ((q >> 1) != h) return;
  const int cb = (pw >= 4) ? 32 : 0;
  const uint32_t taddr = tacc + (uint32_t(q * 32) << 16) + uint32_t(64 * t + cb);
  uint32_t w[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]),
        "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15]), "=r"(w[16]),
        "=r"(w[17]), "=r"(w[18]), "=r"(w[19]), "=r"(w[20]), "=r"(w[21]), "=r"(w[22]), "=r"(w[23]), "=r"(w[24]),
        "=r"(w[25]), "=r"(w[26]), "=r"(w[27]), "=r"(w[28]), "=r"(w[29]), "=r"(w[30]), "=r"(w[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  const int row = 32 * q - 64 * h + (threadIdx.x & 31);
#pragma unroll
  for (int c = 0; c < 32; ++c) f(row, cb + c, __uint_as_float(w[c]));
}

// optional phase timing (p.prof != nullptr): cycles per section, accumulated by thread 64
enum { PF_WAIT = 0, PF_LOAD = 1, PF_S1 = 2, PF_S2 = 3, PF_S3 = 4, PF_END = 5, PF_ITEMS = 6, PF_N = 8 };
struct Timer {
  long long* acc;
  long long t0;
  __device__ void start() {
    if (acc) t0 = clock64();
  }
  __device__ void lap(int k) {
    if (acc) {
      const long long t = clock64();
      acc[k] += t - t0;
      t0 = t;
    }
  }
};

// ---------------------------------------------------------------- step schedule
// Steps tau = 0, 1, 2, ... alternate between slot 0 and slot 1; step ss = tau >> 1 of a slot is
// panel ss % nblk of its item ss / nblk.  The slots' items: this CTA's items blockIdx.x + m G
// (G = gridDim.x), m even for slot 0, odd for slot 1.  Item i = (matrix i >> 1, sweep i & 1) when
// both sweeps are requested.
struct Step {
  int slot, ss, sweep, b, I;
  bool active, last;  // last: neither slot has an item at this round
};
__device__ __forceinline__ Step step_of(const Params& p, int64_t tau, int64_t items) {
  Step st;
  const int ns = p.nslots;
  st.slot = int(tau % ns);
  st.ss = int(tau / ns);
  const int64_t round = st.ss / p.nblk;
  const int64_t item = blockIdx.x + (ns * round + st.slot) * gridDim.x;
  st.active = item < items;
  st.last = blockIdx.x + ns * round * gridDim.x >= items;
  const bool both = (p.mode & 3) == 3;
  st.b = int(both ? item >> 1 : item);
  st.sweep = both ? int(item & 1) : ((p.mode & 1) ? 0 : 1);
  const int panel = st.ss % p.nblk;
  st.I = st.sweep == 0 ? p.nblk - 1 - panel : panel;
  return st;
}

// tensor-core jobs of a step: tiles t0 .. nt-1 of 128 rows, nch K chunks of 32 each
struct Jobs {
  int kind, I, k, t0, nt, nch;
  __device__ __forceinline__ int count() const { return (nt - t0) * nch; }
};
__device__ __forceinline__ Jobs jobs_of(const Params& p, const Step& st) {
  const int NT = (p.n + 127) / 128;
  if (st.sweep == 0) {  // R1: rows / K columns k .. n
    const int k = NBK * (st.I + 1), pr = p.n - k;
    return Jobs{0, st.I, k, (st.I + 1) >> 1, NT, pr > 0 ? pr / BK : 0};
  }
  const int j = NBK * st.I;  // F1: rows j .. n, K = 2 j (two segments)
  return Jobs{1, st.I, j + NBK, st.I >> 1, NT, 2 * (j / BK)};
}

// A operand major of a reverse job: 1 = MN-major (columns of T / S), 0 = K-major (rows of T)
__device__ __forceinline__ int rev_a_mn(int t, int C) { return (C <= 2 * t) ? 1 : 0; }

__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, int c0, int c1, int b, uint64_t* bar) {
  tma_load_3d(dst, m, c0, c1, b, bar);
}

// Handshakes.  full / empty: the TMA -> MMA operand ring.  acc_ready[slot] (mbarrier, one phase per
// active step of the slot, committed by the MMA thread): the step's accumulators are in TMEM.
// panel_cnt[slot] (shared counter, release / acquire): panels of the slot completed -- the TMA
// thread loads step ss of a slot only when panel_cnt >= ss (its operands T / Ldot are published
// and the slot's TMEM rows drained), and the MMA thread commits an empty step's acc_ready only
// then, so acc_ready never runs two phases ahead of the panel warps.
struct Bars {
  uint64_t *full, *empty, *acc_ready;
  uint32_t* panel_cnt;
};
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];\n" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;\n" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_panels(const uint32_t* cnt, uint32_t need) {
  uint32_t spins = 0;
  uint64_t t0 = 0;
  while (ld_acquire(cnt) < need) {
    if (CD_WATCHDOG_NS != 0 && (++spins & 0xFFFFu) == 0) {  // protocol-error watchdog (gemm_tc32.cuh)
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > uint64_t(CD_WATCHDOG_NS)) __trap();
    }
  }
}

// ---------------------------------------------------------------- TMA producer (warp 0, lane 0)
__device__ void tma_role(const Params& p, const Maps& tm, unsigned char* ring, const Bars& br, int64_t items) {
  uint32_t it = 0;
  for (int64_t tau = 0;; ++tau) {
    const Step st = step_of(p, tau, items);
    if (st.last) break;
    if (!st.active) continue;
    const Jobs jb = jobs_of(p, st);
    const int nj = jb.count();
    if (nj == 0) continue;
    // the slot's previous panels have published T / Ldot and drained its TMEM rows
    wait_panels(&br.panel_cnt[st.slot], uint32_t(st.ss));
    const int b = st.b;
    for (int q = 0; q < nj; ++q, ++it) {
      const uint32_t s = it % STAGES;
      if (it >= STAGES) tc_wait(&br.empty[s], ((it / STAGES) - 1) & 1);
      const int t = jb.t0 + q / jb.nch, c = q % jb.nch;
      unsigned char* a = ring + s * STAGE_BYTES;
      unsigned char* bb = a + A_BYTES;
      uint64_t* bar = &br.full[s];
      mbar_expect_tx(bar, STAGE_BYTES);
      if (jb.kind == 0) {
        const int kc = jb.k + 32 * c, C = kc >> 6;
        if (C < 2 * t) {  // T below the diagonal: columns of T, MN-major
          for (int x = 0; x < 4; ++x) tma3(a + x * 4096, &tm.tr_mn, 128 * t + 32 * x, kc, b, bar);
        } else if (C > 2 * t + 1) {  // above: rows of T (T^T), K-major
          for (int h = 0; h < 2; ++h) tma3(a + h * 8192, &tm.tr_k, kc, 128 * t + 64 * h, b, bar);
        } else if (C == 2 * t) {  // rows of block C: S_C; rows of block C+1: T below
          for (int x = 0; x < 2; ++x) tma3(a + x * 4096, &tm.s_mn, 32 * x, kc, b, bar);
          for (int x = 2; x < 4; ++x) tma3(a + x * 4096, &tm.tr_mn, 128 * t + 32 * x, kc, b, bar);
        } else {  // C == 2t+1: rows of block C-1: T^T (K-major); rows of block C: S_C (symmetric)
          tma3(a, &tm.tr_k, kc, 128 * t, b, bar);
          tma3(a + 8192, &tm.s_k, kc - 64 * C, 64 * C, b, bar);
        }
        tma3(bb, &tm.lr_k, kc, 64 * jb.I, b, bar);
      } else {
        const int half = jb.nch / 2, seg = c / half, kk = 32 * (c % half), j = 64 * jb.I;
        const CUtensorMap* am = seg == 0 ? &tm.ldr_mn : &tm.lr_mn;
        const CUtensorMap* bm = seg == 0 ? &tm.lr_mn : &tm.ldr_mn;
        for (int x = 0; x < 4; ++x) tma3(a + x * 4096, am, 128 * t + 32 * x, kk, b, bar);
        for (int h = 0; h < 2; ++h) tma3(bb + h * 4096, bm, j + 32 * h, kk, b, bar);
      }
    }
  }
}

// ---------------------------------------------------------------- MMA issuer (warp 1, lane 0)
__device__ void mma_role(const Params& p, unsigned char* ring, const Bars& br, uint32_t tmem, int64_t items) {
  uint32_t it = 0;
  for (int64_t tau = 0;; ++tau) {
    const Step st = step_of(p, tau, items);
    if (st.last) break;
    if (!st.active) continue;
    const Jobs jb = jobs_of(p, st);
    const int nj = jb.count();
    const uint32_t tacc = tmem + uint32_t(256 * st.slot);
    if (nj == 0) wait_panels(&br.panel_cnt[st.slot], uint32_t(st.ss));  // (see Bars)
    for (int q = 0; q < nj; ++q, ++it) {
      const uint32_t s = it % STAGES;
      tc_wait(&br.full[s], (it / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const int t = jb.t0 + q / jb.nch, c = q % jb.nch;
      const int a_mn = jb.kind == 0 ? rev_a_mn(t, (jb.k + 32 * c) >> 6) : 1;
      const int b_mn = jb.kind == 0 ? 0 : 1;
      const uint32_t idesc = tc_idesc(a_mn, b_mn, NBK);
      const uint32_t sa = smem_u32(ring + s * STAGE_BYTES), sb = sa + A_BYTES;
      const uint32_t d = tacc + uint32_t(64 * t);
#pragma unroll
      for (int k8 = 0; k8 < BK / 8; ++k8) {
        const uint64_t da = a_mn ? umma_desc(sa + k8 * 1024, 4096, 512, 1) : umma_desc(sa + k8 * 32, 16, 1024, 2);
        const uint64_t db = b_mn ? umma_desc(sb + k8 * 1024, 4096, 512, 1) : umma_desc(sb + k8 * 32, 16, 1024, 2);
        const uint32_t accum = (c > 0 || k8 > 0) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred P;\nsetp.ne.b32 P, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, P;\n}\n" ::"r"(d),
            "l"(da), "l"(db), "r"(idesc), "r"(accum));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       smem_u32(&br.empty[s]))
                   : "memory");
    }
    // every step signals its accumulators (an empty step too: the panel waits on it uniformly)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(&br.acc_ready[st.slot]))
                 : "memory");
  }
}

// ---------------------------------------------------------------- reverse panel step
__device__ void rev_panel(const Params& p, const Step& st, uint32_t tacc, uint32_t buf, int warp, int pw, int pt,
                          Timer& tmr) {
  const int n = p.n, I = st.I, b = st.b;
  const int k = NBK * (I + 1), pr = n - k, c0 = NBK * I;
  const float* L = p.L + b * p.sL;
  float* A = p.Ab + b * p.sA;
  float* Tr = p.Tr + int64_t(b) * n * n;
  const float* Dinv = p.Dinv + int64_t(b) * NBK * n;
  float* S = p.S + int64_t(b) * NBK * n;
  // buffers: bDi = D^{-1}, bLb = tril(Lbar[I, I]) -> Dbar', bC = the chunk (in - acc), bC2 = Cbar of
  // the chunk, bL0 / bL1 = C = L chunks (double-buffered); after the chunk loop bC = D
  const uint32_t bDi = buf, bLb = bDi + 4 * SCR, bC = bLb + 4 * SCR, bC2 = bC + 4 * SCR, bL0 = bC2 + 4 * SCR,
                 bL1 = bL0 + 4 * SCR;
  const int nch = pr / NBK;
  {
    Tile64 t0, t1, t2, t3;
    t0.load(Dinv + int64_t(c0) * NBK, NBK, pt, false);
    t1.load(A + c0 + int64_t(c0) * p.lda, p.lda, pt, true);
    if (nch > 0) {
      t2.load(A + k + int64_t(c0) * p.lda, p.lda, pt, false);  // Lbar chunk 0
      t3.load(L + k + int64_t(c0) * p.ldl, p.ldl, pt, false);  // C chunk 0
    }
    t0.store(bDi, pt);
    t1.store(bLb, pt);
    if (nch > 0) {
      t2.store(bC, pt);
      t3.store(bL0, pt);
    }
  }
  panel_sync();
  tmr.lap(PF_LOAD);
  // G = Cbar^T C accumulated over the chunks; each warp owns a 16 x 32 block of G
  const int gr0 = 16 * (pw >> 1), gc0 = 32 * (pw & 1);
  float g[4][4];
  zero(g);
  for (int ch = 0; ch < nch; ++ch) {
    const int r0 = k + NBK * ch;  // global row of the chunk
    const uint32_t bL = (ch & 1) ? bL1 : bL0, bLn = (ch & 1) ? bL0 : bL1;
    // next chunk's inputs in flight while this one is processed
    Tile64 nin, nl;
    const bool more = ch + 1 < nch;
    if (more) {
      nin.load(A + (r0 + NBK) + int64_t(c0) * p.lda, p.lda, pt, false);
      nl.load(L + (r0 + NBK) + int64_t(c0) * p.ldl, p.ldl, pt, false);
    }
    // R2: bC = Lbar rows - acc rows (TMEM)
    tmem_rows64(tacc, r0, warp, pw, [&](int r, int c, float v) {
      const uint32_t a = el(bC, r, c);
      sts(a, lds(a) - v);
    });
    panel_sync();
    // R3: Cbar = bC D^{-1} -> bC2, A[rows, I] (fp32) and Tr (tf32-rounded)
    gemm64(pw, rowmajor(bC), rowmajor(bDi), [&](int r, int c, float v) {
      sts(el(bC2, r, c), v);
      __stcg(A + (r0 + r) + int64_t(c0 + c) * p.lda, v);
      __stcg(Tr + (r0 + r) + int64_t(c0 + c) * n, rnd(v));
    });
    panel_sync();
    // R4 (partial): G += Cbar_chunk^T C_chunk
    warp_mma<4>(g, NBK, rowmajor(bC2).tr().sub(gr0, 0), rowmajor(bL).sub(0, gc0));
    if (more) {
      nin.store(bC, pt);
      nl.store(bLn, pt);
    }
    panel_sync();
  }
  tmr.lap(PF_S1);
  // Dbar' = Lbar[I, I] - tril(G) (in bLb), then D -> bC
  for_acc(g, [&](int r, int c, float v) {
    const int i = gr0 + r, j = gc0 + c;
    const uint32_t a = el(bLb, i, j);
    if (i >= j) sts(a, lds(a) - v);
  });
  {
    Tile64 td;
    td.load(L + c0 + int64_t(c0) * p.ldl, p.ldl, pt, true);
    td.store(bC, pt);
  }
  panel_sync();
  tmr.lap(PF_S2);
  // R5: Eq. 10.  P = D^T Dbar' -> bC2
  gemm64(pw, rowmajor(bC).tr(), rowmajor(bLb), [&](int r, int c, float v) { sts(el(bC2, r, c), v); });
  panel_sync();
  // Psym = Phi(P) + Phi(P)^T: strict lower mirrored, diagonal P_ii -> bL0
  for (int q = 0; q < 16; ++q) {
    int i, j;
    tile_rc(pt, q, i, j);
    sts(el(bL0, i, j), i >= j ? lds(el(bC2, i, j)) : lds(el(bC2, j, i)));
  }
  panel_sync();
  // X1 = D^{-T} Psym -> bL1
  gemm64(pw, rowmajor(bDi).tr(), rowmajor(bL0), [&](int r, int c, float v) { sts(el(bL1, r, c), v); });
  panel_sync();
  // X = X1 D^{-1}; Dbar = Phi(X) -> A[I, I] (lower) and Tr; S_I = Phi(X) + Phi(X)^T (rounded)
  gemm64(pw, rowmajor(bL1), rowmajor(bDi), [&](int i, int j, float v) {
    if (i > j) {
      __stcg(A + (c0 + i) + int64_t(c0 + j) * p.lda, v);
      __stcg(Tr + (c0 + i) + int64_t(c0 + j) * n, rnd(v));
      __stcg(S + i + int64_t(c0 + j) * NBK, rnd(v));
      __stcg(S + j + int64_t(c0 + i) * NBK, rnd(v));
    } else if (i == j) {
      __stcg(A + (c0 + i) + int64_t(c0 + i) * p.lda, 0.5f * v);
      __stcg(Tr + (c0 + i) + int64_t(c0 + i) * n, rnd(0.5f * v));
      __stcg(S + i + int64_t(c0 + i) * NBK, rnd(v));
    }
  });
  tmr.lap(PF_S3);
}

// ---------------------------------------------------------------- forward panel step
__device__ void fwd_panel(const Params& p, const Step& st, uint32_t tacc, uint32_t buf, int warp, int pw, int pt,
                          Timer& tmr) {
  const int n = p.n, I = st.I, b = st.b;
  const int j = NBK * I, k = j + NBK, pr = n - k;
  const float* L = p.L + b * p.sL;
  float* A = p.Ad + b * p.sD;
  float* Ldr = p.Ldr + int64_t(b) * n * n;
  const float* Dinv = p.Dinv + int64_t(b) * NBK * n;
  // buffers: bDi = D^{-1}, bD = D, bDd = Ddot (zero above), bIn = chunk, bT = temp, bL0 / bL1 = C chunks
  const uint32_t bDi = buf, bD = bDi + 4 * SCR, bDd = bD + 4 * SCR, bIn = bDd + 4 * SCR, bT = bIn + 4 * SCR,
                 bL0 = bT + 4 * SCR, bL1 = bL0 + 4 * SCR;
  const int nch = pr / NBK;
  {
    Tile64 t0, t1, t2;
    t0.load(Dinv + int64_t(j) * NBK, NBK, pt, false);
    t1.load(L + j + int64_t(j) * p.ldl, p.ldl, pt, true);
    t2.load(A + j + int64_t(j) * p.ldd, p.ldd, pt, true);  // Sigma_dot[I, I] (lower)
    t0.store(bDi, pt);
    t1.store(bD, pt);
    t2.store(bIn, pt);
  }
  panel_sync();
  // F2 (diagonal rows): Ddot' = Sigma_dot[I, I] - tril(acc rows j .. j+63)
  if (I > 0) {
    tmem_rows64(tacc, j, warp, pw, [&](int r, int c, float v) {
      const uint32_t a = el(bIn, r, c);
      if (c <= r) sts(a, lds(a) - v);
    });
    panel_sync();
  }
  tmr.lap(PF_LOAD);
  // F3 (Eq. 8): Ddot_sym (mirror of the lower triangle) -> bT
  for (int q = 0; q < 16; ++q) {
    int i, c;
    tile_rc(pt, q, i, c);
    sts(el(bT, i, c), i >= c ? lds(el(bIn, i, c)) : lds(el(bIn, c, i)));
  }
  panel_sync();
  // Y = D^{-1} Ddot_sym -> bIn
  gemm64(pw, rowmajor(bDi), rowmajor(bT), [&](int r, int c, float v) { sts(el(bIn, r, c), v); });
  panel_sync();
  // Z = Phi(Y D^{-T}) -> bT
  gemm64(pw, rowmajor(bIn), rowmajor(bDi).tr(), [&](int r, int c, float v) {
    sts(el(bT, r, c), (r > c) ? v : (r == c ? 0.5f * v : 0.f));
  });
  panel_sync();
  // Ddot = D Z (lower) -> A[I, I], Ldr and bDd (zero above: the operand of F4)
  gemm64(pw, rowmajor(bD), rowmajor(bT), [&](int r, int c, float v) {
    sts(el(bDd, r, c), r >= c ? v : 0.f);
    if (r >= c) {
      __stcg(A + (j + r) + int64_t(j + c) * p.ldd, v);
      __stcg(Ldr + (j + r) + int64_t(j + c) * n, rnd(v));
    }
  });
  if (nch > 0) {  // chunk 0 inputs
    Tile64 ti, tl;
    ti.load(A + k + int64_t(j) * p.ldd, p.ldd, pt, false);
    tl.load(L + k + int64_t(j) * p.ldl, p.ldl, pt, false);
    ti.store(bIn, pt);
    tl.store(bL0, pt);
  }
  panel_sync();
  tmr.lap(PF_S1);
  // F4 by 64-row chunks: Cdot' = Sigma_dot rows - acc rows; Cdot = (Cdot' - C Ddot^T) D^{-T}
  for (int ch = 0; ch < nch; ++ch) {
    const int r0 = k + NBK * ch;
    const uint32_t bL = (ch & 1) ? bL1 : bL0, bLn = (ch & 1) ? bL0 : bL1;
    Tile64 nin, nl;
    const bool more = ch + 1 < nch;
    if (more) {
      nin.load(A + (r0 + NBK) + int64_t(j) * p.ldd, p.ldd, pt, false);
      nl.load(L + (r0 + NBK) + int64_t(j) * p.ldl, p.ldl, pt, false);
    }
    if (I > 0) {
      tmem_rows64(tacc, r0, warp, pw, [&](int r, int c, float v) {
        const uint32_t a = el(bIn, r, c);
        sts(a, lds(a) - v);
      });
      panel_sync();
    }
    // bIn -= C Ddot^T (each warp its own 16 x 32 block)
    gemm64(pw, rowmajor(bL), rowmajor(bDd).tr(), [&](int r, int c, float v) {
      const uint32_t a = el(bIn, r, c);
      sts(a, lds(a) - v);
    });
    panel_sync();
    // Cdot = bIn D^{-T} -> A (fp32) and Ldr (rounded)
    gemm64(pw, rowmajor(bIn), rowmajor(bDi).tr(), [&](int r, int c, float v) {
      __stcg(A + (r0 + r) + int64_t(j + c) * p.ldd, v);
      __stcg(Ldr + (r0 + r) + int64_t(j + c) * n, rnd(v));
    });
    panel_sync();
    if (more) {
      nin.store(bIn, pt);
      nl.store(bLn, pt);
    }
    panel_sync();
  }
  tmr.lap(PF_S2);
}

// ---------------------------------------------------------------- panel warps (2..9)
__device__ void panel_role(const Params& p, uint32_t buf, const Bars& br, uint32_t tmem, int warp, int64_t items) {
  const int pw = warp - W_P0, pt = threadIdx.x - W_P0 * 32;
  Timer tmr{(p.prof && pt == 0) ? p.prof + blockIdx.x * PF_N : nullptr, 0};
  tmr.start();
  for (int64_t tau = 0;; ++tau) {
    const Step st = step_of(p, tau, items);
    if (st.last) break;
    if (!st.active) continue;
    tc_wait(&br.acc_ready[st.slot], st.ss & 1);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    tmr.lap(PF_WAIT);
    const uint32_t tacc = tmem + uint32_t(256 * st.slot);
    if (st.sweep == 0) rev_panel(p, st, tacc, buf, warp, pw, pt, tmr);
    else fwd_panel(p, st, tacc, buf, warp, pw, pt, tmr);
    // publish: results (global, generic proxy) become visible to the next update's TMA loads; the
    // slot's TMEM rows are drained
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    panel_sync();
    if (pt == 0) st_release(&br.panel_cnt[st.slot], uint32_t(st.ss + 1));
    tmr.lap(PF_END);
    if (tmr.acc && st.ss % p.nblk == p.nblk - 1) tmr.acc[PF_ITEMS] += 1;
  }
}

__global__ void __launch_bounds__(THREADS, 1) k_rf32(const Params p, const __grid_constant__ Maps tm) {
  extern __shared__ __align__(1024) unsigned char smem_rf[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_rf) + 1023) & ~uintptr_t(1023));
  unsigned char* ring = base;
  const uint32_t buf = smem_u32(base + RING_BYTES);
  Bars br;
  br.full = reinterpret_cast<uint64_t*>(base + RING_BYTES + BUF_BYTES);
  br.empty = br.full + STAGES;
  br.acc_ready = br.empty + STAGES;
  br.panel_cnt = reinterpret_cast<uint32_t*>(br.acc_ready + 2);
  uint32_t* tmem_slot = br.panel_cnt + 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&br.full[s], 1);
      mbar_init(&br.empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&br.acc_ready[s], 1);
      br.panel_cnt[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {  // TMEM: 2 slots x 4 accumulator tiles x 64 fp32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int64_t items = ((p.mode & 3) == 3) ? 2 * p.batch : p.batch;
  if (warp == 0) {
    if (lane == 0) tma_role(p, tm, ring, br, items);
  } else if (warp == 1) {
    if (lane == 0) mma_role(p, ring, br, tmem, items);
  } else {
    panel_role(p, buf, br, tmem, warp, items);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}


// ---------------------------------------------------------------- diagonal blocks of the layered
// fp32 schedule (N_b = 64): one CTA of 256 threads per matrix, the same Eq. 10 / Eq. 8 products as
// the fused kernel's R5 / F3 on mma.sync from shared memory (replaces the fp64-DMMA 8 x 8 blocked
// sweeps k_rev_dmma_cta / k_fwd_dmma_cta for these blocks).
//   rev: tril(A) = Dbar' -> Dbar = Phi(X), X = D^{-T}(P + P^T)D^{-1}, P = Phi(D^T Dbar');
//        S (optional, dense) = Dbar + Dbar^T = Phi(X) + Phi(X)^T
//   fwd: tril(A) = Ddot' -> Ddot = D Phi(D^{-1} Ddot'_sym D^{-T}); S (optional) = tril(Ddot),
//        zeros above
struct Diag64 {
  const float* L;
  int64_t ldl, sL;
  float* A;
  int64_t lda, sA;
  const float* Dinv;  // 64 x 64 blocks, ld 64 (128 x 128, ld ldi, for k_rf_diag128), batch stride dstride
  int64_t dstride;
  float* S;
  int64_t lds, sS;
  int rev;
  int64_t ldi;
};
// Eq. 10 on one 64 x 64 block: D in bD, D^{-1} in bDi, Dbar' (lower, zeros above) in bIn -- all three
// tf32-rounded (the products take pre-rounded operands); scratch bT (P, then X1) and bU (Psym).
// out(i, j, v) receives every element of the symmetric X = D^{-T} (P + P^T) D^{-1},
// P = Phi(D^T Dbar'); the result is Dbar = Phi(X), S = Phi(X) + Phi(X)^T
template <class F>
__device__ __forceinline__ void eq10_64(int pw, int pt, uint32_t bD, uint32_t bDi, uint32_t bIn, uint32_t bT,
                                        uint32_t bU, F out) {
  gemm64<true>(pw, rowmajor(bD).tr(), rowmajor(bIn), [&](int r, int c, float v) { sts(el(bT, r, c), v); });  // P
  panel_sync();
  for (int q = 0; q < 16; ++q) {  // Psym
    int i, j;
    tile_rc(pt, q, i, j);
    sts(el(bU, i, j), rnd(i >= j ? lds(el(bT, i, j)) : lds(el(bT, j, i))));
  }
  panel_sync();
  gemm64<true>(pw, rowmajor(bDi).tr(), rowmajor(bU), [&](int r, int c, float v) { sts(el(bT, r, c), rnd(v)); });  // X1
  panel_sync();
  gemm64<true>(pw, rowmajor(bT), rowmajor(bDi), out);  // X
}

// Eq. 8 on one 64 x 64 block: D in bD, D^{-1} in bDi (both tf32-rounded), Ddot' (lower) in bIn;
// scratch bT; bIn is overwritten.  out(r, c, v) receives every element of
// Ddot = D Phi(D^{-1} Ddot'_sym D^{-T}) (lower triangular: zero above the diagonal)
template <class F>
__device__ __forceinline__ void eq8_64(int pw, int pt, uint32_t bD, uint32_t bDi, uint32_t bIn, uint32_t bT, F out) {
  for (int q = 0; q < 16; ++q) {  // Ddot'_sym
    int i, c;
    tile_rc(pt, q, i, c);
    sts(el(bT, i, c), rnd(i >= c ? lds(el(bIn, i, c)) : lds(el(bIn, c, i))));
  }
  panel_sync();
  gemm64<true>(pw, rowmajor(bDi), rowmajor(bT), [&](int r, int c, float v) { sts(el(bIn, r, c), rnd(v)); });  // Y
  panel_sync();
  gemm64<true>(pw, rowmajor(bIn), rowmajor(bDi).tr(), [&](int r, int c, float v) {  // Z = Phi(Y D^{-T})
    sts(el(bT, r, c), rnd((r > c) ? v : (r == c ? 0.5f * v : 0.f)));
  });
  panel_sync();
  gemm64<true>(pw, rowmajor(bD), rowmajor(bT), out);  // Ddot = D Z
}

__global__ void __launch_bounds__(PANEL_THREADS) k_rf_diag64(const Diag64 q) {
  extern __shared__ __align__(16) unsigned char smem_d64[];
  const uint32_t b0 = smem_u32(smem_d64), b1 = b0 + 4 * SCR, b2 = b1 + 4 * SCR, b3 = b2 + 4 * SCR, b4 = b3 + 4 * SCR;
  const int pt = threadIdx.x, pw = pt >> 5;
  const int64_t b = blockIdx.x;
  const float* L = q.L + b * q.sL;
  float* A = q.A + b * q.sA;
  float* S = q.S ? q.S + b * q.sS : nullptr;
  {
    Tile64 td, ti, ta;
    td.load(L, q.ldl, pt, true);                     // D
    ti.load(q.Dinv + b * q.dstride, NBK, pt, false);  // D^{-1}
    ta.load(A, q.lda, pt, true);                     // Dbar' / Ddot' (lower)
    td.store(b1, pt, true);
    ti.store(b2, pt, true);
    ta.store(b0, pt, true);
  }
  panel_sync();
  if (q.rev) {
    eq10_64(pw, pt, b1, b2, b0, b3, b4, [&](int i, int j, float v) {
      if (i > j) {
        A[i + int64_t(j) * q.lda] = v;
        if (S) {
          S[i + int64_t(j) * q.lds] = v;
          S[j + int64_t(i) * q.lds] = v;
        }
      } else if (i == j) {
        A[i + int64_t(i) * q.lda] = 0.5f * v;
        if (S) S[i + int64_t(i) * q.lds] = v;
      }
    });
  } else {
    eq8_64(pw, pt, b1, b2, b0, b3, [&](int r, int c, float v) {
      if (r >= c) A[r + int64_t(c) * q.lda] = v;
      if (S) S[r + int64_t(c) * q.lds] = r >= c ? v : 0.f;
    });
  }
}

// 64 x 64 x 128 product over the 8 panel warps: A1 B1 + A2 B2 (same warp layout as gemm64)
template <class FOUT>
__device__ __forceinline__ void gemm64x2(int pw, const SV& A1, const SV& B1, const SV& A2, const SV& B2, FOUT out) {
  const int r0 = 16 * (pw >> 1), c0 = 32 * (pw & 1);
  float acc[4][4];
  zero(acc);
  warp_mma<4, true>(acc, NBK, A1.sub(r0, 0), B1.sub(0, c0));
  warp_mma<4, true>(acc, NBK, A2.sub(r0, 0), B2.sub(0, c0));
  for_acc(acc, [&](int r, int c, float v) { out(r0 + r, c0 + c, v); });
}

// ---------------------------------------------------------------- 128-wide diagonal blocks of the
// layered fp32 schedule (N_b = 128 for the trailing updates): the 128 x 128 block's own sweep as
// the blocked algorithm with two 64-wide steps (PAPER.md:689-701 / 655-666 on the block), every
// product on mma.sync from shared memory, one CTA of 256 threads per matrix.  With the block
// [D11 0; L21 D22], inverses D11^{-1}, D22^{-1} (the diagonal blocks of the 128-wide inverse):
//   rev:  Dbar22 = Eq10(D22, Dbar22');  Dbar21 -= S22 L21  (S22 = Dbar22 + Dbar22^T);
//         Cbar = Dbar21 D11^{-1};  Dbar11' -= tril(Cbar^T L21);  Dbar11 = Eq10(D11, Dbar11')
//         S (128 x 128, dense) = Dbar + Dbar^T = [S11 Cbar^T; Cbar S22]
//   fwd:  Ddot11 = Eq8(D11, Ddot11');  Ddot21 = (Ddot21' - L21 tril(Ddot11)^T) D11^{-T};
//         Ddot22' -= tril(Ddot21 L21^T + L21 Ddot21^T);  Ddot22 = Eq8(D22, Ddot22')
//         S (128 x 128) = tril(Ddot), zeros above
// Six 64 x 64 buffers (108 KB): two CTAs per SM.  The next step's operands are prefetched into
// registers while the current step's products run.
__global__ void __launch_bounds__(PANEL_THREADS, 2) k_rf_diag128(const Diag64 q) {
  extern __shared__ __align__(16) unsigned char smem_d128[];
  const uint32_t B0 = smem_u32(smem_d128), B1 = B0 + 4 * SCR, B2 = B1 + 4 * SCR, B3 = B2 + 4 * SCR,
                 B4 = B3 + 4 * SCR, B5 = B4 + 4 * SCR;
  const int pt = threadIdx.x, pw = pt >> 5;
  const int64_t b = blockIdx.x;
  const float* L = q.L + b * q.sL;
  float* A = q.A + b * q.sA;
  float* S = q.S ? q.S + b * q.sS : nullptr;
  const float* Di = q.Dinv + b * q.dstride;  // 128 x 128, ld q.ldi
  const int64_t ldl = q.ldl, lda = q.lda, lds_ = q.lds, ldi = q.ldi;
  const float* D11 = L;
  const float* L21 = L + 64;
  const float* D22 = L + 64 + 64 * ldl;
  const float* Di11 = Di;
  const float* Di22 = Di + 64 + 64 * ldi;
  float* A11 = A;
  float* A21 = A + 64;
  float* A22 = A + 64 + 64 * lda;
  if (q.rev) {
    {
      Tile64 t0, t1, t2;
      t0.load(D22, ldl, pt, true);
      t1.load(Di22, ldi, pt, false);
      t2.load(A22, lda, pt, true);
      t0.store(B1, pt, true);
      t1.store(B2, pt, true);
      t2.store(B0, pt, true);
    }
    Tile64 p0, p1;
    p0.load(L21, ldl, pt, false);
    p1.load(A21, lda, pt, false);
    panel_sync();
    eq10_64(pw, pt, B1, B2, B0, B3, B4, [&](int i, int j, float v) {  // Dbar22, S22
      if (i >= j) {
        A22[i + int64_t(j) * lda] = i == j ? 0.5f * v : v;
        sts(el(B5, i, j), rnd(v));
        sts(el(B5, j, i), rnd(v));
        if (S) {
          S[64 + i + (64 + j) * lds_] = v;
          S[64 + j + (64 + i) * lds_] = v;
        }
      }
    });
    panel_sync();
    p0.store(B1, pt, true);  // L21
    p1.store(B0, pt);        // Dbar21' (exact: updated below)
    Tile64 q0;
    q0.load(Di11, ldi, pt, false);
    panel_sync();
    gemm64<true>(pw, rowmajor(B5), rowmajor(B1), [&](int r, int c, float v) {  // Dbar21 -= S22 L21
      sts(el(B0, r, c), rnd(lds(el(B0, r, c)) - v));
    });
    q0.store(B2, pt, true);  // D11^{-1} (B2 is not read by that product)
    Tile64 q1, q2;
    q1.load(D11, ldl, pt, true);
    q2.load(A11, lda, pt, true);
    panel_sync();
    q1.store(B5, pt, true);  // D11 (S22 consumed)
    gemm64<true>(pw, rowmajor(B0), rowmajor(B2), [&](int r, int c, float v) {  // Cbar = Dbar21 D11^{-1}
      sts(el(B3, r, c), rnd(v));
      A21[r + int64_t(c) * lda] = v;
      if (S) {
        S[64 + r + int64_t(c) * lds_] = v;
        S[c + int64_t(64 + r) * lds_] = v;
      }
    });
    q2.store(B4, pt);  // Dbar11'
    panel_sync();
    gemm64<true>(pw, rowmajor(B3).tr(), rowmajor(B1), [&](int r, int c, float v) {  // Dbar11' -= tril(Cbar^T L21)
      if (r >= c) sts(el(B4, r, c), rnd(lds(el(B4, r, c)) - v));
    });
    panel_sync();
    eq10_64(pw, pt, B5, B2, B4, B0, B1, [&](int i, int j, float v) {  // Dbar11, S11
      if (i >= j) {
        A11[i + int64_t(j) * lda] = i == j ? 0.5f * v : v;
        if (S) {
          S[i + int64_t(j) * lds_] = v;
          S[j + int64_t(i) * lds_] = v;
        }
      }
    });
  } else {
    {
      Tile64 t0, t1, t2;
      t0.load(D11, ldl, pt, true);
      t1.load(Di11, ldi, pt, false);
      t2.load(A11, lda, pt, true);
      t0.store(B1, pt, true);
      t1.store(B2, pt, true);
      t2.store(B0, pt);
    }
    Tile64 p0, p1;
    p0.load(L21, ldl, pt, false);
    p1.load(A21, lda, pt, false);
    panel_sync();
    eq8_64(pw, pt, B1, B2, B0, B3, [&](int r, int c, float v) {  // Ddot11; tril copy in B4
      const float t = r >= c ? v : 0.f;
      if (r >= c) A11[r + int64_t(c) * lda] = v;
      sts(el(B4, r, c), rnd(t));
      if (S) {
        S[r + int64_t(c) * lds_] = t;
        S[r + int64_t(64 + c) * lds_] = 0.f;
      }
    });
    panel_sync();
    p0.store(B5, pt, true);  // L21
    p1.store(B0, pt);        // Ddot21' (exact: updated below)
    Tile64 q2;
    q2.load(A22, lda, pt, true);
    panel_sync();
    gemm64<true>(pw, rowmajor(B5), rowmajor(B4).tr(), [&](int r, int c, float v) {  // W = Ddot21' - L21 tril(Ddot11)^T
      sts(el(B0, r, c), rnd(lds(el(B0, r, c)) - v));
    });
    Tile64 q0, q1;
    q0.load(Di22, ldi, pt, false);
    q1.load(D22, ldl, pt, true);
    panel_sync();
    q2.store(B4, pt);  // Ddot22' (tril(Ddot11) consumed)
    gemm64<true>(pw, rowmajor(B0), rowmajor(B2).tr(), [&](int r, int c, float v) {  // Ddot21 = W D11^{-T}
      sts(el(B3, r, c), rnd(v));
      A21[r + int64_t(c) * lda] = v;
      if (S) S[64 + r + int64_t(c) * lds_] = v;
    });
    panel_sync();
    q1.store(B1, pt, true);  // D22
    q0.store(B2, pt, true);  // D22^{-1}
    gemm64x2(pw, rowmajor(B3), rowmajor(B5).tr(), rowmajor(B5), rowmajor(B3).tr(),
             [&](int r, int c, float v) {  // Ddot22' -= tril(Ddot21 L21^T + L21 Ddot21^T)
               if (r >= c) sts(el(B4, r, c), lds(el(B4, r, c)) - v);
             });
    panel_sync();
    eq8_64(pw, pt, B1, B2, B4, B0, [&](int r, int c, float v) {  // Ddot22
      if (r >= c) A22[r + int64_t(c) * lda] = v;
      if (S) S[64 + r + int64_t(64 + c) * lds_] = r >= c ? v : 0.f;
    });
  }
}

// 3xTF32 product (fp32-faithful): a b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi, hi = rna(x), lo = rna(x - hi)
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = rna(x);
  lo = rna(x - __uint_as_float(hi));
}
// one warp: acc[16 x 32] += A[16 x 64] B[64 x 32] in 3xTF32
__device__ __forceinline__ void warp_mma3(float (&acc)[4][4], const SV& A, const SV& B) {
  const FragBase fb = frag_base(A, B);
#pragma unroll 2
  for (int k0 = 0; k0 < NBK; k0 += 8) {
    Frag<4> f;
    frag_load(f, fb, k0);
    uint32_t ah[4], al[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) split_tf32(f.a[i], ah[i], al[i]);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      uint32_t bh[2], bl[2];
      split_tf32(f.b[nt][0], bh[0], bl[0]);
      split_tf32(f.b[nt][1], bh[1], bl[1]);
      mma8(acc[nt], al, bh);
      mma8(acc[nt], ah, bl);
      mma8(acc[nt], ah, bh);
    }
  }
}

// The 128-wide block inverses from the 64-wide ones already on their diagonal (k_trinv_dmma with
// odd_off): [D11 0; L21 D22]^{-1} = [D11^{-1} 0; -D22^{-1} L21 D11^{-1}  D22^{-1}], the two products
// on mma.sync in 3xTF32 (fp32-faithful); one CTA of 256 threads per block.  Dinv: 128 x 128 blocks,
// ld 128, nblk2 per matrix.
__global__ void __launch_bounds__(PANEL_THREADS) k_rf_inv128(int nblk2, const float* __restrict__ L, int64_t ldl,
                                                            int64_t sL, float* __restrict__ Dinv) {
  extern __shared__ __align__(16) unsigned char smem_i128[];
  const uint32_t b0 = smem_u32(smem_i128), b1 = b0 + 4 * SCR, b2 = b1 + 4 * SCR;
  const int pt = threadIdx.x, pw = pt >> 5;
  const int64_t blk = blockIdx.x;
  const int64_t b = blk / nblk2;
  const int Q = int(blk - b * nblk2);
  float* X = Dinv + blk * (128 * 128);
  {
    Tile64 ta, tl;
    ta.load(X, 128, pt, false);                                                    // D11^{-1}
    tl.load(L + b * sL + (128 * Q + 64) + int64_t(128 * Q) * ldl, ldl, pt, false);  // L21
    ta.store(b0, pt);
    tl.store(b1, pt);
  }
  Tile64 tc;
  tc.load(X + 64 + 64 * 128, 128, pt, false);  // D22^{-1}
#pragma unroll
  for (int q = 0; q < 16; ++q) {  // upper-right block
    const int e = pt + q * PANEL_THREADS;
    X[(e & 63) + ((e >> 6) + 64) * 128] = 0.f;
  }
  panel_sync();
  const int r0 = 16 * (pw >> 1), c0 = 32 * (pw & 1);
  {
    float acc[4][4];
    zero(acc);
    warp_mma3(acc, rowmajor(b1).sub(r0, 0), rowmajor(b0).sub(0, c0));  // T = L21 D11^{-1}
    tc.store(b2, pt);
    panel_sync();
    for_acc(acc, [&](int r, int c, float v) { sts(el(b1, r0 + r, c0 + c), v); });
  }
  panel_sync();
  float acc[4][4];
  zero(acc);
  warp_mma3(acc, rowmajor(b2).sub(r0, 0), rowmajor(b1).sub(0, c0));  // D22^{-1} T
  for_acc(acc, [&](int r, int c, float v) { X[64 + r0 + r + (c0 + c) * 128] = -v; });
}

// one warp: acc[16 x 8 NT] += A[16 x K] B[K x 8 NT] in 3xTF32 (K a multiple of 8)
// (k-steps [k_lo, k_hi) only: the caller skips the zero blocks of a triangular operand)
template <int NT>
__device__ __forceinline__ void warp_mma3k(float (&acc)[NT][4], int k_lo, int k_hi, const SV& A, const SV& B) {
  const FragBase fb = frag_base(A, B);
#pragma unroll 1
  for (int k0 = k_lo; k0 < k_hi; k0 += 8) {
    Frag<NT> f;
    frag_load(f, fb, k0);
    uint32_t ah[4], al[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) split_tf32(f.a[i], ah[i], al[i]);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      uint32_t bh[2], bl[2];
      split_tf32(f.b[nt][0], bh[0], bl[0]);
      split_tf32(f.b[nt][1], bh[1], bl[1]);
      mma8(acc[nt], al, bh);
      mma8(acc[nt], ah, bl);
      mma8(acc[nt], ah, bh);
    }
  }
}

// The 128-wide diagonal-block inverses of the layered fp32 schedule in one kernel, one CTA of 256
// threads per 128 x 128 block (the inverses the panel solves C D^{-1} and the Eq. 10 / Eq. 8 block
// steps use), by recursive doubling on the block:
//   [D11 0; L21 D22]^{-1} = [X11 0; X21 X22],  X21 = -X22 (L21 X11)
// applied at widths 16 -> 32 -> 64 -> 128: the sixteen 16 x 16 diagonal inverses by forward
// substitution in fp32 (one thread per column), every combination on mma.sync in 3xTF32
// (fp32-faithful products).  Replaces the fp64-DMMA 64-wide inverses + k_rf_inv128 (two launches,
// ~300 us for configs[3]).  Buffers: D11, L21, D22 and X11, X21, X22 (six swizzled 64 x 64 tiles,
// 108 KB: two CTAs per SM).  Out: Dinv, 128 x 128 blocks (ld 128), nblk2 per matrix, zero above
// the diagonal.
__global__ void __launch_bounds__(PANEL_THREADS, 2) k_rf_trinv128(int nblk2, const float* __restrict__ L,
                                                                   int64_t ldl, int64_t sL, float* __restrict__ Dinv) {
  extern __shared__ __align__(16) unsigned char smem_t128[];
  const uint32_t bD1 = smem_u32(smem_t128), bL21 = bD1 + 4 * SCR, bD2 = bL21 + 4 * SCR, bX1 = bD2 + 4 * SCR,
                 bX21 = bX1 + 4 * SCR, bX2 = bX21 + 4 * SCR;
  const int pt = threadIdx.x, pw = pt >> 5, lane = pt & 31;
  const int64_t blk = blockIdx.x;
  const int64_t b = blk / nblk2;
  const int Q = int(blk - b * nblk2);
  const float* D = L + b * sL + 128 * Q + int64_t(128 * Q) * ldl;
  {
    Tile64 t0, t1, t2;
    t0.load(D, ldl, pt, true);                // D11 (zero above the diagonal)
    t1.load(D + 64, ldl, pt, false);          // L21
    t2.load(D + 64 + 64 * ldl, ldl, pt, true);  // D22
    t0.store(bD1, pt);
    t1.store(bL21, pt);
    t2.store(bD2, pt);
#pragma unroll
    for (int q = 0; q < 16; ++q) {  // X buffers start at zero (the upper triangles stay zero)
      int r, c;
      tile_rc(pt, q, r, c);
      sts(el(bX1, r, c), 0.f);
      sts(el(bX2, r, c), 0.f);
    }
  }
  panel_sync();
  // width 16: the diagonal 16 x 16 blocks, thread (block, column c): D x = e_c by substitution
  if (pt < 128) {
    const int q = pt >> 4, c = pt & 15;
    const uint32_t bD = q < 4 ? bD1 : bD2, bX = q < 4 ? bX1 : bX2;
    const int o = 16 * (q & 3);
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float s = (i == c) ? 1.f : 0.f;
#pragma unroll
      for (int m = 0; m < i; ++m) s = fmaf(-lds(el(bD, o + i, o + m)), x[m], s);
      x[i] = (i >= c) ? s / lds(el(bD, o + i, o + i)) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i >= c) sts(el(bX, o + i, o + c), x[i]);
  }
  panel_sync();
  // width 32 (four combinations, warps 0..3) and 64 (two, warps 0..3 as two pairs): T = L21 X11 into
  // X21's place, then X21 = -X22 T (read fully before the in-place store)
#pragma unroll 1
  for (int lev = 0; lev < 2; ++lev) {
    const int h = lev == 0 ? 16 : 32;  // width of the halves being combined
    float acc[4][4];
    zero(acc);
    bool on = false;
    uint32_t bD = 0, bX = 0;
    int o = 0, rr = 0;
    if (lev == 0 && pw < 4) {  // combination pw: half pw >> 1, 32-block pw & 1; one warp, 16 x 16
      on = true;
      bD = pw < 2 ? bD1 : bD2, bX = pw < 2 ? bX1 : bX2, o = 32 * (pw & 1), rr = 0;
    } else if (lev == 1 && pw < 4) {  // combination pw >> 1, rows 16 (pw & 1); 16 x 32 per warp
      on = true;
      bD = pw < 2 ? bD1 : bD2, bX = pw < 2 ? bX1 : bX2, o = 0, rr = 16 * (pw & 1);
    }
    const SV L21v = SV{bD, o + h + rr, o, false}, X11v = SV{bX, o, o, false};
    const SV X22v = SV{bX, o + h + rr, o + h, false}, Tv = SV{bX, o + h, o, false};
    if (on) {
      if (lev == 0) {
        float a2[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        warp_mma3k<2>(a2, 0, h, L21v, X11v);
        for_acc(a2, [&](int r, int c, float v) { sts(Tv.sub(rr, 0).at(r, c), v); });
      } else {
        warp_mma3k<4>(acc, 0, h, L21v, X11v);
        for_acc(acc, [&](int r, int c, float v) { sts(Tv.sub(rr, 0).at(r, c), v); });
      }
    }
    panel_sync();
    if (on) {
      if (lev == 0) {
        float a2[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        warp_mma3k<2>(a2, 0, h, X22v, Tv);
        panel_sync();
        for_acc(a2, [&](int r, int c, float v) { sts(Tv.sub(rr, 0).at(r, c), -v); });
      } else {
        zero(acc);
        warp_mma3k<4>(acc, 0, rr + 16, X22v, Tv);  // X22 rows rr..rr+15: zero beyond column rr+15
        panel_sync();
        for_acc(acc, [&](int r, int c, float v) { sts(Tv.sub(rr, 0).at(r, c), -v); });
      }
    } else {
      panel_sync();
    }
    panel_sync();
  }
  // width 128: T = L21 X11 (8 warps, 16 x 32 each) -> bX21, then X21 = -X22 T in place
  const int r0 = 16 * (pw >> 1), c0 = 32 * (pw & 1);
  {
    float acc[4][4];
    zero(acc);
    warp_mma3k<4>(acc, c0, NBK, rowmajor(bL21).sub(r0, 0), rowmajor(bX1).sub(0, c0));  // X11(k, c) = 0 for k < c
    for_acc(acc, [&](int r, int c, float v) { sts(el(bX21, r0 + r, c0 + c), v); });
  }
  panel_sync();
  {
    float acc[4][4];
    zero(acc);
    warp_mma3k<4>(acc, 0, r0 + 16, rowmajor(bX2).sub(r0, 0), rowmajor(bX21).sub(0, c0));  // X22(r, k) = 0 for k > r
    panel_sync();
    for_acc(acc, [&](int r, int c, float v) { sts(el(bX21, r0 + r, c0 + c), -v); });
  }
  panel_sync();
  // out: [X11 0; X21 X22], coalesced along columns
  float* X = Dinv + blk * (128 * 128);
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    int r, c;
    tile_rc(pt, q, r, c);
    X[r + c * 128] = lds(el(bX1, r, c));
    X[r + (64 + c) * 128] = 0.f;
    X[64 + r + c * 128] = lds(el(bX21, r, c));
    X[64 + r + (64 + c) * 128] = lds(el(bX2, r, c));
  }
  (void)lane;
}

// Block inverses D_J^{-1} (fp32 forward substitution, one CTA of 64 threads per 64 x 64 block;
// thread c solves D x = e_c with four partial sums).  Out: 64 x n per matrix, column-major.
__global__ void __launch_bounds__(64) k_rf_trinv(int n, int nblk, const float* __restrict__ L, int64_t ldl,
                                                 int64_t sL, float* __restrict__ Dinv) {
  __shared__ float D[64 * 65];
  __shared__ float X[64 * 65];
  const int64_t blk = blockIdx.x;
  const int b = int(blk / nblk), J = int(blk % nblk);
  const float* src = L + b * sL + NBK * J + int64_t(NBK * J) * ldl;
  const int c = threadIdx.x;
  for (int e = c; e < 64 * 64; e += 64) {  // coalesced along columns
    const int i = e & 63, col = e >> 6;
    D[i * 65 + col] = (i >= col) ? src[i + int64_t(col) * ldl] : 0.f;
  }
  __syncthreads();
  for (int i = 0; i < c; ++i) X[i * 65 + c] = 0.f;
  for (int i = c; i < 64; ++i) {
    float s0 = (i == c) ? 1.f : 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int m = c;
    for (; m + 4 <= i; m += 4) {
      s0 -= D[i * 65 + m] * X[m * 65 + c];
      s1 -= D[i * 65 + m + 1] * X[(m + 1) * 65 + c];
      s2 -= D[i * 65 + m + 2] * X[(m + 2) * 65 + c];
      s3 -= D[i * 65 + m + 3] * X[(m + 3) * 65 + c];
    }
    for (; m < i; ++m) s0 -= D[i * 65 + m] * X[m * 65 + c];
    X[i * 65 + c] = ((s0 + s1) + (s2 + s3)) / D[i * 65 + i];
  }
  __syncthreads();
  float* dst = Dinv + int64_t(b) * NBK * n + int64_t(NBK * J) * NBK;
  for (int e = c; e < 64 * 64; e += 64) dst[e] = X[(e & 63) * 65 + (e >> 6)];
}

// L_r = tf32-rounded copy of tril(L) (dense n x n per matrix, ld n; the upper part is not read)
__global__ void k_rf_round(int n, int64_t batch, const float* __restrict__ L, int64_t ldl, int64_t sL,
                           float* __restrict__ Lr) {
  const int64_t nn = int64_t(n) * n, total = nn * batch;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = e / nn, r = e - b * nn;
    const int c = int(r / n), i = int(r - int64_t(c) * n);
    if (i >= c) Lr[e] = tf32_rna(__ldcs(L + b * sL + i + int64_t(c) * ldl));
  }
}

}  // namespace rf

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 rf_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
  }();
  return fn;
}

// 3-D fp32 map (rows, cols, batch) of column-major matrices, 128-byte swizzle (32-byte atoms for
// the MN-major tf32 operand layout)
static bool rf_map(CUtensorMap* m, const void* p, int64_t rows, int64_t cols, int64_t ld, int64_t bstride,
                   int64_t batch, int box0, int box1, bool atom32) {
  auto enc = rf_encoder();
  if (!enc) return false;
  cuuint64_t dims[3] = {cuuint64_t(rows), cuuint64_t(cols), cuuint64_t(batch)};
  cuuint64_t strides[2] = {cuuint64_t(ld * 4), cuuint64_t(std::max<int64_t>(bstride, 1) * 4)};
  cuuint32_t box[3] = {cuuint32_t(box0), cuuint32_t(box1), 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// CD_RF32_PROF=1: per-CTA section cycles of the last launch, read back with cd_rf32_prof_read
// (measurement only; tools/time_rf32.py)
static long long* g_rf_prof = nullptr;
static long long* rf_prof_buffer() {
  static const bool on = getenv("CD_RF32_PROF") != nullptr;
  if (!on) return nullptr;
  if (!g_rf_prof && cudaMalloc(&g_rf_prof, sizeof(long long) * 1024 * rf::PF_N) != cudaSuccess) g_rf_prof = nullptr;
  if (g_rf_prof) cudaMemset(g_rf_prof, 0, sizeof(long long) * 1024 * rf::PF_N);
  return g_rf_prof;
}

bool rf32_fused_supported(const RF32Call& c) {
  if (c.n <= 128 || c.n > rf::NMAX || c.n % rf::NBK || c.batch < 1 || !rf_encoder()) return false;
  if (!al16(c.L) || c.ldl % 4 || (c.batch > 1 && c.sL % 4)) return false;
  if ((c.mode & 1) && (!c.Ab || !al16(c.Ab) || c.lda % 4 || (c.batch > 1 && c.sA % 4))) return false;
  if ((c.mode & 2) && (!c.Ad || !al16(c.Ad) || c.ldd % 4 || (c.batch > 1 && c.sD % 4))) return false;
  return (c.mode & 3) != 0;
}

// workspace: D^{-1} and S (64 x n per matrix each), L_r, T_r, Ldot_r (n x n per matrix each)
size_t rf32_fused_ws(int n, int64_t batch) {
  return (2 * size_t(rf::NBK) * size_t(n) + 3 * size_t(n) * size_t(n)) * size_t(batch) * sizeof(float) + 1024;
}

cudaError_t rf32_fused_launch(const RF32Call& c, void* ws, cudaStream_t st, int sms, int64_t* launches) {
  using namespace rf;
  Params p;
  p.n = c.n;
  p.nblk = c.n / NBK;
  p.mode = c.mode;
  p.batch = c.batch;
  p.L = c.L;
  p.ldl = c.ldl;
  p.sL = c.batch > 1 ? c.sL : c.ldl * c.n;
  p.Ab = c.Ab;
  p.lda = c.lda;
  p.sA = c.batch > 1 ? c.sA : c.lda * c.n;
  p.Ad = c.Ad;
  p.ldd = c.ldd;
  p.sD = c.batch > 1 ? c.sD : c.ldd * c.n;
  const int64_t n = c.n, B = c.batch, nn = n * n;
  float* w = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  float* Dinv = w;
  float* S = Dinv + B * NBK * n;
  float* Lr = S + B * NBK * n;
  float* Tr = Lr + B * nn;
  float* Ldr = Tr + B * nn;
  p.Dinv = Dinv;
  p.S = S;
  p.Tr = Tr;
  p.Ldr = Ldr;
  p.prof = rf_prof_buffer();
  Maps tm;
  memset(&tm, 0, sizeof(tm));
  bool ok = rf_map(&tm.lr_mn, Lr, n, n, n, nn, B, 32, 32, true) && rf_map(&tm.lr_k, Lr, n, n, n, nn, B, 32, 64, false) &&
            rf_map(&tm.s_mn, S, NBK, n, NBK, NBK * n, B, 32, 32, true) &&
            rf_map(&tm.s_k, S, NBK, n, NBK, NBK * n, B, 32, 64, false) &&
            rf_map(&tm.tr_mn, Tr, n, n, n, nn, B, 32, 32, true) && rf_map(&tm.tr_k, Tr, n, n, n, nn, B, 32, 64, false) &&
            rf_map(&tm.ldr_mn, Ldr, n, n, n, nn, B, 32, 32, true);
  if (!ok) return cudaErrorInvalidValue;
  k_rf_trinv<<<unsigned(B * p.nblk), 64, 0, st>>>(c.n, p.nblk, c.L, c.ldl, p.sL, Dinv);
  ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t total = B * nn;
  k_rf_round<<<unsigned(std::min<int64_t>((total + 255) / 256, int64_t(sms) * 16)), 256, 0, st>>>(c.n, B, c.L, c.ldl,
                                                                                                  p.sL, Lr);
  ++*launches;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_rf32, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM));
    attr = true;
  }
  const int64_t items = ((c.mode & 3) == 3) ? 2 * B : B;
  // NSLOTS items per CTA at a time (CD_RF32_SLOTS, measurement switch; default 2)
  static const int nslots = getenv("CD_RF32_SLOTS") ? std::max(1, std::min(2, atoi(getenv("CD_RF32_SLOTS")))) : 2;
  p.nslots = nslots;
  const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>((items + nslots - 1) / nslots, sms)));
  k_rf32<<<grid, THREADS, SMEM, st>>>(p, tm);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t rf32_diag64(bool rev, int64_t batch, const float* L, int64_t ldl, int64_t sL, float* A, int64_t lda,
                        int64_t sA, const float* Dinv, int64_t dstride, float* S, int64_t lds, int64_t sS,
                        cudaStream_t st) {
  using namespace rf;
  Diag64 q{L, ldl, sL, A, lda, sA, Dinv, dstride, S, lds, sS, rev ? 1 : 0, NBK};
  constexpr size_t smem = 5 * SCR * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_rf_diag64, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr = true;
  }
  k_rf_diag64<<<unsigned(batch), PANEL_THREADS, smem, st>>>(q);
  return cudaGetLastError();
}

cudaError_t rf32_diag128(bool rev, int64_t batch, const float* L, int64_t ldl, int64_t sL, float* A, int64_t lda,
                         int64_t sA, const float* Dinv, int64_t ldi, int64_t dstride, float* S, int64_t lds,
                         int64_t sS, cudaStream_t st) {
  using namespace rf;
  Diag64 q{L, ldl, sL, A, lda, sA, Dinv, dstride, S, lds, sS, rev ? 1 : 0, ldi};
  constexpr size_t smem = 6 * SCR * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_rf_diag128, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr = true;
  }
  k_rf_diag128<<<unsigned(batch), PANEL_THREADS, smem, st>>>(q);
  return cudaGetLastError();
}

cudaError_t rf32_trinv128(int n, int64_t batch, const float* L, int64_t ldl, int64_t sL, float* Dinv, cudaStream_t st) {
  const int nblk2 = n / 128;
  constexpr size_t smem = 6 * rf::SCR * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(rf::k_rf_trinv128, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr = true;
  }
  rf::k_rf_trinv128<<<unsigned(batch * nblk2), rf::PANEL_THREADS, smem, st>>>(nblk2, L, ldl, sL, Dinv);
  return cudaGetLastError();
}

cudaError_t rf32_inv128(int n, int64_t batch, const float* L, int64_t ldl, int64_t sL, float* Dinv, cudaStream_t st) {
  const int nblk2 = n / 128;
  constexpr size_t smem = 3 * rf::SCR * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(rf::k_rf_inv128, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr = true;
  }
  rf::k_rf_inv128<<<unsigned(batch * nblk2), rf::PANEL_THREADS, smem, st>>>(nblk2, L, ldl, sL, Dinv);
  return cudaGetLastError();
}

}  // namespace cd

// measurement hook (not part of the documented ABI): sums over CTAs of the section cycles of the
// last fused launch with CD_RF32_PROF set (indices: see rf::PF_*)
extern "C" int cd_rf32_prof_read(long long* out, int grid) {
  if (!cd::g_rf_prof) return -1;
  long long h[1024 * cd::rf::PF_N];
  if (cudaMemcpy(h, cd::g_rf_prof, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return -2;
  for (int k = 0; k < cd::rf::PF_N; ++k) {
    out[k] = 0;
    for (int g = 0; g < grid && g < 1024; ++g) out[k] += h[g * cd::rf::PF_N + k];
  }
  return 0;
}
