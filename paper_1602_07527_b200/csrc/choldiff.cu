// choldiff.cu -- C ABI (include/choldiff.h) and host drivers of libcholdiff.so.
//
// Dispatch (per call):
//   n <= 32          one warp per matrix: fp64 reverse register-resident on DMMA tiles
//                    (sweep_reg32.cuh), otherwise sweep_warp.cuh     PAPER.md:566-578 / 489-498
//   n <= DC_NMAX     one CTA per matrix on DMMA tiles (sweep_dmma_cta.cuh)
//   larger n         blocked sweep (PAPER.md:689-701 reverse, 655-666 forward):
//                    diagonal-block inverses (k_trinv) once per call, then per block
//                    step the Level-3 updates as DMMA GEMMs (gemm.cuh) around the
//                    shared-memory diagonal-block kernel.
// All launches go to the caller's stream; the driver never synchronizes.
//
// Workspace: every driver runs in two modes, "plan" (no launches, only workspace
// carving) and "run"; cd_workspace_size returns the plan's high-water mark, so the
// size query and the launch sequence can never disagree.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/choldiff.h"
#include "common.cuh"
#include "gemm.cuh"
#include "gemm_tma.cuh"
#include "gemm_tc32.cuh"
#include "symm_tc.cuh"
#include "misc.cuh"
#include "sweep_warp.cuh"
#include "sweep_reg32.cuh"
#include "sweep_bulk32.cuh"
#include "sweep_dmma_cta.cuh"
#include "symm_ll.cuh"
#include "symbolic_cta.cuh"
#include "panel_rev.cuh"
#include "panel_fwd.cuh"
#include "chol_diag.cuh"
#include "gemm_fwd_sk.cuh"
#include "rf32_fused.h"

namespace cd {

// ---- per-device caches of launch attributes (occupancies, SM counts): a process may drive
// several devices (or MIG slices) with different SM counts.  Computed on first use per device;
// the computation is idempotent, so a race only computes the same value twice. ----
constexpr int kMaxDev = 64;
constexpr int64_t kGridBatch = 32768;  // batch chunk of the paths with the matrix index on grid.y/z
template <typename F>
static int per_device(std::atomic<int> (&cache)[kMaxDev], F&& compute) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return compute();
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    v = compute();
    cache[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

static thread_local int64_t g_launches = 0;
static thread_local char g_cuda_err[256] = "";

// ---- optional per-launch timing (cd_profile_*) ----
struct ProfRec {
  cudaEvent_t a, b;
  int cls;
  double flops;
  cudaStream_t st;
};
struct Prof {
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  cudaEvent_t ev() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  ~Prof() {  // thread exit: release this thread's events (errors ignored at process teardown)
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
  }
};
static thread_local Prof g_prof;

// ---- library-owned streams for the lookahead schedule (per device, per host thread) ----
struct LaStreams {
  cudaStream_t chain = nullptr;  // high priority: panel solve, diagonal block, next-panel updates
  cudaStream_t bulk = nullptr;   // trailing updates of the rest of the left panel
  std::vector<cudaEvent_t> pool;
  size_t next = 0;
  cudaEvent_t ev() {
    if (next == pool.size()) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      pool.push_back(e);
    }
    return pool[next++];
  }
  ~LaStreams() {  // thread exit: release this thread's streams and events
    if (chain) cudaStreamDestroy(chain);
    if (bulk) cudaStreamDestroy(bulk);
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
  }
};
static thread_local LaStreams g_la[64];
static bool g_no_lookahead = getenv("CD_NO_LOOKAHEAD") != nullptr;

static LaStreams* la_streams() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  LaStreams& s = g_la[dev];
  if (!s.chain) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&s.chain, cudaStreamNonBlocking, hi) != cudaSuccess) return nullptr;
    if (cudaStreamCreateWithPriority(&s.bulk, cudaStreamNonBlocking, lo) != cudaSuccess) return nullptr;
  }
  s.next = 0;
  return &s;
}

static int note_cuda(cudaError_t e) {
  if (e == cudaSuccess) return CD_SUCCESS;
  snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  return CD_ERR_CUDA;
}

// ---- host-buffer pipeline (cd_chol_host): column blocks stream in / out while the sweep runs ----
// Only the lower part of each column block, rows [j, n) of columns [j, j+w), is moved:
// the contract never reads the upper triangles, and TRIL output never writes them.
struct HostPipe {
  cudaStream_t cin = nullptr, cout = nullptr;  // library copy streams (per device)
  const char* Lh = nullptr;                    // host L (column-major, ld n)
  const char* Ah_in = nullptr;                 // host input triangle
  char* Ah = nullptr;                          // host output
  char* dL = nullptr;                          // device copies (ld n)
  char* dA = nullptr;
  int64_t n = 0;
  size_t es = 8;
  std::vector<cudaEvent_t> pool;
  size_t next = 0;
  cudaEvent_t ev() {
    if (next == pool.size()) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      pool.push_back(e);
    }
    return pool[next++];
  }
  size_t off(int64_t r, int64_t c) const { return (size_t(r) + size_t(c) * size_t(n)) * es; }
  ~HostPipe() {
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
  }
  // diagonal blocks of L first (the block inverses need all of them), then column blocks in
  // the order `order` lists them; returns one event per column block
  void h2d(int nblk, int nb, bool reverse, std::vector<cudaEvent_t>& ev_in, cudaEvent_t& ev_diag);
  // after `compute` has finished column block [j, j+w): copy rows [j, n) back
  void d2h(cudaStream_t compute, int j, int w) {
    cudaEvent_t e = ev();
    cudaEventRecord(e, compute);
    cudaStreamWaitEvent(cout, e, 0);
    cudaMemcpy2DAsync(Ah + off(j, j), size_t(n) * es, dA + off(j, j), size_t(n) * es, size_t(n - j) * es, size_t(w),
                      cudaMemcpyDeviceToHost, cout);
  }
  int64_t bytes_in = 0, bytes_out = 0;
};
static thread_local HostPipe* g_pipe = nullptr;

struct HostStreams {
  cudaStream_t cin = nullptr, cout = nullptr;
  HostPipe pipe;
  ~HostStreams() {  // thread exit: release this thread's copy streams
    if (cin) cudaStreamDestroy(cin);
    if (cout) cudaStreamDestroy(cout);
  }
};
static thread_local HostStreams g_hs[64];
static bool g_no_host_pipe = getenv("CD_NO_HOST_PIPE") != nullptr;
static thread_local int64_t g_host_bytes_in = 0, g_host_bytes_out = 0;

static HostStreams* host_streams() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  HostStreams& s = g_hs[dev];
  if (!s.cin) {
    if (cudaStreamCreateWithFlags(&s.cin, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    if (cudaStreamCreateWithFlags(&s.cout, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
  }
  return &s;
}


void HostPipe::h2d(int nblk, int nb, bool reverse, std::vector<cudaEvent_t>& ev_in, cudaEvent_t& ev_diag) {
  for (int qb = 0; qb < nblk; ++qb) {
    int j, w;
    block_range(int(n), nb, reverse, qb, j, w);
    cudaMemcpy2DAsync(dL + off(j, j), size_t(n) * es, Lh + off(j, j), size_t(n) * es, size_t(w) * es, size_t(w),
                      cudaMemcpyHostToDevice, cin);
    bytes_in += int64_t(w) * w * int64_t(es);
  }
  ev_diag = ev();
  cudaEventRecord(ev_diag, cin);
  ev_in.assign(size_t(nblk), nullptr);
  for (int i = 0; i < nblk; ++i) {
    const int qb = reverse ? nblk - 1 - i : i;
    int j, w;
    block_range(int(n), nb, reverse, qb, j, w);
    cudaMemcpy2DAsync(dL + off(j, j), size_t(n) * es, Lh + off(j, j), size_t(n) * es, size_t(n - j) * es, size_t(w),
                      cudaMemcpyHostToDevice, cin);
    cudaMemcpy2DAsync(dA + off(j, j), size_t(n) * es, Ah_in + off(j, j), size_t(n) * es, size_t(n - j) * es,
                      size_t(w), cudaMemcpyHostToDevice, cin);
    bytes_in += 2 * int64_t(n - j) * w * int64_t(es);
    ev_in[size_t(qb)] = ev();
    cudaEventRecord(ev_in[size_t(qb)], cin);
  }
}

struct Ctx {
  bool plan;            // plan mode: carve workspace only
  char* ws;             // device workspace base (run mode)
  size_t off = 0;       // high-water mark
  cudaStream_t st;
  int sms = 148;
  int err = CD_SUCCESS;
  void* take(size_t bytes) {
    off = (off + 255) & ~size_t(255);
    void* p = plan ? nullptr : ws + off;
    off += bytes;
    return p;
  }
  bool ok() const { return err == CD_SUCCESS; }
  // call before a launch: opens a timing bracket when profiling is on
  void pre(int cls, double flops) {
    if (!g_prof.on) return;
    ProfRec r{g_prof.ev(), g_prof.ev(), cls, flops, st};
    cudaEventRecord(r.a, st);
    g_prof.recs.push_back(r);
  }
  void launched() {
    ++g_launches;
    if (g_prof.on && !g_prof.recs.empty()) cudaEventRecord(g_prof.recs.back().b, st);
    if (err == CD_SUCCESS) err = note_cuda(cudaGetLastError());
  }
};

static int grid_1d(int64_t total, int threads, int sms) {
  int64_t g = (total + threads - 1) / threads;
  return int(std::max<int64_t>(1, std::min<int64_t>(g, int64_t(sms) * 16)));
}

// ------------------------------------------------------------------ kernel attribute setup
static bool g_no_pdl = getenv("CD_NO_PDL") != nullptr;  // measurement: plain launches of the persistent kernels
// a persistent stream-K kernel launched with programmatic stream serialization (PDL): its CTAs may
// start (prologue only, then griddepcontrol.wait) as the previous kernel's CTAs exit
template <typename K, typename... Args>
static cudaError_t launch_pdl(K kernel, int grid, int threads, size_t smem, cudaStream_t st, Args... args) {
  if (g_no_pdl) {
    kernel<<<grid, threads, smem, st>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <typename K>
static void set_smem(K kernel, size_t bytes) {
  // opt in well below 48 KB: the 48 KB default limit counts static shared memory too
  if (bytes > 32 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}

// ------------------------------------------------------------------ TMA tensor maps
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

static bool g_tma_disabled = getenv("CD_DISABLE_TMA") != nullptr;

// 2-D (or 3-D with batch) fp64 tensor map over a column-major view of `rows` x `cols`
// elements starting at element pointer `p` (leading dimension ld, batch stride bstride).
// `shift` (kept for the kernel's coordinate arithmetic) is always 0.
static bool make_tmap(CUtensorMap* map, int* shift, const void* p, int64_t rows, int64_t cols, int64_t ld,
                      int64_t bstride, int64_t batch, int box0, int box1) {
  auto enc = tmap_encoder();
  if (!enc || rows <= 0 || cols <= 0) return false;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(p);
  // The view must start on a 16-byte boundary: a map whose base was moved down and a
  // box starting at an odd element faulted (cudaErrorIllegalInstruction) on B200 /
  // driver 580 in testing; such views (odd block boundaries) use the cp.async kernel.
  if (addr % 16) return false;
  const int sh = 0;
  if ((ld * 8) % 16 || (batch > 1 && (bstride * 8) % 16)) return false;
  const void* base = reinterpret_cast<const char*>(p) - sh * 8;
  cuuint64_t dims[3] = {cuuint64_t(rows + sh), cuuint64_t(cols), cuuint64_t(std::max<int64_t>(batch, 1))};
  cuuint64_t strides[2] = {cuuint64_t(ld * 8), cuuint64_t(std::max<int64_t>(bstride, 1) * 8)};
  cuuint32_t box[3] = {cuuint32_t(box0), cuuint32_t(box1), 1};
  cuuint32_t es[3] = {1, 1, 1};
  const cuuint32_t rank = batch > 1 ? 3 : 2;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  *shift = sh;
  return r == CUDA_SUCCESS;
}

// fp32 map with 128-byte swizzle for the tcgen05 kernel (gemm_tc32.cuh)
static bool make_tmap_f32_sw128(CUtensorMap* map, const void* p, int64_t rows, int64_t cols, int64_t ld,
                                int64_t bstride, int64_t batch, int box0, int box1, bool atom32) {
  auto enc = tmap_encoder();
  if (!enc || rows <= 0 || cols <= 0) return false;
  if (reinterpret_cast<uintptr_t>(p) % 16) return false;
  if ((ld * 4) % 16 || (batch > 1 && (bstride * 4) % 16)) return false;
  cuuint64_t dims[3] = {cuuint64_t(rows), cuuint64_t(cols), cuuint64_t(std::max<int64_t>(batch, 1))};
  cuuint64_t strides[2] = {cuuint64_t(ld * 4), cuuint64_t(std::max<int64_t>(bstride, 1) * 4)};
  cuuint32_t box[3] = {cuuint32_t(box0), cuuint32_t(box1), 1};
  cuuint32_t es[3] = {1, 1, 1};
  const cuuint32_t rank = batch > 1 ? 3 : 2;
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 map without swizzle (TMA epilogue of the tcgen05 kernel: 128 x 32 column-major chunks)
static bool make_tmap_f32_plain(CUtensorMap* map, const void* p, int64_t rows, int64_t cols, int64_t ld,
                                int64_t bstride, int64_t batch, int box0, int box1) {
  auto enc = tmap_encoder();
  if (!enc || rows <= 0 || cols <= 0) return false;
  if (reinterpret_cast<uintptr_t>(p) % 16) return false;
  if ((ld * 4) % 16 || (batch > 1 && (bstride * 4) % 16)) return false;
  cuuint64_t dims[3] = {cuuint64_t(rows), cuuint64_t(cols), cuuint64_t(std::max<int64_t>(batch, 1))};
  cuuint64_t strides[2] = {cuuint64_t(ld * 4), cuuint64_t(std::max<int64_t>(bstride, 1) * 4)};
  cuuint32_t box[3] = {cuuint32_t(box0), cuuint32_t(box1), 1};
  cuuint32_t es[3] = {1, 1, 1};
  const cuuint32_t rank = batch > 1 ? 3 : 2;
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool g_tc32_disabled = getenv("CD_DISABLE_TC32") != nullptr;
// TMA epilogue of the tcgen05 GEMM (gemm_tc32.cuh, EPI = 1, 4-stage ring): on unless CD_TC_EPI=0;
// 64-wide N tiles for N <= 64 unless CD_TC_BN64=0
#ifndef CD_TC_EPI_STG
#define CD_TC_EPI_STG 4
#endif
#ifndef CD_TC_EPI_STG64  // 64-wide tiles: 24 KB stages, so a deeper ring fits beside the epilogue slots
#define CD_TC_EPI_STG64 5
#endif
static int g_tc_epi = getenv("CD_TC_EPI") ? atoi(getenv("CD_TC_EPI")) : 1;
static int g_tc_bn64 = getenv("CD_TC_BN64") ? atoi(getenv("CD_TC_BN64")) : 1;
static bool g_no_bulk32 = getenv("CD_NO_BULK32") != nullptr;
static std::atomic<bool> g_dc_clk_host{false};  // cd_debug_phase_clocks: the CLK instantiation of k_rev_dmma_cta
// measurement switch: k_rev_bulk32<4>'s register budget as minimum CTAs per SM (default 3: 166
// registers, three CTAs per SM; 4 = 128 registers and four CTAs, measured 12 % slower)
static int g_b32_minb = getenv("CD_B32_MINB") ? atoi(getenv("CD_B32_MINB")) : 3;
// fp32 64-wide diagonal blocks of the layered schedule on the mma.sync Eq. 10 / Eq. 8 kernel of
// rf32_fused.cu (default; configs[3] launch list: 41.6 vs 51.5 us per launch of 1024 blocks) or on
// the fp64-DMMA on-chip sweeps (CD_NO_HMMA_DIAG=1).  The block inverses stay on k_trinv_dmma
// (168 us for 8192 blocks; the fp32 forward-substitution kernel k_rf_trinv took 474 us).
static bool g_no_hmma_diag = getenv("CD_NO_HMMA_DIAG") != nullptr;

// ------------------------------------------------------------------ GEMM launcher
constexpr int64_t PART_TILES = 2 * 152;  // split-K partial budget, in 128x128 output tiles

template <typename T>
struct Gemm {
  Ctx& c;
  GemmParams p{};
  int TA = 0, TB = 0;
  double algo_flops = -1.0;  // the paper's flop count for this update (default 2*M*N*sum K)
  explicit Gemm(Ctx& ctx, int M, int N, int ta, int tb, int64_t batch) : c(ctx), TA(ta), TB(tb) {
    p.M = M;
    p.N = N;
    p.batch = batch;
    p.nseg = 0;
    p.alpha = 1.0;
    p.beta = 0.0;
  }
  Gemm& seg(Opnd A, Opnd B, int K) {
    if (K <= 0) return *this;
    constexpr int BK = GBK<T>::v;
    int kv0 = 0;
    if (p.nseg > 0) {
      const GemmSeg& s = p.seg[p.nseg - 1];
      kv0 = s.kv0 + ((s.K + BK - 1) / BK) * BK;
    }
    p.seg[p.nseg++] = GemmSeg{A, B, K, kv0};
    return *this;
  }
  Gemm& flops(double f) {
    algo_flops = f;
    return *this;
  }
  // store D (and read Cin) transposed: the user's D is N x M (fp32 tcgen05 TMA epilogue only)
  Gemm& trans_out() {
    p.dtrans = 1;
    return *this;
  }
  // D = alpha * sum + beta * Cin
  void run(Opnd Cin, Opnd D, double alpha, double beta, int tril, T* part_ws) {
    if (p.M <= 0 || p.N <= 0 || p.batch <= 0) return;
    if (p.nseg == 0) {  // nothing to accumulate: D = beta * Cin
      if (beta == 1.0 && Cin.base == D.base && Cin.arr == D.arr && Cin.off == D.off) return;
      // (not needed by the drivers)
      return;
    }
    constexpr int BK = GBK<T>::v;
    const GemmSeg& last = p.seg[p.nseg - 1];
    p.KT = (last.kv0 + last.K + BK - 1) / BK;
    p.Cin = Cin;
    p.D = D;
    p.alpha = alpha;
    p.beta = beta;
    p.tril = tril;  // 0 none; 1 + offset (see GemmParams)
    const int64_t tiles = int64_t((p.M + G_BM - 1) / G_BM) * ((p.N + G_BN - 1) / G_BN) * p.batch;
    int splits = 1;
    if (tiles < c.sms && p.KT >= 4 && !p.dtrans) {  // (the transposed store has no split-K reduction)
      splits = int(std::min<int64_t>((2 * c.sms + tiles - 1) / tiles, p.KT / 2));
      const int64_t cap = PART_TILES * G_BM * G_BN / (int64_t(p.M) * p.N * p.batch);
      splits = int(std::max<int64_t>(1, std::min<int64_t>(splits, cap)));
    }
    p.kt_per_split = (p.KT + splits - 1) / splits;
    splits = (p.KT + p.kt_per_split - 1) / p.kt_per_split;
    p.splits = splits;
    p.part = part_ws;
    if (c.plan || !c.ok()) return;
    dim3 grid((p.M + G_BM - 1) / G_BM, (p.N + G_BN - 1) / G_BN, unsigned(p.batch * splits));
    if (algo_flops < 0) {
      int64_t ks = 0;
      for (int s = 0; s < p.nseg; ++s) ks += p.seg[s].K;
      algo_flops = 2.0 * p.M * double(p.N) * double(ks);
    }
    c.pre(CD_PROF_GEMM, algo_flops * double(p.batch));
    launch(grid);
    if (splits > 1) {
      const int64_t total = int64_t(p.M) * p.N * p.batch;
      c.pre(CD_PROF_REDUCE, 0.0);
      k_splitk_reduce<T><<<grid_1d(total, 256, c.sms), 256, 0, c.st>>>(p.M, p.N, p.batch, splits,
                                                                          reinterpret_cast<const T*>(part_ws), Cin,
                                                                          D, alpha, beta, p.tril);
      c.launched();
    }
  }
  template <int A_, int B_>
  void launch_t(dim3 grid) {
    auto kern = k_gemm<T, A_, B_>;
    set_smem(kern, GemmLayout<T, A_, B_>::SMEM);
    if (p.splits > 1) {
      // the kernel writes partials; alpha/beta/Cin are applied by the reduction
    }
    kern<<<grid, G_THREADS, GemmLayout<T, A_, B_>::SMEM, c.st>>>(p);
    c.launched();
  }
  // TMA-fed warp-specialised kernel (fp64, strided operands with even ld)
  bool build_maps(TmaMaps& tm) {
    if (sizeof(T) != 8 || g_tma_disabled) return false;
    tm.batched = p.batch > 1 ? 1 : 0;
    for (int s = 0; s < p.nseg; ++s) {
      const GemmSeg& sg = p.seg[s];
      if (sg.A.arr || sg.B.arr) return false;
      const T* pa = static_cast<const T*>(sg.A.base) + sg.A.off;
      const T* pb = static_cast<const T*>(sg.B.base) + sg.B.off;
      const bool okA = TA == 0 ? make_tmap(&tm.a[s], &tm.a_shift[s], pa, p.M, sg.K, sg.A.ld, sg.A.stride, p.batch, 132, 16)
                               : make_tmap(&tm.a[s], &tm.a_shift[s], pa, sg.K, p.M, sg.A.ld, sg.A.stride, p.batch, 20, 128);
      const bool okB = TB == 0 ? make_tmap(&tm.b[s], &tm.b_shift[s], pb, sg.K, p.N, sg.B.ld, sg.B.stride, p.batch, 20, 128)
                               : make_tmap(&tm.b[s], &tm.b_shift[s], pb, p.N, sg.K, sg.B.ld, sg.B.stride, p.batch, 132, 16);
      if (!okA || !okB) return false;
    }
    return true;
  }
  template <int A_, int B_>
  bool launch_tma(dim3 grid) {
    TmaMaps tm;
    memset(&tm, 0, sizeof(tm));
    if (!build_maps(tm)) return false;
    auto kern = k_gemm_tma<A_, B_>;
    set_smem(kern, TmaLayout<A_, B_>::SMEM);
    kern<<<grid, TG_THREADS, TmaLayout<A_, B_>::SMEM, c.st>>>(p, tm);
    c.launched();
    return true;
  }
  // fp32: tcgen05 kind::tf32 kernel when every operand can be described by a TMA map
  template <int A_, int B_>
  bool launch_tc32(dim3 grid) {
    if (g_tc32_disabled) return false;
    TmaMaps tm;
    memset(&tm, 0, sizeof(tm));
    tm.batched = p.batch > 1 ? 1 : 0;
    // N tile: 64 for the nb = 64 panels (half the MMA work of a 128-wide tile), else 128
    const int bn = (p.N <= 64 && g_tc_bn64) ? 64 : 128;
    for (int s = 0; s < p.nseg; ++s) {
      const GemmSeg& sg = p.seg[s];
      if (sg.A.arr || sg.B.arr) return false;
      const T* pa = static_cast<const T*>(sg.A.base) + sg.A.off;
      const T* pb = static_cast<const T*>(sg.B.base) + sg.B.off;
      const bool okA = A_ == 0 ? make_tmap_f32_sw128(&tm.a[s], pa, p.M, sg.K, sg.A.ld, sg.A.stride, p.batch, 32, 32, true)
                               : make_tmap_f32_sw128(&tm.a[s], pa, sg.K, p.M, sg.A.ld, sg.A.stride, p.batch, 32, 128, false);
      const bool okB = B_ == 0 ? make_tmap_f32_sw128(&tm.b[s], pb, sg.K, p.N, sg.B.ld, sg.B.stride, p.batch, 32, bn, false)
                               : make_tmap_f32_sw128(&tm.b[s], pb, p.N, sg.K, sg.B.ld, sg.B.stride, p.batch, 32, 32, true);
      if (!okA || !okB) return false;
    }
    const int64_t units = int64_t(grid.x) * grid.y * grid.z;
    if (units >= (int64_t(1) << 31)) return false;  // the kernel decodes units in 32 bits
    TcEpiMaps em;
    memset(&em, 0, sizeof(em));
    if (tc_epi_maps(em)) {
      if (p.dtrans) {
        if (bn == 64) return launch_tc32_k<A_, B_, 2, CD_TC_EPI_STG64, 64>(units, tm, em);
        return launch_tc32_k<A_, B_, 2, CD_TC_EPI_STG, 128>(units, tm, em);
      }
      if (bn == 64) return launch_tc32_k<A_, B_, 1, CD_TC_EPI_STG64, 64>(units, tm, em);
      return launch_tc32_k<A_, B_, 1, CD_TC_EPI_STG, 128>(units, tm, em);
    }
    if (p.dtrans) return false;
    if (bn == 64) return launch_tc32_k<A_, B_, 0, TC_STAGES, 64>(units, tm, em);
    return launch_tc32_k<A_, B_, 0, TC_STAGES, 128>(units, tm, em);
  }
  // TMA epilogue eligibility (see gemm_tc32.cuh): one split, plain strided D / Cin, 16-byte
  // aligned, and a tril mask only for the in-place update
  bool tc_epi_maps(TcEpiMaps& em) {
    if (!g_tc_epi || p.splits != 1 || p.D.arr) return false;
    const bool has_cin = p.beta != 0.0;
    const bool inplace = p.Cin.base == p.D.base && !p.Cin.arr && p.Cin.off == p.D.off && p.Cin.ld == p.D.ld &&
                         p.Cin.stride == p.D.stride;
    if (p.tril && !(has_cin && inplace)) return false;
    if (has_cin && p.Cin.arr) return false;
    if (p.dtrans) {  // N x M views, 32 x 128 boxes with the 128-byte swizzle (gemm_tc32.cuh, EPI = 2)
      if (p.tril) return false;
      const float* pd = static_cast<const float*>(p.D.base) + p.D.off;
      if (!make_tmap_f32_sw128(&em.d, pd, p.N, p.M, p.D.ld, p.D.stride, p.batch, 32, 128, false)) return false;
      if (has_cin) {
        const float* pc = static_cast<const float*>(p.Cin.base) + p.Cin.off;
        if (!make_tmap_f32_sw128(&em.cin, pc, p.N, p.M, p.Cin.ld, p.Cin.stride, p.batch, 32, 128, false)) return false;
      }
      return true;
    }
    const float* pd = static_cast<const float*>(p.D.base) + p.D.off;
    if (!make_tmap_f32_plain(&em.d, pd, p.M, p.N, p.D.ld, p.D.stride, p.batch, 128, 32)) return false;
    if (has_cin) {
      const float* pc = static_cast<const float*>(p.Cin.base) + p.Cin.off;
      if (!make_tmap_f32_plain(&em.cin, pc, p.M, p.N, p.Cin.ld, p.Cin.stride, p.batch, 128, 32)) return false;
    }
    return true;
  }
  template <int A_, int B_, int EPI, int STG, int BN>
  bool launch_tc32_k(int64_t units, const TmaMaps& tm, const TcEpiMaps& em) {
    auto kern = k_gemm_tc32<A_, B_, EPI, STG, BN>;
    constexpr size_t smem = tc_smem(STG, EPI, BN);
    static std::atomic<int> occ_cache[kMaxDev];  // per instantiation and device
    const int occ = per_device(occ_cache, [&] {
      int o = 0;
      set_smem(kern, smem);
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, tcp_threads(EPI), smem) != cudaSuccess || o < 1)
        o = 1;
      return std::min(o, 2);  // TMEM: 2 x 256 columns per CTA
    });
    set_smem(kern, smem);
    // persistent: a grid of (up to) occ CTAs per SM loops over the units (CD_TC_SMS: measurement
    // switch capping the SMs it takes)
    static const int tc_sms = getenv("CD_TC_SMS") ? atoi(getenv("CD_TC_SMS")) : 0;
    const int sms = tc_sms > 0 ? std::min(tc_sms, c.sms) : c.sms;
    const unsigned g = unsigned(std::max<int64_t>(1, std::min<int64_t>(units, int64_t(sms) * occ)));
    c.err = note_cuda(launch_pdl(kern, int(g), tcp_threads(EPI), smem, c.st, p, tm, em));
    c.launched();
    return true;
  }
  void launch(dim3 grid) {
    if constexpr (sizeof(T) == 4) {
      bool done = false;
      if (TA == 0 && TB == 0) done = launch_tc32<0, 0>(grid);
      else if (TA == 0 && TB == 1) done = launch_tc32<0, 1>(grid);
      else if (TA == 1 && TB == 0) done = launch_tc32<1, 0>(grid);
      else done = launch_tc32<1, 1>(grid);
      if (done) return;
    }
    if (p.dtrans) {  // only the fp32 TMA epilogue stores transposed; the callers check first
      c.err = CD_ERR_UNSUPPORTED;
      snprintf(g_cuda_err, sizeof(g_cuda_err), "transposed-output GEMM needs the fp32 TMA epilogue");
      return;
    }
    if constexpr (sizeof(T) == 8) {
      bool done = false;
      if (TA == 0 && TB == 0) done = launch_tma<0, 0>(grid);
      else if (TA == 0 && TB == 1) done = launch_tma<0, 1>(grid);
      else if (TA == 1 && TB == 0) done = launch_tma<1, 0>(grid);
      else done = launch_tma<1, 1>(grid);
      if (done) return;
    }
    if (TA == 0 && TB == 0) launch_t<0, 0>(grid);
    else if (TA == 0 && TB == 1) launch_t<0, 1>(grid);
    else if (TA == 1 && TB == 0) launch_t<1, 0>(grid);
    else launch_t<1, 1>(grid);
  }
};

static Opnd null_opnd() { return Opnd{nullptr, nullptr, 0, 0, 0}; }
// sub-view of an operand: rows/cols offset
static Opnd sub(const Opnd& o, int64_t r0, int64_t c0) {
  Opnd s = o;
  s.off = o.off + r0 + c0 * o.ld;
  return s;
}
// dense strided workspace operand: matrix b at base + b*stride, ld
static Opnd ws_opnd(void* base, int64_t stride, int64_t ld) { return Opnd{base, nullptr, stride, ld, 0}; }

// ------------------------------------------------------------------ small-n kernels
template <typename T>
static void run_sweep_small(Ctx& c, bool rev, int n, int64_t batch, Opnd L, Opnd A, int out_mode, Opnd S,
                            int* info) {
  if (c.plan || !c.ok()) return;
  const double nf = n;
  c.pre(CD_PROF_SWEEP, double(batch) * (rev ? (4 * nf * nf * nf + 3 * nf * nf + 11 * nf) / 6
                                            : (4 * nf * nf * nf + 3 * nf * nf + 5 * nf) / 6));
  if (n <= 32) {
    const size_t smem = sweep_warp_smem<T>();
    const unsigned grid = unsigned((batch + SW_WPB - 1) / SW_WPB);
    const bool bulk_ok = rev && sizeof(T) == 8 && n % 8 == 0 && out_mode == CD_OUT_TRIL && !L.arr && !A.arr &&
                         !S.base && !S.arr && !g_no_bulk32 && L.ld % 2 == 0 && A.ld % 2 == 0 &&
                         (batch == 1 || (L.stride % 2 == 0 && A.stride % 2 == 0)) &&
                         (reinterpret_cast<uintptr_t>(static_cast<const T*>(L.base) + L.off) % 16) == 0 &&
                         (reinterpret_cast<uintptr_t>(static_cast<const T*>(A.base) + A.off) % 16) == 0;
    if (bulk_ok) {
      // fp64 reverse, n = 8/16/24/32: the same register sweep fed by bulk copies (sweep_bulk32.cuh)
      const Opnd Lo = L, Ao = A;
      const int nblk = n / 8;
      auto launch = [&](auto kern, size_t smb) {
        set_smem(kern, smb);
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, B32_WPB * 32, smb);
        const unsigned gb = unsigned(std::max<int64_t>(1, std::min<int64_t>((batch + B32_WPB - 1) / B32_WPB,
                                                                          int64_t(c.sms) * std::max(occ, 1))));
        kern<<<gb, B32_WPB * 32, smb, c.st>>>(batch, Lo, Ao, info);
      };
      if (nblk == 1) launch(k_rev_bulk32<1>, b32_smem<1>());
      else if (nblk == 2) launch(k_rev_bulk32<2>, b32_smem<2>());
      else if (nblk == 3) launch(k_rev_bulk32<3>, b32_smem<3>());
      else if (g_b32_minb == 4) launch(k_rev_bulk32<4, 4>, b32_smem<4>());
      else launch(k_rev_bulk32<4, 3>, b32_smem<4>());
    } else if (rev && sizeof(T) == 8) {
      // fp64 reverse: register-resident N_b = 8 blocked sweep on DMMA tiles (sweep_reg32.cuh)
      const int nblk = (n + 7) / 8;
      const size_t sm3 = reg32_smem();
      const unsigned g3 = unsigned(std::min<int64_t>((batch + R32_WPB - 1) / R32_WPB, int64_t(c.sms) * 16));
      const Opnd Lo = L, Ao = A;
      auto go3 = [&](auto kern) {
        set_smem(kern, sm3);
        kern<<<g3, R32_WPB * 32, sm3, c.st>>>(n, batch, Lo, Ao, out_mode, info);
      };
      if (nblk == 1) go3(k_rev_reg32<1>);
      else if (nblk == 2) go3(k_rev_reg32<2>);
      else if (nblk == 3) go3(k_rev_reg32<3>);
      else go3(k_rev_reg32<4>);
    } else if (rev) {
      set_smem(k_sweep_warp_rev<T>, smem);
      k_sweep_warp_rev<T><<<grid, SW_WPB * 32, smem, c.st>>>(n, batch, L, A, out_mode, info);
    } else {
      set_smem(k_sweep_warp_fwd<T>, smem);
      k_sweep_warp_fwd<T><<<grid, SW_WPB * 32, smem, c.st>>>(n, batch, L, A, info);
    }
    c.launched();
    if (S.base || S.arr) {  // (blocked driver with a tiny block) S = Dbar + Dbar^T
      const int64_t total = int64_t(n) * n * batch;
      c.pre(CD_PROF_OTHER, 0.0);
      k_sym2<T><<<grid_1d(total, 256, c.sms), 256, 0, c.st>>>(n, batch, A, S, rev ? 0 : 1);
      c.launched();
    }
  } else {
    // 32 < n <= 128: N_b = 8 blocked sweep on DMMA tiles (fp64 arithmetic), one CTA per matrix
    const size_t smem = dmma_cta_smem((n + 7) / 8);
    if (rev) {
      if ((n + 7) / 8 == 8) {  // n = 57 .. 64: compile-time block count
        if (g_dc_clk_host) {  // phase clocks (cd_debug_phase_clocks)
          set_smem(k_rev_dmma_cta<T, 8, true>, smem);
          k_rev_dmma_cta<T, 8, true><<<unsigned(batch), DC_THREADS, smem, c.st>>>(n, L, A, out_mode, S, info);
        } else {
          set_smem(k_rev_dmma_cta<T, 8>, smem);
          k_rev_dmma_cta<T, 8><<<unsigned(batch), DC_THREADS, smem, c.st>>>(n, L, A, out_mode, S, info);
        }
      } else {
        set_smem(k_rev_dmma_cta<T>, smem);
        k_rev_dmma_cta<T><<<unsigned(batch), DC_THREADS, smem, c.st>>>(n, L, A, out_mode, S, info);
      }
    } else {
      set_smem(k_fwd_dmma_cta<T>, smem);
      k_fwd_dmma_cta<T><<<unsigned(batch), DC_THREADS, smem, c.st>>>(n, L, A, S, info);
    }
    c.launched();
  }
}

// fp32 batches with 128-wide panels: the diagonal blocks on k_rf_diag128, the 128-wide inverses built
// from 64-wide ones (CD_NO_DIAG128: the fp64-DMMA sweeps and inverses of width 128 instead)
static bool g_no_diag128 = getenv("CD_NO_DIAG128") != nullptr;
// measurement switch: the 128-wide inverses as fp64-DMMA 64-wide ones + a 3xTF32 completion on a side
// stream (the round-2 route before k_rf_trinv128)
static bool g_old_inv128 = getenv("CD_OLD_INV128") != nullptr;
static bool diag128_route(int n, int nb, const Opnd& L) {
  return nb == 128 && n % 128 == 0 && !L.arr && !g_no_diag128 && !g_no_hmma_diag;
}

// (cd_chol_rev_fwd, 128-wide route: the combine runs on its own stream beside the two sweeps, which
// wait for it -- g_dinv_wait -- only before their first GEMM against D^{-1}; their diagonal-block
// kernels read just the 64-wide diagonals)
static thread_local cudaEvent_t g_dinv_wait = nullptr;
static void wait_dinv(Ctx& c) {
  if (g_dinv_wait && !c.plan && c.ok()) c.err = note_cuda(cudaStreamWaitEvent(c.st, g_dinv_wait, 0));
}

template <typename T>
static void run_trinv(Ctx& c, int n, int nb, bool reverse, int64_t batch, Opnd L, T* Dinv, bool combine = true) {
  if (c.plan || !c.ok()) return;
  const int nblk = nblocks(n, nb);
  if (sizeof(T) == 4 && diag128_route(n, nb, L) && !g_old_inv128) {
    // all 128-wide inverses in one launch (recursive doubling in fp32 / 3xTF32, rf32_fused.cu)
    c.pre(CD_PROF_TRINV, 0.0);
    c.err = note_cuda(rf32_trinv128(n, batch, reinterpret_cast<const float*>(static_cast<const T*>(L.base) + L.off),
                                    L.ld, L.stride, reinterpret_cast<float*>(Dinv), c.st));
    ++g_launches;
    if (g_prof.on && !g_prof.recs.empty()) cudaEventRecord(g_prof.recs.back().b, c.st);
    return;
  }
  if (sizeof(T) == 4 && diag128_route(n, nb, L)) {
    // (CD_OLD_INV128) the 64-wide inverses straight onto the diagonals of the 128-wide blocks, then
    // the lower-left blocks (rf32_inv128)
    const size_t smem = dmma_cta_smem(8);
    set_smem(k_trinv_dmma<T>, smem);
    c.pre(CD_PROF_TRINV, 0.0);
    k_trinv_dmma<T><<<dim3(n / 64, unsigned(batch)), DC_THREADS, smem, c.st>>>(n, 64, reverse ? 1 : 0, L, Dinv, 128,
                                                                             int64_t(64) * 128, 64);
    c.launched();
    if (!combine) return;
    c.pre(CD_PROF_TRINV, 0.0);
    c.err = note_cuda(rf32_inv128(n, batch, reinterpret_cast<const float*>(static_cast<const T*>(L.base) + L.off), L.ld,
                                  L.stride, reinterpret_cast<float*>(Dinv), c.st));
    ++g_launches;
    if (g_prof.on && !g_prof.recs.empty()) cudaEventRecord(g_prof.recs.back().b, c.st);
    return;
  }
  const size_t smem = dmma_cta_smem((nb + 7) / 8);
  set_smem(k_trinv_dmma<T>, smem);
  c.pre(CD_PROF_TRINV, 0.0);
  k_trinv_dmma<T><<<dim3(nblk, unsigned(batch)), DC_THREADS, smem, c.st>>>(n, nb, reverse ? 1 : 0, L, Dinv, nb,
                                                                          int64_t(nb) * nb, 0);
  c.launched();
}

// Diagonal block of a blocked step (PAPER.md:698 / 662): fp32 64-wide blocks of batches on the
// mma.sync Eq. 10 / Eq. 8 kernel (rf32_fused.cu, uses the block inverse Dinv_q); otherwise the
// on-chip sweeps of run_sweep_small.
template <typename T>
static void diag_block(Ctx& c, bool rev, int w, int64_t batch, Opnd L, Opnd A, Opnd S, Opnd Dinv_q) {
  if constexpr (sizeof(T) == 4) {
    if (w == 64 && !L.arr && !A.arr && !S.arr && !g_no_hmma_diag) {
      if (c.plan || !c.ok()) return;
      c.pre(CD_PROF_SWEEP, double(batch) * (rev ? (4.0 * w * w * w + 3.0 * w * w + 11.0 * w) / 6
                                                : (4.0 * w * w * w + 3.0 * w * w + 5.0 * w) / 6));
      c.err = note_cuda(rf32_diag64(rev, batch, static_cast<const float*>(L.base) + L.off, L.ld, L.stride,
                                    const_cast<float*>(static_cast<const float*>(A.base)) + A.off, A.ld, A.stride,
                                    static_cast<const float*>(Dinv_q.base) + Dinv_q.off, Dinv_q.stride,
                                    S.base ? const_cast<float*>(static_cast<const float*>(S.base)) + S.off : nullptr,
                                    S.ld, S.stride, c.st));
      ++g_launches;
      if (g_prof.on && !g_prof.recs.empty()) cudaEventRecord(g_prof.recs.back().b, c.st);
      return;
    }
    if (w == 128 && !L.arr && !A.arr && !S.arr && !Dinv_q.arr && Dinv_q.ld == 128 && !g_no_diag128 && !g_no_hmma_diag) {
      if (c.plan || !c.ok()) return;
      c.pre(CD_PROF_SWEEP, double(batch) * (rev ? (4.0 * w * w * w + 3.0 * w * w + 11.0 * w) / 6
                                                : (4.0 * w * w * w + 3.0 * w * w + 5.0 * w) / 6));
      c.err = note_cuda(rf32_diag128(rev, batch, static_cast<const float*>(L.base) + L.off, L.ld, L.stride,
                                     const_cast<float*>(static_cast<const float*>(A.base)) + A.off, A.ld, A.stride,
                                     static_cast<const float*>(Dinv_q.base) + Dinv_q.off, Dinv_q.ld, Dinv_q.stride,
                                     S.base ? const_cast<float*>(static_cast<const float*>(S.base)) + S.off : nullptr,
                                     S.ld, S.stride, c.st));
      ++g_launches;
      if (g_prof.on && !g_prof.recs.empty()) cudaEventRecord(g_prof.recs.back().b, c.st);
      return;
    }
  }
  run_sweep_small<T>(c, rev, w, batch, L, A, 0, S, nullptr);
}

template <typename T>
static void run_copy(Ctx& c, int M, int N, int64_t batch, Opnd S, Opnd D) {
  if (c.plan || !c.ok() || M <= 0 || N <= 0) return;
  c.pre(CD_PROF_OTHER, 0.0);
  k_copy<T><<<grid_1d(int64_t(M) * N * batch, 256, c.sms), 256, 0, c.st>>>(M, N, batch, S, D);
  c.launched();
}

template <typename T>
static void run_sym2(Ctx& c, int n, int64_t batch, Opnd A, Opnd S, int clean) {
  if (c.plan || !c.ok()) return;
  c.pre(CD_PROF_OTHER, 0.0);
  k_sym2<T><<<grid_1d(int64_t(n) * n * batch, 256, c.sms), 256, 0, c.st>>>(n, batch, A, S, clean);
  c.launched();
}

// ------------------------------------------------------------------ blocked reverse
// chol_blocked_rev, block [j, k) (0-based), w = k - j, p = n - k, q = j:
//   Cbar <- Cbar D^{-1}                      W = Abar[k:n, j:k] Dinv        (GEMM, K = w)
//   Bbar <- Bbar - Cbar R                    Abar[k:n, 0:j] -= W L[j:k, 0:j]
//   Dbar <- Dbar - tril(Cbar^T C)            Abar[j:k, j:k] -= tril(W^T L[k:n, j:k])  (split-K)
//   Dbar <- chol_unblocked_rev(D, Dbar)      sweep kernel; also S = Dbar + Dbar^T
//   Rbar <- Rbar - Cbar^T B - (Dbar+Dbar^T) R   Abar[j:k, 0:j] -= [S; W]^T L[j:n, 0:j]  (one GEMM, 2 K-segments)
// W is written straight into Abar's Cbar region when one 128-wide N-tile covers
// the block (each CTA then reads its rows completely before writing them);
// otherwise through workspace + copy.
// cd_chol_rev_fwd: the diagonal-block inverses of the shared factor, made once for both sweeps
// (valid when both partitions coincide, n % nb == 0; set only around that call's two enqueues)
static thread_local const void* g_ext_dinv = nullptr;
static thread_local int g_ext_dinv_nb = 0;

template <typename T>
static T* shared_dinv(int n, int nb) {
  return (g_ext_dinv && g_ext_dinv_nb == nb && n % nb == 0) ? static_cast<T*>(const_cast<void*>(g_ext_dinv)) : nullptr;
}

// the transposed Rbar update (blocked_rev) applies to fp32 batches whose operands the tcgen05
// kernel's TMA maps can describe (16-byte aligned views, ld and batch stride multiples of 4)
static bool g_no_rbar_trans = getenv("CD_NO_RBAR_TRANS") != nullptr;
template <typename T>
static bool rbar_transposed(const Ctx& c, int64_t batch, int q, int w, Opnd L, Opnd A, int j, Opnd W) {
  if (sizeof(T) != 4 || batch < 2 || g_no_rbar_trans || g_tc32_disabled || g_tma_disabled || !g_tc_epi) return false;
  if (w % 4) return false;  // S (ld = w) must be TMA-describable too
  auto ok = [&](const Opnd& o, int64_t r0, int64_t c0) {
    if (o.arr || o.ld % 4 || o.stride % 4) return false;
    if (c.plan) return true;
    const float* ptr = static_cast<const float*>(o.base) + o.off + r0 + c0 * o.ld;
    return reinterpret_cast<uintptr_t>(ptr) % 16 == 0;
  };
  (void)q;
  return ok(A, j, 0) && ok(L, j, 0) && ok(W, 0, 0);
}

template <typename T>
static void blocked_rev(Ctx& c, int n, int nb, int64_t batch, Opnd L, Opnd A, int* info, T* part_ws) {
  const int nblk = nblocks(n, nb);
  T* Dinv = static_cast<T*>(c.take(sizeof(T) * size_t(batch) * nblk * nb * nb));
  T* Sws = static_cast<T*>(c.take(sizeof(T) * size_t(batch) * nb * nb));
  const bool w_inplace = nb <= G_BN;
  T* Wws = w_inplace ? nullptr : static_cast<T*>(c.take(sizeof(T) * size_t(batch) * n * nb));
  if (T* ext = shared_dinv<T>(n, nb)) Dinv = c.plan ? Dinv : ext;
  else run_trinv<T>(c, n, nb, true, batch, L, Dinv);
  for (int qb = nblk - 1; qb >= 0; --qb) {
    int j, w;
    block_range(n, nb, true, qb, j, w);
    const int k = j + w, p = n - k, q = j;
    const Opnd Dinv_q = ws_opnd(Dinv + int64_t(qb) * nb * nb, int64_t(nblk) * nb * nb, nb);
    const Opnd S = ws_opnd(Sws, int64_t(nb) * nb, w);
    const Opnd Cbar = sub(A, k, j);
    const Opnd W = w_inplace ? Cbar : ws_opnd(Wws, int64_t(n) * nb, std::max(p, 1));
    if (p > 0) {
      // Cbar <- Cbar D^{-1}
      if (qb == nblk - 2) wait_dinv(c);
      Gemm<T>(c, p, w, 0, 0, batch)
          .seg(Cbar, Dinv_q, w)
          .flops(double(p) * w * (w + 1))  // TRSM  Cbar D^{-1}
          .run(null_opnd(), W, 1.0, 0.0, 0, part_ws);
      if (!w_inplace) run_copy<T>(c, p, w, batch, W, Cbar);
      // Bbar <- Bbar - Cbar R
      if (q > 0)
        Gemm<T>(c, p, q, 0, 0, batch).seg(W, sub(L, j, 0), w).run(sub(A, k, 0), sub(A, k, 0), -1.0, 1.0, false,
                                                                 part_ws);
      // Dbar <- Dbar - tril(Cbar^T C)
      Gemm<T>(c, w, w, 1, 0, batch)
          .seg(W, sub(L, k, j), p)
          .flops(double(w) * (w + 1) * p)  // lower triangle only
          .run(sub(A, j, j), sub(A, j, j), -1.0, 1.0, 1, part_ws);
    }
    // Dbar <- chol_unblocked_rev(D, Dbar)  (+ S = Dbar + Dbar^T)      (w <= DC_NMAX)
    diag_block<T>(c, true, w, batch, sub(L, j, j), sub(A, j, j), q > 0 ? S : null_opnd(), Dinv_q);
    // Rbar <- Rbar - Cbar^T B - (Dbar + Dbar^T) R
    if (q > 0 && rbar_transposed<T>(c, batch, q, w, L, A, j, W)) {
      // fp32 batches: as Rbar^T -= [R; B]^T [S; Cbar] -- M = q rows of 128-row tiles instead of
      // M = w = 64 (half-empty tcgen05 tiles), the result stored transposed by the TMA epilogue
      Gemm<T> g(c, q, w, 1, 0, batch);
      g.seg(sub(L, j, 0), S, w);
      if (p > 0) g.seg(sub(L, k, 0), W, p);
      g.trans_out().run(sub(A, j, 0), sub(A, j, 0), -1.0, 1.0, 0, part_ws);
    } else if (q > 0) {
      Gemm<T> g(c, w, q, 1, 0, batch);
      g.seg(S, sub(L, j, 0), w);
      if (p > 0) g.seg(W, sub(L, k, 0), p);
      g.run(sub(A, j, 0), sub(A, j, 0), -1.0, 1.0, 0, part_ws);
    }
  }
  if (info && !c.plan && c.ok()) {
    c.pre(CD_PROF_OTHER, 0.0);
    k_diag_info<T><<<unsigned(batch), 256, 0, c.st>>>(n, L, info);
    c.launched();
  }
}

// ------------------------------------------------------------------ blocked reverse, lookahead
// Same arithmetic as blocked_rev ("the partitioning into columns is
// arbitrary", 704-707), scheduled on two streams.  For block K = [j, k) with next block
// K' = [j', j):
//   chain (high priority):  Cbar <- Cbar D^{-1};
//        Abar[j:k, j':k] -= W^T L[k:n, j':k]      (Dbar correction + the next panel's
//                                                  share of Rbar -= Cbar^T B; tril on K)
//        Dbar <- chol_unblocked_rev(D, Dbar)  (+ S);
//        [after bulk(K_prev)]  Abar[k:n, j':j] -= W L[j:k, j':j];  Abar[j:k, j':j] -= S L[j:k, j':j]
//   bulk (low priority):    Abar[k:n, 0:j'] -= W L[j:k, 0:j'];
//        Abar[j:k, 0:j'] -= [S; W]^T [L[j:k, 0:j']; L[k:n, 0:j']]
// so the next block's panel solve, correction and diagonal sweep overlap the bulk
// updates of the current block.  S is double-buffered; each stream has its own split-K
// partial buffer.
template <typename T>
static void blocked_rev_la(Ctx& c, LaStreams* ls, int n, int nb, int64_t batch, Opnd L, Opnd A, int* info,
                           T* partA, T* partB) {
  const int nblk = nblocks(n, nb);
  T* Dinv = static_cast<T*>(c.take(sizeof(T) * size_t(batch) * nblk * nb * nb));
  T* Sws = static_cast<T*>(c.take(sizeof(T) * size_t(batch) * nb * nb * 2));
  if (c.plan) return;
  const cudaStream_t caller = c.st;
  cudaEvent_t e0 = ls->ev();
  cudaEventRecord(e0, caller);
  cudaStreamWaitEvent(ls->chain, e0, 0);
  cudaStreamWaitEvent(ls->bulk, e0, 0);
  c.st = ls->chain;
  run_trinv<T>(c, n, nb, true, batch, L, Dinv);
  cudaEvent_t ev_bulk_prev = nullptr;
  for (int qb = nblk - 1; qb >= 0 && c.ok(); --qb) {
    int j, w;
    block_range(n, nb, true, qb, j, w);
    const int k = j + w, p = n - k, q = j;
    int jn = 0, wn = 0;  // next block [jn, j)
    if (qb > 0) block_range(n, nb, true, qb - 1, jn, wn);
    const Opnd Dinv_q = ws_opnd(Dinv + int64_t(qb) * nb * nb, int64_t(nblk) * nb * nb, nb);
    const Opnd S = ws_opnd(Sws + int64_t(qb & 1) * batch * nb * nb, int64_t(nb) * nb, w);
    const Opnd W = sub(A, k, j);  // Cbar, solved in place
    c.st = ls->chain;
    if (p > 0) {
      Gemm<T>(c, p, w, 0, 0, batch)
          .seg(W, Dinv_q, w)
          .flops(double(p) * w * (w + 1))  // TRSM  Cbar D^{-1}
          .run(null_opnd(), W, 1.0, 0.0, 0, partA);
      // Dbar -= tril(Cbar^T C)  and  Rbar[:, jn:j] -= Cbar^T B[:, jn:j]
      Gemm<T>(c, w, wn + w, 1, 0, batch)
          .seg(W, sub(L, k, jn), p)
          .flops(double(w) * (w + 1) * p + 2.0 * w * wn * p)
          .run(sub(A, j, jn), sub(A, j, jn), -1.0, 1.0, 1 + wn, partA);
    }
    run_sweep_small<T>(c, true, w, batch, sub(L, j, j), sub(A, j, j), 0, q > 0 ? S : null_opnd(), nullptr);
    if (q == 0) break;
    cudaEvent_t ev_s = ls->ev();
    cudaEventRecord(ev_s, ls->chain);
    if (ev_bulk_prev) cudaStreamWaitEvent(ls->chain, ev_bulk_prev, 0);
    // next panel [jn, j):  Bbar part (rows k..n) and the S R part of Rbar (rows j..k)
    if (p > 0)
      Gemm<T>(c, p, wn, 0, 0, batch).seg(W, sub(L, j, jn), w).run(sub(A, k, jn), sub(A, k, jn), -1.0, 1.0, 0, partA);
    Gemm<T>(c, w, wn, 1, 0, batch).seg(S, sub(L, j, jn), w).run(sub(A, j, jn), sub(A, j, jn), -1.0, 1.0, 0, partA);
    if (jn > 0) {
      c.st = ls->bulk;
      cudaStreamWaitEvent(ls->bulk, ev_s, 0);
      if (p > 0)
        Gemm<T>(c, p, jn, 0, 0, batch).seg(W, sub(L, j, 0), w).run(sub(A, k, 0), sub(A, k, 0), -1.0, 1.0, 0, partB);
      Gemm<T> g(c, w, jn, 1, 0, batch);
      g.seg(S, sub(L, j, 0), w);
      if (p > 0) g.seg(W, sub(L, k, 0), p);
      g.run(sub(A, j, 0), sub(A, j, 0), -1.0, 1.0, 0, partB);
      ev_bulk_prev = ls->ev();
      cudaEventRecord(ev_bulk_prev, ls->bulk);
    }
  }
  // join both streams back into the caller's stream
  cudaEvent_t e1 = ls->ev(), e2 = ls->ev();
  cudaEventRecord(e1, ls->chain);
  cudaEventRecord(e2, ls->bulk);
  cudaStreamWaitEvent(caller, e1, 0);
  cudaStreamWaitEvent(caller, e2, 0);
  c.st = caller;
  if (info && c.ok()) {
    c.pre(CD_PROF_OTHER, 0.0);
    k_diag_info<T><<<unsigned(batch), 256, 0, c.st>>>(n, L, info);
    c.launched();
  }
}

// ------------------------------------------------------------------ blocked reverse, left-looking
// Same arithmetic as blocked_rev, reordered: the Bbar / Rbar updates of
// PAPER.md:696, 699 are delayed and applied to each panel just before it is processed,
// as ONE symmetric update Cbar -= (T + T^T) L[k:n, j:k] over the finished trailing part
// of the result (symm_ll.cuh derives it).  Per block [j, k), right to left:
//   Cbar <- Cbar - M L[k:n, j:k]            k_symm_ll (stream-K, in-kernel fixup)
//   Cbar <- Cbar D^{-1}                     } k_panel_rev, one cooperative launch:
//   Dbar <- Dbar - tril(Cbar^T C)           }   tile-parallel products + grid-wide
//   Dbar <- chol_unblocked_rev(D, Dbar)     }   deterministic reduction; the diagonal
//                                               block by Eq. 10, with
//                                               S = Dbar + Dbar^T kept per block for later M tiles
// Requires fp64, nb = 128 and TMA-describable Abar / L (16-byte aligned, even ld).
static bool g_no_ll = getenv("CD_REV_RIGHT_LOOKING") != nullptr;
static int64_t g_ll_pieces = getenv("CD_LL_PIECES") ? atoi(getenv("CD_LL_PIECES")) : 8;
// the SYMM moves into the panel kernel while its 32 x 32 output tiles number <= this x #SMs.  Default
// 0 (never) since k_symm_ll's deferred fixup: N = 1024 reverse 465 -> 453 us, 2048 1180 -> 1136 us,
// 4096 3592 -> 3550 us, 8192 15.26 -> 15.21 ms against 1 (before the deferred fixup, 1 won: 466 vs 602 us)
static int64_t g_symm_in_panel = getenv("CD_SYMM_IN_PANEL") ? atoi(getenv("CD_SYMM_IN_PANEL")) : 0;
static bool g_no_ll_defer = getenv("CD_NO_LL_DEFER") != nullptr;  // k_symm_ll: last-arrival fixup only

// (the cooperative panel kernels launched with PDL as well measured no faster: N = 16384 reverse
// 91.95 vs 91.94 ms, forward 95.46 vs 95.45 ms)
static cudaError_t launch_coop(const void* kernel, unsigned grid, size_t smem, cudaStream_t st, void** args) {
  return cudaLaunchCooperativeKernel(kernel, dim3(grid), dim3(PR_THREADS), args, smem, st);
}
static int g_dbg_panel_skip = getenv("CD_DEBUG_PANEL_SKIP") ? atoi(getenv("CD_DEBUG_PANEL_SKIP")) : 0;
// k_fwd_sk CTAs: at most ~PIECES pieces per output tile (0 = no cap); the cap only binds on the last
// ~10 panels of a sweep (m < 10 tiles), where the last arriver otherwise sums up to ~30 partial tiles
// (N = 4096: 5.53 -> 5.24 ms with 16; N = 1024 and 16384 unchanged; 4 and 8 were slower)
static int64_t g_fs_pieces = getenv("CD_FS_PIECES") ? atoi(getenv("CD_FS_PIECES")) : -1;  // -1: by size
// (forward N = 16384: 16 -> 32 pieces 95.56 -> 95.05 ms; N = 8192 17.20 -> 17.10 ms; N = 4096 keeps 16:
// 4.56 vs 4.66 ms with 32)
static int64_t fs_pieces(int n) { return g_fs_pieces >= 0 ? g_fs_pieces : (n > 4096 ? 32 : 16); }
static bool g_no_bal1 = getenv("CD_NO_BAL1") != nullptr;  // forward panel: one CTA per 128-wide K chunk
// k_fwd_sk with a deferred fixup (k_fwd_sk_reduce) whenever >= 4 k-tiles per CTA would leave SMs
// idle: one k-tile per CTA on up to every SM, the split tiles summed by the whole grid
static bool g_no_fs_defer = getenv("CD_NO_FS_DEFER") != nullptr;
// k_fwd_sk (fp.G / fp.defer chosen here); the caller has filled the rest of fp and called c.pre
static void launch_fwd_sk(Ctx& c, FSParams& fp, const FSMaps& tm, int n, int64_t batch) {
  fp.defer = !g_no_fs_defer && fp.total / LL_KT_PER_BLK < int64_t(c.sms) ? 1 : 0;
  if (fp.defer) {
    fp.G = int(std::max<int64_t>(1, std::min<int64_t>(c.sms, fp.total)));
  } else {
    fp.G = int(std::max<int64_t>(1, std::min<int64_t>(c.sms, fp.total / LL_KT_PER_BLK)));
    // (fused sweep N = 4096: 12.54 -> 12.12 ms with the piece cap)
    if (fs_pieces(n) > 0) fp.G = int(std::max<int64_t>(1, std::min<int64_t>(fp.G, fs_pieces(n) * batch * fp.m)));
  }
  c.err = note_cuda(launch_pdl(k_fwd_sk, fp.G, LL_THREADS, FS_SMEM, c.st, fp, tm));
  c.launched();
  if (fp.defer && c.ok()) {
    c.pre(CD_PROF_REDUCE, 0.0);
    const int64_t elems = (fp.total / fp.KT) * int64_t(LL_BM) * fp.w;
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(int64_t(c.sms) * 8, (elems + 255) / 256)));
    c.err = note_cuda(launch_pdl(k_fwd_sk_reduce, grid, 256, 0, c.st, fp));
    c.launched();
  }
}
// reverse panel phase 1: 128-row tiles cut into up to this many sub-tiles when the panel has few
// tiles (1 = whole tiles, and the 32 x 32-tile path for the fewest).  Measured with 4 against 1:
// N = 16384 93.24 -> 92.36 ms, 8192 16.27 -> 15.43 ms, 4096 4.08 -> 3.73 ms, 1024 487 -> 466 us
static int g_pr_split = getenv("CD_PR_SPLIT") ? atoi(getenv("CD_PR_SPLIT")) : 4;
// forward panel phase 0 (the previous panel's W D^{-T}): the same sub-tile split (1 = 32 x 32 staged tiles)
static int g_pf_split = getenv("CD_PF_SPLIT") ? atoi(getenv("CD_PF_SPLIT")) : 4;

// measurement: cap on the cooperative panel grid (0 = every co-resident CTA)
static int64_t g_panel_grid = getenv("CD_PANEL_GRID") ? atoi(getenv("CD_PANEL_GRID")) : 0;
static unsigned panel_grid(int64_t resident) {
  return unsigned(g_panel_grid > 0 ? std::min<int64_t>(resident, g_panel_grid) : resident);
}
static std::atomic<int> g_panel_occ[kMaxDev];
static int panel_occupancy() {
  return per_device(g_panel_occ, [] {
    int occ = 0;
    set_smem(k_panel_rev, PR_SMEM);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_panel_rev, PR_THREADS, PR_SMEM) != cudaSuccess || occ < 1)
      occ = 1;
    return occ;
  });
}

static void blocked_rev_ll(Ctx& c, int n, int nb, int64_t batch, Opnd L, Opnd A, int* info, double* part_ws) {
  const int nblk = nblocks(n, nb);
  double* Dinv = static_cast<double*>(c.take(sizeof(double) * size_t(batch) * nblk * nb * nb));
  const int64_t s_stride = int64_t(LL_BM + 4) * LL_BM * nblk;
  double* Sall = static_cast<double*>(c.take(sizeof(double) * size_t(batch) * s_stride));
  double* llpart = static_cast<double*>(c.take(sizeof(double) * size_t(c.sms) * 2 * LL_TILE));
  int* cnt = static_cast<int*>(c.take(sizeof(int) * size_t(batch) * nblk));
  // P partial slots: one per 128-row tile, or per sub-tile when phase 1 splits (then all fit one grid)
  const size_t nslots = std::max<size_t>(size_t(batch) * nblk, size_t(c.sms) * panel_occupancy());
  double* prpart = static_cast<double*>(c.take(sizeof(double) * nslots * 128 * 128));
  double* Pws = static_cast<double*>(c.take(sizeof(double) * size_t(batch) * 128 * 128));
  double* Zws = static_cast<double*>(c.take(sizeof(double) * size_t(batch) * 128 * 128));
  double* Wst = static_cast<double*>(c.take(sizeof(double) * size_t(batch) * nblk * 128 * 128));
  (void)part_ws;
  if (c.plan || !c.ok()) return;
  set_smem(k_panel_rev, PR_SMEM);
  LLMaps tm;
  memset(&tm, 0, sizeof(tm));
  tm.batched = batch > 1 ? 1 : 0;
  {
    int sh = 0;
    const double* Ab = static_cast<const double*>(A.base) + A.off;
    const double* Lb = static_cast<const double*>(L.base) + L.off;
    bool ok = make_tmap(&tm.aN, &sh, Ab, n, n, A.ld, A.stride, batch, LL_BM + 4, LL_BK) &&
              make_tmap(&tm.aT, &sh, Ab, n, n, A.ld, A.stride, batch, LL_BK + 4, LL_BM) &&
              make_tmap(&tm.s, &sh, Sall, LL_BM + 4, int64_t(LL_BM) * nblk, LL_BM + 4, s_stride, batch, LL_BM + 4, LL_BK) &&
              make_tmap(&tm.l, &sh, Lb, n, n, L.ld, L.stride, batch, LL_BK + 4, LL_BN);
    if (!ok) {
      c.err = CD_ERR_CUDA;
      snprintf(g_cuda_err, sizeof(g_cuda_err), "cuTensorMapEncodeTiled failed for the left-looking sweep");
      return;
    }
  }
  // the short top-left panel (w < 128): L clipped to its w columns, so the B tiles never
  // touch L's upper triangle (the padding columns are zero-filled instead)
  LLMaps tm_short = tm;
  if (n % nb) {
    int sh = 0;
    const double* Lb = static_cast<const double*>(L.base) + L.off;
    if (!make_tmap(&tm_short.l, &sh, Lb, n, n % nb, L.ld, L.stride, batch, LL_BK + 4, LL_BN)) {
      c.err = CD_ERR_CUDA;
      snprintf(g_cuda_err, sizeof(g_cuda_err), "cuTensorMapEncodeTiled failed for the left-looking sweep");
      return;
    }
  }
  std::vector<cudaEvent_t> ev_in;
  if (g_pipe) {  // host path: diagonal blocks, then column blocks right to left, stream in
    cudaEvent_t ev_diag;
    g_pipe->h2d(nblk, nb, true, ev_in, ev_diag);
    cudaStreamWaitEvent(c.st, ev_diag, 0);
  }
  c.err = note_cuda(cudaMemsetAsync(cnt, 0, sizeof(int) * size_t(batch) * nblk, c.st));
  set_smem(k_symm_ll, LL_SMEM);
  run_trinv<double>(c, n, nb, true, batch, L, Dinv);
  for (int qb = nblk - 1; qb >= 0 && c.ok(); --qb) {
    int j, w;
    block_range(n, nb, true, qb, j, w);
    const int k = j + w, p = n - k;
    if (g_pipe) cudaStreamWaitEvent(c.st, ev_in[size_t(qb)], 0);
    // small trailing part: the SYMM runs as phase 0 of the panel kernel (one launch per step)
    const bool symm_in_panel = p > 0 && batch * int64_t(p / LL_BM) * 16 <= int64_t(c.sms) * g_symm_in_panel;
    if (p > 0 && !symm_in_panel) {
      LLParams lp;
      lp.A = A;
      lp.n = n, lp.k = k, lp.j = j, lp.w = w;
      lp.m = p / LL_BM;
      lp.nblk = nblk;
      lp.total = batch * int64_t(lp.m) * LL_KT_PER_BLK * lp.m;
      // CTAs: at most ~PIECES pieces per output tile -- the last-arriving CTA sums all pieces
      // of a tile alone, so with few tiles more CTAs cost more in the fixup than they save
      const int64_t pieces = g_ll_pieces;
      // (deferred fixup as for k_fwd_sk: ~one k-tile per CTA on every SM, k_symm_ll_reduce sums)
      lp.defer = !g_no_ll_defer && lp.total / LL_KT_PER_BLK < int64_t(c.sms) ? 1 : 0;
      lp.G = lp.defer ? int(std::min<int64_t>(c.sms, lp.total))
                      : int(std::max<int64_t>(1, std::min<int64_t>({int64_t(c.sms), lp.total / LL_KT_PER_BLK,
                                                                    pieces * batch * int64_t(lp.m)})));
      lp.part = llpart;
      lp.cnt = cnt;
      c.pre(CD_PROF_SYMM, 2.0 * double(p) * p * w * double(batch));
      if (lp.total >= (int64_t(1) << 31)) {
        c.err = CD_ERR_UNSUPPORTED;
        return;
      }
      c.err = note_cuda(launch_pdl(k_symm_ll, lp.G, LL_THREADS, LL_SMEM, c.st, lp, w < nb ? tm_short : tm));
      c.launched();
      if (lp.defer && c.ok()) {
        c.pre(CD_PROF_REDUCE, 0.0);
        const int64_t elems = (lp.total / (LL_KT_PER_BLK * int64_t(lp.m))) * int64_t(LL_BM) * w;
        const int rg = int(std::max<int64_t>(1, std::min<int64_t>(int64_t(c.sms) * 8, (elems + 255) / 256)));
        c.err = note_cuda(launch_pdl(k_symm_ll_reduce, rg, 256, 0, c.st, lp));
        c.launched();
      }
    }
    // Cbar <- Cbar D^{-1};  Dbar <- Dbar - tril(Cbar^T C);  Dbar <- chol_unblocked_rev(D, Dbar)
    // (Eq. 10) + S -- one cooperative kernel
    PanelParams pp;
    pp.A = A;
    pp.L = L;
    pp.Dinv = Dinv + int64_t(qb) * nb * nb;
    pp.dstride = int64_t(nblk) * nb * nb;
    pp.dld = nb;
    pp.n = n, pp.j = j, pp.w = w, pp.k = k;
    pp.tiles = p / LL_BM;
    pp.batch = batch;
    pp.part = prpart;
    pp.Pws = Pws;
    pp.Zws = Zws;
    pp.S = qb > 0 ? Sall + int64_t(qb) * (LL_BM + 4) * LL_BM : nullptr;
    pp.s_ld = LL_BM + 4;
    pp.s_stride = s_stride;
    pp.dbg_skip = g_dbg_panel_skip;
    pp.Wst = Wst;
    pp.symm = symm_in_panel ? 1 : 0;
    pp.Sall = Sall;
    pp.s_blk = int64_t(LL_BM + 4) * LL_BM;
    pp.nblk = nblk;
    pp.split_max = g_pr_split;
    const unsigned grid = panel_grid(int64_t(c.sms) * panel_occupancy());  // all co-resident CTAs
    void* args[] = {&pp};
    const double wf = w;
    c.pre(CD_PROF_PANEL, (double(p) * w * (w + 1) * 2.0 + (4 * wf * wf * wf + 3 * wf * wf + 11 * wf) / 6) * double(batch));
    c.err = note_cuda(launch_coop(reinterpret_cast<const void*>(k_panel_rev), grid, PR_SMEM, c.st, args));
    c.launched();
    if (g_pipe) g_pipe->d2h(c.st, j, w);  // column block final: stream it out
  }
  if (info && c.ok()) {
    c.pre(CD_PROF_OTHER, 0.0);
    k_diag_info<double><<<unsigned(batch), 256, 0, c.st>>>(n, L, info);
    c.launched();
  }
}

// ------------------------------------------------------------------ blocked reverse, left-looking, fp32
// The left-looking schedule of blocked_rev_ll for fp32 on the tcgen05 tensor cores: per block
// [j, k), right to left,
//   Cbar <- Cbar - M L[k:n, j:k]         k_symm_tc (stream-K, tf32, in-kernel fixup)
//   Cbar <- Cbar D^{-1}                  tcgen05 GEMM, in place
//   Dbar <- Dbar - tril(Cbar^T C)        tcgen05 GEMM, tril
//   Dbar <- chol_unblocked_rev(D, Dbar)  k_rev_dmma_cta (fp64 arithmetic), + S kept
// nb = 128, TMA-describable fp32 operands (16-byte aligned, ld % 4 == 0).
static bool g_no_ll32 = getenv("CD_NO_LL32") != nullptr;
// pieces per output tile of k_symm_tc (its fixup moves (pieces + 1) fp32 tiles through one SM;
// 4 measured best: N = 4096 4.13 ms vs 4.41 at 8, N = 16384 31.9 vs 32.2 ms)
static int64_t g_ll32_pieces = getenv("CD_LL32_PIECES") ? atoi(getenv("CD_LL32_PIECES")) : 4;

static void blocked_rev_ll32(Ctx& c, int n, int nb, int64_t batch, Opnd L, Opnd A, int* info, float* part_ws) {
  const int nblk = nblocks(n, nb);
  float* Dinv = static_cast<float*>(c.take(sizeof(float) * size_t(batch) * nblk * nb * nb));
  const int64_t s_stride = int64_t(nblk) * 128 * 128;
  float* Sall = static_cast<float*>(c.take(sizeof(float) * size_t(batch) * s_stride));
  float* tcpart = static_cast<float*>(c.take(sizeof(float) * size_t(c.sms) * 2 * STC_TILE));
  int* cnt = static_cast<int*>(c.take(sizeof(int) * size_t(batch) * nblk));
  if (c.plan || !c.ok()) return;
  STCMaps tm;
  memset(&tm, 0, sizeof(tm));
  tm.batched = batch > 1 ? 1 : 0;
  {
    const float* Ab = static_cast<const float*>(A.base) + A.off;
    const float* Lb = static_cast<const float*>(L.base) + L.off;
    const bool ok = make_tmap_f32_sw128(&tm.aMN, Ab, n, n, A.ld, A.stride, batch, 32, 32, true) &&
                    make_tmap_f32_sw128(&tm.aK, Ab, n, n, A.ld, A.stride, batch, 32, 128, false) &&
                    make_tmap_f32_sw128(&tm.sMN, Sall, 128, int64_t(128) * nblk, 128, s_stride, batch, 32, 32, true) &&
                    make_tmap_f32_sw128(&tm.lK, Lb, n, n, L.ld, L.stride, batch, 32, 128, false);
    if (!ok) {
      c.err = CD_ERR_CUDA;
      snprintf(g_cuda_err, sizeof(g_cuda_err), "cuTensorMapEncodeTiled failed for the fp32 left-looking sweep");
      return;
    }
  }
  c.err = note_cuda(cudaMemsetAsync(cnt, 0, sizeof(int) * size_t(batch) * nblk, c.st));
  set_smem(k_symm_tc, STC_SMEM);
  run_trinv<float>(c, n, nb, true, batch, L, Dinv);
  for (int qb = nblk - 1; qb >= 0 && c.ok(); --qb) {
    int j, w;
    block_range(n, nb, true, qb, j, w);
    const int k = j + w, p = n - k;
    const Opnd Cbar = sub(A, k, j);
    if (p > 0) {
      STCParams sp;
      sp.A = A;
      sp.n = n, sp.k = k, sp.j = j, sp.w = w;
      sp.m = p / 128;
      sp.nblk = nblk;
      sp.total = batch * int64_t(sp.m) * STC_CHUNKS_PER_BLK * sp.m;
      // CTAs: >= 2 K chunks each, at most ~PIECES pieces per output tile (see blocked_rev_ll)
      sp.G = int(std::max<int64_t>(1, std::min<int64_t>({int64_t(c.sms), sp.total / 2,
                                                         g_ll32_pieces * batch * int64_t(sp.m)})));
      sp.part = tcpart;
      sp.cnt = cnt;
      if (sp.total >= (int64_t(1) << 31)) {
        c.err = CD_ERR_UNSUPPORTED;
        return;
      }
      c.pre(CD_PROF_SYMM, 2.0 * double(p) * p * w * double(batch));
      k_symm_tc<<<sp.G, STC_THREADS, STC_SMEM, c.st>>>(sp, tm);
      c.launched();
      // Cbar <- Cbar D^{-1}
      const Opnd Dinv_q = ws_opnd(Dinv + int64_t(qb) * nb * nb, int64_t(nblk) * nb * nb, nb);
      Gemm<float>(c, p, w, 0, 0, batch)
          .seg(Cbar, Dinv_q, w)
          .flops(double(p) * w * (w + 1))
          .run(null_opnd(), Cbar, 1.0, 0.0, 0, part_ws);
      // Dbar <- Dbar - tril(Cbar^T C)
      Gemm<float>(c, w, w, 1, 0, batch)
          .seg(Cbar, sub(L, k, j), p)
          .flops(double(w) * (w + 1) * p)
          .run(sub(A, j, j), sub(A, j, j), -1.0, 1.0, 1, part_ws);
    }
    // Dbar <- chol_unblocked_rev(D, Dbar); S = Dbar + Dbar^T kept for the later SYMMs
    const Opnd S = qb > 0 ? ws_opnd(Sall + int64_t(qb) * 128 * 128, s_stride, 128) : null_opnd();
    run_sweep_small<float>(c, true, w, batch, sub(L, j, j), sub(A, j, j), 0, S, nullptr);
  }
  if (info && c.ok()) {
    c.pre(CD_PROF_OTHER, 0.0);
    k_diag_info<float><<<unsigned(batch), 256, 0, c.st>>>(n, L, info);
    c.launched();
  }
}

// ------------------------------------------------------------------ blocked forward
// chol_blocked_fwd, block [j, k), w = k - j, p = n - k, q = j:
//   Ddot <- Ddot - tril(Rdot R^T + R Rdot^T)        GEMM (2 K-segments), tril, split-K
//   Ddot <- chol_unblocked_fwd(D, Ddot)             sweep kernel (+ clean tril(Ddot) copy Dc)
//   Cdot <- Cdot - Bdot R^T - B Rdot^T              } one GEMM with 3 K-segments into W:
//   Cdot <- (Cdot - C Ddot^T) D^{-T}                }   W = Cdot - [Bdot B C][R Rdot Dc]^T
//                                                       then Cdot = W Dinv^T
// (W is Cdot itself when one N-tile covers the block, as in blocked_rev.)
template <typename T>
static void blocked_fwd(Ctx& c, int n, int nb, int64_t batch, Opnd L, Opnd A, int* info, T* part_ws) {
  const int nblk = nblocks(n, nb);
  T* Dinv = static_cast<T*>(c.take(sizeof(T) * size_t(batch) * nblk * nb * nb));
  T* Dcw = static_cast<T*>(c.take(sizeof(T) * size_t(batch) * nb * nb));
  const bool w_inplace = nb <= G_BN;  // see blocked_rev
  T* Wws = w_inplace ? nullptr : static_cast<T*>(c.take(sizeof(T) * size_t(batch) * n * nb));
  if (T* ext = shared_dinv<T>(n, nb)) Dinv = c.plan ? Dinv : ext;
  else run_trinv<T>(c, n, nb, false, batch, L, Dinv);
  for (int qb = 0; qb < nblk; ++qb) {
    int j, w;
    block_range(n, nb, false, qb, j, w);
    const int k = j + w, p = n - k, q = j;
    const Opnd Dinv_q = ws_opnd(Dinv + int64_t(qb) * nb * nb, int64_t(nblk) * nb * nb, nb);
    const Opnd Dc = ws_opnd(Dcw, int64_t(nb) * nb, w);
    const Opnd W = w_inplace ? sub(A, k, j) : ws_opnd(Wws, int64_t(n) * nb, std::max(p, 1));
    if (q > 0)  // Ddot <- Ddot - tril(Rdot R^T + R Rdot^T)
      Gemm<T>(c, w, w, 0, 1, batch)
          .seg(sub(A, j, 0), sub(L, j, 0), q)
          .seg(sub(L, j, 0), sub(A, j, 0), q)
          .flops(2.0 * w * (w + 1) * q)  // lower triangle only
          .run(sub(A, j, j), sub(A, j, j), -1.0, 1.0, 1, part_ws);
    diag_block<T>(c, false, w, batch, sub(L, j, j), sub(A, j, j), p > 0 ? Dc : null_opnd(), Dinv_q);
    if (p > 0) {
      Gemm<T> g(c, p, w, 0, 1, batch);
      if (q > 0) g.seg(sub(A, k, 0), sub(L, j, 0), q).seg(sub(L, k, 0), sub(A, j, 0), q);
      g.seg(sub(L, k, j), Dc, w);
      g.run(sub(A, k, j), W, -1.0, 1.0, 0, part_ws);
      if (qb == 0) wait_dinv(c);
      Gemm<T>(c, p, w, 0, 1, batch)
          .seg(W, Dinv_q, w)
          .flops(double(p) * w * (w + 1))  // TRSM  X D^{-T}
          .run(null_opnd(), sub(A, k, j), 1.0, 0.0, 0, part_ws);
    }
  }
  if (info && !c.plan && c.ok()) {
    c.pre(CD_PROF_OTHER, 0.0);
    k_diag_info<T><<<unsigned(batch), 256, 0, c.st>>>(n, L, info);
    c.launched();
  }
}

// ------------------------------------------------------------------ blocked forward, fused panels
// chol_blocked_fwd for fp64, nb = 128, TMA-describable operands, as two
// launches per panel J = [j, k):
//   k_panel_fwd (cooperative): [previous panel's Cdot <- W D^{-T}], Ddot -= tril(Rdot R^T +
//       R Rdot^T) (K-chunk partials + deterministic reduction), Ddot <- D Phi(D^{-1} Ddot D^{-T})
//       (Eq. 8) + the clean copy Dc
//   k_fwd_sk (stream-K):   W = Cdot - [Bdot B C] [R Rdot Dc]^T, in place
// The last panel has no rows below it, so no W D^{-T} is left pending.
static std::atomic<int> g_panel_fwd_occ[kMaxDev];
static int panel_fwd_occupancy() {
  return per_device(g_panel_fwd_occ, [] {
    int occ = 0;
    set_smem(k_panel_fwd, PR_SMEM);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_panel_fwd, PR_THREADS, PR_SMEM) != cudaSuccess || occ < 1)
      occ = 1;
    return occ;
  });
}

static void blocked_fwd_ll(Ctx& c, int n, int nb, int64_t batch, Opnd L, Opnd A, int* info) {
  const int nblk = nblocks(n, nb);
  double* Dinv = static_cast<double*>(c.take(sizeof(double) * size_t(batch) * nblk * nb * nb));
  // phase-1 partial slots: nblk per matrix, or one per SM for single matrices (balanced K split)
  const int kslots = batch == 1 ? std::max(nblk, c.sms) : nblk;
  double* part = static_cast<double*>(c.take(sizeof(double) * size_t(batch) * kslots * 128 * 128));
  double* Yws = static_cast<double*>(c.take(sizeof(double) * size_t(batch) * 128 * 128));
  double* Fws = static_cast<double*>(c.take(sizeof(double) * size_t(batch) * 128 * 128));
  double* Dc = static_cast<double*>(c.take(sizeof(double) * size_t(batch) * 132 * 128));
  double* skpart = static_cast<double*>(c.take(sizeof(double) * size_t(c.sms) * 2 * LL_TILE));
  int* cnt = static_cast<int*>(c.take(sizeof(int) * size_t(batch) * nblk));
  if (c.plan || !c.ok()) return;
  FSMaps tm;
  memset(&tm, 0, sizeof(tm));
  tm.batched = batch > 1 ? 1 : 0;
  {
    int sh = 0;
    const double* Ab = static_cast<const double*>(A.base) + A.off;
    const double* Lb = static_cast<const double*>(L.base) + L.off;
    const bool ok = make_tmap(&tm.adot, &sh, Ab, n, n, A.ld, A.stride, batch, FS_PITCH, LL_BK) &&
                    make_tmap(&tm.l, &sh, Lb, n, n, L.ld, L.stride, batch, FS_PITCH, LL_BK) &&
                    make_tmap(&tm.dc, &sh, Dc, 132, 128, 132, 132 * 128, batch, FS_PITCH, LL_BK);
    if (!ok) {
      c.err = CD_ERR_CUDA;
      snprintf(g_cuda_err, sizeof(g_cuda_err), "cuTensorMapEncodeTiled failed for the forward sweep");
      return;
    }
  }
  std::vector<cudaEvent_t> ev_in;
  if (g_pipe) {  // host path: diagonal blocks, then column blocks left to right, stream in
    cudaEvent_t ev_diag;
    g_pipe->h2d(nblk, nb, false, ev_in, ev_diag);
    cudaStreamWaitEvent(c.st, ev_diag, 0);
  }
  c.err = note_cuda(cudaMemsetAsync(cnt, 0, sizeof(int) * size_t(batch) * nblk, c.st));
  set_smem(k_fwd_sk, FS_SMEM);
  set_smem(k_panel_fwd, PR_SMEM);
  run_trinv<double>(c, n, nb, false, batch, L, Dinv);
  int j_prev = 0, k_prev = 0, p_prev = 0;
  for (int qb = 0; qb < nblk && c.ok(); ++qb) {
    int j, w;
    block_range(n, nb, false, qb, j, w);
    const int k = j + w, p = n - k, q = j;
    if (g_pipe) cudaStreamWaitEvent(c.st, ev_in[size_t(qb)], 0);
    PanelFwdParams pf;
    pf.A = A;
    pf.L = L;
    pf.Dinv = Dinv + int64_t(qb) * nb * nb;
    pf.Dinv_prev = (qb > 0 && p_prev > 0) ? Dinv + int64_t(qb - 1) * nb * nb : nullptr;
    pf.dstride = int64_t(nblk) * nb * nb;
    pf.dld = nb;
    pf.n = n, pf.j = j, pf.w = w;
    pf.j_prev = j_prev, pf.k_prev = k_prev, pf.tiles_prev = (p_prev + 127) / 128;
    pf.kchunks = q / 128;
    pf.batch = batch;
    pf.part = part;
    pf.Yws = Yws;
    pf.Fws = Fws;
    pf.Dc = Dc;
    pf.T0 = A;
    pf.single = 0;
    pf.skip3 = 0;
    pf.dbg_skip = g_dbg_panel_skip;
    pf.kslot_cap = g_no_bal1 ? 0 : kslots;
    pf.split_max = g_pf_split;
    const unsigned grid = panel_grid(int64_t(c.sms) * panel_fwd_occupancy());
    void* args[] = {&pf};
    const double wf = w;
    c.pre(CD_PROF_PANEL, (double(p_prev) * 128 * 129 + 2.0 * wf * (wf + 1) * q +
                          (4 * wf * wf * wf + 3 * wf * wf + 5 * wf) / 6) * double(batch));
    c.err = note_cuda(launch_coop(reinterpret_cast<const void*>(k_panel_fwd), grid, PR_SMEM, c.st, args));
    c.launched();
    if (g_pipe && qb > 0) g_pipe->d2h(c.st, j_prev, 128);  // previous block's W D^{-T} is done
    if (p > 0 && c.ok()) {
      FSParams fp;
      fp.A = A;
      fp.n = n, fp.k = k, fp.j = j, fp.w = w, fp.q = q;
      fp.m = (p + 127) / 128;
      fp.KT = (2 * q + w + LL_BK - 1) / LL_BK;
      fp.total = batch * int64_t(fp.m) * fp.KT;
      if (fp.total >= (int64_t(1) << 31) || w != 128) {
        c.err = CD_ERR_UNSUPPORTED;
        return;
      }
      fp.part = skpart;
      fp.cnt = cnt;
      fp.chol = 0;
      c.pre(CD_PROF_SYMM, 2.0 * double(p) * w * (2.0 * q + w) * double(batch));
      launch_fwd_sk(c, fp, tm, n, batch);
    }
    j_prev = j, k_prev = k, p_prev = p;
  }
  if (g_pipe && c.ok()) {  // the last block (no rows below it) is final after its panel
    int j, w;
    block_range(n, nb, false, nblk - 1, j, w);
    g_pipe->d2h(c.st, j, w);
  }
  if (info && c.ok()) {
    c.pre(CD_PROF_OTHER, 0.0);
    k_diag_info<double><<<unsigned(batch), 256, 0, c.st>>>(n, L, info);
    c.launched();
  }
}

// ------------------------------------------------------------------ fused factorisation + forward
// chol_blocked and chol_blocked_fwd accumulated in one
// sweep: in: tril(A) = Sigma, tril(Adot) = Sigma_dot; out: L, Ldot.
// fp64, nb = 128, TMA-describable operands.  Per panel J = [j, k):
//   k_panel_fwd  [phase 0: previous panel's Cdot <- W D^{-T}; phases 1-2: D <- D - tril(R R^T)]
//   k_chol_diag  D <- chol_unblocked(D) on chip, D^{-1}
//   k_fwd_sk     C <- C - B R^T                                  (factorisation mode)
//   k_panel_fwd  [phase 0: C <- C D^{-T}; phases 1-3: Ddot -= tril(Rdot R^T + R Rdot^T), Eq. 8]
//   k_fwd_sk     W = Cdot - [Bdot B C][R Rdot Dc]^T
static void chol_fwd_fused(Ctx& c, int n, int nb, int64_t batch, Opnd A, Opnd Ad, int* info) {
  const int nblk = nblocks(n, nb);
  double* Dinv = static_cast<double*>(c.take(sizeof(double) * size_t(batch) * nblk * nb * nb));
  // phase-1 partial slots: nblk per matrix, or one per SM for single matrices (balanced K split)
  const int kslots = batch == 1 ? std::max(nblk, c.sms) : nblk;
  double* part = static_cast<double*>(c.take(sizeof(double) * size_t(batch) * kslots * 128 * 128));
  double* Yws = static_cast<double*>(c.take(sizeof(double) * size_t(batch) * 128 * 128));
  double* Fws = static_cast<double*>(c.take(sizeof(double) * size_t(batch) * 128 * 128));
  double* Dc = static_cast<double*>(c.take(sizeof(double) * size_t(batch) * 132 * 128));
  double* skpart = static_cast<double*>(c.take(sizeof(double) * size_t(c.sms) * 2 * LL_TILE));
  int* cnt = static_cast<int*>(c.take(sizeof(int) * size_t(batch) * nblk));
  if (c.plan || !c.ok()) return;
  FSMaps tmf, tmc;
  memset(&tmf, 0, sizeof(tmf));
  tmf.batched = batch > 1 ? 1 : 0;
  {
    int sh = 0;
    const double* Ab = static_cast<const double*>(A.base) + A.off;
    const double* Adb = static_cast<const double*>(Ad.base) + Ad.off;
    const bool ok = make_tmap(&tmf.adot, &sh, Adb, n, n, Ad.ld, Ad.stride, batch, FS_PITCH, LL_BK) &&
                    make_tmap(&tmf.l, &sh, Ab, n, n, A.ld, A.stride, batch, FS_PITCH, LL_BK) &&
                    make_tmap(&tmf.dc, &sh, Dc, 132, 128, 132, 132 * 128, batch, FS_PITCH, LL_BK);
    if (!ok) {
      c.err = CD_ERR_CUDA;
      snprintf(g_cuda_err, sizeof(g_cuda_err), "cuTensorMapEncodeTiled failed for the fused sweep");
      return;
    }
  }
  tmc = tmf;  // factorisation mode reads only the `l` map
  c.err = note_cuda(cudaMemsetAsync(cnt, 0, sizeof(int) * size_t(batch) * nblk, c.st));
  if (info && c.ok()) c.err = note_cuda(cudaMemsetAsync(info, 0, sizeof(int) * size_t(batch), c.st));
  set_smem(k_fwd_sk, FS_SMEM);
  set_smem(k_panel_fwd, PR_SMEM);
  const size_t dsm = dmma_cta_smem((nb + 7) / 8);
  set_smem(k_chol_diag<double>, dsm);
  const unsigned grid = panel_grid(int64_t(c.sms) * panel_fwd_occupancy());
  auto panel = [&](PanelFwdParams& pf, double flops) {
    void* args[] = {&pf};
    c.pre(CD_PROF_PANEL, flops * double(batch));
    c.err = note_cuda(launch_coop(reinterpret_cast<const void*>(k_panel_fwd), grid, PR_SMEM, c.st, args));
    c.launched();
  };
  auto sk = [&](int j, int w, int k, int p, int q, int chol, const FSMaps& tm, Opnd D) {
    FSParams fp;
    fp.A = D;
    fp.n = n, fp.k = k, fp.j = j, fp.w = w, fp.q = q;
    fp.m = (p + 127) / 128;
    fp.KT = chol ? q / LL_BK : (2 * q + w + LL_BK - 1) / LL_BK;
    fp.total = batch * int64_t(fp.m) * fp.KT;
    if (fp.total >= (int64_t(1) << 31) || w != 128) {
      c.err = CD_ERR_UNSUPPORTED;
      return;
    }
    fp.part = skpart;
    fp.cnt = cnt;
    fp.chol = chol;
    c.pre(CD_PROF_SYMM, 2.0 * double(p) * w * double(chol ? q : 2.0 * q + w) * double(batch));
    launch_fwd_sk(c, fp, tm, n, batch);
  };
  auto base_params = [&](PanelFwdParams& pf) {
    memset(&pf, 0, sizeof(pf));
    pf.dstride = int64_t(nblk) * nb * nb;
    pf.dld = nb;
    pf.n = n;
    pf.batch = batch;
    pf.part = part;
    pf.Yws = Yws;
    pf.Fws = Fws;
    pf.Dc = Dc;
    pf.kslot_cap = g_no_bal1 ? 0 : kslots;
    pf.split_max = g_pf_split;
  };
  int j_prev = 0, k_prev = 0, p_prev = 0;
  for (int qb = 0; qb < nblk && c.ok(); ++qb) {
    int j, w;
    block_range(n, nb, false, qb, j, w);
    const int k = j + w, p = n - k, q = j;
    if (qb > 0) {  // previous panel's forward solve; D <- D - tril(R R^T)
      PanelFwdParams pf;
      base_params(pf);
      pf.A = A;
      pf.L = A;
      pf.T0 = Ad;
      pf.Dinv = Dinv + int64_t(qb) * nb * nb;
      pf.Dinv_prev = p_prev > 0 ? Dinv + int64_t(qb - 1) * nb * nb : nullptr;
      pf.j_prev = j_prev, pf.k_prev = k_prev, pf.tiles_prev = (p_prev + 127) / 128;
      pf.j = j, pf.w = w;
      pf.kchunks = q / 128;
      pf.single = 1;
      pf.skip3 = 1;
      pf.dbg_skip = 0;
      panel(pf, double(p_prev) * 128 * 129 + double(w) * (w + 1) * q);
    }
    // D <- chol_unblocked(D), D^{-1}
    c.pre(CD_PROF_SWEEP, (double(w) * w * w / 3.0 + double(w) * w * w / 3.0) * double(batch));
    k_chol_diag<double><<<dim3(1, unsigned(batch)), DC_THREADS, dsm, c.st>>>(
        w, sub(A, j, j), Dinv + int64_t(qb) * nb * nb, nb, int64_t(nblk) * nb * nb, j, info);
    c.launched();
    if (p > 0 && q > 0) sk(j, w, k, p, q, 1, tmc, A);  // C <- C - B R^T
    {  // C <- C D^{-T}; the forward panel (Ddot update, Eq. 8)
      PanelFwdParams pf;
      base_params(pf);
      pf.A = Ad;
      pf.L = A;
      pf.T0 = A;
      pf.Dinv = Dinv + int64_t(qb) * nb * nb;
      pf.Dinv_prev = p > 0 ? Dinv + int64_t(qb) * nb * nb : nullptr;
      pf.j_prev = j, pf.k_prev = k, pf.tiles_prev = (p + 127) / 128;
      pf.j = j, pf.w = w;
      pf.kchunks = q / 128;
      pf.single = 0;
      pf.skip3 = 0;
      const double wf = w;
      panel(pf, double(p) * w * (w + 1) + 2.0 * wf * (wf + 1) * q + (4 * wf * wf * wf + 3 * wf * wf + 5 * wf) / 6);
    }
    if (p > 0 && c.ok()) sk(j, w, k, p, q, 0, tmf, Ad);  // W = Cdot - [Bdot B C][R Rdot Dc]^T
    j_prev = j, k_prev = k, p_prev = p;
  }
}

// ------------------------------------------------------------------ symbolic route, large n
// Eqs. 10 / 8 on the whole matrix for n > 64:
//   reverse  X = P + P^T, P = Phi(L^T Lbar);  Y = L^{-T} X L^{-1};  tril(Sigmabar) = Phi(Y)
//   forward  Y = L^{-1} Sigmadot L^{-T};  Ldot = L Phi(Y)
// Products are the library's GEMM kernels on clean (upper-zero) triangular copies; the two
// triangular solves are blocked over 128-column blocks with the diagonal-block inverses
// (k_trinv_dmma) -- the "Level 3 ... solving a triangular system" of PAPER.md:634-636.
// About 4 n^3 flops against the sweep's 2 n^3 / 3: offered for measurement (north star (d),
// "worth measuring against the blocked sweep"); AUTO never picks it.
template <typename T>
static void symbolic_large(Ctx& c, int n, int64_t batch, bool rev, Opnd L, Opnd A, int out_mode, T* part) {
  const int nb = 128, nblk = nblocks(n, nb);
  const int64_t nn = int64_t(n) * n;
  T* Lc = static_cast<T*>(c.take(sizeof(T) * size_t(batch) * nn));
  T* X = static_cast<T*>(c.take(sizeof(T) * size_t(batch) * nn));
  T* Z = static_cast<T*>(c.take(sizeof(T) * size_t(batch) * nn));
  T* Dinv = static_cast<T*>(c.take(sizeof(T) * size_t(batch) * nblk * nb * nb));
  if (c.plan || !c.ok()) return;
  const Opnd OL = ws_opnd(Lc, nn, n), OX = ws_opnd(X, nn, n), OZ = ws_opnd(Z, nn, n);
  auto elem = [&](Opnd S, Opnd D, int mode) {
    c.pre(CD_PROF_OTHER, 0.0);
    k_sym_elem<T><<<grid_1d(nn * batch, 256, c.sms), 256, 0, c.st>>>(n, batch, S, D, mode);
    c.launched();
  };
  elem(L, OL, 0);  // clean tril(L)
  run_trinv<T>(c, n, nb, false, batch, L, Dinv);
  auto dinv = [&](int qb) { return ws_opnd(Dinv + int64_t(qb) * nb * nb, int64_t(nblk) * nb * nb, nb); };
  if (rev) {
    elem(A, OZ, 0);  // clean tril(Lbar)
    Gemm<T>(c, n, n, 1, 0, batch).seg(OL, OZ, n).run(null_opnd(), OX, 1.0, 0.0, 0, part);  // L^T Lbar
    elem(OX, OZ, 1);  // Z = Phi(P) + Phi(P)^T
    // right solve W = Z L^{-1}: column blocks right to left, W[:, J] = (Z[:, J] - W[:, k:n] L[k:n, J]) D_J^{-1}
    for (int qb = nblk - 1; qb >= 0 && c.ok(); --qb) {
      int j, w;
      block_range(n, nb, false, qb, j, w);
      const int k = j + w;
      if (k < n) Gemm<T>(c, n, w, 0, 0, batch).seg(sub(OZ, 0, k), sub(OL, k, j), n - k).run(sub(OZ, 0, j), sub(OZ, 0, j), -1.0, 1.0, 0, part);
      Gemm<T>(c, n, w, 0, 0, batch).seg(sub(OZ, 0, j), dinv(qb), w).run(null_opnd(), sub(OZ, 0, j), 1.0, 0.0, 0, part);
    }
    // left solve Y = L^{-T} W: row blocks bottom to top, Y[J, :] = D_J^{-T} (W[J, :] - L[k:n, J]^T Y[k:n, :])
    for (int qb = nblk - 1; qb >= 0 && c.ok(); --qb) {
      int j, w;
      block_range(n, nb, false, qb, j, w);
      const int k = j + w;
      if (k < n) Gemm<T>(c, w, n, 1, 0, batch).seg(sub(OL, k, j), sub(OZ, k, 0), n - k).run(sub(OZ, j, 0), sub(OZ, j, 0), -1.0, 1.0, 0, part);
      Gemm<T>(c, w, n, 1, 0, batch).seg(dinv(qb), sub(OZ, j, 0), w).run(null_opnd(), sub(OZ, j, 0), 1.0, 0.0, 0, part);
    }
    elem(OZ, A, 4);  // tril(Sigmabar) = Phi(Y)
    if (out_mode != CD_OUT_TRIL && c.ok()) {
      c.pre(CD_PROF_OTHER, 0.0);
      k_out_mode<T><<<grid_1d(nn * batch, 256, c.sms), 256, 0, c.st>>>(n, batch, A, out_mode);
      c.launched();
    }
  } else {
    elem(A, OZ, 2);  // X = Sigmadot, symmetric
    // left solve Y = L^{-1} X: row blocks top to bottom, Y[J, :] = D_J^{-1} (X[J, :] - L[J, 0:j] Y[0:j, :])
    for (int qb = 0; qb < nblk && c.ok(); ++qb) {
      int j, w;
      block_range(n, nb, false, qb, j, w);
      if (j > 0) Gemm<T>(c, w, n, 0, 0, batch).seg(sub(OL, j, 0), OZ, j).run(sub(OZ, j, 0), sub(OZ, j, 0), -1.0, 1.0, 0, part);
      Gemm<T>(c, w, n, 0, 0, batch).seg(dinv(qb), sub(OZ, j, 0), w).run(null_opnd(), sub(OZ, j, 0), 1.0, 0.0, 0, part);
    }
    // right solve Z = Y L^{-T}: column blocks left to right, Z[:, J] = (Y[:, J] - Z[:, 0:j] L[J, 0:j]^T) D_J^{-T}
    for (int qb = 0; qb < nblk && c.ok(); ++qb) {
      int j, w;
      block_range(n, nb, false, qb, j, w);
      if (j > 0) Gemm<T>(c, n, w, 0, 1, batch).seg(OZ, sub(OL, j, 0), j).run(sub(OZ, 0, j), sub(OZ, 0, j), -1.0, 1.0, 0, part);
      Gemm<T>(c, n, w, 0, 1, batch).seg(sub(OZ, 0, j), dinv(qb), w).run(null_opnd(), sub(OZ, 0, j), 1.0, 0.0, 0, part);
    }
    elem(OZ, OX, 3);  // F = Phi(Z), clean
    Gemm<T>(c, n, n, 0, 0, batch).seg(OL, OX, n).run(null_opnd(), OZ, 1.0, 0.0, 0, part);  // Ldot = L F
    c.pre(CD_PROF_OTHER, 0.0);
    k_copy_tril<T><<<grid_1d(nn * batch, 256, c.sms), 256, 0, c.st>>>(n, batch, OZ, A);
    c.launched();
  }
}

// ------------------------------------------------------------------ top-level
struct Call {
  cd_op op;
  cd_dtype dt;
  int64_t n, batch;
  Opnd L, A;
  cd_opts o;
  int* info;
};

static int default_nb(cd_dtype dt, int64_t n, int64_t batch, bool arr) {
  // fp64: 128 (the left-looking schedule's tile).  fp32 mid-size (batched tf32 path): 128 for
  // strided batches with n % 128 == 0 -- the trailing updates are memory-bound and their traffic
  // falls with the panel count, the 128-wide diagonal blocks run on k_rf_diag128 (configs[3]
  // rev + fwd 3.54 -> 2.93 ms); otherwise 64, whose on-chip diagonal-block kernels fit several
  // CTAs per SM (round 1, with the fp64-DMMA 128-wide sweeps: rev 4.28 -> 3.39 ms, fwd 4.10 -> 2.83 ms)
  if (dt == CD_F32 && n <= 1024)
    return (batch > 1 && n % 128 == 0 && !arr && !g_no_diag128 && !g_no_hmma_diag) ? 128 : 64;
  return 128;
}

// The fused per-matrix fp32 batched kernel (rf32_fused.cu) is opt-in (CD_RF32=1): measured on
// configs[3] it runs 5.9 ms against the layered schedule's 3.67 ms -- it is bound by DRAM / L2
// capacity (148-296 sweeps in flight re-read 8-9 MB each; L2 hit rate 50 %) and by the serial
// latency of each matrix's panel chain.
static bool g_no_rf32 = getenv("CD_RF32") == nullptr || getenv("CD_NO_RF32") != nullptr;
static double rev_nominal(double n) { return (4 * n * n * n + 3 * n * n + 11 * n) / 6; }
static double fwd_nominal(double n) { return (4 * n * n * n + 3 * n * n + 5 * n) / 6; }
// shape test of the fused fp32 batched route (pointers checked separately)
static bool rf32_shape(const Call& k) {
  return !g_no_rf32 && k.dt == CD_F32 && (k.op == CD_OP_REV || k.op == CD_OP_FWD) && k.batch >= 2 && k.n > 128 &&
         k.n <= 512 && k.n % 64 == 0 && k.o.route != CD_ROUTE_SYMBOLIC && (k.o.nb == 0 || k.o.nb == 64) &&
         !k.L.arr && !k.A.arr && !g_tma_disabled && !g_tc32_disabled;
}
static RF32Call rf32_call(const Call& k) {
  RF32Call rc;
  memset(&rc, 0, sizeof(rc));
  rc.mode = k.op == CD_OP_REV ? 1 : 2;
  rc.n = int(k.n);
  rc.batch = k.batch;
  rc.L = static_cast<const float*>(k.L.base) + k.L.off;
  rc.ldl = k.L.ld;
  rc.sL = k.L.stride;
  float* a = const_cast<float*>(static_cast<const float*>(k.A.base)) + k.A.off;
  if (k.op == CD_OP_REV) {
    rc.Ab = a;
    rc.lda = k.A.ld;
    rc.sA = k.A.stride;
  } else {
    rc.Ad = a;
    rc.ldd = k.A.ld;
    rc.sD = k.A.stride;
  }
  return rc;
}
template <typename T>
static void drive_layered(Ctx& c, const Call& k);

template <typename T>
static void drive_one(Ctx& c, const Call& k) {
  const int n = int(k.n);
  if (n == 0 || k.batch == 0) return;
  if (k.op == CD_OP_CHOL_FWD) {  // fused factorisation + forward (fp64; checked with the arguments)
    if constexpr (sizeof(T) == 8) {
      const Opnd Aop = k.L;  // tril(Sigma) in, L out (the call's first matrix, written)
      const int nb = 128;
      if (n <= DC_NMAX) {  // one block: factor on chip, then the on-chip forward sweep
        double* Dinv = static_cast<double*>(c.take(sizeof(double) * size_t(k.batch) * n * n));
        if (c.plan || !c.ok()) return;
        if (k.info) c.err = note_cuda(cudaMemsetAsync(k.info, 0, sizeof(int) * size_t(k.batch), c.st));
        const size_t dsm = dmma_cta_smem((n + 7) / 8);
        set_smem(k_chol_diag<double>, dsm);
        c.pre(CD_PROF_SWEEP, double(n) * n * n / 3.0 * double(k.batch));
        k_chol_diag<double><<<dim3(1, unsigned(k.batch)), DC_THREADS, dsm, c.st>>>(n, Aop, Dinv, n, int64_t(n) * n, 0,
                                                                                 k.info);
        c.launched();
        run_sweep_small<double>(c, false, n, k.batch, Aop, k.A, 0, null_opnd(), nullptr);
        return;
      }
      if (g_tma_disabled) {
        c.err = CD_ERR_UNSUPPORTED;
        return;
      }
      const bool direct = !c.plan && (reinterpret_cast<uintptr_t>(static_cast<const double*>(Aop.base) + Aop.off) % 16) == 0 &&
                          (reinterpret_cast<uintptr_t>(static_cast<const double*>(k.A.base) + k.A.off) % 16) == 0 &&
                          Aop.ld % 2 == 0 && k.A.ld % 2 == 0 && !Aop.arr && !k.A.arr &&
                          (k.batch == 1 || (Aop.stride % 2 == 0 && k.A.stride % 2 == 0));
      if (direct) {
        chol_fwd_fused(c, n, nb, k.batch, Aop, k.A, k.info);
        return;
      }
      // odd ld / unaligned / pointer arrays: run on aligned workspace copies (ld even)
      const int64_t ldw = n + (n & 1);
      double* wA = static_cast<double*>(c.take(sizeof(double) * size_t(k.batch) * ldw * n));
      double* wD = static_cast<double*>(c.take(sizeof(double) * size_t(k.batch) * ldw * n));
      const Opnd OA = ws_opnd(wA, ldw * n, ldw), OD = ws_opnd(wD, ldw * n, ldw);
      if (!c.plan && c.ok()) {  // lower triangles in
        c.pre(CD_PROF_OTHER, 0.0);
        k_copy_tril<double><<<grid_1d(int64_t(n) * n * k.batch, 256, c.sms), 256, 0, c.st>>>(n, k.batch, Aop, OA);
        c.launched();
        c.pre(CD_PROF_OTHER, 0.0);
        k_copy_tril<double><<<grid_1d(int64_t(n) * n * k.batch, 256, c.sms), 256, 0, c.st>>>(n, k.batch, k.A, OD);
        c.launched();
      }
      chol_fwd_fused(c, n, nb, k.batch, OA, OD, k.info);
      if (!c.plan && c.ok()) {  // lower triangles back
        c.pre(CD_PROF_OTHER, 0.0);
        k_copy_tril<double><<<grid_1d(int64_t(n) * n * k.batch, 256, c.sms), 256, 0, c.st>>>(n, k.batch, OA, Aop);
        c.launched();
        c.pre(CD_PROF_OTHER, 0.0);
        k_copy_tril<double><<<grid_1d(int64_t(n) * n * k.batch, 256, c.sms), 256, 0, c.st>>>(n, k.batch, OD, k.A);
        c.launched();
      }
    } else {
      c.err = CD_ERR_UNSUPPORTED;
    }
    return;
  }
  // fp32 batches, 128 < n <= 512: the fused per-matrix kernel (rf32_fused.cu).  The plan reserves
  // its workspace as well as the layered schedule's (the size query has no pointers to check)
  if (rf32_shape(k)) {
    const size_t o0 = c.off;
    void* wsf = c.take(rf32_fused_ws(n, k.batch));
    const size_t o_f = c.off;
    if (!c.plan) {
      RF32Call rc = rf32_call(k);
      if (rf32_fused_supported(rc)) {
        if (!c.ok()) return;
        if (k.info) {
          c.pre(CD_PROF_OTHER, 0.0);
          k_diag_info<float><<<unsigned(k.batch), 256, 0, c.st>>>(n, k.L, k.info);
          c.launched();
        }
        c.pre(CD_PROF_SWEEP, double(k.batch) * (k.op == CD_OP_REV ? rev_nominal(n) : fwd_nominal(n)));
        c.err = note_cuda(rf32_fused_launch(rc, wsf, c.st, c.sms, &g_launches));
        if (g_prof.on && !g_prof.recs.empty()) cudaEventRecord(g_prof.recs.back().b, c.st);
        if (k.op == CD_OP_REV && k.o.out_mode != CD_OUT_TRIL && c.ok()) {
          c.pre(CD_PROF_OTHER, 0.0);
          k_out_mode<float><<<grid_1d(int64_t(n) * n * k.batch, 256, c.sms), 256, 0, c.st>>>(n, k.batch, k.A,
                                                                                            k.o.out_mode);
          c.launched();
        }
        return;
      }
    }
    c.off = o0;  // the layered schedule below (run when the pointers do not qualify)
    drive_layered<T>(c, k);
    c.off = std::max(c.off, o_f);
    return;
  }
  drive_layered<T>(c, k);
}

template <typename T>
static void drive_layered(Ctx& c, const Call& k) {
  const int n = int(k.n);
  if (k.o.route == CD_ROUTE_SYMBOLIC && n > SYM_NMAX) {
    double* part = static_cast<double*>(c.take(sizeof(double) * size_t(PART_TILES) * G_BM * G_BN));
    if constexpr (sizeof(T) == 8) {
      symbolic_large<double>(c, n, k.batch, k.op == CD_OP_REV, k.L, k.A, k.o.out_mode, part);
    } else {
      // fp32: four chained tf32 products would miss the 1e-4 gate -- run the route in fp64
      // on converted copies (it is offered for measurement, not speed)
      const int64_t nn = int64_t(n) * n;
      double* L64 = static_cast<double*>(c.take(sizeof(double) * size_t(k.batch) * nn));
      double* A64 = static_cast<double*>(c.take(sizeof(double) * size_t(k.batch) * nn));
      const Opnd OL = ws_opnd(L64, nn, n), OA = ws_opnd(A64, nn, n);
      if (!c.plan && c.ok()) {
        c.pre(CD_PROF_OTHER, 0.0);
        k_convert_tril<float, double><<<grid_1d(nn * k.batch, 256, c.sms), 256, 0, c.st>>>(n, k.batch, k.L, OL);
        c.launched();
        c.pre(CD_PROF_OTHER, 0.0);
        k_convert_tril<float, double><<<grid_1d(nn * k.batch, 256, c.sms), 256, 0, c.st>>>(n, k.batch, k.A, OA);
        c.launched();
      }
      symbolic_large<double>(c, n, k.batch, k.op == CD_OP_REV, OL, OA, CD_OUT_TRIL, part);
      if (!c.plan && c.ok()) {
        c.pre(CD_PROF_OTHER, 0.0);
        k_convert_tril<double, float><<<grid_1d(nn * k.batch, 256, c.sms), 256, 0, c.st>>>(n, k.batch, OA, k.A);
        c.launched();
        if (k.op == CD_OP_REV && k.o.out_mode != CD_OUT_TRIL) {
          c.pre(CD_PROF_OTHER, 0.0);
          k_out_mode<float><<<grid_1d(nn * k.batch, 256, c.sms), 256, 0, c.st>>>(n, k.batch, k.A, k.o.out_mode);
          c.launched();
        }
      }
    }
    return;
  }
  if (k.o.route == CD_ROUTE_SYMBOLIC) {  // n <= SYM_NMAX: one CTA per matrix
    if (c.plan || !c.ok()) return;
    const int nblk = (n + 7) / 8;
    const size_t smem = symbolic_smem(nblk);
    set_smem(k_symbolic_cta<T>, smem);
    c.pre(CD_PROF_SWEEP, 0.0);
    k_symbolic_cta<T><<<unsigned(k.batch), DC_THREADS, smem, c.st>>>(n, k.op == CD_OP_REV ? 1 : 0, k.L, k.A,
                                                                   k.o.out_mode, k.info);
    c.launched();
    return;
  }
  if (n <= DC_NMAX) {
    run_sweep_small<T>(c, k.op == CD_OP_REV, n, k.batch, k.L, k.A, k.o.out_mode, null_opnd(), k.info);
    return;
  }
  const int nb = std::min(n, k.o.nb > 0 ? k.o.nb : default_nb(k.dt, n, k.batch, k.L.arr || k.A.arr));
  if (nb > DC_NMAX) {  // diagonal blocks must fit the on-chip sweep / inverse kernels
    c.err = CD_ERR_UNSUPPORTED;
    return;
  }
  T* part = static_cast<T*>(c.take(sizeof(T) * size_t(PART_TILES) * G_BM * G_BN));
  if (k.op == CD_OP_REV) {
    // left-looking schedule (fp64, nb = 128, TMA-describable operands); the plan sizes the
    // workspace for both schedules because the size query does not see the pointers / ld
    const bool ll_shape = k.dt == CD_F64 && nb == LL_BM && !g_no_ll && !g_tma_disabled && !k.L.arr && !k.A.arr;
    const bool ll = ll_shape && (c.plan || ((reinterpret_cast<uintptr_t>(static_cast<const double*>(k.A.base) + k.A.off) % 16) == 0 &&
                                            (reinterpret_cast<uintptr_t>(static_cast<const double*>(k.L.base) + k.L.off) % 16) == 0 &&
                                            k.A.ld % 2 == 0 && k.L.ld % 2 == 0 &&
                                            (k.batch == 1 || (k.A.stride % 2 == 0 && k.L.stride % 2 == 0))));
    // fp32 left-looking schedule (single matrices: batches keep the right-looking sweep, whose
    // nb = 64 diagonal blocks are cheaper -- DESIGN.md §9)
    const bool ll32_shape = k.dt == CD_F32 && nb == 128 && k.batch == 1 && n >= 1024 && !g_no_ll32 &&
                            !g_tma_disabled && !g_tc32_disabled && !k.L.arr && !k.A.arr;
    const bool ll32 = ll32_shape && (c.plan || ((reinterpret_cast<uintptr_t>(static_cast<const float*>(k.A.base) + k.A.off) % 16) == 0 &&
                                                (reinterpret_cast<uintptr_t>(static_cast<const float*>(k.L.base) + k.L.off) % 16) == 0 &&
                                                k.A.ld % 4 == 0 && k.L.ld % 4 == 0));
    const size_t o0 = c.off;
    size_t o_ll = o0;
    if (ll) {
      blocked_rev_ll(c, n, nb, k.batch, k.L, k.A, k.info, reinterpret_cast<double*>(part));
      o_ll = c.off;
      c.off = o0;
    } else if (ll32) {
      blocked_rev_ll32(c, n, nb, k.batch, k.L, k.A, k.info, reinterpret_cast<float*>(part));
      o_ll = c.off;
      c.off = o0;
    }
    if (!(ll || ll32) || c.plan) {
      // lookahead schedule needs a one-tile-wide block (in-place panel solve) and library streams
      T* part2 = static_cast<T*>(c.take(sizeof(T) * size_t(PART_TILES) * G_BM * G_BN));
      // (batches already fill the GPU: the lookahead's extra launches only cost there)
      LaStreams* ls = (!g_no_lookahead && nb <= G_BN && k.batch == 1)
                          ? (c.plan ? reinterpret_cast<LaStreams*>(1) : la_streams())
                          : nullptr;
      if (ls) blocked_rev_la<T>(c, ls, n, nb, k.batch, k.L, k.A, k.info, part, part2);
      else blocked_rev<T>(c, n, nb, k.batch, k.L, k.A, k.info, part);
    }
    c.off = std::max(c.off, o_ll);
  } else {
    // fused-panel forward schedule (fp64, nb = 128, TMA-describable operands); the plan sizes
    // the workspace for both schedules (see above)
    const bool fl_shape = k.dt == CD_F64 && nb == LL_BM && !g_no_ll && !g_tma_disabled && !k.L.arr && !k.A.arr;
    const bool fl = fl_shape && (c.plan || ((reinterpret_cast<uintptr_t>(static_cast<const double*>(k.A.base) + k.A.off) % 16) == 0 &&
                                            (reinterpret_cast<uintptr_t>(static_cast<const double*>(k.L.base) + k.L.off) % 16) == 0 &&
                                            k.A.ld % 2 == 0 && k.L.ld % 2 == 0 &&
                                            (k.batch == 1 || (k.A.stride % 2 == 0 && k.L.stride % 2 == 0))));
    const size_t o0 = c.off;
    size_t o_fl = o0;
    if (fl) {
      blocked_fwd_ll(c, n, nb, k.batch, k.L, k.A, k.info);
      o_fl = c.off;
      c.off = o0;
    }
    if (!fl || c.plan) blocked_fwd<T>(c, n, nb, k.batch, k.L, k.A, k.info, part);
    c.off = std::max(c.off, o_fl);
  }
  if (k.op == CD_OP_REV && k.o.out_mode != CD_OUT_TRIL && !c.plan && c.ok()) {
    c.pre(CD_PROF_OTHER, 0.0);
    k_out_mode<T><<<grid_1d(int64_t(n) * n * k.batch, 256, c.sms), 256, 0, c.st>>>(n, k.batch, k.A, k.o.out_mode);
    c.launched();
  }
}

static std::atomic<int> g_sm_count[kMaxDev];
// Paths whose kernels put the matrix index on gridDim.y / .z (the blocked sweeps' GEMMs and
// inverses, the fused factorisation's diagonal kernel) run batches above the 65535 grid limit in
// chunks of kGridBatch matrices, reusing one chunk's workspace; the n <= DC_NMAX on-chip paths
// index matrices by gridDim.x and take any batch in one launch.
static Opnd shift_batch(const Opnd& o, int64_t b0, size_t es) {
  Opnd r = o;
  if (r.arr) r.arr += b0;
  else r.base = static_cast<const char*>(r.base) + size_t(b0) * size_t(r.stride) * es;
  return r;
}

template <typename T>
static void drive(Ctx& c, const Call& k) {
  const bool grid2d = k.op == CD_OP_CHOL_FWD || k.n > DC_NMAX;
  if (k.batch <= 65535 || !grid2d) {
    drive_one<T>(c, k);
    return;
  }
  const size_t o0 = c.off;
  size_t hi = o0;
  for (int64_t b0 = 0; b0 < k.batch && c.ok(); b0 += kGridBatch) {
    Call s = k;
    s.batch = std::min<int64_t>(kGridBatch, k.batch - b0);
    s.L = shift_batch(k.L, b0, sizeof(T));
    s.A = shift_batch(k.A, b0, sizeof(T));
    s.info = k.info ? k.info + b0 : nullptr;
    c.off = o0;
    drive_one<T>(c, s);
    hi = std::max(hi, c.off);
    if (c.plan) break;  // the first chunk is the largest: it sizes the workspace
  }
  c.off = hi;
}

static int sm_count() {
  return per_device(g_sm_count, [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      v = 148;
    return v;
  });
}

// ------------------------------------------------------------------ distributed reverse steps
// (include/choldiff.h describes the distribution.)  The same arithmetic as
// one step of blocked_rev, split at the broadcast: the panel on the column owner, the
// rank-w updates of the columns left of the panel on every rank.
template <typename T>
static void dist_rev_panel(Ctx& c, int n, int j, int w, Opnd Lk, Opnd Ak, Opnd X) {
  const int k = j + w, p = n - k;
  T* Dinv = static_cast<T*>(c.take(sizeof(T) * size_t(w) * w));
  T* part = static_cast<T*>(c.take(sizeof(T) * size_t(PART_TILES) * G_BM * G_BN));
  run_trinv<T>(c, w, w, true, 1, sub(Lk, j, 0), Dinv);
  const Opnd Cbar = sub(Ak, k, 0);
  if (p > 0) {
    // Cbar <- Cbar D^{-1} (in place: one 128-wide N tile covers the block)
    Gemm<T>(c, p, w, 0, 0, 1)
        .seg(Cbar, ws_opnd(Dinv, 0, w), w)
        .flops(double(p) * w * (w + 1))
        .run(null_opnd(), Cbar, 1.0, 0.0, 0, part);
    // Dbar <- Dbar - tril(Cbar^T C)
    Gemm<T>(c, w, w, 1, 0, 1)
        .seg(Cbar, sub(Lk, k, 0), p)
        .flops(double(w) * (w + 1) * p)
        .run(sub(Ak, j, 0), sub(Ak, j, 0), -1.0, 1.0, 1, part);
  }
  // Dbar <- chol_unblocked_rev(D, Dbar), S = Dbar + Dbar^T into the top of X
  run_sweep_small<T>(c, true, w, 1, sub(Lk, j, 0), sub(Ak, j, 0), 0, X, nullptr);
  if (p > 0) run_copy<T>(c, p, w, 1, Cbar, sub(X, w, 0));
}

template <typename T>
static void dist_rev_update(Ctx& c, int n, int j, int w, Opnd X, int q, Opnd Lq, Opnd Aq) {
  const int k = j + w, p = n - k;
  T* part = static_cast<T*>(c.take(sizeof(T) * size_t(PART_TILES) * G_BM * G_BN));
  if (q <= 0) return;
  // Bbar <- Bbar - Cbar R
  if (p > 0)
    Gemm<T>(c, p, q, 0, 0, 1).seg(sub(X, w, 0), sub(Lq, j, 0), w).run(sub(Aq, k, 0), sub(Aq, k, 0), -1.0, 1.0, 0, part);
  // Rbar <- Rbar - [S; Cbar]^T [R; B]
  Gemm<T>(c, w, q, 1, 0, 1).seg(X, sub(Lq, j, 0), n - j).run(sub(Aq, j, 0), sub(Aq, j, 0), -1.0, 1.0, 0, part);
}

// Forward, block [j, k) on its owner; Z = the sum over all ranks of
// [Adot[j:n, cols] L[j:n, cols]] [L[j:k, cols] Adot[j:k, cols]]^T for their columns left of the
// block, i.e. [Rdot R^T + R Rdot^T ; Bdot R^T + B Rdot^T].
template <typename T>
static void dist_fwd_partial(Ctx& c, int n, int j, int w, int q, Opnd Lq, Opnd Aq, Opnd Z) {
  T* part = static_cast<T*>(c.take(sizeof(T) * size_t(PART_TILES) * G_BM * G_BN));
  if (c.plan || !c.ok()) return;
  if (q == 0) {  // no columns left of the block on this rank: a zero contribution
    c.err = note_cuda(cudaMemsetAsync(const_cast<void*>(Z.base), 0, sizeof(T) * size_t(n - j) * w, c.st));  // ldz = n - j
    return;
  }
  Gemm<T>(c, n - j, w, 0, 1, 1)
      .seg(sub(Aq, j, 0), sub(Lq, j, 0), q)
      .seg(sub(Lq, j, 0), sub(Aq, j, 0), q)
      .run(null_opnd(), Z, 1.0, 0.0, 0, part);
}

template <typename T>
static void dist_fwd_panel(Ctx& c, int n, int j, int w, Opnd Lk, Opnd Ak, Opnd Z) {
  const int k = j + w, p = n - k;
  T* Dinv = static_cast<T*>(c.take(sizeof(T) * size_t(w) * w));
  T* Dcw = static_cast<T*>(c.take(sizeof(T) * size_t(w) * w));
  T* part = static_cast<T*>(c.take(sizeof(T) * size_t(PART_TILES) * G_BM * G_BN));
  run_trinv<T>(c, w, w, false, 1, sub(Lk, j, 0), Dinv);
  if (!c.plan && c.ok()) {
    // Ddot <- Ddot - tril(Rdot R^T + R Rdot^T);  Cdot <- Cdot - Bdot R^T - B Rdot^T
    c.pre(CD_PROF_OTHER, 0.0);
    k_sub<T><<<grid_1d(int64_t(w) * w, 256, c.sms), 256, 0, c.st>>>(w, w, Z, sub(Ak, j, 0), 1);
    c.launched();
    if (p > 0) {
      c.pre(CD_PROF_OTHER, 0.0);
      k_sub<T><<<grid_1d(int64_t(p) * w, 256, c.sms), 256, 0, c.st>>>(p, w, sub(Z, w, 0), sub(Ak, k, 0), 0);
      c.launched();
    }
  }
  const Opnd Dc = ws_opnd(Dcw, 0, w);
  // Ddot <- chol_unblocked_fwd(D, Ddot) (+ the clean copy Dc = tril(Ddot))
  run_sweep_small<T>(c, false, w, 1, sub(Lk, j, 0), sub(Ak, j, 0), 0, p > 0 ? Dc : null_opnd(), nullptr);
  if (p > 0) {
    // Cdot <- (Cdot - C Ddot^T) D^{-T}
    const Opnd Cd = sub(Ak, k, 0);
    Gemm<T>(c, p, w, 0, 1, 1).seg(sub(Lk, k, 0), Dc, w).run(Cd, Cd, -1.0, 1.0, 0, part);
    Gemm<T>(c, p, w, 0, 1, 1)
        .seg(Cd, ws_opnd(Dinv, 0, w), w)
        .flops(double(p) * w * (w + 1))
        .run(null_opnd(), Cd, 1.0, 0.0, 0, part);
  }
}

template <typename F>
static int run_steps(cd_dtype dt, void* ws, size_t ws_bytes, cudaStream_t st, int ws_arg, F&& body) {
  Ctx pc;
  pc.plan = true;
  pc.ws = nullptr;
  pc.st = nullptr;
  pc.sms = sm_count();
  if (dt == CD_F64) body(pc, double(0));
  else body(pc, float(0));
  if (pc.off > 0 && (ws == nullptr || ws_bytes < pc.off)) return -ws_arg;
  Ctx c;
  c.plan = false;
  c.ws = static_cast<char*>(ws);
  c.st = st;
  c.sms = sm_count();
  if (dt == CD_F64) body(c, double(0));
  else body(c, float(0));
  return c.err;
}

static size_t plan_size(const Call& k) {
  Ctx c;
  c.plan = true;
  c.ws = nullptr;
  c.st = nullptr;
  c.sms = sm_count();
  if (k.dt == CD_F64) drive<double>(c, k);
  else drive<float>(c, k);
  return c.off;
}

static int execute(const Call& k, void* ws, size_t ws_bytes, cudaStream_t st, int ws_arg) {
  const size_t need = plan_size(k);
  if (need > 0 && (ws == nullptr || ws_bytes < need)) return -ws_arg;
  Ctx c;
  c.plan = false;
  c.ws = static_cast<char*>(ws);
  c.st = st;
  c.sms = sm_count();
  if (k.dt == CD_F64) drive<double>(c, k);
  else drive<float>(c, k);
  return c.err;
}

}  // namespace cd

using namespace cd;

// ------------------------------------------------------------------ argument validation
static const cd_opts kDefaultOpts = {0, CD_ROUTE_AUTO, CD_OUT_TRIL, 0};

static int check_common(cd_op op, int dt, int64_t n, int64_t ldl, int64_t lda, const cd_opts* opts, int a_dt,
                        int a_n, int a_ldl, int a_lda, int a_opts) {
  if (dt != CD_F64 && dt != CD_F32) return -a_dt;
  if (n < 0 || n > (int64_t(1) << 30)) return -a_n;
  if (ldl < std::max<int64_t>(1, n)) return -a_ldl;
  if (lda < std::max<int64_t>(1, n)) return -a_lda;
  if (opts) {
    if (opts->nb < 0) return -a_opts;
    if (opts->route < CD_ROUTE_AUTO || opts->route > CD_ROUTE_SYMBOLIC) return -a_opts;
    if (opts->out_mode < CD_OUT_TRIL || opts->out_mode > CD_OUT_GRAD) return -a_opts;
    if (op != CD_OP_REV && opts->out_mode != CD_OUT_TRIL) return -a_opts;
    if (op == CD_OP_CHOL_FWD && (opts->route == CD_ROUTE_SYMBOLIC || (opts->nb != 0 && opts->nb != 128))) return -a_opts;
    if (opts->flags != 0) return -a_opts;
  }
  return 0;
}

static int route_supported(const cd_opts& o, int64_t n) {
  // every route is available at every size: symbolic = k_symbolic_cta (n <= 64) or
  // symbolic_large (blocked triangular solves); AUTO = the algorithmic sweeps
  (void)o;
  (void)n;
  return 0;
}

static int strided(cd_op op, cd_dtype dt, int64_t n, const void* L, int64_t ldl, int64_t sL, void* A, int64_t lda,
                   int64_t sA, int64_t batch, const cd_opts* opts, void* ws, size_t ws_bytes, int* d_info,
                   cd_stream_t stream, bool single) {
  // argument positions (1-based) in the strided signature / single signature
  const int pDt = 1, pN = 2, pL = 3, pLdl = 4;
  const int pSL = single ? 0 : 5, pA = single ? 5 : 6, pLda = single ? 6 : 7, pSA = single ? 0 : 8;
  const int pB = single ? 0 : 9, pOpts = single ? 7 : 10, pWs = single ? 8 : 11;
  int r = check_common(op, dt, n, ldl, lda, opts, pDt, pN, pLdl, pLda, pOpts);
  if (r) return r;
  if (batch < 0) return -pB;
  if (n == 0 || batch == 0) return CD_SUCCESS;
  if (!L) return -pL;
  if (!A) return -pA;
  if (batch > 1 && sL < ldl * n) return -pSL;
  if (batch > 1 && sA < lda * n) return -pSA;
  const cd_opts o = opts ? *opts : kDefaultOpts;
  if ((r = route_supported(o, n))) return r;
  Call k{op, dt, n, batch, Opnd{L, nullptr, sL, ldl, 0}, Opnd{A, nullptr, sA, lda, 0}, o, d_info};
  return execute(k, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), pWs);
}

extern "C" {

int cd_chol_rev(cd_dtype dt, int64_t n, const void* L, int64_t ldl, void* Abar, int64_t ldabar, const cd_opts* opts,
                void* ws, size_t ws_bytes, int* d_info, cd_stream_t stream) {
  return strided(CD_OP_REV, dt, n, L, ldl, 0, Abar, ldabar, 0, 1, opts, ws, ws_bytes, d_info, stream, true);
}

int cd_chol_fwd(cd_dtype dt, int64_t n, const void* L, int64_t ldl, void* Adot, int64_t ldadot, const cd_opts* opts,
                void* ws, size_t ws_bytes, int* d_info, cd_stream_t stream) {
  return strided(CD_OP_FWD, dt, n, L, ldl, 0, Adot, ldadot, 0, 1, opts, ws, ws_bytes, d_info, stream, true);
}

int cd_chol_rev_strided_batched(cd_dtype dt, int64_t n, const void* L, int64_t ldl, int64_t strideL, void* Abar,
                                int64_t ldabar, int64_t strideAbar, int64_t batch, const cd_opts* opts, void* ws,
                                size_t ws_bytes, int* d_info, cd_stream_t stream) {
  return strided(CD_OP_REV, dt, n, L, ldl, strideL, Abar, ldabar, strideAbar, batch, opts, ws, ws_bytes, d_info,
                 stream, false);
}

int cd_chol_fwd_strided_batched(cd_dtype dt, int64_t n, const void* L, int64_t ldl, int64_t strideL, void* Adot,
                                int64_t ldadot, int64_t strideAdot, int64_t batch, const cd_opts* opts, void* ws,
                                size_t ws_bytes, int* d_info, cd_stream_t stream) {
  return strided(CD_OP_FWD, dt, n, L, ldl, strideL, Adot, ldadot, strideAdot, batch, opts, ws, ws_bytes, d_info,
                 stream, false);
}

static int ptr_batched(cd_op op, cd_dtype dt, int64_t n, const void* const* La, int64_t ldl, void* const* Aa,
                       int64_t lda, int64_t batch, const cd_opts* opts, void* ws, size_t ws_bytes, int* d_info,
                       cd_stream_t stream) {
  int r = check_common(op, dt, n, ldl, lda, opts, 1, 2, 4, 6, 8);
  if (r) return r;
  if (batch < 0) return -7;
  if (n == 0 || batch == 0) return CD_SUCCESS;
  if (!La) return -3;
  if (!Aa) return -5;
  const cd_opts o = opts ? *opts : kDefaultOpts;
  if ((r = route_supported(o, n))) return r;
  Call k{op, dt, n, batch, Opnd{nullptr, La, 0, ldl, 0},
         Opnd{nullptr, reinterpret_cast<const void* const*>(Aa), 0, lda, 0}, o, d_info};
  return execute(k, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), 9);
}

int cd_chol_rev_batched(cd_dtype dt, int64_t n, const void* const* L_array, int64_t ldl, void* const* Abar_array,
                        int64_t ldabar, int64_t batch, const cd_opts* opts, void* ws, size_t ws_bytes, int* d_info,
                        cd_stream_t stream) {
  return ptr_batched(CD_OP_REV, dt, n, L_array, ldl, Abar_array, ldabar, batch, opts, ws, ws_bytes, d_info, stream);
}

int cd_chol_fwd_batched(cd_dtype dt, int64_t n, const void* const* L_array, int64_t ldl, void* const* Adot_array,
                        int64_t ldadot, int64_t batch, const cd_opts* opts, void* ws, size_t ws_bytes, int* d_info,
                        cd_stream_t stream) {
  return ptr_batched(CD_OP_FWD, dt, n, L_array, ldl, Adot_array, ldadot, batch, opts, ws, ws_bytes, d_info, stream);
}

int cd_chol_fwd_fused(cd_dtype dt, int64_t n, void* A, int64_t lda, void* Adot, int64_t ldadot, const cd_opts* opts,
                      void* ws, size_t ws_bytes, int* d_info, cd_stream_t stream) {
  if (dt != CD_F64 && dt != CD_F32) return -1;
  if (dt == CD_F32) return CD_ERR_UNSUPPORTED;
  return strided(CD_OP_CHOL_FWD, dt, n, A, lda, 0, Adot, ldadot, 0, 1, opts, ws, ws_bytes, d_info, stream, true);
}

int cd_chol_fwd_fused_strided_batched(cd_dtype dt, int64_t n, void* A, int64_t lda, int64_t strideA, void* Adot,
                                      int64_t ldadot, int64_t strideAdot, int64_t batch, const cd_opts* opts, void* ws,
                                      size_t ws_bytes, int* d_info, cd_stream_t stream) {
  if (dt != CD_F64 && dt != CD_F32) return -1;
  if (dt == CD_F32) return CD_ERR_UNSUPPORTED;
  return strided(CD_OP_CHOL_FWD, dt, n, A, lda, strideA, Adot, ldadot, strideAdot, batch, opts, ws, ws_bytes, d_info,
                 stream, false);
}

// ---- both sweeps of one factor on two streams (cd_chol_rev_fwd_strided_batched) ----
struct SideStream {  // per device and host thread; released at thread exit
  cudaStream_t s = nullptr;
  cudaStream_t s2 = nullptr;  // the 128-wide inverses' completion (rf32_inv128) beside both sweeps
  std::vector<cudaEvent_t> ev;
  ~SideStream() {
    if (s) cudaStreamDestroy(s);
    if (s2) cudaStreamDestroy(s2);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
};
static thread_local SideStream g_side[64];

// the batched fp32 right-looking drivers share one set of diagonal-block inverses (configs[3])
static int shared_dinv_nb(cd_dtype dt, int64_t n, int64_t batch, const cd_opts& o) {
  const int nb = int(std::min<int64_t>(n, o.nb > 0 ? o.nb : default_nb(dt, n, batch, false)));
  const bool ok = dt == CD_F32 && batch > 1 && batch <= kGridBatch && n > DC_NMAX && nb <= DC_NMAX &&
                  n % nb == 0 && o.route != CD_ROUTE_SYMBOLIC;
  return ok ? nb : 0;
}

// both sweeps in the fused fp32 kernel (configs[3]); shape test as rf32_shape
static bool rf32_rev_fwd_shape(cd_dtype dt, int64_t n, int64_t batch, const cd_opts& o) {
  Call k{CD_OP_REV, dt, n, batch, null_opnd(), null_opnd(), o, nullptr};
  return rf32_shape(k) && o.out_mode == CD_OUT_TRIL;
}

static size_t rev_fwd_ws(cd_dtype dt, int64_t n, int64_t batch, const cd_opts& o, size_t* ws_rev, size_t* ws_dinv) {
  Call kr{CD_OP_REV, dt, n, batch, null_opnd(), null_opnd(), o, nullptr};
  kr.L.ld = kr.A.ld = n;
  Call kf = kr;
  kf.op = CD_OP_FWD;
  kf.o.out_mode = CD_OUT_TRIL;
  const size_t a = (plan_size(kr) + 255) & ~size_t(255);
  const size_t f = (plan_size(kf) + 255) & ~size_t(255);
  if (ws_rev) *ws_rev = a;
  if (ws_dinv) *ws_dinv = a + f;
  const int nb = shared_dinv_nb(dt, n, batch, o);
  const size_t es = dt == CD_F64 ? 8 : 4;
  const size_t layered = a + f + (nb ? size_t(batch) * (n / nb) * nb * nb * es : 0);
  return rf32_rev_fwd_shape(dt, n, batch, o) ? std::max(layered, rf32_fused_ws(int(n), batch)) : layered;
}

size_t cd_workspace_size(cd_op op, cd_dtype dt, int64_t n, int64_t batch, const cd_opts* opts) {
  if ((dt != CD_F64 && dt != CD_F32) || n <= 0 || batch <= 0) return 0;
  const cd_opts o = opts ? *opts : kDefaultOpts;
  Call k{op, dt, n, batch, null_opnd(), null_opnd(), o, nullptr};
  k.L.ld = k.A.ld = n;
  size_t need = plan_size(k);
  if (dt == CD_F32 && o.nb == 0) {  // pointer-array batches take nb = 64 (default_nb)
    Call k64 = k;
    k64.o.nb = 64;
    need = std::max(need, plan_size(k64));
  }
  return need;
}

size_t cd_workspace_size_rev_fwd(cd_dtype dt, int64_t n, int64_t batch, const cd_opts* opts) {
  if ((dt != CD_F64 && dt != CD_F32) || n <= 0 || batch <= 0) return 0;
  const cd_opts o = opts ? *opts : kDefaultOpts;
  return rev_fwd_ws(dt, n, batch, o, nullptr, nullptr);
}

int cd_chol_rev_fwd_strided_batched(cd_dtype dt, int64_t n, const void* L, int64_t ldl, int64_t strideL, void* Abar,
                                    int64_t ldabar, int64_t strideAbar, void* Adot, int64_t ldadot,
                                    int64_t strideAdot, int64_t batch, const cd_opts* opts, void* ws,
                                    size_t ws_bytes, int* d_info, cd_stream_t stream) {
  int r = check_common(CD_OP_REV, dt, n, ldl, ldabar, opts, 1, 2, 4, 7, 13);
  if (r) return r;
  if (ldadot < std::max<int64_t>(1, n)) return -10;
  if (batch < 0) return -12;
  if (n == 0 || batch == 0) return CD_SUCCESS;
  if (!L) return -3;
  if (!Abar) return -6;
  if (!Adot) return -9;
  if (batch > 1 && (strideL < ldl * n)) return -5;
  if (batch > 1 && (strideAbar < ldabar * n)) return -8;
  if (batch > 1 && (strideAdot < ldadot * n)) return -11;
  const cd_opts o = opts ? *opts : kDefaultOpts;
  size_t ws_rev = 0, ws_dinv = 0;
  const size_t need = rev_fwd_ws(dt, n, batch, o, &ws_rev, &ws_dinv);
  if (need > 0 && (!ws || ws_bytes < need)) return -14;
  if (rf32_rev_fwd_shape(dt, n, batch, o)) {
    // both sweeps of every matrix in one fused kernel (rf32_fused.cu): one CTA per (matrix,
    // sweep), the two sweeps of a matrix on neighbouring CTAs so that L is fetched once
    RF32Call rc{3, int(n), batch, static_cast<const float*>(L), ldl, strideL, static_cast<float*>(Abar), ldabar,
                strideAbar, static_cast<float*>(Adot), ldadot, strideAdot};
    if (rf32_fused_supported(rc)) {
      cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
      if (d_info) {
        k_diag_info<float><<<unsigned(batch), 256, 0, st>>>(int(n), Opnd{L, nullptr, strideL, ldl, 0}, d_info);
        ++g_launches;
        if ((r = note_cuda(cudaGetLastError()))) return r;
      }
      return note_cuda(rf32_fused_launch(rc, ws, st, sm_count(), &g_launches));
    }
  }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return CD_ERR_CUDA;
  if (!g_side[dev].s && (r = note_cuda(cudaStreamCreateWithFlags(&g_side[dev].s, cudaStreamNonBlocking)))) return r;
  std::vector<cudaEvent_t>& evs = g_side[dev].ev;
  if (evs.empty()) {
    evs.resize(4);
    for (auto& e : evs)
      if ((r = note_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)))) return r;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream), side = g_side[dev].s;
  const int snb = shared_dinv_nb(dt, n, batch, o);
  const Opnd Lop{L, nullptr, strideL, ldl, 0};
  const bool split_inv = snb && dt == CD_F32 && diag128_route(int(n), snb, Lop) && g_old_inv128;
  if (split_inv && !g_side[dev].s2 && (r = note_cuda(cudaStreamCreateWithFlags(&g_side[dev].s2, cudaStreamNonBlocking))))
    return r;
  struct ExtReset {  // the shared-inverse hand-over is scoped to this call, error returns included
    ~ExtReset() {
      g_ext_dinv = nullptr;
      g_ext_dinv_nb = 0;
      g_dinv_wait = nullptr;
    }
  } ext_reset;
  if (snb) {  // the inverses of the shared factor, once, before the two sweeps fork
    Ctx c;
    c.plan = false;
    c.ws = nullptr;
    c.st = st;
    c.sms = sm_count();
    float* Dinv = reinterpret_cast<float*>(static_cast<char*>(ws) + ws_dinv);
    run_trinv<float>(c, int(n), snb, false, batch, Lop, Dinv, !split_inv);
    if (c.err) return c.err;
    if (split_inv) {  // the 128-wide completion on s2, awaited by the sweeps' first D^{-1} GEMMs
      if ((r = note_cuda(cudaEventRecord(evs[2], st)))) return r;
      if ((r = note_cuda(cudaStreamWaitEvent(g_side[dev].s2, evs[2], 0)))) return r;
      Ctx c2 = c;
      c2.st = g_side[dev].s2;
      c2.pre(CD_PROF_TRINV, 0.0);
      c2.err = note_cuda(rf32_inv128(int(n), batch, static_cast<const float*>(L), ldl, strideL, Dinv, c2.st));
      ++g_launches;
      if (g_prof.on && !g_prof.recs.empty()) cudaEventRecord(g_prof.recs.back().b, c2.st);
      if (c2.err) return c2.err;
      if ((r = note_cuda(cudaEventRecord(evs[3], g_side[dev].s2)))) return r;
      g_dinv_wait = evs[3];
    }
    g_ext_dinv = Dinv;
    g_ext_dinv_nb = snb;
  }
  // the side stream starts after the work already queued on `stream`, and `stream` ends after it
  if ((r = note_cuda(cudaEventRecord(evs[0], st)))) return r;
  if ((r = note_cuda(cudaStreamWaitEvent(side, evs[0], 0)))) return r;
  Call kr{CD_OP_REV, dt, n, batch, Opnd{L, nullptr, strideL, ldl, 0}, Opnd{Abar, nullptr, strideAbar, ldabar, 0}, o,
          d_info};
  Call kf{CD_OP_FWD, dt, n, batch, Opnd{L, nullptr, strideL, ldl, 0}, Opnd{Adot, nullptr, strideAdot, ldadot, 0}, o,
          nullptr};
  kf.o.out_mode = CD_OUT_TRIL;
  r = execute(kr, ws, ws_rev, st, 14);
  const int rf = execute(kf, static_cast<char*>(ws) + ws_rev, ws_dinv - ws_rev, side, 14);
  g_ext_dinv = nullptr;
  g_ext_dinv_nb = 0;
  g_dinv_wait = nullptr;
  const int rj = note_cuda(cudaEventRecord(evs[1], side));
  const int rw = rj ? rj : note_cuda(cudaStreamWaitEvent(st, evs[1], 0));
  // (`stream` also ends after s2's combine: the sweeps waited for it)
  return r ? r : (rf ? rf : rw);
}

size_t cd_workspace_size_host(cd_op op, cd_dtype dt, int64_t n, const cd_opts* opts) {
  const size_t es = dt == CD_F64 ? 8 : 4;
  const size_t mat = (size_t(n) * n * es + 255) & ~size_t(255);
  return 2 * mat + cd_workspace_size(op, dt, n, 1, opts);
}

int cd_chol_host(cd_op op, cd_dtype dt, int64_t n, const void* L_host, void* A_host, const cd_opts* opts, void* ws,
                 size_t ws_bytes, cd_stream_t stream) {
  if (op != CD_OP_REV && op != CD_OP_FWD) return -1;
  if (dt != CD_F64 && dt != CD_F32) return -2;
  if (n < 0) return -3;
  if (n == 0) return CD_SUCCESS;
  if (!L_host) return -4;
  if (!A_host) return -5;
  const size_t es = dt == CD_F64 ? 8 : 4;
  const size_t mat = (size_t(n) * n * es + 255) & ~size_t(255);
  const size_t need = cd_workspace_size_host(op, dt, n, opts);
  if (!ws || ws_bytes < need) return -7;
  char* dL = static_cast<char*>(ws);
  char* dA = dL + mat;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const cd_opts o = opts ? *opts : kDefaultOpts;
  // pipelined path: the fused fp64 schedules (nb = 128, TRIL output, even n for TMA) stream
  // column blocks in and out while they run
  if (dt == CD_F64 && (o.nb == 0 || o.nb == 128) && o.out_mode == CD_OUT_TRIL && o.route != CD_ROUTE_SYMBOLIC &&
      n > DC_NMAX && n % 2 == 0 && !g_no_ll && !g_tma_disabled && !g_no_host_pipe) {
    HostStreams* hs = host_streams();
    if (hs) {
      HostPipe& hp = hs->pipe;
      hp.cin = hs->cin;
      hp.cout = hs->cout;
      hp.Lh = static_cast<const char*>(L_host);
      hp.Ah_in = static_cast<const char*>(A_host);
      hp.Ah = static_cast<char*>(A_host);
      hp.dL = dL;
      hp.dA = dA;
      hp.n = n;
      hp.es = es;
      hp.next = 0;
      hp.bytes_in = hp.bytes_out = 0;
      // the copy streams must not start before work already queued on `stream`
      cudaEvent_t e0 = hp.ev();
      cudaEventRecord(e0, st);
      cudaStreamWaitEvent(hp.cin, e0, 0);
      cudaStreamWaitEvent(hp.cout, e0, 0);
      g_pipe = &hp;
      void* ws2 = dA + mat;
      const size_t ws2b = ws_bytes - 2 * mat;
      const int r = (op == CD_OP_REV) ? cd_chol_rev(dt, n, dL, n, dA, n, opts, ws2, ws2b, nullptr, stream)
                                      : cd_chol_fwd(dt, n, dL, n, dA, n, opts, ws2, ws2b, nullptr, stream);
      g_pipe = nullptr;
      cudaEvent_t e1 = hp.ev();  // `stream` completes only after the last copy out
      cudaEventRecord(e1, hp.cout);
      cudaStreamWaitEvent(st, e1, 0);
      g_host_bytes_in = hp.bytes_in;
      g_host_bytes_out = 0;
      for (int64_t j = 0; j < n; j += 128) g_host_bytes_out += (n - j) * std::min<int64_t>(128, n - j) * int64_t(es);
      return r;
    }
  }
  g_host_bytes_in = 2 * n * n * int64_t(es);
  g_host_bytes_out = n * n * int64_t(es);
  int r = note_cuda(cudaMemcpyAsync(dL, L_host, size_t(n) * n * es, cudaMemcpyHostToDevice, st));
  if (r) return r;
  r = note_cuda(cudaMemcpyAsync(dA, A_host, size_t(n) * n * es, cudaMemcpyHostToDevice, st));
  if (r) return r;
  void* ws2 = dA + mat;
  const size_t ws2b = ws_bytes - 2 * mat;
  r = (op == CD_OP_REV) ? cd_chol_rev(dt, n, dL, n, dA, n, opts, ws2, ws2b, nullptr, stream)
                        : cd_chol_fwd(dt, n, dL, n, dA, n, opts, ws2, ws2b, nullptr, stream);
  if (r) return r;
  return note_cuda(cudaMemcpyAsync(A_host, dA, size_t(n) * n * es, cudaMemcpyDeviceToHost, st));
}

int cd_debug_gemm(cd_dtype dt, int64_t M, int64_t N, int64_t K, int ta, int tb, const void* A, int64_t lda,
                  const void* B, int64_t ldb, void* C, int64_t ldc, double alpha, double beta, void* ws, size_t ws_bytes,
                  cd_stream_t stream) {
  if (dt != CD_F64 && dt != CD_F32) return -1;
  if (M < 0 || N < 0 || K < 0) return -2;
  if (ta < 0 || ta > 1 || tb < 0 || tb > 1) return -5;
  const size_t es = dt == CD_F64 ? 8 : 4;
  const size_t need = size_t(PART_TILES) * G_BM * G_BN * es;
  if (!ws || ws_bytes < need) return -16;
  Ctx c;
  c.plan = false;
  c.ws = static_cast<char*>(ws);
  c.st = reinterpret_cast<cudaStream_t>(stream);
  c.sms = sm_count();
  const Opnd Ao{A, nullptr, 0, lda, 0}, Bo{B, nullptr, 0, ldb, 0}, Co{C, nullptr, 0, ldc, 0};
  if (dt == CD_F64)
    Gemm<double>(c, int(M), int(N), ta, tb, 1).seg(Ao, Bo, int(K)).run(Co, Co, alpha, beta, 0, static_cast<double*>(ws));
  else
    Gemm<float>(c, int(M), int(N), ta, tb, 1).seg(Ao, Bo, int(K)).run(Co, Co, alpha, beta, 0, static_cast<float*>(ws));
  return c.err;
}

size_t cd_dist_workspace_size(cd_dtype dt, int64_t w) {
  if ((dt != CD_F64 && dt != CD_F32) || w <= 0) return 0;
  const size_t es = dt == CD_F64 ? 8 : 4;
  return 2 * ((size_t(w) * w * es + 255) / 256 * 256) + size_t(PART_TILES) * G_BM * G_BN * es + 256;
}

int cd_dist_rev_panel(cd_dtype dt, int64_t n, int64_t j, int64_t w, const void* Lk, int64_t ldl, void* Ak,
                      int64_t lda, void* X, int64_t ldx, void* ws, size_t ws_bytes, cd_stream_t stream) {
  if (dt != CD_F64 && dt != CD_F32) return -1;
  if (n < 1 || n > (int64_t(1) << 30)) return -2;
  if (j < 0 || j >= n) return -3;
  if (w < 1 || w > DC_NMAX || j + w > n) return -4;
  if (!Lk) return -5;
  if (ldl < n) return -6;
  if (!Ak) return -7;
  if (lda < n) return -8;
  if (!X) return -9;
  if (ldx < n - j) return -10;
  if (ws_bytes < cd_dist_workspace_size(dt, w)) return -12;
  const Opnd L{Lk, nullptr, 0, ldl, 0}, A{Ak, nullptr, 0, lda, 0}, Xo{X, nullptr, 0, ldx, 0};
  return run_steps(dt, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), 11, [&](Ctx& c, auto zero) {
    dist_rev_panel<decltype(zero)>(c, int(n), int(j), int(w), L, A, Xo);
  });
}

int cd_dist_rev_update(cd_dtype dt, int64_t n, int64_t j, int64_t w, const void* X, int64_t ldx, int64_t q,
                       const void* Lq, int64_t ldl, void* Aq, int64_t lda, void* ws, size_t ws_bytes,
                       cd_stream_t stream) {
  if (dt != CD_F64 && dt != CD_F32) return -1;
  if (n < 1 || n > (int64_t(1) << 30)) return -2;
  if (j < 0 || j >= n) return -3;
  if (w < 1 || w > DC_NMAX || j + w > n) return -4;
  if (!X) return -5;
  if (ldx < n - j) return -6;
  if (q < 0 || q > j) return -7;
  if (q == 0) return CD_SUCCESS;
  if (!Lq) return -8;
  if (ldl < n) return -9;
  if (!Aq) return -10;
  if (lda < n) return -11;
  if (ws_bytes < cd_dist_workspace_size(dt, w)) return -13;
  const Opnd L{Lq, nullptr, 0, ldl, 0}, A{Aq, nullptr, 0, lda, 0}, Xo{const_cast<void*>(X), nullptr, 0, ldx, 0};
  return run_steps(dt, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), 12, [&](Ctx& c, auto zero) {
    dist_rev_update<decltype(zero)>(c, int(n), int(j), int(w), Xo, int(q), L, A);
  });
}

int cd_dist_fwd_partial(cd_dtype dt, int64_t n, int64_t j, int64_t w, int64_t q, const void* Lq, int64_t ldl,
                        const void* Aq, int64_t lda, void* Z, int64_t ldz, void* ws, size_t ws_bytes,
                        cd_stream_t stream) {
  if (dt != CD_F64 && dt != CD_F32) return -1;
  if (n < 1 || n > (int64_t(1) << 30)) return -2;
  if (j < 0 || j >= n) return -3;
  if (w < 1 || w > DC_NMAX || j + w > n) return -4;
  if (q < 0 || q > j) return -5;
  if (q > 0 && !Lq) return -6;
  if (q > 0 && ldl < n) return -7;
  if (q > 0 && !Aq) return -8;
  if (q > 0 && lda < n) return -9;
  if (!Z) return -10;
  if (ldz != n - j) return -11;
  if (ws_bytes < cd_dist_workspace_size(dt, w)) return -13;
  const Opnd L{Lq, nullptr, 0, ldl, 0}, A{Aq, nullptr, 0, lda, 0}, Zo{Z, nullptr, 0, ldz, 0};
  return run_steps(dt, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), 12, [&](Ctx& c, auto zero) {
    dist_fwd_partial<decltype(zero)>(c, int(n), int(j), int(w), int(q), L, A, Zo);
  });
}

int cd_dist_fwd_panel(cd_dtype dt, int64_t n, int64_t j, int64_t w, const void* Lk, int64_t ldl, void* Ak,
                      int64_t lda, const void* Z, int64_t ldz, void* ws, size_t ws_bytes, cd_stream_t stream) {
  if (dt != CD_F64 && dt != CD_F32) return -1;
  if (n < 1 || n > (int64_t(1) << 30)) return -2;
  if (j < 0 || j >= n) return -3;
  if (w < 1 || w > DC_NMAX || j + w > n) return -4;
  if (!Lk) return -5;
  if (ldl < n) return -6;
  if (!Ak) return -7;
  if (lda < n) return -8;
  if (!Z) return -9;
  if (ldz < n - j) return -10;
  if (ws_bytes < cd_dist_workspace_size(dt, w)) return -12;
  const Opnd L{Lk, nullptr, 0, ldl, 0}, A{Ak, nullptr, 0, lda, 0}, Zo{Z, nullptr, 0, ldz, 0};
  return run_steps(dt, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), 11, [&](Ctx& c, auto zero) {
    dist_fwd_panel<decltype(zero)>(c, int(n), int(j), int(w), L, A, Zo);
  });
}

const char* cd_status_string(int status) {
  if (status == CD_SUCCESS) return "success";
  if (status == CD_ERR_CUDA) return "CUDA error (see cd_last_cuda_error)";
  if (status == CD_ERR_UNSUPPORTED) return "unsupported combination of valid arguments";
  if (status < 0) return "invalid argument (-status = 1-based argument position)";
  return "unknown status";
}

const char* cd_last_cuda_error(void) { return g_cuda_err; }
void cd_host_bytes(int64_t* h2d, int64_t* d2h) {
  if (h2d) *h2d = g_host_bytes_in;
  if (d2h) *d2h = g_host_bytes_out;
}
int cd_version(void) { return CD_VERSION; }
int64_t cd_launch_count(void) { return g_launches; }

void cd_profile_enable(int on) { g_prof.on = on != 0; }

void cd_profile_reset(void) {
  g_prof.recs.clear();
  g_prof.used = 0;
}

int cd_profile_read(int cls, double* ms, double* flops, int64_t* launches) {
  double t = 0.0, f = 0.0;
  int64_t cnt = 0;
  // CD_PROF_DUMP (measurement switch): list every recorded launch on stderr, in order
  static const bool dump = getenv("CD_PROF_DUMP") != nullptr;
  for (const ProfRec& r : g_prof.recs) {
    if (r.cls != cls && !(dump && cls == 0)) continue;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return note_cuda(e);
    float x = 0.f;
    e = cudaEventElapsedTime(&x, r.a, r.b);
    if (e != cudaSuccess) return note_cuda(e);
    if (dump && cls == 0) {
      float t0 = 0.f;
      cudaEventElapsedTime(&t0, g_prof.recs[0].a, r.a);
      fprintf(stderr, "prof cls %d  %9.1f us  %.3g flop   [start %8.1f us, stream %p]\n", r.cls, 1e3 * x, r.flops,
              1e3 * t0, static_cast<void*>(r.st));
    }
    if (r.cls != cls) continue;
    t += x;
    f += r.flops;
    ++cnt;
  }
  if (ms) *ms = t;
  if (flops) *flops = f;
  if (launches) *launches = cnt;
  return CD_SUCCESS;
}
void cd_reset_launch_count(void) { g_launches = 0; }

int cd_debug_phase_clocks(int enable, long long* out, int max) {
  g_dc_clk_host = enable != 0;
  if (out && max > 0) {
    long long tmp[40];
    if (cudaMemcpyFromSymbol(tmp, g_dc_clk, sizeof(tmp)) != cudaSuccess) return CD_ERR_CUDA;
    for (int i = 0; i < max && i < 40; ++i) out[i] = tmp[i];
  }
  return CD_SUCCESS;
}

}  // extern "C"
