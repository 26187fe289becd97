// ipm_api.cu — the C ABI of libipm (include/ipm.h): argument validation, launch geometry, dispatch of the 30
// legal (op, dtype) kernels, the data environment (present table), and the host-streaming path.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "ipm.h"
#include "ipm_internal.h"
#include "ipm_kernels.cuh"
#include "ipm_fused.cuh"

namespace ipm {

// ------------------------------------------------------------------------------------------ errors
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
ipm_status cuda_fail(cudaError_t e, const char* where) {
  set_error(std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
  return IPM_E_CUDA;
}
#define CK(call)                                            \
  do {                                                      \
    cudaError_t e_ = (call);                                \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);     \
  } while (0)

// ------------------------------------------------------------------------------------------ device facts
int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int s = 0;
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = s > 0 ? s : 148;
  }
  return cache[dev];
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

// tuning (compile-time kernel shapes, run-time grid sizing)
constexpr int FLAT_BLOCK = 256;
constexpr int FLAT_U = 4;    // static / dynamic k_flat: 4 x 32 B loads per thread per tile
constexpr int GUIDED_U = 2;  // k_flat_guided: 2 x 32 B per tile, software-pipelined (2-4 loads in flight)
// run-time options (ipm_set_option); defaults chosen by tools/sweep_flat.cu measurements
// process-wide, set from any thread: atomics (a launch reads each once)
static std::atomic<int> g_opt_flat_cps{-1};  // CTAs per SM for k_flat (-1: IPM_CTAS_PER_SM env or 4)
static std::atomic<int> g_opt_seg_kernel{0}; // 0 auto (= 1), 1 warp per row (direct loads), 2 warp per row (TMA ring)
static std::atomic<int> g_opt_deterministic{1};  // 1: guided deterministic schedule for the flat kernel
static std::atomic<int> g_opt_dist_mode{0};      // 0: fused peer-memory exchange when mapped, 1: NCCL AllGather
static std::atomic<long long> g_opt_dist_timeout_ms{30000};
static std::atomic<int> g_opt_ragged_kernel{0};  // 0 auto (= 1), 1 one warp per element range, 2 CTA tiles
static int flat_ctas_per_sm() {
  const int c = g_opt_flat_cps.load(std::memory_order_relaxed);
  if (c > 0) return c;
  static int v = std::max(1, std::min(8, env_int("IPM_CTAS_PER_SM", 4)));
  return v;
}
constexpr int SEG_WARPS = 8;
constexpr int SEG_U = 8;
// CTAs for k_seg_warp: warps take rows in grid-stride rounds, so when the rows do not fill the last round
// some warps run one row longer while the rest idle (C3, 65536 rows: 592 CTAs -> 13.84 rows per warp, 6.75 TB/s;
// 512 CTAs -> 16 rows per warp exactly, 6.92 TB/s, profiles/r01_sweep_segtail.txt). Take the CTA count in
// [3/4, 1] x one resident wave (occ CTAs per SM) whose warps divide the rows most evenly (the smallest such
// count), one row per warp if the rows fit in one wave.
static int seg_grid(int64_t rows, int sms, int occ) {
  const int64_t need = (rows + SEG_WARPS - 1) / SEG_WARPS;
  const int64_t gmax = (int64_t)sms * occ;
  if (need <= gmax) return (int)std::max<int64_t>(1, need);
  const int64_t glo = std::max<int64_t>(1, gmax * 3 / 4);
  int64_t best = gmax;
  double best_eff = 0.0;
  for (int64_t g = glo; g <= gmax; ++g) {
    const int64_t nw = g * SEG_WARPS;
    const double eff = (double)rows / (double)(((rows + nw - 1) / nw) * nw);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = g;
    }
  }
  return (int)best;
}
constexpr int TMA_WARPS = 8, TMA_S = 4, TMA_CH = 4096;

size_t esize(ipm_dtype dt) {
  switch (dt) {
    case IPM_I32: case IPM_F32: return 4;
    case IPM_I64: case IPM_F64: return 8;
    default: return 0;
  }
}

ipm_status validate(ipm_op op, ipm_dtype dt) {
  if ((int)dt < 0 || (int)dt > IPM_F64) {
    set_error("unknown dtype");
    return IPM_E_DTYPE;
  }
  if ((int)op < 0 || (int)op > IPM_LOR) {
    set_error("unknown reduction operator");
    return IPM_E_REDOP;
  }
  if ((dt == IPM_F32 || dt == IPM_F64) && (op == IPM_BAND || op == IPM_BOR || op == IPM_BXOR)) {
    set_error("bitwise reduction operators are illegal on floating-point types");
    return IPM_E_REDOP;
  }
  return IPM_OK;
}

uint64_t scalar_bits(ipm_dtype dt, const void* s) {
  if (!s) return 0;
  if (esize(dt) == 4) {
    uint32_t u;
    memcpy(&u, s, 4);
    return u;
  }
  uint64_t u;
  memcpy(&u, s, 8);
  return u;
}

static int64_t flat_grid(ipm_dtype dt, int64_t n) {
  const int64_t vw = 32 / (int64_t)esize(dt);
  const int64_t tiles = (n / vw + (int64_t)FLAT_BLOCK * FLAT_U - 1) / ((int64_t)FLAT_BLOCK * FLAT_U);
  int64_t g = std::min<int64_t>((int64_t)sm_count() * flat_ctas_per_sm(), tiles);
  return std::max<int64_t>(1, std::min<int64_t>(g, WS_MAX_PARTIALS));
}

// ------------------------------------------------------------------------------------------ kernel timing
struct Prof {
  bool on = false;
  int max = 0, used = 0;
  cudaEvent_t* ev = nullptr;  // 2 per record
  int* kind = nullptr;
};
static Prof g_prof;

struct ProfScope {  // records an event pair around one kernel launch when profiling is enabled
  int slot = -1;
  cudaStream_t st;
  ProfScope(cudaStream_t s, int kind) : st(s) {
    if (g_prof.on && g_prof.used < g_prof.max) {
      slot = g_prof.used++;
      g_prof.kind[slot] = kind;
      cudaEventRecord(g_prof.ev[2 * slot], st);
    }
  }
  ~ProfScope() {
    if (slot >= 0) cudaEventRecord(g_prof.ev[2 * slot + 1], st);
  }
};

static void prof_free() {
  for (int i = 0; i < 2 * g_prof.max; ++i) cudaEventDestroy(g_prof.ev[i]);
  delete[] g_prof.ev;
  delete[] g_prof.kind;
  g_prof = Prof();
}

int dist_mode_option() { return g_opt_dist_mode.load(std::memory_order_relaxed); }
long long dist_timeout_ns() { return g_opt_dist_timeout_ms.load(std::memory_order_relaxed) * 1000000ll; }

// ------------------------------------------------------------------------------------------ dispatch
#define IPM_LEGAL(X)                                                                                       \
  X(IPM_ADD, IPM_I32) X(IPM_MUL, IPM_I32) X(IPM_MAX, IPM_I32) X(IPM_MIN, IPM_I32) X(IPM_BAND, IPM_I32)     \
  X(IPM_BOR, IPM_I32) X(IPM_BXOR, IPM_I32) X(IPM_LAND, IPM_I32) X(IPM_LOR, IPM_I32)                        \
  X(IPM_ADD, IPM_I64) X(IPM_MUL, IPM_I64) X(IPM_MAX, IPM_I64) X(IPM_MIN, IPM_I64) X(IPM_BAND, IPM_I64)     \
  X(IPM_BOR, IPM_I64) X(IPM_BXOR, IPM_I64) X(IPM_LAND, IPM_I64) X(IPM_LOR, IPM_I64)                        \
  X(IPM_ADD, IPM_F32) X(IPM_MUL, IPM_F32) X(IPM_MAX, IPM_F32) X(IPM_MIN, IPM_F32) X(IPM_LAND, IPM_F32)     \
  X(IPM_LOR, IPM_F32)                                                                                      \
  X(IPM_ADD, IPM_F64) X(IPM_MUL, IPM_F64) X(IPM_MAX, IPM_F64) X(IPM_MIN, IPM_F64) X(IPM_LAND, IPM_F64)     \
  X(IPM_LOR, IPM_F64)

// Which flat kernel a launch takes (the one decision both Launch::flat and ipm_flat_schedule use). The flat
// clause uses the guided schedule (k_flat_guided: ~90% of the tiles static, the rest in chunks claimed
// dynamically, one partial slot per element range) — load-balanced and bit-reproducible for every operator.
// IPM_OPT_DETERMINISTIC = 0 selects the purely dynamic tile schedule instead (float + and * may then differ in
// the last bits between runs). Multi-row launches (grid.y > 1), the per-block partials mode and inputs up to
// 64 MiB (latency-bound: the static schedule saves the chunk claims, C1: 12.4 -> 10.3 us) keep the static
// grid-stride schedule.
enum { SCHED_STATIC = 0, SCHED_GUIDED = 1, SCHED_DYNAMIC = 2 };
static int flat_schedule(size_t es, int64_t n, unsigned grid_x, unsigned grid_y, bool has_counter) {
  const bool small = n * (int64_t)es <= (64ll << 20);
  const int det = g_opt_deterministic.load(std::memory_order_relaxed);
  if (has_counter && grid_y == 1 && grid_x > 1 && det != 2 && !small) return det ? SCHED_GUIDED : SCHED_DYNAMIC;
  return SCHED_STATIC;
}

template <int OP, int DT>
struct Launch {
  using R = Red<OP, DT>;
  static void flat(const FlatParams& p, dim3 grid, cudaStream_t st) {
    switch (flat_schedule(sizeof(typename R::B), p.n, grid.x, grid.y, p.counter != nullptr)) {
      case SCHED_GUIDED: k_flat_guided<R, FLAT_BLOCK, GUIDED_U, true><<<grid, FLAT_BLOCK, 0, st>>>(p); break;
      case SCHED_DYNAMIC: k_flat<R, FLAT_BLOCK, FLAT_U, 0, 2><<<grid, FLAT_BLOCK, 0, st>>>(p); break;
      default: k_flat<R, FLAT_BLOCK, FLAT_U, 0, 0><<<grid, FLAT_BLOCK, 0, st>>>(p); break;
    }
  }
  static void seg_warp(const SegParams& p, int sms, cudaStream_t st) {
    static const int occ = [] {
      int m = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m, k_seg_warp<R, SEG_WARPS, SEG_U>, SEG_WARPS * 32, 0);
      return m > 0 ? m : 1;
    }();
    k_seg_warp<R, SEG_WARPS, SEG_U><<<seg_grid(p.rows, sms, occ), SEG_WARPS * 32, 0, st>>>(p);
  }
  // CTA-tile ragged kernel (default): 128 threads x 4 vectors per thread per tile (32 float32 / 16 float64
  // elements per thread), L2 bulk prefetch 2 tiles ahead, 4 CTAs per SM
  static constexpr int RT_BLOCK = 128, RT_VPT = 4, RT_MINB = 4, RT_PFD = 2;
  static cudaError_t ragged_tile(const RaggedParams& p, int blocks, cudaStream_t st) {
    constexpr int smem = RaggedTile<R, RT_BLOCK, RT_VPT>::SMEM;
    auto kern = k_ragged_tile<R, RT_BLOCK, RT_VPT, RT_MINB, RT_PFD>;
    static const cudaError_t attr = [&] {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 (int)cudaSharedmemCarveoutMaxShared);
      return e;
    }();
    if (attr != cudaSuccess) return attr;
    kern<<<blocks, RT_BLOCK, smem, st>>>(p);
    k_ragged_fix<R><<<(unsigned)((blocks + 7) / 8), 256, 0, st>>>(p, blocks);
    return cudaSuccess;
  }
  // the warp kernel's shape: 2 vectors per lane at 8 CTAs x 4 warps per SM for 4-byte elements; 8-byte elements 4
  // vectors at IPM_RV_8B = 6 CTAs (same-box A/B: compare / bitwise / logical folds profiles/r02_ab_ragged_vec_cmp8.txt,
  // float64 max/min +25-29 %, int64 max +11-14 %, int64 && +8-11 %, 7 CTAs slightly slower; + and *
  // profiles/r02_ab_ragged_vec_8b_add.txt, int64 + +6-9 %, float64 + * +1-6 %, -3..6 % on 4-element rows); 4-byte
  // folds lose at 4 vectors (-2..16 %, profiles/r02_ab_ragged_vec_4b.txt). The float64 max/min instantiations keep a
  // 4-byte spill outside the chunk loop (tests/test_build_report.py)
#ifndef IPM_RV_8B
#define IPM_RV_8B 6
#endif
#ifndef IPM_RV_4B
#define IPM_RV_4B 8
#endif
  static constexpr bool RV_8B = sizeof(typename R::B) == 8;
  static constexpr int RV_VPL = RV_8B ? 4 : 2, RV_MINB = RV_8B ? IPM_RV_8B : IPM_RV_4B;
  static int64_t ragged_vec_warps(int sms) { return std::min<int64_t>((int64_t)sms * 4 * RV_MINB, WS_MAX_RAGGED_WARPS); }
  static void ragged_vec_only(const RaggedParams& p, int blocks, cudaStream_t st) {
    // 25 KiB of static shared memory per CTA: ask for the largest carveout so 8 CTAs fit on an SM
    // L2 prefetch of the next chunk (profiles/r01_sweep_ragged_5_l2prefetch.txt: +13-16 % on long rows, +1-7 % on
    // the power-law graph); for the widened float32 + * fold (issue-bound on short rows) only inside long rows
    constexpr int PFV = sizeof(typename R::A) > sizeof(typename R::B) ? -1 : 1;
    static const bool carveout = cudaFuncSetAttribute(k_ragged_vec<R, 4, RV_MINB, RV_VPL, true, PFV>,
                                                      cudaFuncAttributePreferredSharedMemoryCarveout,
                                                      (int)cudaSharedmemCarveoutMaxShared) == cudaSuccess;
    (void)carveout;
    k_ragged_vec<R, 4, RV_MINB, RV_VPL, true, PFV><<<blocks, 128, 0, st>>>(p);  // RV_MINB CTAs x 4 warps per SM
  }
  static void ragged(const RaggedParams& p, int blocks, int64_t nw, cudaStream_t st) {
    ragged_vec_only(p, blocks, st);
    k_ragged_fix<R><<<(unsigned)((nw + 7) / 8), 256, 0, st>>>(p, nw);
  }
  // rank-order ragged kernel: RR_WARPS warps per CTA, 2 vectors per lane, offset ring of RR_NR windows; as many CTAs
  // per SM as fit (shared memory bound), the grid one full wave of them
#ifndef IPM_RR_WARPS
#define IPM_RR_WARPS 4
#endif
#ifndef IPM_RR_MINB
#define IPM_RR_MINB 6
#endif
#ifndef IPM_RR_NR
#define IPM_RR_NR 8
#endif
#ifndef IPM_RR_K
#define IPM_RR_K 8
#endif
  static constexpr int RR_WARPS = IPM_RR_WARPS, RR_MINB = IPM_RR_MINB, RR_VPL = 2, RR_NR = IPM_RR_NR, RR_K = IPM_RR_K;
  static constexpr int RR_PFV = sizeof(typename R::A) > sizeof(typename R::B) ? -1 : 1;
  static int ragged_rank_ctas_per_sm() {
    static const int occ = [] {
      auto kern = k_ragged_rank<R, RR_WARPS, RR_MINB, RR_VPL, RR_NR, RR_PFV>;
      cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
      int m = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m, kern, RR_WARPS * 32, 0);
      return m > 0 ? m : 1;
    }();
    return occ;
  }
  static void ragged_rank(const RaggedParams& p, int blocks, int64_t nw, cudaStream_t st) {
    k_ragged_rank<R, RR_WARPS, RR_MINB, RR_VPL, RR_NR, RR_PFV><<<blocks, RR_WARPS * 32, 0, st>>>(p);
    k_ragged_fix<R><<<(unsigned)((nw + 7) / 8), 256, 0, st>>>(p, nw);
  }
  // lane-per-row ragged kernel: windows of <= 32 rows spanning <= LP_CAPB bytes staged in shared memory by cp.async
#ifndef IPM_LP_WARPS
#define IPM_LP_WARPS 4
#endif
#ifndef IPM_LP_MINB
#define IPM_LP_MINB 8
#endif
#ifndef IPM_LP_CAPB
#define IPM_LP_CAPB 4096
#endif
#ifndef IPM_LP_T
#define IPM_LP_T 32
#endif
  static void ragged_lpr(const RaggedParams& p, int blocks, int64_t nw, cudaStream_t st) {
    k_ragged_lpr<R, IPM_LP_WARPS, IPM_LP_MINB, IPM_LP_CAPB, 8, IPM_LP_T><<<blocks, IPM_LP_WARPS * 32, 0, st>>>(p);
    k_ragged_fix<R><<<(unsigned)((nw + 7) / 8), 256, 0, st>>>(p, nw);
  }
  // auto: the warp kernel below RA_LONG elements per row on average (the whole input), the lane-per-row kernel at or
  // above; both launched, the other one returns at once (gate on off[0], off[rows]). The crossover measured on one
  // box (profiles/r02_time_ragged_cross.txt, rows of 128 .. 2048 elements): 256 elements for 4-byte types, 128 for
  // 8-byte ones
#ifndef IPM_RA_LONG
#define IPM_RA_LONG (sizeof(typename R::B) == 8 ? 128 : 256)
#endif
  // each candidate on its own grid (the warp kernel: one wave of its shape; the lane-per-row kernel: 8 CTAs x 4
  // warps per SM); the one that runs publishes its warp count (a workspace word) for the fix-up
  static void ragged_auto(const RaggedParams& p0, int sms, cudaStream_t st) {
    RaggedParams p = p0;
    p.nw_dev = (int64_t*)((char*)p.head_row - WS_RAGGED + WS_RAGGED_NW);
    const int64_t nw_vec = ragged_vec_warps(sms);
    const int64_t nw_lpr = std::min<int64_t>((int64_t)sms * 32, WS_MAX_RAGGED_WARPS);
    p.gate_len = IPM_RA_LONG;
    p.gate = 1;
    ragged_vec_only(p, (int)(nw_vec / 4), st);
    p.gate = 2;
    k_ragged_lpr<R, IPM_LP_WARPS, IPM_LP_MINB, IPM_LP_CAPB, 8, IPM_LP_T>
        <<<(unsigned)(nw_lpr / IPM_LP_WARPS), IPM_LP_WARPS * 32, 0, st>>>(p);
    const int64_t nw = std::max(nw_vec, nw_lpr);
    k_ragged_fix<R><<<(unsigned)((nw + 7) / 8), 256, 0, st>>>(p, nw);
  }
  // marked rows (two passes, k_ragged_mark + k_ragged_mk, then the fix-up): chunks of 512 elements (4-byte) / 256
  // (8-byte), 8 CTAs x 4 warps per SM; the scratch (bitmap + chunk counts) is zeroed in stream order first
  // shape per fold (same-box A/B, profiles/r02_ab_marked_{1,3,4}.txt): folds with 8-byte accumulators on 4-byte
  // elements (float32 + * in float64, float32 max/min pairs) 4 vectors per lane at 6 CTAs per SM (shared memory
  // bound); 8-byte compare / bitwise / logical folds 4 at 7 (+3..31 %); the rest (4-byte folds, 8-byte + *) 2 at 8;
  // every fold asks L2 for the chunk after the next (profiles/r02_ab_marked_1.txt)
  static constexpr bool MK_WIDE = sizeof(typename R::A) > sizeof(typename R::B);
  static constexpr bool MK_CMP8 = sizeof(typename R::B) == 8 && OP != IPM_ADD && OP != IPM_MUL;
#ifndef IPM_MK_VPL
#define IPM_MK_VPL (MK_WIDE || MK_CMP8 ? 4 : 2)
#endif
#ifndef IPM_MK_MINB
#define IPM_MK_MINB (MK_WIDE ? 6 : MK_CMP8 ? 7 : 8)
#endif
#ifndef IPM_MK_PFD
#define IPM_MK_PFD 1
#endif
  static constexpr int MK_VPL = IPM_MK_VPL, MK_MINB = IPM_MK_MINB, MK_PFD = IPM_MK_PFD;
  static int64_t ragged_mk_warps(int sms) {
    return std::min<int64_t>((int64_t)sms * 4 * MK_MINB, WS_MAX_RAGGED_WARPS);  // one wave of 4-warp CTAs
  }
  static constexpr int MK_CH = 32 * Vec<typename R::B>::W * MK_VPL;
  static cudaError_t ragged_mk(const RaggedParams& p, const RaggedMarks& m, size_t zero_bytes, int sms, int64_t nw,
                               cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(m.bits, 0, zero_bytes, st);
    if (e != cudaSuccess) return e;
#ifndef IPM_MK_RPL
#define IPM_MK_RPL 8
#endif
    // 8 warps x 32 x RPL rows per CTA step; one wave of the CTAs that fit (74 registers: 3 per SM at RPL 8). RPL 8
    // against 4: power-law +2-3 %, uniform rows +2-4 %, 4-element rows +4-6 %, 64-element rows -1..4 %
    // (profiles/r02_ab_mark_rpl.txt)
    static const int occ0 = [] {
      int n = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_ragged_mark<R, MK_CH, IPM_MK_RPL>, 256, 0);
      return n > 0 ? n : 1;
    }();
    const int64_t blocks0 = std::min<int64_t>((p.rows + 256 * IPM_MK_RPL - 1) / (256 * IPM_MK_RPL), (int64_t)sms * occ0);
    k_ragged_mark<R, MK_CH, IPM_MK_RPL><<<(unsigned)blocks0, 256, 0, st>>>(p, m);
    static const bool carveout = cudaFuncSetAttribute(k_ragged_mk<R, 4, MK_MINB, MK_VPL, MK_PFD>,
                                                      cudaFuncAttributePreferredSharedMemoryCarveout,
                                                      (int)cudaSharedmemCarveoutMaxShared) == cudaSuccess;
    (void)carveout;
    k_ragged_mk<R, 4, MK_MINB, MK_VPL, MK_PFD><<<(unsigned)(nw / 4), 128, 0, st>>>(p, m);
    k_ragged_fix<R><<<(unsigned)((nw + 7) / 8), 256, 0, st>>>(p, nw);
    return cudaSuccess;
  }
  // 8-byte folds run 3 CTAs x 256 per SM with up to 85 registers (+1-3 % over 4 CTAs at 64 registers; 4-byte folds
  // lose up to 17 % that way, profiles/r01_ab_2d_minb.txt). max_grid = SMs x the resident CTAs per SM.
  static constexpr int TWO_D_MINB = sizeof(typename R::B) == 8 ? 3 : 4;
  static void two_d(const Params2D& q, int max_items_grid, int sms, cudaStream_t st) {
    const int grid = std::max(1, std::min(max_items_grid, sms * TWO_D_MINB));
    k_2d<R, FLAT_BLOCK, 4, 0, TWO_D_MINB><<<grid, FLAT_BLOCK, 0, st>>>(q);
  }
  static cudaError_t seg_tma(const SegParams& p, int grid, cudaStream_t st) {
    constexpr int smem = SegTma<R, TMA_WARPS, TMA_S, TMA_CH>::SMEM;
    static cudaError_t attr =
        cudaFuncSetAttribute(k_seg_tma<R, TMA_WARPS, TMA_S, TMA_CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (attr != cudaSuccess) return attr;
    k_seg_tma<R, TMA_WARPS, TMA_S, TMA_CH><<<grid, TMA_WARPS * 32, smem, st>>>(p);
    return cudaSuccess;
  }
  static void seg_group(const SegParams& p, int G, int grid, cudaStream_t st) {
    switch (G) {
      case 1: k_seg_group<R, 1><<<grid, 256, 0, st>>>(p); break;
      case 2: k_seg_group<R, 2><<<grid, 256, 0, st>>>(p); break;
      case 4: k_seg_group<R, 4><<<grid, 256, 0, st>>>(p); break;
      case 8: k_seg_group<R, 8><<<grid, 256, 0, st>>>(p); break;
      default: k_seg_group<R, 16><<<grid, 256, 0, st>>>(p); break;
    }
  }
  static void exchange(const FlatParams& p, const uint64_t* acc, cudaStream_t st) {
    k_exchange<R><<<1, 32, 0, st>>>(p, acc);
  }
  static void finalize(const uint64_t* slots, int P, uint64_t init, int has_init, void* out, cudaStream_t st) {
    k_finalize<R><<<1, 32, 0, st>>>(slots, P, init, has_init, out);
  }
};

struct Table {
  void (*flat)(const FlatParams&, dim3, cudaStream_t);
  void (*two_d)(const Params2D&, int, int, cudaStream_t);  // (params, grid bound by the items, SM count, stream)
  void (*ragged)(const RaggedParams&, int, int64_t, cudaStream_t);
  cudaError_t (*ragged_tile)(const RaggedParams&, int, cudaStream_t);
  void (*ragged_rank)(const RaggedParams&, int, int64_t, cudaStream_t);
  void (*ragged_lpr)(const RaggedParams&, int, int64_t, cudaStream_t);
  void (*ragged_auto)(const RaggedParams&, int, cudaStream_t);
  int (*ragged_rank_ctas_per_sm)();
  cudaError_t (*ragged_mk)(const RaggedParams&, const RaggedMarks&, size_t, int, int64_t, cudaStream_t);
  int64_t (*ragged_mk_warps)(int);
  int64_t (*ragged_vec_warps)(int);
  void (*seg_warp)(const SegParams&, int, cudaStream_t);  // (params, SM count, stream)
  cudaError_t (*seg_tma)(const SegParams&, int, cudaStream_t);
  void (*seg_group)(const SegParams&, int, int, cudaStream_t);
  void (*finalize)(const uint64_t*, int, uint64_t, int, void*, cudaStream_t);
  void (*exchange)(const FlatParams&, const uint64_t*, cudaStream_t);
};

static const Table* table(ipm_op op, ipm_dtype dt) {
#define IPM_ENTRY(O, D)                                                                                  \
  if (op == O && dt == D) {                                                                            \
    static const Table t = {&Launch<O, D>::flat, &Launch<O, D>::two_d, &Launch<O, D>::ragged, &Launch<O, D>::ragged_tile, &Launch<O, D>::ragged_rank, &Launch<O, D>::ragged_lpr, &Launch<O, D>::ragged_auto, &Launch<O, D>::ragged_rank_ctas_per_sm, &Launch<O, D>::ragged_mk, &Launch<O, D>::ragged_mk_warps, &Launch<O, D>::ragged_vec_warps, &Launch<O, D>::seg_warp, &Launch<O, D>::seg_tma,     \
                            &Launch<O, D>::seg_group, &Launch<O, D>::finalize, &Launch<O, D>::exchange};\
    return &t;                                                                                         \
  }
  IPM_LEGAL(IPM_ENTRY)
#undef IPM_ENTRY
  return nullptr;
}

static ipm_status check_ws(void* ws) {
  if (!ws || ((uintptr_t)ws & 255u)) {
    set_error("workspace must be a non-NULL, 256-byte aligned device buffer of ipm_workspace_bytes() bytes");
    return IPM_E_WORKSPACE;
  }
  return IPM_OK;
}

static ipm_status check_array(ipm_dtype dt, const void* dev, int64_t n) {
  if (n < 0) {
    set_error("negative element count");
    return IPM_E_SIZE;
  }
  if (n > 0 && !dev) {
    set_error("NULL device array with n > 0");
    return IPM_E_NULL;
  }
  if (dev && ((uintptr_t)dev % esize(dt))) {
    set_error("device array not aligned to its element size");
    return IPM_E_ALIGN;
  }
  return IPM_OK;
}

ipm_status launch_flat(ipm_op op, ipm_dtype dt, const void* dev, int64_t n, uint64_t init, int has_init, int mode,
                       void* out, void* ws, cudaStream_t st, const DistArgs* dist, unsigned long long* done,
                       unsigned long long done_seq) {
  const Table* t = table(op, dt);
  FlatParams p;
  p.a = dev;
  p.n = n;
  p.row_stride = 0;
  p.init = init;
  p.has_init = has_init;
  p.mode = mode;
  p.out = out;
  p.partials = (uint64_t*)((char*)ws + WS_PARTIALS);
  p.tickets = (unsigned*)((char*)ws + WS_TICKETS);
  p.counter = (unsigned long long*)((char*)ws + WS_COUNTER);
  p.packed = (unsigned long long*)((char*)ws + WS_PACKED);
  p.done = mode == MODE_RESULT ? done : nullptr;
  p.done_seq = done_seq;
  const int64_t grid = flat_grid(dt, n);
  p.max_chunks = std::max<int64_t>(1, WS_MAX_PARTIALS - grid - 1);
  p.peers = dist ? dist->peers : nullptr;
  p.rank = dist ? dist->rank : 0;
  p.world = dist ? dist->world : 1;
  p.timeout_ns = dist ? dist->timeout_ns : 0;
  {
    ProfScope ps(st, 0);
    t->flat(p, dim3((unsigned)grid, 1, 1), st);
  }
  CK(cudaGetLastError());
  return IPM_OK;
}

ipm_status launch_finalize(ipm_op op, ipm_dtype dt, const uint64_t* slots, int P, uint64_t init, int has_init,
                           void* out, cudaStream_t st) {
  table(op, dt)->finalize(slots, P, init, has_init, out, st);
  CK(cudaGetLastError());
  return IPM_OK;
}

ipm_status launch_exchange(ipm_op op, ipm_dtype dt, const uint64_t* acc, uint64_t init, int has_init, void* out,
                           const DistArgs* dist, cudaStream_t st) {
  FlatParams p;
  memset(&p, 0, sizeof p);
  p.init = init;
  p.has_init = has_init;
  p.mode = MODE_DIST;
  p.out = out;
  p.peers = dist->peers;
  p.rank = dist->rank;
  p.world = dist->world;
  p.timeout_ns = dist->timeout_ns;
  table(op, dt)->exchange(p, acc, st);
  CK(cudaGetLastError());
  return IPM_OK;
}

// ------------------------------------------------------------------------------------------ fused
// 32-byte vectors per thread per tile: 4 for one stream, 2 per stream for two (x*y); same-box A/B
// (profiles/r02_ab_fused_u.txt): one stream at U = 4 vs 2 +1.2 % (float32 stats) .. +6.6 % (float64 stats), x*y at
// U = 4 -4 %; U = 6 / 8 no better (r02_ab_fused_u1.txt)
#ifndef IPM_FUSED_U1
#define IPM_FUSED_U1 4
#endif
#ifndef IPM_FUSED_U2
#define IPM_FUSED_U2 2
#endif
template <int DT>
struct FusedLaunch {
  using ADDX = Comp<Red<IPM_ADD, DT>, EX>;
  using ADDXX = Comp<Red<IPM_ADD, DT>, EXX>;
  using ADDXY = Comp<Red<IPM_ADD, DT>, EXY>;
  using MINX = Comp<Red<IPM_MIN, DT>, EX>;
  using MAXX = Comp<Red<IPM_MAX, DT>, EX>;
  template <class C0, class C1, class C2, class C3, bool TWO>
  static void go(const FusedParams& p, bool vec, int grid, cudaStream_t st) {
    using S = Sig<C0, C1, C2, C3>;
    // int64 keeps U = 2 for one stream too: its 64-bit x*x products at U = 4 spill (ptxas)
    constexpr int U = TWO || DT == IPM_I64 ? IPM_FUSED_U2 : IPM_FUSED_U1;
    if (vec) k_fused<S, C0, C1, C2, C3, TWO, true, FLAT_BLOCK, U><<<grid, FLAT_BLOCK, 0, st>>>(p);
    else k_fused<S, C0, C1, C2, C3, TWO, false, FLAT_BLOCK, U><<<grid, FLAT_BLOCK, 0, st>>>(p);
  }
  static void launch(ipm_fused f, const FusedParams& p, bool vec, int grid, cudaStream_t st) {
    switch (f) {
      case IPM_FUSED_SUM_SUMSQ: go<ADDX, ADDXX, NoComp, NoComp, false>(p, vec, grid, st); break;
      case IPM_FUSED_DOT: go<ADDXY, NoComp, NoComp, NoComp, true>(p, vec, grid, st); break;
      case IPM_FUSED_MINMAX: go<MINX, MAXX, NoComp, NoComp, false>(p, vec, grid, st); break;
      case IPM_FUSED_STATS: go<ADDX, ADDXX, MINX, MAXX, false>(p, vec, grid, st); break;
    }
  }
};

static int fused_nvars(ipm_fused f) {
  switch (f) {
    case IPM_FUSED_SUM_SUMSQ: return 2;
    case IPM_FUSED_DOT: return 1;
    case IPM_FUSED_MINMAX: return 2;
    case IPM_FUSED_STATS: return 4;
  }
  return 0;
}

// ------------------------------------------------------------------------------------------ allocator
static std::mutex g_mu;
static ipm_allocator g_alloc = {nullptr, nullptr, nullptr};

static void* dev_alloc(size_t bytes, cudaStream_t st) {
  if (g_alloc.alloc) return g_alloc.alloc(bytes, (void*)st, g_alloc.ctx);
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, st) != cudaSuccess) return nullptr;
  return p;
}
static void dev_free(void* p, cudaStream_t st) {
  if (!p) return;
  if (g_alloc.free) g_alloc.free(p, (void*)st, g_alloc.ctx);
  else cudaFreeAsync(p, st);
}

// ------------------------------------------------------------------------------------------ present table
struct Entry {
  size_t bytes;
  void* dev;
  int ref;
};
static std::map<uintptr_t, Entry> g_present;  // host start -> entry

// the entry whose host range covers [h, h+bytes), or end()
static std::map<uintptr_t, Entry>::iterator find_cover(uintptr_t h, size_t bytes) {
  auto it = g_present.upper_bound(h);
  if (it == g_present.begin()) return g_present.end();
  --it;
  if (h >= it->first && h + bytes <= it->first + it->second.bytes) return it;
  return g_present.end();
}

// ------------------------------------------------------------------------------------------ host staging
struct Staging {
  void* buf[2] = {nullptr, nullptr};
  size_t bytes = 0;
  cudaStream_t copy = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
  int device = -1;
};
static Staging g_stage;

static ipm_status release_staging_locked() {
  for (int i = 0; i < 2; ++i) {
    if (g_stage.buf[i]) {
      cudaStreamSynchronize(g_stage.copy);
      if (g_stage.consumed[i]) cudaEventSynchronize(g_stage.consumed[i]);  // the last reader (any caller's stream)
      dev_free(g_stage.buf[i], g_stage.copy);
      g_stage.buf[i] = nullptr;
    }
    if (g_stage.copied[i]) cudaEventDestroy(g_stage.copied[i]);
    if (g_stage.consumed[i]) cudaEventDestroy(g_stage.consumed[i]);
    g_stage.copied[i] = g_stage.consumed[i] = nullptr;
  }
  if (g_stage.copy) {
    cudaStreamSynchronize(g_stage.copy);
    cudaStreamDestroy(g_stage.copy);
  }
  g_stage.copy = nullptr;
  g_stage.bytes = 0;
  g_stage.device = -1;
  return IPM_OK;
}

}  // namespace ipm

using namespace ipm;

// ============================================================================================ C ABI
// Synchronous calls deliver the 8-byte result through a small pinned, device-mapped host buffer per host thread
// and device: the finishing kernel stores the result straight into host memory, so the call is launch + stream
// synchronize (no separate device-to-host copy through a pageable staging buffer). One per thread suffices: a
// thread has at most one synchronous call in flight.
namespace ipm {
namespace {
struct Mailbox {
  void* host[64] = {nullptr};
  void* dev[64] = {nullptr};
  unsigned long long seq[64] = {0};  // the last done flag value asked of a kernel (word 1 of the buffer)
};
thread_local Mailbox tl_mail;
}  // namespace

ipm_status result_mailbox(void** host, void** dev) {
  int d = 0;
  CK(cudaGetDevice(&d));
  if (d < 0 || d >= 64) {
    set_error("device index out of range for the result mailbox");
    return IPM_E_ARG;
  }
  if (!tl_mail.host[d]) {
    void* h = nullptr;
    CK(cudaHostAlloc(&h, 64, cudaHostAllocMapped | cudaHostAllocPortable));
    memset(h, 0, 64);  // word 1 is the done flag: no stale value may match a sequence number
    void* dp = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(&dp, h, 0);
    if (e != cudaSuccess) {
      cudaFreeHost(h);
      return cuda_fail(e, "cudaHostGetDevicePointer");
    }
    tl_mail.host[d] = h;
    tl_mail.dev[d] = dp;
  }
  *host = tl_mail.host[d];
  *dev = tl_mail.dev[d];
  return IPM_OK;
}

// the next done-flag value for this thread's mailbox on the current device (result_mailbox called first)
unsigned long long mailbox_next_seq() {
  int d = 0;
  cudaGetDevice(&d);
  return ++tl_mail.seq[d];
}

// Wait for a synchronous call's result: poll the mailbox's done flag (the kernel stores it with system-scope
// release after the result, so the result is visible once the flag is), at most POLL_NS, then fall back to a stream
// synchronize (long kernels, and errors: a failed kernel never sets the flag). Polling skips the driver's wake-up
// path of cudaStreamSynchronize on the latency-bound small calls (BASELINE config 1).
ipm_status wait_mailbox(void* host, unsigned long long seq, cudaStream_t st) {
  constexpr long long POLL_NS = 200000;
  volatile unsigned long long* flag = (volatile unsigned long long*)host + 1;
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0;; ++i) {
    if (__atomic_load_n((const unsigned long long*)flag, __ATOMIC_ACQUIRE) == seq) return IPM_OK;
    if ((i & 255) == 255 &&
        std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count() > POLL_NS)
      break;
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  CK(cudaStreamSynchronize(st));
  return IPM_OK;
}
}  // namespace ipm

extern "C" {

const char* ipm_status_str(ipm_status s) {
  switch (s) {
    case IPM_OK: return "IPM_OK";
    case IPM_E_REDOP: return "IPM_E_REDOP";
    case IPM_E_DTYPE: return "IPM_E_DTYPE";
    case IPM_E_NULL: return "IPM_E_NULL";
    case IPM_E_SIZE: return "IPM_E_SIZE";
    case IPM_E_PRESENT: return "IPM_E_PRESENT";
    case IPM_E_ALIGN: return "IPM_E_ALIGN";
    case IPM_E_WORKSPACE: return "IPM_E_WORKSPACE";
    case IPM_E_CUDA: return "IPM_E_CUDA";
    case IPM_E_NCCL: return "IPM_E_NCCL";
    case IPM_E_ARG: return "IPM_E_ARG";
  }
  return "IPM_E_UNKNOWN";
}

const char* ipm_last_error_message(void) { return g_err.c_str(); }
int ipm_version(void) { return 100; }
int ipm_op_legal(ipm_op op, ipm_dtype dt) { return validate(op, dt) == IPM_OK ? 1 : 0; }
size_t ipm_dtype_size(ipm_dtype dt) { return esize(dt); }
size_t ipm_workspace_bytes(void) { return WS_BYTES; }

ipm_status ipm_workspace_init(void* ws, void* stream) {
  ipm_status s = check_ws(ws);
  if (s) return s;
  CK(cudaMemsetAsync(ws, 0, WS_BYTES, (cudaStream_t)stream));
  return IPM_OK;
}

ipm_status ipm_set_allocator(const ipm_allocator* a) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (a && (!a->alloc || !a->free)) {
    set_error("allocator needs both alloc and free");
    return IPM_E_NULL;
  }
  g_alloc = a ? *a : ipm_allocator{nullptr, nullptr, nullptr};
  return IPM_OK;
}

ipm_status ipm_set_option(ipm_option key, int64_t value) {
  switch (key) {
    case IPM_OPT_FLAT_CTAS_PER_SM:
      if (value < -1 || value > 8 || value == 0) break;
      g_opt_flat_cps = (int)value;
      return IPM_OK;
    case IPM_OPT_SEG_KERNEL:
      if (value < 0 || value > 2) break;
      g_opt_seg_kernel = (int)value;
      return IPM_OK;
    case IPM_OPT_DETERMINISTIC:
      if (value < 0 || value > 2) break;
      g_opt_deterministic = (int)value;
      return IPM_OK;
    case IPM_OPT_DIST_MODE:
      if (value < 0 || value > 1) break;
      g_opt_dist_mode = (int)value;
      return IPM_OK;
    case IPM_OPT_DIST_TIMEOUT_MS:
      if (value < 1) break;
      g_opt_dist_timeout_ms = value;
      return IPM_OK;
    case IPM_OPT_RAGGED_KERNEL:
      if (value < 0 || value > 4) break;
      g_opt_ragged_kernel = (int)value;
      return IPM_OK;
  }
  set_error("unknown option or value out of range");
  return IPM_E_ARG;
}

ipm_status ipm_profile_enable(int max_records) {
  if (max_records < 1 || max_records > (1 << 20)) {
    set_error("max_records out of range");
    return IPM_E_ARG;
  }
  prof_free();
  g_prof.ev = new cudaEvent_t[2 * max_records];
  g_prof.kind = new int[max_records];
  for (int i = 0; i < 2 * max_records; ++i) {
    cudaError_t e = cudaEventCreate(&g_prof.ev[i]);
    if (e != cudaSuccess) {
      g_prof.max = i / 2;
      prof_free();
      return cuda_fail(e, "cudaEventCreate");
    }
  }
  g_prof.max = max_records;
  g_prof.used = 0;
  g_prof.on = true;
  return IPM_OK;
}

ipm_status ipm_profile_read(float* ms, int* kinds, int max, int* count) {
  if (!count) return IPM_E_NULL;
  const int n = std::min(max, g_prof.used);
  for (int i = 0; i < n; ++i) {
    CK(cudaEventSynchronize(g_prof.ev[2 * i + 1]));
    if (ms) CK(cudaEventElapsedTime(&ms[i], g_prof.ev[2 * i], g_prof.ev[2 * i + 1]));
    if (kinds) kinds[i] = g_prof.kind[i];
  }
  *count = g_prof.used;
  return IPM_OK;
}

ipm_status ipm_profile_disable(void) {
  prof_free();
  return IPM_OK;
}

ipm_status ipm_flat_geometry(ipm_dtype dt, int64_t n, int* grid, int* block) {
  if (!esize(dt)) return IPM_E_DTYPE;
  if (n < 0) return IPM_E_SIZE;
  if (grid) *grid = (int)flat_grid(dt, n);
  if (block) *block = FLAT_BLOCK;
  return IPM_OK;
}

ipm_status ipm_flat_schedule(ipm_dtype dt, int64_t n, int* schedule) {
  if (!esize(dt)) return IPM_E_DTYPE;
  if (n < 0) return IPM_E_SIZE;
  if (!schedule) return IPM_E_NULL;
  *schedule = n == 0 ? -1 : flat_schedule(esize(dt), n, (unsigned)flat_grid(dt, n), 1, true);
  return IPM_OK;
}

// identities of the nine operators ("per-thread private v initialized to op's identity"; DESIGN.md
// R2: -inf / +inf for float max / min) as element bits; the device-side Red<>::id() of the kernels agrees with
// it (tests/test_gpu_parity.py: the n = 0 finalize kernel writes exactly these bits)
ipm_status ipm_identity(ipm_op op, ipm_dtype dt, void* out) {
  ipm_status s;
  if ((s = validate(op, dt))) return s;
  if (!out) {
    set_error("NULL out");
    return IPM_E_NULL;
  }
  const bool w4 = esize(dt) == 4, fl = dt == IPM_F32 || dt == IPM_F64;
  uint64_t b = 0;
  switch (op) {
    case IPM_ADD: case IPM_BOR: case IPM_BXOR: case IPM_LOR: b = 0; break;
    case IPM_MUL: case IPM_LAND: b = fl ? (w4 ? 0x3F800000ull : 0x3FF0000000000000ull) : 1ull; break;
    case IPM_MAX: b = fl ? (w4 ? 0xFF800000ull : 0xFFF0000000000000ull) : (w4 ? 0x80000000ull : 1ull << 63); break;
    case IPM_MIN: b = fl ? (w4 ? 0x7F800000ull : 0x7FF0000000000000ull) : (w4 ? 0x7FFFFFFFull : ~0ull >> 1); break;
    case IPM_BAND: b = w4 ? 0xFFFFFFFFull : ~0ull; break;
  }
  if (w4) {
    const uint32_t u = (uint32_t)b;
    memcpy(out, &u, 4);
  } else {
    memcpy(out, &b, 8);
  }
  return IPM_OK;
}

// ---------------------------------------------------------------------------------- reductions
ipm_status ipm_reduce_async(ipm_op op, ipm_dtype dt, const void* dev, int64_t n, const void* init,
                            void* dev_result, void* ws, void* stream) {
  ipm_status s;
  if ((s = validate(op, dt)) || (s = check_array(dt, dev, n)) || (s = check_ws(ws))) return s;
  if (!dev_result) {
    set_error("NULL dev_result");
    return IPM_E_NULL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t ib = scalar_bits(dt, init);
  if (n == 0)  // zero-trip loop: no reduction kernel; var = init ⊕ identity
    return launch_finalize(op, dt, nullptr, 0, ib, init != nullptr, dev_result, st);
  return launch_flat(op, dt, dev, n, ib, init != nullptr, MODE_RESULT, dev_result, ws, st);
}

ipm_status ipm_reduce(ipm_op op, ipm_dtype dt, const void* dev, int64_t n, void* inout, void* ws, void* stream) {
  if (!inout) {
    set_error("NULL inout");
    return IPM_E_NULL;
  }
  void *mh, *md;
  ipm_status s = result_mailbox(&mh, &md);
  if (s) return s;
  if (n > 0) {  // the flat kernel signals the mailbox: poll it (end of the compute region)
    if ((s = validate(op, dt)) || (s = check_array(dt, dev, n)) || (s = check_ws(ws))) return s;
    const unsigned long long seq = mailbox_next_seq();
    if ((s = launch_flat(op, dt, dev, n, scalar_bits(dt, inout), 1, MODE_RESULT, md, ws, (cudaStream_t)stream,
                         nullptr, (unsigned long long*)md + 1, seq)))
      return s;
    if ((s = wait_mailbox(mh, seq, (cudaStream_t)stream))) return s;
  } else {
    if ((s = ipm_reduce_async(op, dt, dev, n, inout, md, ws, stream))) return s;
    CK(cudaStreamSynchronize((cudaStream_t)stream));
  }
  memcpy(inout, mh, esize(dt));
  return IPM_OK;
}

ipm_status ipm_reduce_segmented(ipm_op op, ipm_dtype dt, const void* dev, int64_t rows, int64_t cols,
                                int64_t row_stride, const void* init, void* dev_out, void* ws, void* stream) {
  ipm_status s;
  if ((s = validate(op, dt))) return s;
  if (rows < 0 || cols < 0 || row_stride < cols) {
    set_error("need rows >= 0, cols >= 0, row_stride >= cols");
    return IPM_E_SIZE;
  }
  if (rows == 0) return IPM_OK;
  if (!dev_out || (cols > 0 && !dev)) {
    set_error("NULL device pointer");
    return IPM_E_NULL;
  }
  if (((uintptr_t)dev_out % esize(dt)) || (dev && ((uintptr_t)dev % esize(dt)))) {
    set_error("device pointer not aligned to its element size");
    return IPM_E_ALIGN;
  }
  if (row_stride > 0 && (rows - 1) > (INT64_MAX - cols) / row_stride) {
    set_error("rows*row_stride overflows");
    return IPM_E_SIZE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const Table* t = table(op, dt);
  const uint64_t ib = scalar_bits(dt, init);
  const int has_init = init != nullptr;
  const int sms = sm_count();
  const int64_t vw = 32 / (int64_t)esize(dt);

  // few long rows: split each row over S CTAs with the flat kernel's cross-CTA finish (gridDim.y = rows)
  const int64_t target_ctas = (int64_t)sms * flat_ctas_per_sm();
  if (rows < 2 * (int64_t)sms && cols >= 64 * vw * FLAT_BLOCK / 8 && rows <= WS_MAX_ROWS) {
    int64_t S = (target_ctas + rows - 1) / rows;
    const int64_t per_cta_vecs = (cols / vw + S - 1) / S;
    if (per_cta_vecs < FLAT_BLOCK) S = std::max<int64_t>(1, cols / vw / FLAT_BLOCK);
    S = std::min<int64_t>(S, WS_MAX_PARTIALS / rows);
    if (S > 1) {
      if ((s = check_ws(ws))) return s;
    }
    FlatParams p;
    p.a = dev;
    p.n = cols;
    p.row_stride = row_stride;
    p.init = ib;
    p.has_init = has_init;
    p.mode = MODE_RESULT;
    p.out = dev_out;
    p.partials = ws ? (uint64_t*)((char*)ws + WS_PARTIALS) : nullptr;
    p.tickets = ws ? (unsigned*)((char*)ws + WS_TICKETS) : nullptr;
    p.counter = nullptr;
    p.packed = nullptr;
    p.done = nullptr;
    p.max_chunks = 0;
    p.peers = nullptr;
    p.rank = 0;
    p.world = 1;
    p.timeout_ns = 0;
    {
      ProfScope ps(st, 1);
      t->flat(p, dim3((unsigned)S, (unsigned)rows, 1), st);
    }
    CK(cudaGetLastError());
    return IPM_OK;
  }
  SegParams p;
  p.a = dev;
  p.rows = rows;
  p.cols = cols;
  p.row_stride = row_stride;
  p.init = ib;
  p.has_init = has_init;
  p.out = dev_out;
  ProfScope ps(st, 1);
  const bool tma = g_opt_seg_kernel.load(std::memory_order_relaxed) == 2 && cols * (int64_t)esize(dt) >= 64;
  if (tma) {         // one warp per row, rows staged by TMA bulk copies (one 128 KiB-ring CTA per SM)
    const int64_t blocks = std::min<int64_t>((rows + TMA_WARPS - 1) / TMA_WARPS, (int64_t)sms);
    CK(t->seg_tma(p, (int)std::max<int64_t>(1, blocks), st));
  } else if (cols >= 32) {  // one warp per row, direct 256-bit loads
    t->seg_warp(p, sms, st);
  } else {           // G lanes per row, G = the power of two >= cols (capped at 16)
    int G = 1;
    while (G < cols && G < 16) G <<= 1;
    const int64_t rows_per_block = 256 / G;
    const int64_t blocks = std::min<int64_t>((rows + rows_per_block - 1) / rows_per_block, (int64_t)sms * 8);
    t->seg_group(p, G, (int)std::max<int64_t>(1, blocks), st);
  }
  CK(cudaGetLastError());
  return IPM_OK;
}

// ---------------------------------------------------------------------------------- two-level pieces
ipm_status ipm_reduce_partials(ipm_op op, ipm_dtype dt, const void* dev, int64_t n, void* dev_partials,
                               int max_partials, int* count, void* stream) {
  ipm_status s;
  if ((s = validate(op, dt)) || (s = check_array(dt, dev, n))) return s;
  if (!dev_partials || !count) {
    set_error("NULL pointer");
    return IPM_E_NULL;
  }
  const int g = (int)flat_grid(dt, n);
  if (max_partials < g) {
    set_error("max_partials smaller than the grid (query ipm_flat_geometry)");
    return IPM_E_SIZE;
  }
  FlatParams p;
  p.a = dev;
  p.n = n;
  p.row_stride = 0;
  p.init = 0;
  p.has_init = 0;
  p.mode = MODE_CTA_PARTIALS;
  p.out = dev_partials;
  p.partials = nullptr;
  p.tickets = nullptr;
  p.counter = nullptr;
  p.packed = nullptr;
  p.done = nullptr;
  p.max_chunks = 0;
  p.peers = nullptr;
  p.rank = 0;
  p.world = 1;
  p.timeout_ns = 0;
  cudaStream_t st = (cudaStream_t)stream;
  {
    ProfScope ps(st, 0);
    table(op, dt)->flat(p, dim3((unsigned)g, 1, 1), st);
  }
  CK(cudaGetLastError());
  *count = g;
  return IPM_OK;
}

ipm_status ipm_finalize_partials(ipm_op op, ipm_dtype dt, const void* dev_partials, int count, const void* init,
                                 void* dev_result, void* stream) {
  ipm_status s;
  if ((s = validate(op, dt))) return s;
  if ((count > 0 && !dev_partials) || !dev_result) {
    set_error("NULL pointer");
    return IPM_E_NULL;
  }
  if (count < 0) {
    set_error("negative count");
    return IPM_E_SIZE;
  }
  return launch_finalize(op, dt, (const uint64_t*)dev_partials, count, scalar_bits(dt, init), init != nullptr,
                         dev_result, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------------- ragged rows
ipm_status ipm_reduce_ragged(ipm_op op, ipm_dtype dt, const void* dev, const int64_t* dev_offsets, int64_t rows,
                             const void* init, void* dev_out, void* ws, void* stream) {
  ipm_status s;
  if ((s = validate(op, dt)) || (s = check_ws(ws))) return s;
  if (rows < 0) {
    set_error("negative row count");
    return IPM_E_SIZE;
  }
  if (rows == 0) return IPM_OK;
  if (rows >= INT32_MAX) {
    set_error("ragged: at most 2^31-2 rows");
    return IPM_E_SIZE;
  }
  if (!dev_offsets || !dev_out) {
    set_error("NULL device pointer");
    return IPM_E_NULL;
  }
  if (((uintptr_t)dev_out % esize(dt)) || (dev && ((uintptr_t)dev % esize(dt))) || ((uintptr_t)dev_offsets & 7u)) {
    set_error("device pointer not aligned to its element size");
    return IPM_E_ALIGN;
  }
  RaggedParams p;
  p.a = dev;
  p.off = dev_offsets;
  p.rows = rows;
  p.init = scalar_bits(dt, init);
  p.has_init = init != nullptr;
  p.out = dev_out;
  p.gate = 0;
  p.gate_len = 0;
  p.nw_dev = nullptr;
  const int kopt = g_opt_ragged_kernel.load(std::memory_order_relaxed);
  const int kern = kopt;  // 0 auto: the warp kernel or, for long rows, the lane-per-row kernel (gated on device)
  const Table* tb = table(op, dt);
  const int64_t nw = kern <= 1 ? tb->ragged_vec_warps(sm_count())  // one wave of the warp kernel's CTAs
                     : kern == 4 ? std::min<int64_t>((int64_t)sm_count() * 32, WS_MAX_RAGGED_WARPS)  // 8 CTAs x 4 warps per SM
                     : kern == 3 ? (int64_t)std::min<int64_t>((int64_t)sm_count() * tb->ragged_rank_ctas_per_sm(),
                                                              WS_MAX_RAGGED_WARPS / IPM_RR_WARPS) *
                                           IPM_RR_WARPS  // one wave of CTAs
                                 : std::min<int64_t>((int64_t)sm_count() * 4, WS_MAX_RAGGED_WARPS);  // 4 CTAs per SM
  int64_t* base = (int64_t*)((char*)ws + WS_RAGGED);
  p.head_row = base;
  p.head_part = (uint64_t*)(base + WS_MAX_RAGGED_WARPS);
  p.tail_row = base + 2 * WS_MAX_RAGGED_WARPS;
  p.tail_part = (uint64_t*)(base + 3 * WS_MAX_RAGGED_WARPS);
  cudaStream_t st = (cudaStream_t)stream;
  {
    ProfScope ps(st, 4);
    if (kern == 0) tb->ragged_auto(p, sm_count(), st);
    else if (kern == 1) tb->ragged(p, (int)(nw / 4), nw, st);
    else if (kern == 3) tb->ragged_rank(p, (int)(nw / IPM_RR_WARPS), nw, st);
    else if (kern == 4) tb->ragged_lpr(p, (int)(nw / IPM_LP_WARPS), nw, st);

    else CK(tb->ragged_tile(p, (int)nw, st));
  }
  CK(cudaGetLastError());
  return IPM_OK;
}

// marked rows: scratch = [bitmap words][chunk counts], each section 256-byte aligned; bounds from the element
// array's length (positions relative to the chunk origin G >= off[0] - 7 reach at most nvalues + 7)
static size_t rmk_bits_bytes(int64_t nvalues) { return (((size_t)(nvalues + 64) / 32 + 1) * 4 + 255) & ~(size_t)255; }
static size_t rmk_cnt_bytes(ipm_dtype dt, int64_t nvalues) {
  const int64_t ch = 32 * 32 / (int64_t)esize(dt) * 2;  // the marked kernel's smallest chunk (2 vectors per lane)
  return (((size_t)((nvalues + 64) / ch + 2)) * 4 + 255) & ~(size_t)255;
}
static size_t rmk_ebits_bytes(int64_t rows) { return (((size_t)(rows + 31) / 32 + 1) * 4 + 255) & ~(size_t)255; }
size_t ipm_ragged_scratch_bytes(ipm_dtype dt, int64_t nvalues, int64_t rows) {
  if (nvalues < 0 || rows < 0 || esize(dt) == 0) return 0;
  return rmk_bits_bytes(nvalues) + rmk_cnt_bytes(dt, nvalues) + rmk_ebits_bytes(rows);
}

ipm_status ipm_reduce_ragged_marked(ipm_op op, ipm_dtype dt, const void* dev, int64_t nvalues,
                                    const int64_t* dev_offsets, int64_t rows, const void* init, void* dev_out,
                                    void* ws, void* scratch, size_t scratch_bytes, void* stream) {
  ipm_status s;
  if ((s = validate(op, dt)) || (s = check_ws(ws))) return s;
  if (rows < 0 || nvalues < 0) {
    set_error("negative row or element count");
    return IPM_E_SIZE;
  }
  if (rows == 0) return IPM_OK;
  if (rows >= INT32_MAX) {
    set_error("ragged: at most 2^31-2 rows");
    return IPM_E_SIZE;
  }
  if (!dev_offsets || !dev_out || !scratch || (!dev && nvalues > 0)) {
    set_error("NULL device pointer");
    return IPM_E_NULL;
  }
  if (((uintptr_t)dev_out % esize(dt)) || (dev && ((uintptr_t)dev % esize(dt))) || ((uintptr_t)dev_offsets & 7u) ||
      ((uintptr_t)scratch & 255u)) {
    set_error("device pointer not aligned to its element size (scratch: 256 bytes)");
    return IPM_E_ALIGN;
  }
  if (scratch_bytes < ipm_ragged_scratch_bytes(dt, nvalues, rows)) {
    set_error("ragged scratch smaller than ipm_ragged_scratch_bytes(dt, nvalues, rows)");
    return IPM_E_WORKSPACE;
  }
  RaggedParams p;
  p.a = dev;
  p.off = dev_offsets;
  p.rows = rows;
  p.init = scalar_bits(dt, init);
  p.has_init = init != nullptr;
  p.out = dev_out;
  p.gate = 0;
  p.gate_len = 0;
  p.nw_dev = nullptr;
  int64_t* base = (int64_t*)((char*)ws + WS_RAGGED);
  p.head_row = base;
  p.head_part = (uint64_t*)(base + WS_MAX_RAGGED_WARPS);
  p.tail_row = base + 2 * WS_MAX_RAGGED_WARPS;
  p.tail_part = (uint64_t*)(base + 3 * WS_MAX_RAGGED_WARPS);
  RaggedMarks m;
  m.bits = (uint32_t*)scratch;
  m.cnt = (uint32_t*)((char*)scratch + rmk_bits_bytes(nvalues));
  m.nwords = (int64_t)(rmk_bits_bytes(nvalues) / 4);
  m.nchunks = (int64_t)(rmk_cnt_bytes(dt, nvalues) / 4);
  m.ebits = (uint32_t*)((char*)m.cnt + rmk_cnt_bytes(dt, nvalues));
  m.newords = (int64_t)(rmk_ebits_bytes(rows) / 4);
  const Table* tb = table(op, dt);
  const int64_t nw = tb->ragged_mk_warps(sm_count());
  cudaStream_t st = (cudaStream_t)stream;
  {
    ProfScope ps(st, 4);
    CK(tb->ragged_mk(p, m, rmk_bits_bytes(nvalues) + rmk_cnt_bytes(dt, nvalues), sm_count(), nw, st));
  }
  CK(cudaGetLastError());
  return IPM_OK;
}

// ---------------------------------------------------------------------------------- 2-D collapse
ipm_status ipm_reduce_2d_async(ipm_op op, ipm_dtype dt, const void* dev, int64_t rows, int64_t cols,
                               int64_t row_stride, const void* init, void* dev_result, void* ws, void* stream) {
  ipm_status s;
  if ((s = validate(op, dt)) || (s = check_ws(ws))) return s;
  if (rows < 0 || cols < 0 || row_stride < cols) {
    set_error("need rows >= 0, cols >= 0, row_stride >= cols");
    return IPM_E_SIZE;
  }
  if (row_stride > 0 && rows > 0 && (rows - 1) > (INT64_MAX - cols) / row_stride) {
    set_error("rows*row_stride overflows");
    return IPM_E_SIZE;
  }
  if (rows * cols > 0 && !dev) {
    set_error("NULL device array");
    return IPM_E_NULL;
  }
  if (!dev_result) {
    set_error("NULL dev_result");
    return IPM_E_NULL;
  }
  if (dev && ((uintptr_t)dev % esize(dt))) {
    set_error("device array not aligned to its element size");
    return IPM_E_ALIGN;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t ib = scalar_bits(dt, init);
  if (rows == 0 || cols == 0) return launch_finalize(op, dt, nullptr, 0, ib, init != nullptr, dev_result, st);
  if (row_stride == cols || rows == 1)  // contiguous region: the flat clause
    return launch_flat(op, dt, dev, rows * cols, ib, init != nullptr, MODE_RESULT, dev_result, ws, st);
  Params2D q;
  q.f.a = dev;
  q.f.n = 0;
  q.f.row_stride = 0;
  q.f.init = ib;
  q.f.has_init = init != nullptr;
  q.f.mode = MODE_RESULT;
  q.f.out = dev_result;
  q.f.partials = (uint64_t*)((char*)ws + WS_PARTIALS);
  q.f.tickets = (unsigned*)((char*)ws + WS_TICKETS);
  q.f.counter = nullptr;
  q.f.packed = (unsigned long long*)((char*)ws + WS_PACKED);
  q.f.done = nullptr;
  q.f.max_chunks = 0;
  q.f.peers = nullptr;
  q.f.rank = 0;
  q.f.world = 1;
  q.f.timeout_ns = 0;
  q.rows = rows;
  q.cols = cols;
  q.row_stride = row_stride;
  const int64_t vw = 32 / (int64_t)esize(dt), chv = 32 * 4;
  const int64_t per_row = std::max<int64_t>(1, (cols / vw + chv - 1) / chv);
  const int64_t items = rows * per_row;
  const int64_t item_grid = std::min<int64_t>(INT32_MAX, (items + FLAT_BLOCK / 32 - 1) / (FLAT_BLOCK / 32));
  {
    ProfScope ps(st, 3);
    table(op, dt)->two_d(q, (int)item_grid, sm_count(), st);
  }
  CK(cudaGetLastError());
  return IPM_OK;
}

ipm_status ipm_reduce_2d(ipm_op op, ipm_dtype dt, const void* dev, int64_t rows, int64_t cols, int64_t row_stride,
                         void* inout, void* ws, void* stream) {
  if (!inout) {
    set_error("NULL inout");
    return IPM_E_NULL;
  }
  void *mh, *md;
  ipm_status s = result_mailbox(&mh, &md);
  if (s) return s;
  if ((s = ipm_reduce_2d_async(op, dt, dev, rows, cols, row_stride, inout, md, ws, stream))) return s;
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  memcpy(inout, mh, esize(dt));
  return IPM_OK;
}

// ---------------------------------------------------------------------------------- fused (multi-variable)
int ipm_fused_nvars(ipm_fused f) { return fused_nvars(f); }

ipm_status ipm_reduce_fused_async(ipm_fused f, ipm_dtype dt, const void* x, const void* y, int64_t n,
                                  const void* init, void* dev_result, void* ws, void* stream) {
  ipm_status s;
  const int nv = fused_nvars(f);
  if (!nv) {
    set_error("unknown fused signature");
    return IPM_E_ARG;
  }
  if (!esize(dt)) {
    set_error("unknown dtype");
    return IPM_E_DTYPE;
  }
  if ((s = check_array(dt, x, n)) || (s = check_ws(ws))) return s;
  if (f == IPM_FUSED_DOT && (s = check_array(dt, y, n))) return s;
  if (!dev_result) {
    set_error("NULL dev_result");
    return IPM_E_NULL;
  }
  FusedParams p;
  p.x = x;
  p.y = f == IPM_FUSED_DOT ? y : nullptr;
  p.n = n;
  for (int v = 0; v < 4; ++v) p.init[v] = v < nv && init ? scalar_bits(dt, (const char*)init + v * esize(dt)) : 0;
  p.has_init = init != nullptr;
  p.out = dev_result;
  p.partials = (uint64_t*)((char*)ws + WS_PARTIALS);
  p.ticket = (unsigned*)((char*)ws + WS_TICKETS);
  const bool vec = f != IPM_FUSED_DOT || (((uintptr_t)x & 31u) == ((uintptr_t)y & 31u));
  int grid = (int)flat_grid(dt, n);
  if (!vec) grid = (int)std::max<int64_t>(1, std::min<int64_t>(grid, (n + FLAT_BLOCK - 1) / FLAT_BLOCK));
  cudaStream_t st = (cudaStream_t)stream;
  {
    ProfScope ps(st, 2);
    switch (dt) {
      case IPM_I32: FusedLaunch<IPM_I32>::launch(f, p, vec, grid, st); break;
      case IPM_I64: FusedLaunch<IPM_I64>::launch(f, p, vec, grid, st); break;
      case IPM_F32: FusedLaunch<IPM_F32>::launch(f, p, vec, grid, st); break;
      case IPM_F64: FusedLaunch<IPM_F64>::launch(f, p, vec, grid, st); break;
    }
  }
  CK(cudaGetLastError());
  return IPM_OK;
}

ipm_status ipm_reduce_fused(ipm_fused f, ipm_dtype dt, const void* x, const void* y, int64_t n, void* inout,
                            void* ws, void* stream) {
  if (!inout) {
    set_error("NULL inout");
    return IPM_E_NULL;
  }
  void *mh, *md;
  ipm_status s = result_mailbox(&mh, &md);
  if (s) return s;
  if ((s = ipm_reduce_fused_async(f, dt, x, y, n, inout, md, ws, stream))) return s;
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  memcpy(inout, mh, esize(dt) * fused_nvars(f));  // <= 4 variables x 8 bytes
  return IPM_OK;
}

// ---------------------------------------------------------------------------------- host streaming
ipm_status ipm_release_staging(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  return release_staging_locked();
}

}  // extern "C"

namespace ipm {
// copyin fused with the reduction: the host array streams through two staging buffers (H2D of chunk c+1 on a
// copy stream overlapping the kernel of chunk c); each chunk's kernel folds into the running accumulator at
// ws + WS_ACC (MODE_ACCUM), so the partial of the whole array stays on the device
ipm_status stream_host_partial(ipm_op op, ipm_dtype dt, const void* host, int64_t n, void* ws, cudaStream_t st) {
  ipm_status s;
  const size_t es = esize(dt);
  uint64_t* acc = (uint64_t*)((char*)ws + WS_ACC);
  std::lock_guard<std::mutex> lk(g_mu);
  if (n == 0) return launch_flat(op, dt, nullptr, 0, 0, 0, MODE_ACCUM_FIRST, acc, ws, st);  // identity
  const size_t chunk_bytes = (size_t)std::max(1, env_int("IPM_STAGE_MB", 64)) << 20;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (g_stage.device != dev || g_stage.bytes != chunk_bytes) {
    release_staging_locked();
    CK(cudaStreamCreateWithFlags(&g_stage.copy, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&g_stage.copied[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&g_stage.consumed[i], cudaEventDisableTiming));
      g_stage.buf[i] = dev_alloc(chunk_bytes, g_stage.copy);
      if (!g_stage.buf[i]) {
        release_staging_locked();
        set_error("staging allocation failed");
        return IPM_E_CUDA;
      }
    }
    CK(cudaStreamSynchronize(g_stage.copy));
    g_stage.bytes = chunk_bytes;
    g_stage.device = dev;
  }
  const int64_t per = (int64_t)(chunk_bytes / es);
  // The staging buffers are shared by every caller (the lock covers enqueueing only, not execution): a buffer is
  // free once the previous caller's last kernel that read it has run (consumed[i], recorded on THAT caller's
  // stream) and everything queued earlier on `st` has run. `st` waits for the former, then consumed[i] is
  // re-recorded on `st` so the copies below wait for both.
  for (int i = 0; i < 2; ++i) {
    CK(cudaStreamWaitEvent(st, g_stage.consumed[i], 0));
    CK(cudaEventRecord(g_stage.consumed[i], st));
  }
  int64_t c = 0;
  for (int64_t off = 0; off < n; off += per, ++c) {
    const int b = (int)(c & 1);
    const int64_t cnt = std::min(per, n - off);
    CK(cudaStreamWaitEvent(g_stage.copy, g_stage.consumed[b], 0));
    CK(cudaMemcpyAsync(g_stage.buf[b], (const char*)host + off * es, cnt * es, cudaMemcpyHostToDevice,
                       g_stage.copy));
    CK(cudaEventRecord(g_stage.copied[b], g_stage.copy));
    CK(cudaStreamWaitEvent(st, g_stage.copied[b], 0));
    if ((s = launch_flat(op, dt, g_stage.buf[b], cnt, 0, 0, c == 0 ? MODE_ACCUM_FIRST : MODE_ACCUM, acc, ws, st)))
      return s;
    CK(cudaEventRecord(g_stage.consumed[b], st));
  }
  return IPM_OK;
}
}  // namespace ipm

extern "C" {

ipm_status ipm_reduce_host(ipm_op op, ipm_dtype dt, const void* host, int64_t n, void* inout, void* ws,
                           void* stream) {
  ipm_status s;
  if ((s = validate(op, dt)) || (s = check_ws(ws))) return s;
  if (n < 0) {
    set_error("negative element count");
    return IPM_E_SIZE;
  }
  if (!inout || (n > 0 && !host)) {
    set_error("NULL host pointer");
    return IPM_E_NULL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  void *mh, *md;
  if ((s = result_mailbox(&mh, &md))) return s;
  if ((s = stream_host_partial(op, dt, host, n, ws, st))) return s;
  if ((s = launch_finalize(op, dt, (const uint64_t*)((char*)ws + WS_ACC), 1, scalar_bits(dt, inout), 1, md, st)))
    return s;
  CK(cudaStreamSynchronize(st));
  memcpy(inout, mh, esize(dt));
  return IPM_OK;
}

// ---------------------------------------------------------------------------------- data environment
static ipm_status present_insert(const void* host, size_t bytes, void** dev, void* stream, bool copy) {
  if (!host || !dev) {
    set_error("NULL pointer");
    return IPM_E_NULL;
  }
  if (bytes == 0) {
    set_error("zero-byte data clause (size unknown)");
    return IPM_E_SIZE;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  const uintptr_t h = (uintptr_t)host;
  auto it = find_cover(h, bytes);
  if (it != g_present.end()) {  // already present: reference only (OpenACC present-or semantics)
    it->second.ref++;
    *dev = (char*)it->second.dev + (h - it->first);
    return IPM_OK;
  }
  // a partial overlap with a live entry is an error (the OpenACC runtime forbids it)
  auto nx = g_present.lower_bound(h);
  if (nx != g_present.end() && nx->first < h + bytes) {
    set_error("data clause range partially overlaps a present range");
    return IPM_E_PRESENT;
  }
  if (nx != g_present.begin()) {
    auto pv = std::prev(nx);
    if (pv->first + pv->second.bytes > h) {
      set_error("data clause range partially overlaps a present range");
      return IPM_E_PRESENT;
    }
  }
  cudaStream_t st = (cudaStream_t)stream;
  void* d = dev_alloc(bytes, st);
  if (!d) {
    set_error("device allocation failed");
    return IPM_E_CUDA;
  }
  if (copy) {
    cudaError_t e = cudaMemcpyAsync(d, host, bytes, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      dev_free(d, st);
      return cuda_fail(e, "copyin");
    }
  }
  g_present[h] = Entry{bytes, d, 1};
  *dev = d;
  return IPM_OK;
}

ipm_status ipm_copyin(const void* host, size_t bytes, void** dev, void* stream) {
  return present_insert(host, bytes, dev, stream, true);
}
ipm_status ipm_create(const void* host, size_t bytes, void** dev, void* stream) {
  return present_insert(host, bytes, dev, stream, false);
}

ipm_status ipm_present(const void* host, size_t bytes, void** dev) {
  if (!host || !dev) {
    set_error("NULL pointer");
    return IPM_E_NULL;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = find_cover((uintptr_t)host, bytes);
  if (it == g_present.end()) {
    set_error("no live device copy for this host range");
    return IPM_E_PRESENT;
  }
  *dev = (char*)it->second.dev + ((uintptr_t)host - it->first);
  return IPM_OK;
}

static ipm_status update(void* host, size_t bytes, void* stream, bool to_device) {
  if (!host) {
    set_error("NULL pointer");
    return IPM_E_NULL;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = find_cover((uintptr_t)host, bytes);
  if (it == g_present.end()) {
    set_error("no live device copy for this host range");
    return IPM_E_PRESENT;
  }
  char* d = (char*)it->second.dev + ((uintptr_t)host - it->first);
  cudaStream_t st = (cudaStream_t)stream;
  if (to_device) CK(cudaMemcpyAsync(d, host, bytes, cudaMemcpyHostToDevice, st));
  else CK(cudaMemcpyAsync(host, d, bytes, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return IPM_OK;
}
ipm_status ipm_update_device(const void* host, size_t bytes, void* stream) {
  return update((void*)host, bytes, stream, true);
}
ipm_status ipm_update_host(void* host, size_t bytes, void* stream) { return update(host, bytes, stream, false); }

static ipm_status release(const void* host, size_t bytes, void* stream, bool copy) {
  if (!host) {
    set_error("NULL pointer");
    return IPM_E_NULL;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_present.find((uintptr_t)host);
  if (it == g_present.end()) {
    set_error("no live device copy starting at this host address");
    return IPM_E_PRESENT;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (copy) {
    if (bytes > it->second.bytes) {
      set_error("copyout larger than the present range");
      return IPM_E_SIZE;
    }
    CK(cudaMemcpyAsync((void*)host, it->second.dev, bytes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  if (--it->second.ref == 0) {
    dev_free(it->second.dev, st);
    g_present.erase(it);
  }
  return IPM_OK;
}
ipm_status ipm_copyout(void* host, size_t bytes, void* stream) { return release(host, bytes, stream, true); }
ipm_status ipm_delete(const void* host, void* stream) { return release(host, 0, stream, false); }

int ipm_present_count(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  return (int)g_present.size();
}

}  // extern "C"
