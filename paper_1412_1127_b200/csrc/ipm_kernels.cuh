// ipm_kernels.cuh — the sm_100a kernels of the reduction clause.
//
//   k_flat      the flat clause (and, with gridDim.y > 1, the few-rows / long-rows segmented clause):
//               a3 vector level: grid-stride over 32-byte vector loads (LDG.E.256), VW private accumulators
//                  per thread (SPEC.md:317 private copy, one per vector lane for ILP)
//               a4 warp combine (REDUX/CREDUX or a shuffle butterfly)
//               a5 CTA combine through shared memory ("[Harris 2006]" block tree, one level)
//               a6 cross-CTA finish: per-CTA partial + ticket; the last CTA folds the partials in index
//                  order (deterministic) and merges the variable's original value ("merges
//                  results across different thread blocks"; PAPER.md:205 does this on the host — see
//                  DESIGN.md "What differs from the paper")
//   k_2d        one scalar over a strided 2-D region (collapsed gang x vector loops)
//   k_seg_warp  the nested gang-outer / vector-inner clause, one warp per row (a8)
//   k_seg_tma   the same with each row staged into shared memory by TMA bulk copies (per-warp ring)
//   k_seg_group the same for short rows: a group of G <= 32 lanes per row
//   k_finalize  fold of P accumulator slots (cross-rank, or cross-chunk) + init, rounding to T (a6/a9)
#pragma once
#include <type_traits>
#include "ipm_ops.cuh"

namespace ipm {

// ------------------------------------------------------------------------------------------ loads
// 256-bit streaming loads (sm_100: LDG.E.ENL2.256): read-only path, no L1 allocation, evict-first in L2,
// 256-byte L2 prefetch granule. Every input byte is read exactly once, so nothing is worth caching.
struct alignas(32) V8 {
  uint32_t w[8];
};
struct alignas(32) V4 {
  uint64_t w[4];
};
template <class B>
struct Vec;
template <>
struct Vec<uint32_t> {
  using T = V8;
  static constexpr int W = 8;
};
template <>
struct Vec<uint64_t> {
  using T = V4;
  static constexpr int W = 4;
};

// HINT selects the cache policy (tools/sweep_flat.cu measures them; the product uses 0):
//   0 ld.global.nc.L1::no_allocate.L2::evict_first.L2::256B   1 ld.global.nc.L1::no_allocate
//   2 ld.global (plain)                                         3 ld.global.nc.L1::no_allocate.L2::256B
// `asm volatile`: a plain asm statement is a pure function to the compiler, which may then hoist or speculate
// the load past the branch that guards it (observed: a guarded tile load executed for an out-of-range tile).
#define IPM_LDV8(Q)                                                                                   \
  asm volatile(Q ".v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                                                   \
      : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]), "=r"(v.w[6]), \
        "=r"(v.w[7])                                                                                  \
      : "l"(p))
#define IPM_LDV4(Q) \
  asm volatile(Q ".v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(v.w[0]), "=l"(v.w[1]), "=l"(v.w[2]), "=l"(v.w[3]) : "l"(p))
template <int HINT = 0>
__device__ __forceinline__ V8 ldv(const V8* p) {
  V8 v;
  if (HINT == 0) IPM_LDV8("ld.global.nc.L1::no_allocate.L2::evict_first.L2::256B");
  else if (HINT == 1) IPM_LDV8("ld.global.nc.L1::no_allocate");
  else if (HINT == 2) IPM_LDV8("ld.global");
  else IPM_LDV8("ld.global.nc.L1::no_allocate.L2::256B");
  return v;
}
template <int HINT = 0>
__device__ __forceinline__ V4 ldv(const V4* p) {
  V4 v;
  if (HINT == 0) IPM_LDV4("ld.global.nc.L1::no_allocate.L2::evict_first.L2::256B");
  else if (HINT == 1) IPM_LDV4("ld.global.nc.L1::no_allocate");
  else if (HINT == 2) IPM_LDV4("ld.global");
  else IPM_LDV4("ld.global.nc.L1::no_allocate.L2::256B");
  return v;
}
#undef IPM_LDV8
#undef IPM_LDV4
__device__ __forceinline__ uint32_t lds(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint64_t lds(const uint64_t* p) { return (uint64_t)__ldg((const unsigned long long*)p); }

// the cross-CTA ticket: one atomic with release (publishes this CTA's partial, stored before it by the same
// thread) and acquire (makes every earlier CTA's partial visible; __syncthreads then extends that to the CTA)
__device__ __forceinline__ unsigned ticket_acq_rel(unsigned* t) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(t) : "memory");
  return old;
}

// ------------------------------------------------------------------------------------------ params
struct FlatParams {
  const void* a;          // row 0 base
  int64_t n;              // elements per row (flat: the whole array)
  int64_t row_stride;     // elements between rows (gridDim.y rows)
  uint64_t init;          // the variable's original value (element bits), merged when has_init
  int has_init;
  int mode;               // MODE_RESULT: write fin(init ⊕ total) as T to out[row]
                          // MODE_PARTIAL: write pack(total) (no init) to out (8 bytes)
                          // MODE_ACCUM_FIRST / MODE_ACCUM: *acc_slot = total / *acc_slot ⊕= total
  void* out;
  uint64_t* partials;     // gridDim.x * gridDim.y slots (unused when gridDim.x == 1)
  unsigned* tickets;      // gridDim.y tickets (unused when gridDim.x == 1); left at zero
  unsigned long long* counter;  // dynamic schedules: tile / chunk counter, left at zero
  unsigned long long* packed;   // int32 +, one row: the CTA count (low word) and the wrapping sum (high word) in
                                // one 64-bit word, left at zero (nullptr: not used)
  unsigned long long* done;     // MODE_RESULT: after the result, done_seq is stored here with system-scope release
  unsigned long long done_seq;  // (the synchronous call's mapped mailbox: the host polls it; nullptr: not used)
  int64_t max_chunks;     // k_flat_guided: partial slots available for dynamic chunks
  // MODE_DIST (multi-GPU, one kernel): the CTA that finishes this rank's shard exchanges the rank partial with
  // every peer through NVLink peer memory (see dist_exchange)
  uint64_t* const* peers; // device array: world pointers to each rank's symmetric slot buffer (own = [rank])
  int rank, world;
  long long timeout_ns;
};
enum { MODE_RESULT = 0, MODE_PARTIAL = 1, MODE_ACCUM_FIRST = 2, MODE_ACCUM = 3, MODE_CTA_PARTIALS = 4, MODE_DIST = 5 };

// symmetric slot buffer layout (uint64 words): [parity 0..1][rank 0..63] x {value, epoch}, then the epoch
// counter and the error flag
constexpr int SYM_RANKS = 64;
constexpr int SYM_EPOCH = 2 * 2 * SYM_RANKS;
constexpr int SYM_ERROR = SYM_EPOCH + 1;
constexpr int SYM_WORDS = SYM_EPOCH + 8;

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long globaltimer_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// a9 fused into the reduction kernel (one thread of the CTA that finished this rank's shard): store the rank's
// accumulator partial into slot [parity][rank] of EVERY rank's symmetric buffer (NVLink peer stores, value then
// epoch with release semantics), wait until all world slots of the own buffer carry this epoch (acquire), fold
// them in rank order, merge the variable's original value and write the result. The epoch is a device-side
// counter in the own buffer (one per call, so the kernel can be captured in a CUDA graph); two parities let a
// fast rank start call e+1 while a slow rank still reads call e. A peer that never arrives sets the error word
// after timeout_ns instead of hanging the GPU.
// (The fields come by value: a reference to the kernel's parameter struct made every kernel copy that struct to
// local memory at entry -- 7-10 MB of DRAM writes per launch over 592 x 256 threads.)
struct DevDistArgs {
  uint64_t* const* peers;
  int rank, world;
  long long timeout_ns;
  uint64_t init;
  int has_init;
  void* out;
};
template <class R>
__device__ __noinline__ void dist_exchange(const DevDistArgs p, typename R::A total) {
  using A = typename R::A;
  using B = typename R::B;
  uint64_t* own = p.peers[p.rank];
  const uint64_t ep = own[SYM_EPOCH] + 1;
  own[SYM_EPOCH] = ep;
  const int base = 2 * (int)(ep & 1u) * SYM_RANKS;
  const uint64_t v = pack(total);
  for (int q = 0; q < p.world; ++q) {
    uint64_t* slot = p.peers[q] + base + 2 * p.rank;
    st_relaxed_sys(slot, v);
    st_release_sys(slot + 1, ep);
  }
  const long long t0 = globaltimer_ns();
  bool timed_out = false;
  for (int q = 0; q < p.world && !timed_out; ++q)
    while (ld_acquire_sys(own + base + 2 * q + 1) != ep) {
      if (globaltimer_ns() - t0 > p.timeout_ns) {
        timed_out = true;
        own[SYM_ERROR] = 1ull;
        break;
      }
    }
  A t = R::id();
  for (int q = 0; q < p.world; ++q) t = R::op(t, unpack<A>(ld_relaxed_sys(own + base + 2 * q)));
  if (p.has_init) t = R::op(R::lift((B)p.init), t);
  *(B*)p.out = R::fin(t);
}

template <class R>
__device__ __forceinline__ void store_out(const FlatParams& p, int64_t row, typename R::A total) {
  using A = typename R::A;
  using B = typename R::B;
  switch (p.mode) {
    case MODE_RESULT: {
      A t = total;
      if (p.has_init) t = R::op(R::lift((B)p.init), total);  // var = var_original ⊕ fold (R1)
      ((B*)p.out)[row] = R::fin(t);
      if (p.done) st_release_sys((uint64_t*)p.done, p.done_seq);  // the result first, then the flag
      break;
    }
    case MODE_PARTIAL: ((uint64_t*)p.out)[row] = pack(total); break;
    case MODE_ACCUM_FIRST: *(uint64_t*)p.out = pack(total); break;
    case MODE_DIST:
      dist_exchange<R>(DevDistArgs{p.peers, p.rank, p.world, p.timeout_ns, p.init, p.has_init, p.out}, total);
      break;
    default: *(uint64_t*)p.out = pack(R::op(unpack<A>(*(uint64_t*)p.out), total)); break;
  }
}

// block-wide ⊕ of one value per thread; result valid in thread 0. `sm` holds BLOCK/32 slots.
template <class R, int BLOCK>
__device__ __forceinline__ typename R::A block_reduce(typename R::A v, typename R::A* sm) {
  using A = typename R::A;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = R::warp(v);
  if (BLOCK == 32) return v;
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  A r = R::id();
  if (warp == 0) {
    r = lane < BLOCK / 32 ? sm[lane] : R::id();
    r = R::warp(r);
  }
  return r;
}

// a6: publish the CTA partial of `row`; the CTA that takes the row's last ticket folds the partials in index
// order (deterministic), merges the original value and stores; the ticket is left at zero for the next launch.
template <class R, int BLOCK>
__device__ __forceinline__ void grid_finish(const FlatParams& p, int64_t row, typename R::A cta, typename R::A* sm) {
  using A = typename R::A;
  __shared__ int s_last;
  if (p.mode == MODE_CTA_PARTIALS) {  // the paper's first level only: one partial per thread block
    if (threadIdx.x == 0) ((uint64_t*)p.out)[blockIdx.x] = pack(cta);
    return;
  }
  if (gridDim.x == 1) {
    if (threadIdx.x == 0) {
      store_out<R>(p, row, cta);
      if (p.counter) *p.counter = 0ull;  // (the single CTA has finished claiming tiles)
    }
    return;
  }
  if constexpr (std::is_same<R, Red<IPM_ADD, IPM_I32>>::value) {
    // int32 + (BASELINE config 1): the CTA's partial rides in the ticket itself, count in the low word and the sum
    // mod 2^32 in the high word of one 64-bit atomic (the count never carries into the sum: at most 2^31 CTAs),
    // so the last CTA has the total without storing and re-loading partials or a CTA reduction: one L2 round trip
    // fewer on the latency-bound small inputs (profiles/r02_c1_breakdown.txt). The sum is exact in any order.
    if (p.packed && gridDim.y == 1) {
      if (threadIdx.x == 0) {
        const unsigned long long old = atomicAdd(p.packed, ((unsigned long long)cta << 32) | 1ull);
        if ((unsigned)old == gridDim.x - 1) {
          *p.packed = 0ull;
          if (p.counter) *p.counter = 0ull;
          store_out<R>(p, row, (A)(old >> 32) + cta);
        }
      }
      return;
    }
  }
  uint64_t* parts = p.partials + row * gridDim.x;
  if (threadIdx.x == 0) {
    __stcg(parts + blockIdx.x, pack(cta));
    s_last = (ticket_acq_rel(p.tickets + row) == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  A v = R::id();
  for (int i = threadIdx.x; i < (int)gridDim.x; i += BLOCK) v = R::op(v, unpack<A>(__ldcg(parts + i)));
  __syncthreads();  // sm reuse
  A total = block_reduce<R, BLOCK>(v, sm);
  if (threadIdx.x == 0) {
    store_out<R>(p, row, total);
    p.tickets[row] = 0u;
    if (p.counter) *p.counter = 0ull;
  }
}

// ------------------------------------------------------------------------------------------ flat
// SCHED: how whole tiles are assigned to CTAs — 0 grid-stride (static, interleaved), 1 one contiguous balanced
// range per CTA, 2 dynamic (an atomic tile counter; absorbs per-SM bandwidth differences). tools/sweep_flat.cu
// measures them.
template <class R, int BLOCK, int U, int HINT = 0, int SCHED = 0>
__global__ void __launch_bounds__(BLOCK, 1024 / BLOCK) k_flat(FlatParams p) {
  using B = typename R::B;
  using A = typename R::A;
  using VT = typename Vec<B>::T;
  constexpr int VW = Vec<B>::W;
  constexpr int64_t TILE = (int64_t)BLOCK * U;
  __shared__ A sm[BLOCK / 32 > 0 ? BLOCK / 32 : 1];

  const int64_t row = blockIdx.y;
  const B* a = (const B*)p.a + row * p.row_stride;
  const int64_t n = p.n;
  // head: elements before the first 32-byte boundary; body: nv whole vectors; tail: the rest
  const uintptr_t addr = (uintptr_t)a;
  int64_t head = (int64_t)(((32u - (addr & 31u)) & 31u) / sizeof(B));
  if (head > n) head = n;
  const int64_t nv = (n - head) / VW;
  const int64_t tail0 = head + nv * VW;
  const VT* vp = (const VT*)(a + head);

  using LC = Loc<R>;
  using L = typename LC::L;
  L acc[VW];
#pragma unroll
  for (int k = 0; k < VW; ++k) acc[k] = LC::id();

  // a3: the hot loop — whole tiles of BLOCK*U vectors, U independent 256-bit loads in flight per thread
  const int64_t ntiles = nv / TILE;
  auto tile = [&](int64_t t) {
    const VT* base = vp + t * TILE + threadIdx.x;
    VT v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldv<HINT>(base + u * BLOCK);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      LC::vec(acc, v[u]);
  };
  if (SCHED == 0) {
    #pragma unroll 1
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) tile(t);
  } else if (SCHED == 3) {  // static grid-stride, software-pipelined: the next tile's loads are issued first
    int64_t t = blockIdx.x;
    VT nx[U];
    if (t < ntiles) {
#pragma unroll
      for (int u = 0; u < U; ++u) nx[u] = ldv<HINT>(vp + t * TILE + threadIdx.x + u * BLOCK);
    }
    #pragma unroll 1
    for (; t < ntiles; t += gridDim.x) {
      VT cu[U];
#pragma unroll
      for (int u = 0; u < U; ++u) cu[u] = nx[u];
      const int64_t tn = t + gridDim.x;
      if (tn < ntiles) {
#pragma unroll
        for (int u = 0; u < U; ++u) nx[u] = ldv<HINT>(vp + tn * TILE + threadIdx.x + u * BLOCK);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        LC::vec(acc, cu[u]);
    }
  } else if (SCHED == 1) {
    const int64_t t1 = (ntiles * (blockIdx.x + 1)) / gridDim.x;
    #pragma unroll 1
    for (int64_t t = (ntiles * blockIdx.x) / gridDim.x; t < t1; ++t) tile(t);
  } else {
    __shared__ long long s_next;
    int64_t t = blockIdx.x;
    while (t < ntiles) {
      if (threadIdx.x == 0) s_next = (long long)atomicAdd(p.counter, 1ull) + gridDim.x;
      tile(t);
      __syncthreads();
      t = s_next;
      __syncthreads();
    }
  }
  // ragged last tile
  for (int64_t i = ntiles * TILE + (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * BLOCK) {
    const VT v = ldv<HINT>(vp + i);
#pragma unroll
    LC::vec(acc, v);
  }
  // head and tail scalars (< VW each)
  const int64_t g = (int64_t)blockIdx.x * BLOCK + threadIdx.x;
  if (g < head) acc[0] = LC::step(acc[0], lds(a + g));
  if (g < n - tail0) acc[VW - 1] = LC::step(acc[VW - 1], lds(a + tail0 + g));

  // fold the private copies in a fixed tree
#pragma unroll
  for (int s = VW / 2; s > 0; s >>= 1)
#pragma unroll
    for (int k = 0; k < s; ++k) acc[k] = LC::comb(acc[k], acc[k + s]);

  // a4 + a5
  A cta = block_reduce<R, BLOCK>(LC::out(acc[0]), sm);
  grid_finish<R, BLOCK>(p, row, cta, sm);
}

// ------------------------------------------------------------------------------------------ flat, guided
// Deterministic AND load-balanced schedule ("guided self-scheduling"): about 90% of the tiles are dealt
// statically, grid-stride (CTA b folds tiles b, b+G, b+2G, ... into partial slot b); the rest is cut into K
// fixed chunks of ct contiguous tiles that CTAs claim from an atomic counter as they finish (chunk c ->
// partial slot G + c), and one last "chunk" K holds the ragged remainder (vectors past the last whole tile,
// head and tail scalars). Every slot's value depends only on its element range and the fixed thread mapping —
// not on which CTA computed it — and the last CTA folds the G + K + 1 slots in slot order, so the result is
// bit-identical run to run while fast SMs absorb the slow ones' share of the tail.
template <class R, int BLOCK, int U, bool PIPE = false>
__global__ void __launch_bounds__(BLOCK, 1024 / BLOCK) k_flat_guided(FlatParams p) {
  using B = typename R::B;
  using A = typename R::A;
  using VT = typename Vec<B>::T;
  constexpr int VW = Vec<B>::W;
  constexpr int64_t TILE = (int64_t)BLOCK * U;
  __shared__ A sm[BLOCK / 32];
  __shared__ long long s_c;
  __shared__ int s_last;
  const B* a = (const B*)p.a;
  const int64_t n = p.n;
  const uintptr_t addr = (uintptr_t)a;
  int64_t head = (int64_t)(((32u - (addr & 31u)) & 31u) / sizeof(B));
  if (head > n) head = n;
  const int64_t nv = (n - head) / VW;
  const int64_t tail0 = head + nv * VW;
  const VT* vp = (const VT*)(a + head);
  const int64_t ntiles = nv / TILE;
  const int64_t G = gridDim.x;
  const int64_t srounds = (ntiles - ntiles / 10) / G;   // static rounds per CTA (~90% of the tiles)
  const int64_t dyn0 = srounds * G;
  const int64_t rem = ntiles - dyn0;
  const int64_t max_chunks = p.max_chunks > 0 ? p.max_chunks : 1;
  // tiles per dynamic chunk: enough chunks to balance; >= 4 tiles each to amortise the per-chunk block
  // reduction when there are at least 4 such chunks per CTA (tools/sweep_flat.cu "chunks": 1-tile chunks cost
  // 2.6% at 1 GiB), single tiles for small inputs (few chunks would leave most CTAs idle)
  int64_t ct = rem > 0 ? (rem + max_chunks - 1) / max_chunks : 1;
  if (ct < 4 && rem >= 4 * G) ct = 4;
  const int64_t K = (rem + ct - 1) / ct;                 // dynamic chunks 0..K-1; chunk K = the remainder
  uint64_t* slots = p.partials;

  using LC = Loc<R>;
  using L = typename LC::L;
  L acc[VW];
  auto reset = [&]() {
#pragma unroll
    for (int k = 0; k < VW; ++k) acc[k] = LC::id();
  };
  auto tile = [&](int64_t t) {
#ifdef IPM_GUIDED_DEBUG
    if (t < 0 || t >= ntiles) {
      printf("OOB tile %lld ntiles %lld block %d thread %d G %lld srounds %lld K %lld ct %lld dyn0 %lld\n",
             (long long)t, (long long)ntiles, blockIdx.x, threadIdx.x, (long long)G, (long long)srounds,
             (long long)K, (long long)ct, (long long)dyn0);
      __trap();
    }
#endif
    const VT* base = vp + t * TILE + threadIdx.x;
    VT v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldv(base + u * BLOCK);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      LC::vec(acc, v[u]);
  };
  auto publish = [&](int64_t slot) {  // fixed tree: VW lanes -> warp -> CTA; one slot per element range
#pragma unroll
    for (int s2 = VW / 2; s2 > 0; s2 >>= 1)
#pragma unroll
      for (int k = 0; k < s2; ++k) acc[k] = LC::comb(acc[k], acc[k + s2]);
    const A t = block_reduce<R, BLOCK>(LC::out(acc[0]), sm);
    if (threadIdx.x == 0) __stcg(slots + slot, pack(t));
    __syncthreads();  // sm reuse
  };

  // static part
  // fold tiles first, first + stride, ... (count of them) with the next tile's loads issued before the
  // current tile is folded (software pipelining: loads stay in flight while the previous tile is consumed)
  auto run = [&](int64_t first, int64_t stride, int64_t count) {
    if (count <= 0) return;
    VT nx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) nx[u] = ldv(vp + first * TILE + threadIdx.x + u * BLOCK);
#pragma unroll 1
    for (int64_t k = 0; k < count; ++k) {
      VT cu[U];
#pragma unroll
      for (int u = 0; u < U; ++u) cu[u] = nx[u];
      if (k + 1 < count) {
        const int64_t tn = first + (k + 1) * stride;
#pragma unroll
        for (int u = 0; u < U; ++u) nx[u] = ldv(vp + tn * TILE + threadIdx.x + u * BLOCK);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        LC::vec(acc, cu[u]);
    }
  };
  reset();
  if (PIPE) run(blockIdx.x, G, srounds);
  else
    for (int64_t k = 0; k < srounds; ++k) tile(blockIdx.x + k * G);
  if (threadIdx.x == 0) s_c = (long long)atomicAdd(p.counter, 1ull);  // claim the first dynamic chunk
  publish(blockIdx.x);
  long long c = s_c;
  // dynamic part: chunks claimed until the counter passes the remainder chunk
  while (c <= K) {
    __syncthreads();  // everyone has read s_c
    if (threadIdx.x == 0) s_c = (long long)atomicAdd(p.counter, 1ull);  // claim the next chunk early
    reset();
    if (c < K) {
      const int64_t e1 = dyn0 + (int64_t)(c + 1) * ct;
      const int64_t t1 = e1 < ntiles ? e1 : ntiles;
      const int64_t t0 = dyn0 + (int64_t)c * ct;
      if (PIPE) run(t0, 1, t1 - t0);
      else
        for (int64_t t = t0; t < t1; ++t) tile(t);
    } else {
      for (int64_t i = ntiles * TILE + threadIdx.x; i < nv; i += BLOCK) {
        const VT v = ldv(vp + i);
#pragma unroll
        LC::vec(acc, v);
      }
      if (threadIdx.x < head) acc[0] = LC::step(acc[0], lds(a + threadIdx.x));
      if (threadIdx.x < n - tail0) acc[VW - 1] = LC::step(acc[VW - 1], lds(a + tail0 + threadIdx.x));
    }
    publish(G + c);
    c = s_c;
  }
  // the CTA that takes the last ticket folds all slots (fixed thread -> slot mapping and tree)
  if (threadIdx.x == 0) s_last = ticket_acq_rel(p.tickets) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  const int64_t nslots = G + K + 1;
  // thousands of slots: 8 independent loads in flight per thread (a dependent load-op chain would cost one L2
  // round trip per slot); fixed thread -> slot mapping and combine order
  A v8[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v8[j] = R::id();
  int64_t i = threadIdx.x;
  for (; i + 7 * BLOCK < nslots; i += 8 * BLOCK) {
    uint64_t w[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) w[j] = __ldcg(slots + i + j * BLOCK);
#pragma unroll
    for (int j = 0; j < 8; ++j) v8[j] = R::op(v8[j], unpack<A>(w[j]));
  }
  for (int j = 0; i < nslots; i += BLOCK, ++j) v8[j & 7] = R::op(v8[j & 7], unpack<A>(__ldcg(slots + i)));
#pragma unroll
  for (int j = 1; j < 8; ++j) v8[0] = R::op(v8[0], v8[j]);
  const A total = block_reduce<R, BLOCK>(v8[0], sm);
  if (threadIdx.x == 0) {
    store_out<R>(p, 0, total);
    *p.tickets = 0u;
    *p.counter = 0ull;
  }
}

// L2 prefetch of a byte range (one bulk-prefetch instruction; only the 16-byte-aligned interior is named, so
// nothing outside [p, p + bytes) is touched). Issued by one lane for data the warp reads next.
__device__ __forceinline__ void l2_prefetch(const void* p, int64_t bytes) {
  const uintptr_t b0 = ((uintptr_t)p + 15u) & ~(uintptr_t)15u;
  const uintptr_t b1 = ((uintptr_t)p + (uintptr_t)bytes) & ~(uintptr_t)15u;
  if (bytes > 0 && b1 > b0) {
    const uint64_t nb = b1 - b0;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b0), "r"((uint32_t)(nb < 0xFFFFFFF0ull ? nb : 0xFFFFFFF0ull))
                 : "memory");
  }
}

// ------------------------------------------------------------------------------------------ 2-D collapse
// One scalar over a strided 2-D region (a gang loop over rows collapsed with the
// vector loop over columns, rows not contiguous when row_stride > cols): work items are (row, chunk of
// 32*U vectors) pairs taken by warps in grid-stride order, so few long rows and many short rows both spread
// over the whole GPU; each row peels its own head/tail to 32-byte alignment. Then a4-a6 as in k_flat.
struct Params2D {
  FlatParams f;   // f.a = base, f.n unused
  int64_t rows, cols, row_stride;
};
template <class R, int BLOCK, int U, int PF = 0, int MINB = 1024 / BLOCK>
__global__ void __launch_bounds__(BLOCK, MINB) k_2d(Params2D q) {
  using B = typename R::B;
  using A = typename R::A;
  using VT = typename Vec<B>::T;
  constexpr int VW = Vec<B>::W;
  constexpr int64_t CHV = 32 * U;  // vectors per work item
  __shared__ A sm[BLOCK / 32];
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * (BLOCK / 32) + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * (BLOCK / 32);
  // vectors per row is the same for every row only if all rows share the alignment; take the maximum
  // (head = 0) and let rows with a head skip their last partial vector through the bounds check
  const int64_t maxv = q.cols / VW;
  const int64_t per_row = maxv > 0 ? (maxv + CHV - 1) / CHV : 1;
  const int64_t items = q.rows * per_row;
  // item it = (row r, chunk c), it = r * per_row + c, stepped by nw without a division per item
  const int64_t dr = nw / per_row, dc = nw - dr * per_row;
  int64_t r = gw / per_row, c = gw - r * per_row;
  using LC = Loc<R>;
  using L = typename LC::L;
  L acc[VW];
#pragma unroll
  for (int k = 0; k < VW; ++k) acc[k] = LC::id();
  for (int64_t it = gw; it < items; it += nw) {
    if (PF && lane == 0 && it + nw < items) {  // the warp's next item (row, chunk) into L2
      int64_t rn = r + dr, cn = c + dc;
      if (cn >= per_row) {
        cn -= per_row;
        ++rn;
      }
      const int64_t e0 = cn * CHV * VW, e1 = e0 + CHV * VW + VW;
      l2_prefetch((const B*)q.f.a + rn * q.row_stride + e0, ((e1 < q.cols ? e1 : q.cols) - e0) * (int64_t)sizeof(B));
    }
    const B* a = (const B*)q.f.a + r * q.row_stride;
    int64_t head = (int64_t)(((32u - ((uintptr_t)a & 31u)) & 31u) / sizeof(B));
    if (head > q.cols) head = q.cols;
    const int64_t nv = (q.cols - head) / VW;
    const int64_t tail0 = head + nv * VW;
    const VT* vp = (const VT*)(a + head);
    const int64_t v0 = c * CHV + lane;
    if (c * CHV + CHV <= nv) {
      VT v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ldv(vp + v0 + u * 32);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        LC::vec(acc, v[u]);
    } else {
      for (int64_t i = v0; i < nv; i += 32) {
        const VT v = ldv(vp + i);
#pragma unroll
        LC::vec(acc, v);
      }
    }
    if (c == 0) {
      if (lane < head) acc[0] = LC::step(acc[0], lds(a + lane));
      if (lane < q.cols - tail0) acc[VW - 1] = LC::step(acc[VW - 1], lds(a + tail0 + lane));
    }
    r += dr;
    c += dc;
    if (c >= per_row) {
      c -= per_row;
      ++r;
    }
  }
#pragma unroll
  for (int s = VW / 2; s > 0; s >>= 1)
#pragma unroll
    for (int k = 0; k < s; ++k) acc[k] = LC::comb(acc[k], acc[k + s]);
  A cta = block_reduce<R, BLOCK>(LC::out(acc[0]), sm);
  grid_finish<R, BLOCK>(q.f, 0, cta, sm);
}

// ------------------------------------------------------------------------------------------ segmented
struct SegParams {
  const void* a;
  int64_t rows, cols, row_stride;
  uint64_t init;
  int has_init;
  void* out;
};

// one warp per row (gang = the grid of warps over rows, vector = the 32 lanes over the row's columns)
template <class R, int WARPS, int U, int HINT = 0, int PF = 0>
__global__ void __launch_bounds__(WARPS * 32) k_seg_warp(SegParams p) {
  using B = typename R::B;
  using A = typename R::A;
  using VT = typename Vec<B>::T;
  constexpr int VW = Vec<B>::W;
  using LC = Loc<R>;
  using L = typename LC::L;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  #pragma unroll 1
  for (int64_t r = gw; r < p.rows; r += nw) {
    if (PF && lane == 0 && r + nw < p.rows)  // the warp's next row into L2
      l2_prefetch((const B*)p.a + (r + nw) * p.row_stride, p.cols * (int64_t)sizeof(B));
    const B* a = (const B*)p.a + r * p.row_stride;
    const int64_t n = p.cols;
    int64_t head = (int64_t)(((32u - ((uintptr_t)a & 31u)) & 31u) / sizeof(B));
    if (head > n) head = n;
    const int64_t nv = (n - head) / VW;
    const int64_t tail0 = head + nv * VW;
    const VT* vp = (const VT*)(a + head);
    L acc[VW];
#pragma unroll
    for (int k = 0; k < VW; ++k) acc[k] = LC::id();
    int64_t i = lane;
    #pragma unroll 1
    for (; i + (U - 1) * 32 < nv; i += U * 32) {
      VT v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ldv<HINT>(vp + i + u * 32);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        LC::vec(acc, v[u]);
    }
    for (; i < nv; i += 32) {
      const VT v = ldv<HINT>(vp + i);
#pragma unroll
      LC::vec(acc, v);
    }
    if (lane < head) acc[0] = LC::step(acc[0], lds(a + lane));
    if (lane < n - tail0) acc[VW - 1] = LC::step(acc[VW - 1], lds(a + tail0 + lane));
#pragma unroll
    for (int s = VW / 2; s > 0; s >>= 1)
#pragma unroll
      for (int k = 0; k < s; ++k) acc[k] = LC::comb(acc[k], acc[k + s]);
    A t = R::warp(LC::out(acc[0]));
    if (lane == 0) {
      if (p.has_init) t = R::op(R::lift((B)p.init), t);
      ((B*)p.out)[r] = R::fin(t);
    }
  }
}

// ------------------------------------------------------------------------------------------ TMA rows
// One warp per row like k_seg_warp, but the row body is staged into shared memory by the bulk-copy engine
// (cp.async.bulk ... mbarrier::complete_tx, SASS UBLKCP) through a per-warp ring of S slots of CH bytes; lane
// 0 keeps S chunks in flight across row boundaries, all 32 lanes fold each landed chunk from shared memory
// with conflict-free 16-byte loads. Requirements: row bodies split at 16-byte boundaries (head/tail elements
// of each row are read directly). No CTA-wide barrier: each warp owns its ring and its mbarriers.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n.reg .pred P;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(0x12F0000000000000ull)  // evict-first policy
      : "memory");
}

template <class R, int WARPS, int S, int CH>
struct SegTma {
  static constexpr int SMEM = WARPS * S * CH + WARPS * S * 8;
};

template <class R, int WARPS, int S, int CH>
__global__ void __launch_bounds__(WARPS * 32) k_seg_tma(SegParams p) {
  using B = typename R::B;
  using A = typename R::A;
  constexpr int EPV = 16 / sizeof(B);  // elements per 16-byte shared-memory load
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned char* ring = smem + (size_t)wid * S * CH;
  uint64_t* bar = (uint64_t*)(smem + (size_t)WARPS * S * CH) + wid * S;
  if (lane == 0)
    for (int i = 0; i < S; ++i) mbar_init(bar + i, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();

  const int64_t gw = (int64_t)blockIdx.x * WARPS + wid;
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  const int es = (int)sizeof(B);
  // per-row body geometry: [head elements][body: multiple of 16 bytes][tail elements]
  auto geom = [&](int64_t r, const B*& a, int64_t& head, int64_t& body_bytes) {
    a = (const B*)p.a + r * p.row_stride;
    head = (int64_t)(((16u - ((uintptr_t)a & 15u)) & 15u) / es);
    if (head > p.cols) head = p.cols;
    body_bytes = ((p.cols - head) * es) & ~(int64_t)15;
  };
  // producer cursor (meaningful in lane 0): row, byte offset in the row body
  int64_t pr = gw, poff = 0;
  const B* pa;
  int64_t phead, pbody;
  if (pr < p.rows) geom(pr, pa, phead, pbody);
  auto produce = [&](int slot) {  // issue the next chunk into `slot`; returns via cursors
    while (pr < p.rows && poff >= pbody) {
      pr += nw;
      poff = 0;
      if (pr < p.rows) geom(pr, pa, phead, pbody);
    }
    if (pr >= p.rows) return;
    const uint32_t bytes = (uint32_t)((pbody - poff) < CH ? (pbody - poff) : CH);
    if (lane == 0) {
      mbar_expect_tx(bar + slot, bytes);
      bulk_g2s(ring + (size_t)slot * CH, (const char*)(pa + phead) + poff, bytes, bar + slot);
    }
    poff += bytes;
  };
  for (int i = 0; i < S; ++i) produce(i);

  int slot = 0;
  uint32_t phase = 0;
  for (int64_t r = gw; r < p.rows; r += nw) {
    const B* a;
    int64_t head, body;
    geom(r, a, head, body);
    A acc[EPV];
#pragma unroll
    for (int k = 0; k < EPV; ++k) acc[k] = R::id();
    for (int64_t off = 0; off < body; off += CH) {
      const int bytes = (int)((body - off) < CH ? (body - off) : CH);
      mbar_wait(bar + slot, phase);
      const unsigned char* c = ring + (size_t)slot * CH;
      for (int o = lane * 16; o < bytes; o += 32 * 16) {
        const uint4 q = *(const uint4*)(c + o);
        if (EPV == 4) {
          acc[0] = R::op(acc[0], R::lift((B)q.x));
          acc[1 % EPV] = R::op(acc[1 % EPV], R::lift((B)q.y));
          acc[2 % EPV] = R::op(acc[2 % EPV], R::lift((B)q.z));
          acc[3 % EPV] = R::op(acc[3 % EPV], R::lift((B)q.w));
        } else {
          acc[0] = R::op(acc[0], R::lift((B)(((uint64_t)q.y << 32) | q.x)));
          acc[1 % EPV] = R::op(acc[1 % EPV], R::lift((B)(((uint64_t)q.w << 32) | q.z)));
        }
      }
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the next async write
      produce(slot);
      if (++slot == S) {
        slot = 0;
        phase ^= 1u;
      }
    }
    // head and tail elements of this row
    const int64_t tail0 = head + body / es;
    if (lane < head) acc[0] = R::op(acc[0], R::lift(lds(a + lane)));
    for (int64_t j = tail0 + lane; j < p.cols; j += 32) acc[EPV - 1] = R::op(acc[EPV - 1], R::lift(lds(a + j)));
#pragma unroll
    for (int s2 = EPV / 2; s2 > 0; s2 >>= 1)
#pragma unroll
      for (int k = 0; k < s2; ++k) acc[k] = R::op(acc[k], acc[k + s2]);
    A t = R::warp(acc[0]);
    if (lane == 0) {
      if (p.has_init) t = R::op(R::lift((B)p.init), t);
      ((B*)p.out)[r] = R::fin(t);
    }
  }
}

// short rows: G lanes per row (G in 1,2,4,8,16), 32/G rows per warp step; scalar loads (coalesced across
// the warp when rows are contiguous)
template <class R, int G>
__global__ void __launch_bounds__(256) k_seg_group(SegParams p) {
  using B = typename R::B;
  using A = typename R::A;
  const int lane = threadIdx.x & 31;
  const int sub = lane % G;
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;  // this group's first row
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  // all lanes of a warp iterate the same number of times (shuffles need the full warp)
  const int64_t warp_first = (((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / G);
  for (int64_t base = warp_first; base < p.rows; base += ngroups) {
    const int64_t r = base + (gid - warp_first);
    A acc = R::id();
    if (r < p.rows) {
      const B* a = (const B*)p.a + r * p.row_stride;
      for (int64_t j = sub; j < p.cols; j += G) acc = R::op(acc, R::lift(lds(a + j)));
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc = R::op(acc, unpack<A>(__shfl_xor_sync(FULL, pack(acc), o)));
    if (sub == 0 && r < p.rows) {
      if (p.has_init) acc = R::op(R::lift((B)p.init), acc);
      ((B*)p.out)[r] = R::fin(acc);
    }
  }
}

// ------------------------------------------------------------------------------------------ exchange
// the multi-GPU exchange of an accumulator partial already in device memory (host-streaming path): one
// thread runs the same store_out as the reduction kernels (MODE_DIST: dist_exchange)
template <class R>
__global__ void __launch_bounds__(32) k_exchange(FlatParams p, const uint64_t* acc) {
  if (threadIdx.x == 0) store_out<R>(p, 0, unpack<typename R::A>(__ldcg(acc)));
}

// ------------------------------------------------------------------------------------------ finalize
// out = fin(init ⊕ slot[0] ⊕ ... ⊕ slot[P-1]) — cross-rank (a9) or cross-chunk fold, in slot order groups
template <class R>
__global__ void __launch_bounds__(32) k_finalize(const uint64_t* slots, int P, uint64_t init, int has_init,
                                                 void* out) {
  using A = typename R::A;
  using B = typename R::B;
  A v = R::id();
  for (int i = threadIdx.x; i < P; i += 32) v = R::op(v, unpack<A>(__ldcg(slots + i)));
  v = R::warp(v);
  if (threadIdx.x == 0) {
    if (has_init) v = R::op(R::lift((B)init), v);
    *(B*)out = R::fin(v);
  }
}

}  // namespace ipm

namespace ipm {

// ------------------------------------------------------------------------------------------ ragged (CSR)
// out[r] = init ⊕ fold a[off[r] .. off[r+1]) for rows with data-dependent lengths (SURVEY.md §8(f) rank 2:
// BFS-style adjacency loops). Load balance by ELEMENTS, not rows: warp w of nw owns the
// element range [lo, hi) = [P0 + w*nnz/nw, P0 + (w+1)*nnz/nw) and every row whose first element (off[r]) lies in
// it. A row that ends inside its owner's range is finished by the owner; a row that runs past hi leaves a
// TAIL record (row, owner's partial) and every later warp whose range it covers leaves a HEAD record; a second
// one-warp-per-record kernel folds tail + heads in warp order (deterministic) and finishes those rows.
struct RaggedParams {
  const void* a;
  const int64_t* off;     // rows + 1 offsets
  int64_t rows;
  uint64_t init;
  int has_init;
  void* out;
  int64_t* head_row;      // per warp: the row continued from the previous warp (-1: none)
  uint64_t* head_part;
  int64_t* tail_row;      // per warp: the owned row that continues into the next warp (-1: none)
  uint64_t* tail_part;
  int gate;               // 0: run; 1: run only below gate_len elements per row on average; 2: only at or above
  int64_t gate_len;
  int64_t* nw_dev;        // non-NULL (auto: gated candidates with different warp counts): the kernel that runs
                          // stores its warp count here and the fix-up kernel scans only that many records
};

// first index r in [0, rows] with off[r] >= x (off non-decreasing); 32-ary search by the whole warp
__device__ __forceinline__ int64_t warp_lower_bound(const int64_t* off, int64_t rows, int64_t x) {
  const int lane = threadIdx.x & 31;
  int64_t lo = 0, hi = rows;  // answer in [lo, hi]
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t idx = min(lo + (int64_t)lane * step, hi);
    const unsigned ge = __ballot_sync(FULL, __ldg(off + idx) >= x);
    // lanes are increasing in idx: the first lane with off >= x bounds the answer from above
    const int f = ge ? __ffs(ge) - 1 : 32;
    const int64_t nhi = f < 32 ? min(lo + (int64_t)f * step, hi) : hi;
    const int64_t nlo = f > 0 ? min(lo + (int64_t)(f - 1) * step, hi) + 1 : lo;
    lo = nlo;
    hi = nhi;
  }
  const int64_t idx = lo + lane;
  const unsigned ge = __ballot_sync(FULL, idx <= hi && __ldg(off + min(idx, hi)) >= x);
  return ge ? lo + (__ffs(ge) - 1) : hi;
}

// Phase 1 (k_ragged_vec, element-parallel): the warp streams
// its element range in chunks of 32 lanes x VW contiguous elements (one 32-byte vector per lane), marks the
// positions where rows start (from a window of 32 row offsets, through a per-warp shared-memory map
// position -> row), folds each lane's VW elements with those breaks, and joins the pieces of rows that cross
// lanes and chunks with a segmented warp scan. Every element is read once with coalesced vector loads
// whatever the row lengths (short rows no longer cost a warp each). FF: a chunk in which no row starts (inside a
// long row) skips the lane fold with breaks and the segmented scan: its elements join the open row through one
// warp reduction (profiles/r01_sweep_ragged_4_flagfree.txt: +7 % on 4096-element rows, +1.5 % power-law).
template <class A>
__device__ __forceinline__ A shfl_up_acc(A v, int d) {
  return unpack<A>(__shfl_up_sync(FULL, pack(v), d));
}
template <class A>
__device__ __forceinline__ A shfl_acc(A v, int src) {
  return unpack<A>(__shfl_sync(FULL, pack(v), src));
}

// the ragged kernels' common prologue: warp w of nw owns the element range [lo, hi) of [P0, P1) and the rows that
// start in it (r0: the first one), hrow is the row that crosses lo from before (-1: none); the warp's head / tail
// records start empty (-2: an empty range, so the fix-up kernel passes over it)
struct RaggedWarp {
  int64_t w, nw, P1, lo, hi, r0, hrow;
};
// p.gate (0: none; 1: only below p.gate_len elements per row on average over the whole input; 2: only at or above):
// false = this kernel does not run for this input and nothing is written. The lane-per-row kernel, idle on the
// common short-row inputs, checks before the row search (EARLY_GATE: it returns after two loads); the warp kernel
// after it (placed before it, ptxas spilled in the warp kernel's chunk loop)
template <bool EARLY_GATE = false>
__device__ __forceinline__ bool ragged_warp(RaggedWarp& g, const RaggedParams& p, int64_t w, int64_t nw) {
  g.w = w;
  g.nw = nw;
  const int64_t P0 = __ldg(p.off);
  g.P1 = __ldg(p.off + p.rows);
  const int64_t nnz = g.P1 - P0;
  if (EARLY_GATE && p.gate && (p.gate == 1) == (nnz >= p.gate_len * p.rows)) return false;
  g.lo = P0 + (int64_t)(((__int128)nnz * w) / nw);
  g.hi = P0 + (int64_t)(((__int128)nnz * (w + 1)) / nw);
  g.r0 = warp_lower_bound(p.off, p.rows, g.lo);
  g.hrow = (g.r0 > 0 && g.lo < g.hi && __ldg(p.off + g.r0 - 1) < g.lo && __ldg(p.off + g.r0) > g.lo) ? g.r0 - 1 : -1;
  if (!EARLY_GATE && p.gate && (p.gate == 1) == (nnz >= p.gate_len * p.rows)) return false;
  if ((threadIdx.x & 31) == 0) {
    p.head_row[w] = g.lo < g.hi ? -1 : -2;
    p.tail_row[w] = -1;
    if (w == 0 && p.nw_dev) *p.nw_dev = nw;
  }
  return true;
}

// per-warp shared memory of ragged_vec_body (one region per warp, carved below)
template <class R, int VPL>
struct RaggedVecSmem {
  static constexpr int CH = 32 * Vec<typename R::B>::W * VPL;
  static constexpr int BYTES = CH * (int)sizeof(int) + CH * (int)sizeof(typename R::A) + 32 * (int)sizeof(unsigned);
};

template <class R, int VPL, bool FF = true, int PFV = 0>
__device__ __forceinline__ void ragged_vec_body(const RaggedParams& p, unsigned char* wsm, const RaggedWarp& g) {
  using B = typename R::B;
  using A = typename R::A;
  using VT = typename Vec<B>::T;
  constexpr int VW = Vec<B>::W;
  constexpr int EPL = VW * VPL;  // elements per lane per chunk (<= 32: one flag bit each)
  constexpr int CH = 32 * EPL;   // elements per chunk
  static_assert(EPL <= 32, "flag word");
  // per warp, column-major by lane (position EPL*l + k at [k*32 + l]: a lane's column is bank-conflict free):
  // chunk position -> (row - r0) starting there (valid where flagged); the value of the segment that ends just
  // before a flagged position; per lane, bit k = a row starts at the lane's element k
  int* const s_rid = (int*)wsm;
  A* const s_val = (A*)(wsm + CH * sizeof(int));
  unsigned* const s_flag = (unsigned*)(wsm + CH * (sizeof(int) + sizeof(A)));
  const int lane = threadIdx.x & 31;
  int* rid_map = s_rid;
  const int* rid_col = s_rid + lane;
  A* val_col = s_val + lane;
  unsigned* flagw = s_flag;
  flagw[lane] = 0u;
  const unsigned lanemask_lt = (1u << lane) - 1u;
  const int64_t w = g.w, nw = g.nw, P1 = g.P1, lo = g.lo, hi = g.hi, r0 = g.r0, hrow = g.hrow;
  const B* a = (const B*)p.a;
  const bool last = (w == nw - 1);
  auto finish = [&](int64_t row, A v) {  // a complete row owned by this warp
    if (p.has_init) v = R::op(R::lift((B)p.init), v);
    ((B*)p.out)[row] = R::fin(v);
  };
  // window of row offsets: lane l holds off[wb + l] and off[wb + l + 1]; the offsets are loaded two windows
  // ahead (one coalesced load per lane per window; the end offsets come from the neighbour lane)
  int64_t wb = r0;
  auto fetch = [&](int64_t base) -> int64_t {
    const int64_t r = base + lane;
    return r <= p.rows ? __ldg(p.off + r) : P1;
  };
  auto ends = [&](int64_t s0, int64_t nxt0) -> int64_t {  // off[wb + lane + 1]
    const int64_t up = __shfl_down_sync(FULL, s0, 1);
    const int64_t n0 = __shfl_sync(FULL, nxt0, 0);
    return lane == 31 ? n0 : up;
  };
  // chunk bases: positions whose address is 32-byte aligned, from q0; window quantities are kept relative to q0
  // in 32 bits (clamped: a row starting past the warp's range only needs to compare as "later")
  const int64_t q0 = lo - (int64_t)(((uintptr_t)(a + lo) & 31u) / sizeof(B));
  int64_t nx = fetch(wb + 32);   // the next window
  int64_t nx2 = fetch(wb + 64);  // and the one after (its first offset closes the next window's last row)
  int wpos;                      // off[wb + lane] - q0
  bool wrow, wfull;              // wb + lane is a row; it is non-empty
  auto window = [&](int64_t sw) {
    const int64_t ew = ends(sw, nx);
    const int64_t d = sw - q0;
    wpos = d < (int64_t)INT32_MAX ? (int)d : INT32_MAX;
    wrow = wb + lane < p.rows;
    wfull = ew > sw;
  };
  window(fetch(wb));
  int64_t open_rid = hrow;
  A open_val = R::id();
  __syncwarp();
  // PFV > 0: lane 0 asks L2 to fetch the chunk PFV chunks ahead (one bulk prefetch, no registers or shared
  // memory held), so the chunk's own loads hit L2 and more HBM bytes are in flight per warp
  // PFV < 0: the same at distance -PFV, only while the previous chunk had no row start (inside long rows;
  // short-row regions are issue-bound and skip the extra instructions)
  constexpr int PFD = PFV < 0 ? -PFV : PFV;
  bool pf_on = PFV > 0;
  auto prefetch = [&](int64_t pb) {
    if (PFV != 0 && lane == 0 && pf_on && pb < hi) {
      const uint32_t bytes = (uint32_t)((hi - pb < CH ? hi - pb : CH) * sizeof(B)) & ~15u;
      if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a + pb), "r"(bytes) : "memory");
    }
  };
  if (lo < hi) {
#pragma unroll 1
    for (int d = 1; d < PFV; ++d) prefetch(q0 + (int64_t)d * CH);
    for (int64_t Bc = q0; Bc < hi; Bc += CH) {
      prefetch(Bc + (int64_t)PFD * CH);
      // valid positions of this chunk, relative to Bc: [rlo_c, rhi_c)
      const int rlo_c = (int)(lo > Bc ? lo - Bc : 0);
      const int rhi_c = (int)(hi - Bc < CH ? hi - Bc : CH);
      const bool interior = rlo_c == 0 && rhi_c == CH;  // warp-uniform
      // this lane's elements, issued first: positions Bc + EPL*lane + k
      const B* pl = a + Bc + EPL * lane;
      B x[EPL];
      if (interior) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          const VT t = ldv((const VT*)(pl + v * VW));
#pragma unroll
          for (int k = 0; k < VW; ++k) x[v * VW + k] = t.w[k];
        }
      } else {
#pragma unroll
        for (int k = 0; k < EPL; ++k) {
          const int rel = EPL * lane + k;
          x[k] = (rel >= rlo_c && rel < rhi_c) ? lds(pl + k) : (B)0;
        }
      }
      // rows starting in the chunk's valid range: flag their start position; empty ones are finished here
      const int cb = (int)(Bc - q0);
      while (true) {
        const int d = wpos - cb;
        const bool inr = wrow && d >= rlo_c && d < rhi_c;
        if (inr && wfull) {
          const unsigned ud = (unsigned)d;  // >= rlo_c >= 0 here
          rid_map[(ud % EPL) * 32 + ud / EPL] = (int)(wb + lane - r0);
          atomicOr(&flagw[ud / EPL], 1u << (ud % EPL));
        }
        if (inr && !wfull) finish(wb + lane, R::id());
        const bool done = !wrow || d < rhi_c;
        if (__all_sync(FULL, done) && wb + 32 < p.rows) {
          wb += 32;
          const int64_t sw = nx;
          nx = nx2;
          nx2 = fetch(wb + 64);
          window(sw);
          continue;
        }
        break;
      }
      __syncwarp();
      const unsigned fl = flagw[lane];
      flagw[lane] = 0u;
      const unsigned bal = __ballot_sync(FULL, fl != 0u);  // lanes with a row start
      if (FF) {
        if (bal == 0u) {  // no row starts in the chunk: every element continues open_rid
          A v = R::id();
          if (interior) {
#pragma unroll
            for (int k = 0; k < EPL; ++k) v = R::op(v, R::lift(x[k]));
          } else {
#pragma unroll
            for (int k = 0; k < EPL; ++k) {
              const int rel = EPL * lane + k;
              v = R::op(v, (rel >= rlo_c && rel < rhi_c) ? R::lift(x[k]) : R::id());
            }
          }
          open_val = R::op(open_val, R::warp(v));  // the open row's lane values join now
          if (PFV < 0) pf_on = true;
          __syncwarp();
          continue;
        }
      }
      if (PFV < 0) pf_on = false;
      // lane-local segmented fold, one pass: at every flagged element the running value (the segment that
      // ends there) is parked in the lane's own shared-memory column and the accumulator restarts
      A acc = R::id();
      if (interior) {
#pragma unroll
        for (int k = 0; k < EPL; ++k) {
          const bool s = (fl >> k) & 1u;
          if (s) val_col[k * 32] = acc;
          acc = R::op(s ? R::id() : acc, R::lift(x[k]));
        }
      } else {
#pragma unroll
        for (int k = 0; k < EPL; ++k) {
          const int rel = EPL * lane + k;
          const bool s = (fl >> k) & 1u;
          if (s) val_col[k * 32] = acc;
          acc = R::op(s ? R::id() : acc, (rel >= rlo_c && rel < rhi_c) ? R::lift(x[k]) : R::id());
        }
      }
      const int kf = fl ? __ffs(fl) - 1 : EPL;
      const int kl = fl ? 31 - __clz(fl) : EPL;
      // head = elements before the first flag, cur = from the last flag on
      const A head = fl ? val_col[kf * 32] : acc;
      const A cur = fl ? acc : R::id();
      // rows that start and end inside this lane: between consecutive flags, value parked at the later one
      for (unsigned m = fl & ~(1u << kl); m; m &= m - 1) {
        const int k0 = __ffs(m) - 1;
        const int k1 = __ffs(fl & ~((2u << k0) - 1u)) - 1;
        finish(r0 + rid_col[k0 * 32], val_col[k1 * 32]);
      }
      const bool flag = fl != 0u;
      const int lastk = kl;
      const long long my_rid = flag ? (long long)(r0 + rid_col[lastk * 32]) : -1;
      // segmented inclusive scan over lanes: a flagged lane starts a segment with its tail value
      const unsigned le = bal & (lanemask_lt | (1u << lane));
      const int start = le ? 31 - __clz(le) : 0;
      A sv = flag ? cur : head;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const A ov = shfl_up_acc(sv, d);
        if (lane - d >= start) sv = R::op(ov, sv);
      }
      // the row open at this lane's start
      const unsigned lt = bal & lanemask_lt;
      A ev = shfl_up_acc(sv, 1);
      const int src = lt ? 31 - __clz(lt) : 0;
      const long long rr = __shfl_sync(FULL, my_rid, src);
      if (!lt) ev = lane == 0 ? open_val : R::op(open_val, ev);
      const long long er = lt ? rr : open_rid;
      if (flag && er >= 0) {  // it ends at this lane's first flag
        const A v = R::op(ev, head);
        if (er == hrow) {
          p.head_row[w] = hrow;
          p.head_part[w] = pack(v);
        } else {
          finish(er, v);
        }
      }
      // carry into the next chunk: the row open at the end of lane 31
      const A lv = shfl_acc(sv, 31);
      const long long lr = __shfl_sync(FULL, my_rid, bal ? 31 - __clz(bal) : 0);
      if (bal) {
        open_val = lv;
        open_rid = lr;
      } else {
        open_val = R::op(open_val, lv);
      }
      __syncwarp();
    }
  }
  // the row still open at hi
  if (lane == 0 && open_rid >= 0) {
    if (open_rid == hrow) {
      p.head_row[w] = hrow;
      p.head_part[w] = pack(open_val);
    } else if (__ldg(p.off + open_rid + 1) <= hi) {
      finish(open_rid, open_val);
    } else {
      p.tail_row[w] = open_rid;
      p.tail_part[w] = pack(open_val);
    }
  }
  // the last warp also owns the empty rows that start at P1 (after every element)
  if (last) {
    const int64_t r = warp_lower_bound(p.off, p.rows, lo < hi ? P1 : lo);
    for (int64_t q = r + lane; q < p.rows; q += 32)
      if (__ldg(p.off + q) == __ldg(p.off + q + 1)) finish(q, R::id());
  }
}

// auto (round 2): both the warp kernel and the lane-per-row kernel are launched; the mean row length of the whole
// input, (off[rows] - off[0]) / rows, picks one of them and the other returns after two offset loads
// (RaggedParams::gate, ragged_warp; profiles/r02_time_ragged_cross.txt)

template <class R, int WARPS, int MINB, int VPL, bool FF = true, int PFV = 0>
__global__ void __launch_bounds__(WARPS * 32, MINB) k_ragged_vec(RaggedParams p) {
  __shared__ __align__(16) unsigned char sm[WARPS * RaggedVecSmem<R, VPL>::BYTES];
  const int wid = threadIdx.x >> 5;
  RaggedWarp g;
  if (!ragged_warp(g, p, (int64_t)blockIdx.x * WARPS + wid, (int64_t)gridDim.x * WARPS)) return;
  ragged_vec_body<R, VPL, FF, PFV>(p, sm + wid * RaggedVecSmem<R, VPL>::BYTES, g);
}

// one warp per phase-1 warp: a warp with a TAIL record finishes that row by folding the HEAD records of the
// following warps (in warp order, 32 at a time with a fixed lane tree) while they continue the same row
template <class R>
__global__ void __launch_bounds__(256) k_ragged_fix(RaggedParams p, int64_t nw) {
  using B = typename R::B;
  using A = typename R::A;
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (p.nw_dev) nw = *(volatile int64_t*)p.nw_dev;  // auto: the warp count of the candidate that ran
  if (w >= nw) return;
  const int64_t row = p.tail_row[w];
  if (row < 0) return;
  A acc = unpack<A>(p.tail_part[w]);
  for (int64_t base = w + 1; base < nw; base += 32) {
    const int64_t j = base + lane;
    const int64_t hr = j < nw ? p.head_row[j] : -1;
    const bool same = hr == row || hr == -2;
    const unsigned m = __ballot_sync(FULL, same);
    const unsigned run = ~m ? (m & ((1u << (__ffs(~m) - 1)) - 1u)) : m;  // contiguous prefix of matches
    const bool take = (run >> lane) & 1u;
    A v = take && hr == row ? unpack<A>(p.head_part[j]) : R::id();
    acc = R::op(acc, R::warp(v));
    if (run != 0xffffffffu) break;
  }
  if (lane == 0) {
    if (p.has_init) acc = R::op(R::lift((B)p.init), acc);
    ((B*)p.out)[row] = R::fin(acc);
  }
}

__device__ __forceinline__ void cp_async8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ------------------------------------------------------------------------------------------ ragged, marked rows
// Two passes (round 2, IPM_OPT_RAGGED_KERNEL = 5 / ipm_reduce_ragged_marked). In k_ragged_vec the
// per-chunk loop over windows of row offsets (find the rows that start in the chunk, flag their positions, map
// position -> row) cost ~70 M of 242 M warp instructions on the power-law graph and held the kernel's main stall
// (profiles/r01_ncu_ragged5_*). Here that work is done once, row-parallel, before the element pass:
//  pass 0 (k_ragged_mark, one lane per row): bit (off[r] - G) of a bitmap over the elements is set for every row
//    (G: the first element's index rounded down to a 32-byte address, the origin of the chunk grid), cnt[c] counts
//    the rows that start in chunk c (CH elements from G; bit 31: one of them is empty), and every EMPTY row is
//    written here (its result is init ⊕ identity);
//  pass 1 (k_ragged_mk, element-parallel): warp w owns whole chunks; per chunk each lane reads its EPL flag bits
//    from the bitmap (one 32-bit load), folds its elements with parking exactly as k_ragged_vec, and names rows by
//    RANK: the k-th flagged position of the chunk starts row R + k, R = rows started before the chunk (a running
//    sum of cnt). In a chunk that holds an empty row (cnt bit 31) a flag's row is the (rank+1)-th non-empty row from
//    the chunk's first row: a clear bit of the empty-row bitmap the row pass also writes (2-3 words prefetched a chunk
//    ahead; a binary search beyond them). Rows crossing warps: head / tail records and k_ragged_fix as for the
//    other kernels.
// Scratch (caller-owned, ipm_ragged_scratch_bytes): the bitmap and the chunk counts, zeroed by the launcher.
struct RaggedMarks {
  uint32_t* bits;  // bit q = some row starts at element G + q
  uint32_t* cnt;   // per chunk: rows starting in it (bits 0..30), one of them empty (bit 31)
  int64_t nwords, nchunks;  // their sizes (checked in the IPM_CHECK_BOUNDS build)
  uint32_t* ebits;  // bit r = row r is empty (every word written by the row pass: no zeroing needed)
  int64_t newords;
};
// IPM_CHECK_BOUNDS (a test build, tools/gpu_bounds.sh; compute-sanitizer is not available on the GPU pool): every
// scratch, output and offsets index of the marked kernels is checked and a violation traps
#ifdef IPM_CHECK_BOUNDS
#define IPM_BOUND(c) \
  do {               \
    if (!(c)) __trap(); \
  } while (0)
#else
#define IPM_BOUND(c) \
  do {               \
  } while (0)
#endif

template <class B>
__device__ __forceinline__ int64_t ragged_origin(const void* a, int64_t P0) {
  return P0 - (int64_t)(((uintptr_t)((const B*)a + P0) & 31u) / sizeof(B));
}

// pass 0: 32 x RPL consecutive rows per warp step, RPL per lane (RPL / 4 32-byte loads of off[] per lane, the next
// step's issued before this one is processed). The row starts' bits are OR-ed into a per-warp shared-memory window
// of the 16 x RPL bitmap words from the step's first row, its row counts into a window of the 2 x RPL chunks from
// the first row's chunk (shared atomics); a row beyond a window (rows longer than 16 elements on average) updates
// global memory itself. Each non-zero word is then written once: plainly if only this step's rows can start in it
// (strictly between its first and last row's words), atomically at the two ends (shared with the neighbouring
// steps); chunk counts are added atomically. Empty rows: result written, chunk flagged (bit 31).
template <class R, int CH, int RPL = 4>
__global__ void __launch_bounds__(256) k_ragged_mark(RaggedParams p, RaggedMarks m) {
  using B = typename R::B;
  static_assert((CH & (CH - 1)) == 0, "chunk: a power of two");
  static_assert(RPL == 4 || RPL == 8, "rows per lane: one or two 32-byte loads");
  constexpr int LCH = __builtin_ctz(CH);
  constexpr int STEP = 32 * RPL, WW = 16 * RPL, CW = 2 * RPL;
  __shared__ uint32_t s_win[8][WW];
  __shared__ uint32_t s_cnt[8][CW];
  const int lane = threadIdx.x & 31;
  uint32_t* win = s_win[threadIdx.x >> 5];
  uint32_t* cwin = s_cnt[threadIdx.x >> 5];
#pragma unroll
  for (int h = 0; h < WW / 32; ++h) win[lane + 32 * h] = 0u;
  if (lane < CW) cwin[lane] = 0u;
  const int64_t rows = p.rows;
  const int64_t P0 = __ldg(p.off);
  const int64_t G = ragged_origin<B>(p.a, P0);
  const B empty_val = R::fin(p.has_init ? R::op(R::lift((B)p.init), R::id()) : R::id());
  const int64_t stride = (int64_t)gridDim.x * 8 * STEP;
  const bool vec = ((uintptr_t)p.off & 31u) == 0;  // 32-byte loads of 4 offsets
  // off[b + RPL lane + u], u < RPL (clamped to off[rows])
  auto loadr = [&](int64_t b, int64_t (&v)[RPL]) {
    const int64_t r = b + RPL * lane;
    if (vec && r + RPL - 1 < rows) {
#pragma unroll
      for (int h = 0; h < RPL / 4; ++h) {
        const V4 t = ldv<1>((const V4*)(p.off + r + 4 * h));
#pragma unroll
        for (int u = 0; u < 4; ++u) v[4 * h + u] = (int64_t)t.w[u];
      }
    } else {
#pragma unroll
      for (int u = 0; u < RPL; ++u) v[u] = __ldg(p.off + (r + u < rows ? r + u : rows));
    }
  };
  int64_t b = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * STEP;
  int64_t nx[RPL], nx_end = 0;  // the next step's offsets and the end of its last row, loaded a step ahead
  if (b < rows) {
    loadr(b, nx);
    nx_end = __ldg(p.off + (b + STEP < rows ? b + STEP : rows));
  }
  __syncwarp();
  for (; b < rows; b += stride) {
    int64_t sv[RPL];
#pragma unroll
    for (int u = 0; u < RPL; ++u) sv[u] = nx[u];
    const int64_t bend = b + STEP < rows ? b + STEP : rows;
    const int64_t s_end = nx_end;  // the end of the step's last row
    if (b + stride < rows) {
      loadr(b + stride, nx);
      nx_end = __ldg(p.off + (b + stride + STEP < rows ? b + stride + STEP : rows));
    }
    const int64_t q0 = __shfl_sync(FULL, sv[0], 0) - G;  // the step's first row start, relative to G
    const int64_t w0 = q0 >> 5, c0 = q0 >> LCH;
    const int64_t nxt = __shfl_down_sync(FULL, sv[0], 1);
    const int64_t e3 = lane == 31 ? s_end : nxt;
    const int nr = (int)(bend - b);                    // rows in this step (<= STEP)
    // the empty-row words of this step (b is a multiple of STEP): lane l holds the bits of rows b + RPL l + u
    {
      uint32_t em = 0u;
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int64_t e = u < RPL - 1 ? sv[u + 1 < RPL ? u + 1 : RPL - 1] : e3;
        if (RPL * lane + u < nr && e == sv[u]) em |= 1u << u;
      }
#pragma unroll
      for (int j = 1; j < 32 / RPL; ++j) {
        const uint32_t o = __shfl_down_sync(FULL, em, j);
        if ((lane & (32 / RPL - 1)) == 0) em |= o << (RPL * j);
      }
      const int64_t ew = (b >> 5) + lane / (32 / RPL);
      if ((lane & (32 / RPL - 1)) == 0 && ew < m.newords) m.ebits[ew] = em;
    }
    const int64_t base = G + (w0 << 5);                // bit 0 of the window's first word
    if (s_end - base < ((int64_t)1 << 31)) {           // warp-uniform: the step spans < 2^31 elements: 32 bits
      const uint32_t offc = (uint32_t)((w0 << 5) - (c0 << LCH));
      const uint32_t blo = (uint32_t)base;
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        if (RPL * lane + u < nr) {
          const uint32_t t = (uint32_t)sv[u] - blo;  // position relative to the window's first word
          const uint32_t e = u < RPL - 1 ? (uint32_t)sv[u + 1 < RPL ? u + 1 : RPL - 1] : (uint32_t)e3;
          const uint32_t dw = t >> 5, dc = (t + offc) >> LCH;
          IPM_BOUND(w0 + dw < m.nwords && c0 + dc < m.nchunks);
          const bool okw = w0 + dw < m.nwords, okc = c0 + dc < m.nchunks;  // (offsets out of contract: no write)
          if (dw < WW) atomicOr(win + dw, 1u << (t & 31));
          else if (okw) atomicOr(m.bits + w0 + dw, 1u << (t & 31));
          if (dc < CW) atomicAdd(cwin + dc, 1u);
          else if (okc) atomicAdd(m.cnt + c0 + dc, 1u);
          if (e == (uint32_t)sv[u]) {
            ((B*)p.out)[b + RPL * lane + u] = empty_val;
            if (okc) atomicOr(m.cnt + c0 + dc, 0x80000000u);
          }
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int64_t r = b + RPL * lane + u;
        if (r < rows) {
          const int64_t q = sv[u] - G;
          const int64_t e = u < RPL - 1 ? sv[u + 1 < RPL ? u + 1 : RPL - 1] : e3;
          const int64_t dw = (q >> 5) - w0, dc = (q >> LCH) - c0;
          const uint32_t bit = 1u << (q & 31);
          IPM_BOUND(q >= 0 && (q >> 5) < m.nwords && (q >> LCH) < m.nchunks && dw >= 0 && dc >= 0);
          const bool okw = q >= 0 && (q >> 5) < m.nwords, okc = q >= 0 && (q >> LCH) < m.nchunks;
          if (dw >= 0 && dw < WW) atomicOr(win + dw, bit);
          else if (okw) atomicOr(m.bits + (q >> 5), bit);
          if (dc >= 0 && dc < CW) atomicAdd(cwin + dc, 1u);
          else if (okc) atomicAdd(m.cnt + (q >> LCH), 1u);
          if (e == sv[u]) {
            ((B*)p.out)[r] = empty_val;
            if (okc) atomicOr(m.cnt + (q >> LCH), 0x80000000u);
          }
        }
      }
    }
    // the step's last row's word, relative to w0
    const int lastl = (nr - 1) / RPL, lastu = (nr - 1) % RPL;
    int64_t pick = sv[0];
#pragma unroll
    for (int u = 1; u < RPL; ++u)
      if (u == lastu) pick = sv[u];
    const int64_t sl = __shfl_sync(FULL, pick, lastl);
    const int64_t dwl = ((sl - G) >> 5) - w0;
    __syncwarp();
#pragma unroll
    for (int h = 0; h < WW / 32; ++h) {
      const int dw = lane + 32 * h;
      const uint32_t word = win[dw];
      win[dw] = 0u;
      if (word && w0 + dw < m.nwords) {
        IPM_BOUND(w0 + dw < m.nwords);
        if (dw == 0 || dw == dwl) atomicOr(m.bits + w0 + dw, word);
        else m.bits[w0 + dw] = word;
      }
    }
    if (lane < CW) {
      const uint32_t c = cwin[lane];
      cwin[lane] = 0u;
      if (c && c0 + lane < m.nchunks) {
        IPM_BOUND(c0 + lane < m.nchunks);
        atomicAdd(m.cnt + c0 + lane, c);
      }
    }
    __syncwarp();
  }
}

template <class R, int WARPS, int MINB, int VPL, int PFD = 0>
__global__ void __launch_bounds__(WARPS * 32, MINB) k_ragged_mk(RaggedParams p, RaggedMarks m) {
  using B = typename R::B;
  using A = typename R::A;
  using VT = typename Vec<B>::T;
  constexpr int VW = Vec<B>::W;
  constexpr int EPL = VW * VPL;  // elements per lane per chunk: 16 (4-byte) / 8 (8-byte) flag bits
  constexpr int CH = 32 * EPL;
  static_assert(EPL == 32 || EPL == 16 || EPL == 8, "a lane's flags are a 32-, 16- or 8-bit field of one bitmap word");
  // per warp, column-major by lane: the value of the segment that ends just before a flagged position
  __shared__ A s_val[WARPS][CH];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  A* const val_col = s_val[wid] + lane;
  // a chunk holding an empty row names a flag's row from the empty-row bitmap: the first EW words from the chunk's
  // first row, loaded at the end of the previous chunk (its count word, which says whether it has empties, arrived
  // a chunk ahead)
  constexpr int EW = CH >= 1024 ? 3 : 2;  // words: the chunk's rows at >= 16 elements per row on average, + 1
  uint32_t ew[EW];
#pragma unroll
  for (int i = 0; i < EW; ++i) ew[i] = 0u;
  bool ew_ready = false;  // warp-uniform: ew holds the current chunk's words
  const int64_t w = (int64_t)blockIdx.x * WARPS + wid, nw = (int64_t)gridDim.x * WARPS;
  const B* a = (const B*)p.a;
  const int64_t P0 = __ldg(p.off), P1 = __ldg(p.off + p.rows);
  const int64_t G = ragged_origin<B>(p.a, P0);
  // chunks holding elements (bounded by the scratch: with off[rows] beyond the caller's nvalues — outside the
  // contract — results are undefined but nothing outside the scratch is read)
  const int64_t NC = min(P1 > P0 ? (P1 - G + CH - 1) / CH : 0, min(m.nchunks, m.nwords * 32 / CH));
  const int64_t c_lo = (int64_t)(((__int128)NC * w) / nw), c_hi = (int64_t)(((__int128)NC * (w + 1)) / nw);
  const int64_t lo = max(P0, G + c_lo * CH), hi = min(P1, G + c_hi * CH);
  if (lane == 0) {
    p.head_row[w] = lo < hi ? -1 : -2;
    p.tail_row[w] = -1;
  }
  if (lo >= hi) return;  // warp-uniform
  const int64_t r0 = warp_lower_bound(p.off, p.rows, lo);
  const int64_t hrow = (r0 > 0 && __ldg(p.off + r0) > lo) ? r0 - 1 : -1;  // off[r0 - 1] < lo
  const bool has_init = p.has_init;
  const A ia = has_init ? R::lift((B)p.init) : R::id();
  auto finish = [&](int64_t row, A v) {
    IPM_BOUND(row >= 0 && row < p.rows);
    ((B*)p.out)[row] = R::fin(has_init ? R::op(ia, v) : v);
  };
  // the EW empty-row words from row R0x's word on (past the bitmap: all empty, never selected)
  auto load_ew = [&](int64_t R0x) {
#pragma unroll
    for (int i = 0; i < EW; ++i) {
      const int64_t wi = (R0x >> 5) + i;
      ew[i] = wi < m.newords ? __ldg(m.ebits + wi) : ~0u;
    }
  };
  const unsigned lanemask_lt = (1u << lane) - 1u;
  constexpr unsigned FMASK = EPL == 32 ? 0xffffffffu : (1u << EPL) - 1u;
  int64_t R0 = r0;  // rows that start before the current chunk
  int64_t open_rid = hrow;
  A open_val = R::id();
  // the chunk's row count and this lane's bitmap word, loaded one chunk ahead (their latency was the kernel's
  // largest stall when loaded in the chunk that uses them)
  const uint32_t* bits_l = m.bits + (EPL * lane >> 5);
  IPM_BOUND(c_hi <= m.nchunks && (((c_hi - 1) * CH) >> 5) + 1 <= m.nwords && r0 <= p.rows);
  uint32_t cw_n = __ldg(m.cnt + c_lo), bw_n = __ldg(bits_l + ((c_lo * CH) >> 5));
#pragma unroll 1
  for (int64_t c = c_lo; c < c_hi; ++c) {
    const uint32_t cw = cw_n, bw = bw_n;
    // PFD > 0: lane 0 asks L2 for the chunk PFD ahead (no registers or shared memory held)
    if (PFD > 0 && lane == 0 && c + PFD < c_hi) {
      const int64_t pb = G + (c + PFD) * CH;
      const int64_t pe = min(hi, pb + CH);
      const uint32_t bytes = (uint32_t)((pe - pb) * (int64_t)sizeof(B)) & ~15u;
      if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a + pb), "r"(bytes) : "memory");
    }
    if (c + 1 < c_hi) {
      cw_n = __ldg(m.cnt + c + 1);
      bw_n = __ldg(bits_l + (((c + 1) * CH) >> 5));
    }
    const int64_t Bc = G + c * CH;
    const int rlo_c = (int)(lo > Bc ? lo - Bc : 0);
    const int rhi_c = (int)(hi - Bc < CH ? hi - Bc : CH);
    const bool interior = rlo_c == 0 && rhi_c == CH;  // warp-uniform
    IPM_BOUND(!interior || (Bc >= lo && Bc + CH <= hi));
    const B* pl = a + Bc + EPL * lane;
    B x[EPL];
    if (interior) {
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const VT t = ldv((const VT*)(pl + v * VW));
#pragma unroll
        for (int k = 0; k < VW; ++k) x[v * VW + k] = t.w[k];
      }
    } else {
#pragma unroll
      for (int k = 0; k < EPL; ++k) {
        const int rel = EPL * lane + k;
        x[k] = (rel >= rlo_c && rel < rhi_c) ? lds(pl + k) : (B)0;
      }
    }
    unsigned fl = (bw >> ((EPL * lane) & 31)) & FMASK;
    if (!interior) {  // flags of positions outside [lo, hi) (before P0, at or after P1 / the next warp's chunks)
      const int b0 = rlo_c - EPL * lane, b1 = rhi_c - EPL * lane;
      const unsigned keep_lo = b0 <= 0 ? FMASK : b0 >= EPL ? 0u : (FMASK & ~((1u << b0) - 1u));
      const unsigned keep_hi = b1 >= EPL ? FMASK : b1 <= 0 ? 0u : ((1u << b1) - 1u);
      fl &= keep_lo & keep_hi;
    }
    const unsigned bal = __ballot_sync(FULL, fl != 0u);
    if (bal == 0u) {  // no row starts in the chunk: every element continues open_rid
      A v = R::id();
      if (interior) {
#pragma unroll
        for (int k = 0; k < EPL; ++k) v = R::op(v, R::lift(x[k]));
      } else {
#pragma unroll
        for (int k = 0; k < EPL; ++k) {
          const int rel = EPL * lane + k;
          v = R::op(v, (rel >= rlo_c && rel < rhi_c) ? R::lift(x[k]) : R::id());
        }
      }
      open_val = R::op(open_val, R::warp(v));
      R0 += cw & 0x7fffffffu;
      ew_ready = c + 1 < c_hi && (cw_n >> 31);
      if (ew_ready) load_ew(R0);
      continue;
    }
    // lane-local segmented fold, one pass, parking at every flag (as k_ragged_vec)
    A acc = R::id();
    if (interior) {
#pragma unroll
      for (int k = 0; k < EPL; ++k) {
        const bool s = (fl >> k) & 1u;
        if (s) val_col[k * 32] = acc;
        acc = R::op(s ? R::id() : acc, R::lift(x[k]));
      }
    } else {
#pragma unroll
      for (int k = 0; k < EPL; ++k) {
        const int rel = EPL * lane + k;
        const bool s = (fl >> k) & 1u;
        if (s) val_col[k * 32] = acc;
        acc = R::op(s ? R::id() : acc, (rel >= rlo_c && rel < rhi_c) ? R::lift(x[k]) : R::id());
      }
    }
    // rank of the lane's first flag in the chunk: exclusive prefix of the flag counts (a per-bit ballot form
    // measured 1-4 % slower, profiles/r02_ab_marked_2.txt)
    const int nf = __popc(fl);
    int pre = nf;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int o = __shfl_up_sync(FULL, pre, d);
      if (lane >= d) pre += o;
    }
    pre -= nf;
    const bool has_empty = (cw >> 31) != 0u;  // warp-uniform
    const int64_t cnt_c = cw & 0x7fffffffu;
    if (has_empty && !ew_ready) load_ew(R0);  // (the warp's first chunk)
    // the row that starts at the lane's flag k (k-th bit): by rank, or (a chunk with an empty row) the (rank+1)-th
    // non-empty row from R0 — the (rank+1)-th clear bit of the empty-row words — and beyond those EW words the last of
    // the chunk's rows that starts at or before the position (binary search)
    auto rid_of = [&](int k, int rank) -> int64_t {
      if (!has_empty) return R0 + rank;
      int kk = rank;
#pragma unroll
      for (int i = 0; i < EW; ++i) {
        const uint32_t z = ~ew[i] & (i == 0 ? ~0u << (R0 & 31) : ~0u);
        const int cz = __popc(z);
        if (kk < cz) return (((R0 >> 5) + i) << 5) + (int64_t)__fns(z, 0, kk + 1);
        kk -= cz;
      }
      const int64_t pos = Bc + EPL * lane + k;
      int64_t l = R0, h = R0 + cnt_c - 1;
      while (l < h) {
        const int64_t mid = (l + h + 1) >> 1;
        if (__ldg(p.off + mid) <= pos) l = mid;
        else h = mid - 1;
      }
      return l;
    };
    const int kf = fl ? __ffs(fl) - 1 : EPL;
    const int kl = fl ? 31 - __clz(fl) : EPL;
    const A head = fl ? val_col[kf * 32] : acc;
    const A cur = fl ? acc : R::id();
    {  // rows that start and end inside this lane: between consecutive flags, value parked at the later one
      int rank = pre;
      for (unsigned mm = fl & ~(1u << kl); mm; mm &= mm - 1, ++rank) {
        const int k0 = __ffs(mm) - 1;
        const int k1 = __ffs(fl & ~((2u << k0) - 1u)) - 1;
        finish(rid_of(k0, rank), val_col[k1 * 32]);
      }
    }
    const bool flag = fl != 0u;
    const long long my_rid = flag ? (long long)rid_of(kl, pre + nf - 1) : -1;
    // segmented inclusive scan over lanes: a flagged lane starts a segment with its tail value
    const unsigned le = bal & (lanemask_lt | (1u << lane));
    const int start = le ? 31 - __clz(le) : 0;
    A sv = flag ? cur : head;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const A ov = shfl_up_acc(sv, d);
      if (lane - d >= start) sv = R::op(ov, sv);
    }
    // the row open at this lane's start
    const unsigned lt = bal & lanemask_lt;
    A ev = shfl_up_acc(sv, 1);
    const int src = lt ? 31 - __clz(lt) : 0;
    const long long rr = __shfl_sync(FULL, my_rid, src);
    if (!lt) ev = lane == 0 ? open_val : R::op(open_val, ev);
    const long long er = lt ? rr : open_rid;
    if (flag && er >= 0) {  // it ends at this lane's first flag
      const A v = R::op(ev, head);
      if (er == hrow) {
        p.head_row[w] = hrow;
        p.head_part[w] = pack(v);
      } else {
        finish(er, v);
      }
    }
    // carry into the next chunk: the row open at the end of lane 31
    open_val = shfl_acc(sv, 31);
    open_rid = __shfl_sync(FULL, my_rid, 31 - __clz(bal));
    R0 += cnt_c;
    ew_ready = c + 1 < c_hi && (cw_n >> 31);
    if (ew_ready) load_ew(R0);
    __syncwarp();
  }
  // the row still open at hi
  if (lane == 0 && open_rid >= 0) {
    if (open_rid == hrow) {
      p.head_row[w] = hrow;
      p.head_part[w] = pack(open_val);
    } else if (__ldg(p.off + open_rid + 1) <= hi) {
      finish(open_rid, open_val);
    } else {
      p.tail_row[w] = open_rid;
      p.tail_part[w] = pack(open_val);
    }
  }
}


// ------------------------------------------------------------------------------------------ ragged, row order
// k_ragged_rank: the ownership rules, chunk shape and lane fold of k_ragged_vec, with the per-chunk row bookkeeping
// rebuilt so that every row is examined once, by one lane, which later finishes it (round 2;
// profiles/r01_ncu_ragged5_*: the window / flag-map loop of k_ragged_vec cost ~175 of ~474 warp instructions per
// chunk, the per-lane finish loop ~65, and 30 % of the stall samples sat on the register copy that shifts the
// offset window; profiles/r02_ncu_rrank_* record the variants measured on the way here):
//  - row offsets come through a per-warp shared-memory ring of NR windows of 32 offsets (entry (r - r0) mod 32*NR
//    holds off[r]), filled by cp.async up to NR-3 windows ahead of the first row not yet examined; no register
//    holds an in-flight offset;
//  - each chunk reads the 64 offsets from its first unexamined row on (two LDS per lane; a chunk in which more
//    than 64 rows start reads further groups): lane i owns rows nxt+i and nxt+32+i, flags their starts (shared
//    atomicOr) and keeps start and end relative to the chunk in registers (later groups re-read them);
//  - the lane fold parks the value of every segment that ends at a flag in the lane's own shared-memory column
//    (as k_ragged_vec); after the segmented warp scan the lane that holds a row's first piece adds the pieces
//    before it; then each owning lane reads its row's value at the row's END position (where the next row
//    starts) and stores out[row]: consecutive rows from consecutive lanes, no per-lane loop, no row map.
//  Positions are kept relative to the chunk and rows relative to r0 in 32 bits.

template <class R, int WARPS, int MINB, int VPL, int NR, int PFV = 0>
__global__ void __launch_bounds__(WARPS * 32, MINB) k_ragged_rank(RaggedParams p) {
  using B = typename R::B;
  using A = typename R::A;
  using VT = typename Vec<B>::T;
  constexpr int VW = Vec<B>::W;
  constexpr int EPL = VW * VPL;  // elements per lane per chunk (one flag bit each)
  constexpr int CH = 32 * EPL;   // elements per chunk
  constexpr int RING = 32 * NR;  // offset ring entries
  static_assert(EPL <= 32 && (EPL & (EPL - 1)) == 0, "flag word");
  static_assert(NR >= 4 && (NR & (NR - 1)) == 0, "offset ring: a power of two >= 4 windows");
  // per warp, column-major by lane (position EPL*l + k at [k*32 + l]: a lane's column is bank-conflict free)
  __shared__ A s_val[WARPS][CH];             // value of the segment that ends just before a flagged position
  __shared__ unsigned s_flag[WARPS][32];     // per lane: bit k = a row starts at the lane's element k
  __shared__ int64_t s_off[WARPS][RING];     // offset ring
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  A* val = s_val[wid];
  A* val_col = s_val[wid] + lane;
  unsigned* flagw = s_flag[wid];
  int64_t* ring = s_off[wid];
  flagw[lane] = 0u;
  const unsigned lanemask_lt = (1u << lane) - 1u;
  const int64_t w = (int64_t)blockIdx.x * WARPS + wid;
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  const B* a = (const B*)p.a;
  const int64_t rows = p.rows;
  const int64_t P0 = __ldg(p.off), P1 = __ldg(p.off + rows);
  const int64_t nnz = P1 - P0;
  const int64_t lo = P0 + (int64_t)(((__int128)nnz * w) / nw);
  const int64_t hi = P0 + (int64_t)(((__int128)nnz * (w + 1)) / nw);
  const int64_t r0 = warp_lower_bound(p.off, rows, lo);
  const int64_t hrow = (r0 > 0 && lo < hi && __ldg(p.off + r0 - 1) < lo && __ldg(p.off + r0) > lo) ? r0 - 1 : -1;
  const int nrel = (int)(rows - r0);  // rows from r0 on (rows < 2^31)
  if (lane == 0) {
    p.head_row[w] = lo < hi ? -1 : -2;
    p.tail_row[w] = -1;
  }
  const bool has_init = p.has_init;
  const A ia = has_init ? R::lift((B)p.init) : R::id();
  B* const outw = (B*)p.out + r0;  // rows relative to r0
  auto fin = [&](A v) { return R::fin(has_init ? R::op(ia, v) : v); };
  auto col = [](unsigned d) { return (d % EPL) * 32 + d / EPL; };  // chunk position -> column address
  // chunk bases are 32-byte aligned positions from q0; positions below are relative to the chunk
  const int64_t q0 = lo - (int64_t)(((uintptr_t)(a + lo) & 31u) / sizeof(B));
  const int hrel = (int)(hi - q0), lrel = (int)(lo - q0);  // warp range relative to q0 (< 2^31)
  // offset ring: window k = rows r0 + 32k .. +31 (offsets clamped to off[rows] = P1) lands in ring[32 (k % NR) ..]
  int nxt = 0;     // first row not yet examined, relative to r0
  int issued = 0;  // windows issued so far
  auto refill = [&]() {  // windows nxt/32 .. nxt/32 + 2 complete, up to NR - 3 more in flight
    const int bw = nxt >> 5;
    if (issued < bw + NR) {
      if (issued < bw + NR - 3) cp_async_wait<0>();  // a jump: no copy may still target a slot reused below
      for (int k = issued > bw ? issued : bw; k < bw + NR; ++k) {
        const int64_t r = r0 + 32 * (int64_t)k + lane;
        cp_async8(&ring[32 * (k & (NR - 1)) + lane], p.off + (r < rows ? r : rows));
        cp_async_commit();
      }
      issued = bw + NR;
    }
    cp_async_wait<NR - 3>();
    __syncwarp();
  };
  long long open_rid = hrow;  // the row open at the chunk start (-1: none)
  A open_val = R::id();
  constexpr int PFD = PFV < 0 ? -PFV : PFV;
  bool pf_on = PFV > 0;
  auto prefetch = [&](int pb) {  // pb relative to q0
    if (PFV != 0 && lane == 0 && pf_on && pb < hrel) {
      const uint32_t bytes = (uint32_t)((hrel - pb < CH ? hrel - pb : CH) * (int)sizeof(B)) & ~15u;
      if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a + q0 + pb), "r"(bytes) : "memory");
    }
  };
  if (lrel < hrel) {
#pragma unroll 1
    for (int d = 1; d < PFV; ++d) prefetch(d * CH);
    const B* pl = a + q0 + EPL * lane;
#pragma unroll 1
    for (int cb = 0; cb < hrel; cb += CH, pl += CH) {
      prefetch(cb + PFD * CH);
      const int rlo_c = lrel > cb ? lrel - cb : 0;
      const int rhi_c = hrel - cb < CH ? hrel - cb : CH;
      const bool interior = rlo_c == 0 && rhi_c == CH;  // warp-uniform
      B x[EPL];
      if (interior) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          const VT t = ldv((const VT*)(pl + v * VW));
#pragma unroll
          for (int k = 0; k < VW; ++k) x[v * VW + k] = t.w[k];
        }
      } else {
#pragma unroll
        for (int k = 0; k < EPL; ++k) {
          const int rel = EPL * lane + k;
          x[k] = (rel >= rlo_c && rel < rhi_c) ? lds(pl + k) : (B)0;
        }
      }
      // rows starting in the chunk's valid range (every unexamined row starts at or after the chunk and lo), in
      // groups of 64 from row c0: lane i holds rows c0 + 64g + i and c0 + 64g + 32 + i (starts d, ends e)
      const int64_t qc = q0 + cb;
      auto rel = [&](int64_t o) { const int64_t d = o - qc; return d < (int64_t)INT32_MAX ? (int)d : INT32_MAX; };
      const int c0 = nxt;
      int dA = 0, eA = 0, dB = 0, eB = 0;  // group 0
      int F = 0;                           // non-empty rows starting in the chunk
      int first_d = 0, last_put = -1;      // start of the first of them, row of the last (relative to r0)
#pragma unroll 1
      for (int g = 0;; ++g) {
        refill();
        const int base = nxt & (RING - 1);
        const int d1 = rel(ring[(base + lane) & (RING - 1)]);
        const int d2 = rel(ring[(base + 32 + lane) & (RING - 1)]);
        const int d3 = rel(ring[(base + 64) & (RING - 1)]);
        const int u1 = __shfl_down_sync(FULL, d1, 1), u2 = __shfl_down_sync(FULL, d2, 1);
        const int f2 = __shfl_sync(FULL, d2, 0);
        const int e1 = lane == 31 ? f2 : u1, e2 = lane == 31 ? d3 : u2;
        const bool in1 = nxt + lane < nrel && d1 < rhi_c;
        const bool in2 = nxt + 32 + lane < nrel && d2 < rhi_c;
        const bool p1 = in1 && e1 > d1, p2 = in2 && e2 > d2;
        if (p1) atomicOr(&flagw[(unsigned)d1 / EPL], 1u << ((unsigned)d1 % EPL));
        if (p2) atomicOr(&flagw[(unsigned)d2 / EPL], 1u << ((unsigned)d2 % EPL));
        const unsigned m1 = __ballot_sync(FULL, p1), m2 = __ballot_sync(FULL, p2);
        if (m1 | m2) {
          if (F == 0) first_d = m1 ? __shfl_sync(FULL, d1, __ffs(m1) - 1) : __shfl_sync(FULL, d2, __ffs(m2) - 1);
          last_put = m2 ? nxt + 63 - __clz(m2) : nxt + 31 - __clz(m1);
        }
        F += __popc(m1) + __popc(m2);
        if (g == 0) {
          dA = d1; eA = e1; dB = d2; eB = e2;
        }
        // the in-range rows are a prefix of the 64
        const int nin = __popc(__ballot_sync(FULL, in1)) + __popc(__ballot_sync(FULL, in2));
        nxt += nin;
        if (nin < 64) break;
      }
      __syncwarp();
      if (F == 0) {  // no row starts in the chunk (empty rows: finished below): every element continues open_rid
        A v = R::id();
        if (interior) {
#pragma unroll
          for (int k = 0; k < EPL; ++k) v = R::op(v, R::lift(x[k]));
        } else {
#pragma unroll
          for (int k = 0; k < EPL; ++k) {
            const int rel = EPL * lane + k;
            v = R::op(v, (rel >= rlo_c && rel < rhi_c) ? R::lift(x[k]) : R::id());
          }
        }
        open_val = R::op(open_val, R::warp(v));
        if (PFV < 0) pf_on = true;
      } else {
        if (PFV < 0) pf_on = false;
        const unsigned fl = flagw[lane];
        flagw[lane] = 0u;
        // lane-local segmented fold, one pass: at every flagged element the running value (the segment that
        // ends there) is parked in the lane's own shared-memory column and the accumulator restarts
        A acc = R::id();
        if (interior) {
#pragma unroll
          for (int k = 0; k < EPL; ++k) {
            const bool s = (fl >> k) & 1u;
            if (s) val_col[k * 32] = acc;
            acc = R::op(s ? R::id() : acc, R::lift(x[k]));
          }
        } else {
#pragma unroll
          for (int k = 0; k < EPL; ++k) {
            const int rel = EPL * lane + k;
            const bool s = (fl >> k) & 1u;
            if (s) val_col[k * 32] = acc;
            acc = R::op(s ? R::id() : acc, (rel >= rlo_c && rel < rhi_c) ? R::lift(x[k]) : R::id());
          }
        }
        // segmented inclusive scan over lanes: a flagged lane starts a segment with its tail value
        const bool flag = fl != 0u;
        const unsigned bal = __ballot_sync(FULL, flag);
        const unsigned le = bal & (lanemask_lt | (1u << lane));
        const int start = le ? 31 - __clz(le) : 0;
        A sv = acc;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const A ov = shfl_up_acc(sv, d);
          if (lane - d >= start) sv = R::op(ov, sv);
        }
        // the pieces before a flagged lane's first row start complete the row open at the lane's start
        A ev = shfl_up_acc(sv, 1);
        if (!(bal & lanemask_lt)) ev = lane == 0 ? open_val : R::op(open_val, ev);
        if (flag) {
          A* h = val_col + (__ffs(fl) - 1) * 32;
          *h = R::op(ev, *h);
        }
        __syncwarp();
        // the row open at the chunk start ends where the chunk's first non-empty row starts
        if (lane == 0 && open_rid >= 0) {
          const A v = val[col((unsigned)first_d)];
          if (open_rid == hrow) {
            p.head_row[w] = hrow;
            p.head_part[w] = pack(v);
          } else {
            ((B*)p.out)[open_rid] = fin(v);
          }
        }
        open_val = shfl_acc(sv, 31);
        open_rid = r0 + last_put;
      }
      // finish the rows examined in this chunk that end inside it (value parked where the next row starts) and
      // the empty ones; a row that ends at or after the chunk's end is the new open row
      const int nrow = nxt - c0;
      if (lane < nrow && eA < rhi_c) outw[c0 + lane] = fin(eA > dA ? val[col((unsigned)eA)] : R::id());
      if (32 + lane < nrow && eB < rhi_c) outw[c0 + 32 + lane] = fin(eB > dB ? val[col((unsigned)eB)] : R::id());
#pragma unroll 1
      for (int j = 64 + lane; j < nrow; j += 32) {  // rows beyond the first 64: offsets re-read
        const int64_t r = r0 + c0 + j;  // < rows
        const int d = rel(__ldg(p.off + r));
        const int e = rel(__ldg(p.off + r + 1));
        if (e < rhi_c) outw[c0 + j] = fin(e > d ? val[col((unsigned)e)] : R::id());
      }
      __syncwarp();
    }
  }
  // the row still open at hi
  if (lane == 0 && open_rid >= 0) {
    if (open_rid == hrow) {
      p.head_row[w] = hrow;
      p.head_part[w] = pack(open_val);
    } else if (__ldg(p.off + open_rid + 1) <= hi) {
      ((B*)p.out)[open_rid] = fin(open_val);
    } else {
      p.tail_row[w] = open_rid;
      p.tail_part[w] = pack(open_val);
    }
  }
  // the last warp also owns the empty rows that start at P1 (after every element)
  if (w == nw - 1) {
    const int64_t r = warp_lower_bound(p.off, rows, lo < hi ? P1 : lo);
    for (int64_t q = r + lane; q < rows; q += 32)
      if (__ldg(p.off + q) == __ldg(p.off + q + 1)) ((B*)p.out)[q] = fin(R::id());
  }
  cp_async_wait<0>();  // no copy may land in shared memory after the warp leaves
}

// ------------------------------------------------------------------------------------------ ragged, lane per row
// k_ragged_lpr: the ownership rules of k_ragged_vec (warp w owns the element range [lo, hi) and the rows that start
// in it; head / tail records for the rows that cross its ends), with rows rather than elements as the lane unit
// (round 2). Rows are taken in WINDOWS of up to 32 consecutive rows whose elements span at most CAPE elements
// (the lanes read the window's offsets from a cp.async shared-memory ring, NR windows of 32 ahead); the window's
// span is copied into shared memory with 16-byte cp.async (zero-filled past the span, no byte outside it read);
// then each lane folds its own row from shared memory if it has at most T elements (one loop for the window,
// maxlen steps), a longer row of the window is folded by the whole warp from shared memory (32 elements a step, a
// warp reduction), and every lane stores its row's result: out[] is written by consecutive lanes. A row longer
// than CAPE is a window of its own, folded by the whole warp from global memory with 32-byte loads. No flags, no
// segmented scan: the work per element is one shared load and one op, the work per row one offset and one store.
__device__ __forceinline__ void cp_async16z(void* s, const void* g, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(s)), "l"(g), "r"(src_bytes) : "memory");
}

// per-warp shared memory of ragged_lpr_body: the staged span (from a 16-byte aligned start), the offset ring
template <class R, int CAPB, int NR>
struct RaggedLprSmem {
  static constexpr int E16 = 16 / (int)sizeof(typename R::B);
  static constexpr int STAGE = (CAPB / (int)sizeof(typename R::B) + 2 * E16) * (int)sizeof(typename R::B);
  static constexpr int BYTES = STAGE + 32 * NR * (int)sizeof(int64_t);
};

template <class R, int CAPB, int NR, int T>
__device__ __forceinline__ void ragged_lpr_body(const RaggedParams& p, unsigned char* wsm, const RaggedWarp& g) {
  using B = typename R::B;
  using A = typename R::A;
  using VT = typename Vec<B>::T;
  constexpr int VW = Vec<B>::W;
  constexpr int CAPE = CAPB / (int)sizeof(B);  // elements per window span
  constexpr int E16 = 16 / (int)sizeof(B);     // elements per 16-byte copy
  constexpr int RING = 32 * NR;
  static_assert(NR >= 4 && (NR & (NR - 1)) == 0, "offset ring: a power of two >= 4 windows");
  static_assert(CAPB % 512 == 0, "span: whole 16-byte copies per lane");
  B* const stage = (B*)wsm;
  int64_t* const ring = (int64_t*)(wsm + RaggedLprSmem<R, CAPB, NR>::STAGE);
  const int lane = threadIdx.x & 31;
  const int64_t w = g.w, nw = g.nw, P1 = g.P1, lo = g.lo, hi = g.hi, r0 = g.r0, hrow = g.hrow;
  const B* a = (const B*)p.a;
  const int64_t rows = p.rows;
  const int nrel = (int)(rows - r0);
  auto fin = [&](A v) { return R::fin(p.has_init ? R::op(R::lift((B)p.init), v) : v); };
  // the whole warp folds a[s, e) from global memory: a scalar head to 32-byte alignment, 32-byte vectors (two in
  // flight per lane), a scalar tail; the warp-reduced value (every lane)
  auto fold_global = [&](int64_t s0, int64_t e0) -> A {
    A v = R::id();
    const int64_t head = ((32 - (int64_t)(((uintptr_t)(a + s0)) & 31u)) & 31) / (int64_t)sizeof(B);
    const int64_t h1 = s0 + (head < e0 - s0 ? head : e0 - s0);
    if (s0 + lane < h1) v = R::lift(lds(a + s0 + lane));
    const VT* vp = (const VT*)(a + h1);
    const int64_t nv = (e0 - h1) / VW;
    using LC = Loc<R>;
    typename LC::L la[VW];
#pragma unroll
    for (int k = 0; k < VW; ++k) la[k] = LC::id();
    int64_t i = lane;
#pragma unroll 1
    for (; i + 32 < nv; i += 64) {
      const VT t0 = ldv(vp + i), t1 = ldv(vp + i + 32);
      LC::vec(la, t0);
      LC::vec(la, t1);
    }
    if (i < nv) LC::vec(la, ldv(vp + i));
#pragma unroll
    for (int k = 1; k < VW; ++k) la[0] = LC::comb(la[0], la[k]);
    v = R::op(v, LC::out(la[0]));
    const int64_t t0 = h1 + nv * VW;
    if (t0 + lane < e0) v = R::op(v, R::lift(lds(a + t0 + lane)));
    return R::warp(v);
  };
  int nxt = 0;     // first row not yet taken, relative to r0
  int issued = 0;  // offset windows issued (window j = rows r0 + 32j ..)
  auto refill = [&]() {  // windows nxt/32 and nxt/32 + 1 complete, up to NR - 2 more in flight
    const int bw = nxt >> 5;
    if (issued < bw + NR) {
      if (issued < bw + NR - 2) cp_async_wait<0>();  // a jump: no copy may still target a slot reused below
      for (int j = issued > bw ? issued : bw; j < bw + NR; ++j) {
        const int64_t r = r0 + 32 * (int64_t)j + lane;
        cp_async8(&ring[32 * (j & (NR - 1)) + lane], p.off + (r < rows ? r : rows));
        cp_async_commit();
      }
      issued = bw + NR;
    }
    cp_async_wait<NR - 2>();
    __syncwarp();
  };
  if (lo < hi) {
    // the row that started before lo: its elements in [lo, min(end, hi)) go to the head record
    if (hrow >= 0) {
      const int64_t e = __ldg(p.off + hrow + 1);
      const A v = fold_global(lo, e < hi ? e : hi);
      if (lane == 0) {
        p.head_row[w] = hrow;
        p.head_part[w] = pack(v);
      }
    }
#pragma unroll 1
    while (nxt < nrel) {
      refill();
      const int base = nxt & (RING - 1);
      const int64_t s_i = ring[(base + lane) & (RING - 1)];   // start of row nxt + lane
      const int64_t s_n = ring[(base + 32) & (RING - 1)];
      const int64_t e_up = __shfl_down_sync(FULL, s_i, 1);
      const int64_t e_raw = lane == 31 ? s_n : e_up;          // its end
      const int64_t s0 = __shfl_sync(FULL, s_i, 0);
      if (s0 >= hi) break;                                      // the rows from here on belong to later warps
      const bool valid = nxt + lane < nrel && s_i < hi;
      const int64_t e_i = e_raw < hi ? e_raw : hi;              // clipped to the warp's range
      const int64_t len = valid ? e_i - s_i : 0;
      const int64_t e0 = __shfl_sync(FULL, e_i, 0);
      if (e0 - s0 > CAPE) {  // a long row: a window of its own, folded from global memory
        const A v = fold_global(s0, e0);
        if (lane == 0) {
          const int64_t r = r0 + nxt;
          if (e_raw > hi) {
            p.tail_row[w] = r;
            p.tail_part[w] = pack(v);
          } else {
            ((B*)p.out)[r] = fin(v);
          }
        }
        ++nxt;
        continue;
      }
      // the window: the leading rows whose span from s0 stays within CAPE elements
      const bool inw = valid && e_i - s0 <= CAPE;
      const unsigned wm = __ballot_sync(FULL, inw);
      const int nwin = __popc(wm);  // a prefix of the lanes (>= 1: lane 0's row fits)
      const int64_t ew = __shfl_sync(FULL, e_i, nwin - 1);
      // stage [s0, ew) from the 16-byte aligned address at or below a + s0 (at most 12 bytes before the span, inside
      // the same allocation: device allocations are 256-byte aligned); zero-filled past ew, nothing after it read
      const int64_t sb = s0 - (int64_t)(((uintptr_t)(a + s0) & 15u) / sizeof(B));
      const int nvec = (int)((ew - sb + E16 - 1) / E16);
      for (int q = lane; q < nvec; q += 32) {
        const int64_t g = sb + (int64_t)q * E16;
        const int64_t rem = ew - g;
        cp_async16z(stage + q * E16, a + g, (int)(rem < E16 ? rem : E16) * (int)sizeof(B));
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncwarp();
      const int off_i = (int)(s_i - sb);
      const int L = inw ? (int)len : 0;
      const bool shrt = L <= T;
      A v = R::id();
      // short rows: lane per row
      const int Ls = shrt ? L : 0;
      const int maxl = __reduce_max_sync(FULL, Ls);
      const B* sp = stage + off_i;
#pragma unroll 1
      for (int j = 0; j < maxl; j += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (j + u < Ls) v = R::op(v, R::lift(sp[j + u]));
      }
      // longer rows of the window: the whole warp from shared memory
      unsigned mm = __ballot_sync(FULL, inw && !shrt);
#pragma unroll 1
      while (mm) {
        const int ln = __ffs(mm) - 1;
        mm &= mm - 1;
        const int o = __shfl_sync(FULL, off_i, ln), n = __shfl_sync(FULL, L, ln);
        A u = R::id();
        for (int j = lane; j < n; j += 32) u = R::op(u, R::lift(stage[o + j]));
        u = R::warp(u);
        if (lane == ln) v = u;
      }
      if (inw) {
        const int64_t r = r0 + nxt + lane;
        if (e_raw > hi) {  // the row continues in the next warp's range
          p.tail_row[w] = r;
          p.tail_part[w] = pack(v);
        } else {
          ((B*)p.out)[r] = fin(v);
        }
      }
      nxt += nwin;
      __syncwarp();
    }
  }
  // the last warp also owns the empty rows that start at P1 (after every element)
  if (w == nw - 1) {
    const int64_t r = warp_lower_bound(p.off, rows, lo < hi ? P1 : lo);
    for (int64_t q = r + lane; q < rows; q += 32)
      if (__ldg(p.off + q) == __ldg(p.off + q + 1)) ((B*)p.out)[q] = fin(R::id());
  }
  cp_async_wait<0>();
}

template <class R, int WARPS, int MINB, int CAPB, int NR, int T>
__global__ void __launch_bounds__(WARPS * 32, MINB) k_ragged_lpr(RaggedParams p) {
  static_assert(RaggedLprSmem<R, CAPB, NR>::BYTES % 16 == 0, "per-warp regions 16-byte aligned");
  __shared__ __align__(16) unsigned char sm[WARPS * RaggedLprSmem<R, CAPB, NR>::BYTES];
  const int wid = threadIdx.x >> 5;
  RaggedWarp g;
  if (!ragged_warp<true>(g, p, (int64_t)blockIdx.x * WARPS + wid, (int64_t)gridDim.x * WARPS)) return;
  ragged_lpr_body<R, CAPB, NR, T>(p, sm + wid * RaggedLprSmem<R, CAPB, NR>::BYTES, g);
}

// ------------------------------------------------------------------------------------------ ragged, CTA tiles
// The same clause and ownership rules as k_ragged_vec, with the CTA (not the warp) as the unit: CTA b owns the
// element range [lo, hi) = [P0 + b*nnz/G, P0 + (b+1)*nnz/G) and every row whose first element lies in it, and
// streams it in tiles of BLOCK x EPT elements (EPT contiguous elements per thread, VPT 32-byte loads issued at the
// start of the tile; thread 0 asks L2 for the tile PFD tiles ahead with one bulk prefetch, so the loads hit L2 and
// HBM bytes stay in flight without holding registers). Per tile:
//   1. row setup, one thread per row: the rows that start in the tile are the next rows in order (rows are
//      sorted by their start), so thread i takes row rs + i (one coalesced 8-byte offset load, the window
//      prefetched during the previous tile), flags the row's first element in the owning thread's 32-bit flag
//      word (atomicOr) and records the row id at that position; an empty row is finished on the spot. A window
//      of BLOCK rows that is entirely inside the tile repeats the step with the next BLOCK rows.
//   2. a tile in which no row starts (inside a long row) is folded into per-thread running values, no scan; they
//      are reduced into the open row's value once, when the next row start (or the range end) comes.
//   3. otherwise the lane fold: each thread folds its EPT elements once; at a flagged element the running value
//      (the segment that ends there) is parked in the thread's shared-memory column and the accumulator restarts;
//      rows that start and end inside the thread are finished from the parked values.
//   4. a segmented scan over the CTA's threads (warp shuffles, then one thread chains the NW warp totals with
//      the open row carried in from the previous tile) gives each flagged thread the value of the row that ends
//      at its first flag.
// Rows continued from the previous CTA or into the next one leave head / tail records, finished by
// k_ragged_fix (one record pair per CTA instead of per warp).
template <class R, int BLOCK, int VPT>
struct RaggedTile {
  static constexpr int EPT = Vec<typename R::B>::W * VPT;
  static constexpr int SMEM = EPT * BLOCK * ((int)sizeof(typename R::A) + 4);
};
template <class R, int BLOCK, int VPT, int MINB, int PFD>
__global__ void __launch_bounds__(BLOCK, MINB) k_ragged_tile(RaggedParams p) {
  using B = typename R::B;
  using A = typename R::A;
  using VT = typename Vec<B>::T;
  constexpr int VW = Vec<B>::W;
  constexpr int EPT = VW * VPT;     // elements per thread per tile (one flag bit each)
  constexpr int TILE = BLOCK * EPT;
  constexpr int NW = BLOCK / 32;
  static_assert(EPT <= 32, "one 32-bit flag word per thread");
  __shared__ unsigned s_flag[BLOCK];      // bit k of word t: a row starts at the thread's element k
  // dynamic shared memory (RaggedTile<>::SMEM bytes):
  //   s_val [k][t]: value of the segment that ends just before a flagged element (column per thread)
  //   s_rid [k][t]: the row starting there (valid where flagged)
  extern __shared__ __align__(16) unsigned char ragged_dsm[];
  A* s_val = (A*)ragged_dsm;
  int* s_rid = (int*)(ragged_dsm + (size_t)EPT * BLOCK * sizeof(A));
  __shared__ A s_wv[NW], s_red[NW];
  __shared__ long long s_wr[NW];
  __shared__ int s_wf[NW];
  __shared__ int s_any[3];                // per tile (mod 3): some row starts in the tile
  __shared__ A s_cv[2];                   // the row open at the end of the last flagged tile, and its id (by the
  __shared__ long long s_cr[2];           // parity q of flagged tiles: read in one, written for the next)
  __shared__ long long s_rs;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const unsigned lanemask_lt = (1u << lane) - 1u;
  const int64_t b = blockIdx.x, G = gridDim.x;
  const B* a = (const B*)p.a;
  const int64_t rows = p.rows;
  const int64_t P0 = __ldg(p.off), P1 = __ldg(p.off + rows);
  const int64_t nnz = P1 - P0;
  const int64_t lo = P0 + (int64_t)(((__int128)nnz * b) / G);
  const int64_t hi = P0 + (int64_t)(((__int128)nnz * (b + 1)) / G);
  if (wid == 0) {
    const int64_t r0 = warp_lower_bound(p.off, rows, lo);  // first row starting at or after lo
    if (lane == 0) s_rs = r0;
  }
  s_flag[t] = 0u;
  if (t == 0) s_any[0] = s_any[1] = s_any[2] = 0;
  __syncthreads();
  int64_t rs = s_rs;
  const int64_t hrow = (rs > 0 && lo < hi && __ldg(p.off + rs) > lo) ? rs - 1 : -1;  // spans lo from before
  if (t == 0) {
    p.head_row[b] = lo < hi ? -1 : -2;
    p.tail_row[b] = -1;
    s_cv[0] = R::id();
    s_cr[0] = hrow;
  }
  auto finish = [&](int64_t row, A v) {
    if (p.has_init) v = R::op(R::lift((B)p.init), v);
    ((B*)p.out)[row] = R::fin(v);
  };
  // tiles start at 32-byte aligned element positions at or below lo
  const int64_t q0 = lo - (int64_t)(((uintptr_t)(a + lo) & 31u) / sizeof(B));
  auto prefetch_tile = [&](int64_t Bc) {  // one thread: the tile's bytes into L2
    if (Bc < hi) {
      const int64_t e0 = Bc > lo ? Bc : lo;
      const int64_t e1 = Bc + TILE < hi ? Bc + TILE : hi;
      l2_prefetch(a + e0, (e1 - e0) * (int64_t)sizeof(B));
    }
  };
  // the first window of row offsets of the next tile: thread i holds off[rs + i] (and lane 31 off[rs + i + 1])
  int64_t wo = 0, wo31 = 0;
  auto fetch_window = [&](int64_t base) {
    const int64_t r = base + t;
    wo = r <= rows ? __ldg(p.off + r) : INT64_MAX;
    wo31 = (lane == 31 && r + 1 <= rows) ? __ldg(p.off + r + 1) : INT64_MAX;
  };
  if (lo < hi) {
    fetch_window(rs);
    if (t == 0)
      for (int d = 1; d < PFD; ++d) prefetch_tile(q0 + (int64_t)d * TILE);
  }
  A run = R::id();          // flag-free tiles: this thread's elements of the open row, not yet in s_cv
  bool pending = false;     // CTA-uniform: some thread's `run` holds elements
  int q = 0;                // CTA-uniform: parity of the flagged tiles so far
  auto flush_runs = [&]() {  // s_cv ⊕= the runs (thread order); ends with a barrier
    const A tot = block_reduce<R, BLOCK>(run, s_red);
    if (t == 0) s_cv[q] = R::op(s_cv[q], tot);
    run = R::id();
    pending = false;
    __syncthreads();
  };
  int par = 0;
#pragma unroll 1
  for (int64_t Bc = q0; Bc < hi; Bc += TILE, par = par == 2 ? 0 : par + 1) {
    const int rlo = (int)(lo > Bc ? lo - Bc : 0);
    const int rhi = (int)(hi - Bc < TILE ? hi - Bc : TILE);
    const bool interior = rlo == 0 && rhi == TILE;  // CTA-uniform
    const int64_t tile_end = Bc + rhi;
    if (t == 0) prefetch_tile(Bc + (int64_t)PFD * TILE);
    // this tile's elements: loads issued now, consumed after the row setup
    B x[EPT];
    {
      const B* pl = a + Bc + (int64_t)t * EPT;
      if (interior) {
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
          const VT w = ldv((const VT*)(pl + v * VW));
#pragma unroll
          for (int k = 0; k < VW; ++k) x[v * VW + k] = w.w[k];
        }
      } else {
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
          const int rel = t * EPT + k;
          x[k] = (rel >= rlo && rel < rhi) ? lds(pl + k) : (B)0;
        }
      }
    }
    // (no barrier here: every thread cleared its own flag word when it read it, and the previous tile's readers of
    // s_rid / s_val / s_any finished before its last barrier)
    // the next tile's word: last read two tiles ago, before the previous tile's row-setup barrier (with two words
    // a thread still reading the previous tile's word could race this store; racecheck, profiles/r02_san_*)
    if (t == 0) s_any[par == 2 ? 0 : par + 1] = 0;
    // 1. row setup
#pragma unroll 1
    while (true) {
      const int64_t r = rs + t;
      const int64_t o = wo;
      const int64_t up = __shfl_down_sync(FULL, o, 1);
      const int64_t e = lane == 31 ? wo31 : up;  // off[r + 1]
      const bool in = r < rows && o < tile_end;
      const bool starts = in && e > o;
      if (starts) {
        const int pos = (int)(o - Bc);
        const int tt = pos / EPT, k = pos - tt * EPT;
        atomicOr(&s_flag[tt], 1u << k);
        s_rid[k * BLOCK + tt] = (int)r;
      } else if (in) {
        finish(r, R::id());  // an empty row
      }
      if (__ballot_sync(FULL, starts) && lane == 0) s_any[par] = 1;
      const int cnt = __syncthreads_count(in);  // also publishes the flags
      rs += cnt;
      if (cnt < BLOCK) break;
      fetch_window(rs);  // every row of the window starts in this tile: the next BLOCK rows
    }
    fetch_window(rs);  // the next tile's first window, in flight while this tile is folded
    if (!s_any[par]) {
      // 2. no row starts here: every element continues the open row
      if (interior) {
#pragma unroll
        for (int k = 0; k < EPT; ++k) run = R::op(run, R::lift(x[k]));
      } else {
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
          const int rel = t * EPT + k;
          run = R::op(run, (rel >= rlo && rel < rhi) ? R::lift(x[k]) : R::id());
        }
      }
      pending = true;
      continue;
    }
    if (pending) flush_runs();
    // 3. lane fold, parking the value of every segment that ends at a flagged element
    const unsigned fl = s_flag[t];
    s_flag[t] = 0u;  // ready for the next tile's setup (which runs after this tile's scan barrier)
    A acc = R::id();
    if (interior) {
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const bool sf = (fl >> k) & 1u;
        if (sf) s_val[k * BLOCK + t] = acc;
        acc = R::op(sf ? R::id() : acc, R::lift(x[k]));
      }
    } else {
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const int rel = t * EPT + k;
        const bool sf = (fl >> k) & 1u;
        if (sf) s_val[k * BLOCK + t] = acc;
        acc = R::op(sf ? R::id() : acc, (rel >= rlo && rel < rhi) ? R::lift(x[k]) : R::id());
      }
    }
    const int kf = fl ? __ffs(fl) - 1 : 0;
    const int kl = fl ? 31 - __clz(fl) : 0;
    const A head = fl ? s_val[kf * BLOCK + t] : acc;  // elements before the first flag
    const A cur = fl ? acc : R::id();                 // from the last flag on
    for (unsigned m = fl & ~(1u << kl); m; m &= m - 1) {  // rows that start and end inside this thread
      const int k0 = __ffs(m) - 1;
      const int k1 = __ffs(fl & ~((2u << k0) - 1u)) - 1;
      finish(s_rid[k0 * BLOCK + t], s_val[k1 * BLOCK + t]);
    }
    const long long my_rid = fl ? (long long)s_rid[kl * BLOCK + t] : -1;
    // 4. segmented scan over the threads: a flagged thread starts a segment with `cur`
    const bool F = fl != 0u;
    const unsigned bal = __ballot_sync(FULL, F);
    const unsigned le = bal & (lanemask_lt | (1u << lane));
    const int start = le ? 31 - __clz(le) : 0;
    A sv = F ? cur : head;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const A ov = shfl_up_acc(sv, d);
      if (lane - d >= start) sv = R::op(ov, sv);
    }
    const long long wlast_rid = __shfl_sync(FULL, my_rid, bal ? 31 - __clz(bal) : 0);
    if (lane == 31) {
      s_wv[wid] = sv;
      s_wf[wid] = bal != 0u;
      s_wr[wid] = wlast_rid;
    }
    __syncthreads();
    // the row open at this warp's start: the tile's carry-in folded with the earlier warps, in warp order
    A P = s_cv[q];
    long long PR = s_cr[q];
    for (int w2 = 0; w2 < wid; ++w2) {
      if (s_wf[w2]) {
        P = s_wv[w2];
        PR = s_wr[w2];
      } else {
        P = R::op(P, s_wv[w2]);
      }
    }
    const unsigned lt = bal & lanemask_lt;
    const A ev = shfl_up_acc(sv, 1);
    const long long rr = __shfl_sync(FULL, my_rid, lt ? 31 - __clz(lt) : 0);
    const A E = lt ? ev : (lane == 0 ? P : R::op(P, ev));  // the row open at this thread's start
    const long long ER = lt ? rr : PR;
    if (F && ER >= 0) {  // ... ends at this thread's first flag
      const A v = R::op(E, head);
      if (ER == hrow) {
        p.head_row[b] = hrow;
        p.head_part[b] = pack(v);
      } else {
        finish(ER, v);
      }
    }
    if (t == BLOCK - 1) {  // the row open at the end of the tile, for the next flagged tile
      s_cv[q ^ 1] = bal ? sv : R::op(P, sv);
      s_cr[q ^ 1] = bal ? wlast_rid : PR;
    }
    q ^= 1;
  }
  if (pending) flush_runs();
  __syncthreads();
  // the row still open at hi
  if (t == 0 && lo < hi) {
    const long long orid = s_cr[q];
    const A ov = s_cv[q];
    if (orid >= 0) {
      if (orid == hrow) {
        p.head_row[b] = hrow;
        p.head_part[b] = pack(ov);
      } else if (__ldg(p.off + orid + 1) <= hi) {
        finish(orid, ov);
      } else {
        p.tail_row[b] = orid;
        p.tail_part[b] = pack(ov);
      }
    }
  }
  // the last CTA also owns the empty rows that start at P1 (after every element)
  if (b == G - 1 && wid == 0) {
    const int64_t r = warp_lower_bound(p.off, rows, P1);
    for (int64_t q = r + lane; q < rows; q += 32)
      if (__ldg(p.off + q) == __ldg(p.off + q + 1)) finish(q, R::id());
  }
}

}  // namespace ipm
