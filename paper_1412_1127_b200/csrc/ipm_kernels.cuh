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
//   k_seg_warp  the nested gang-outer / vector-inner clause, one warp per row (a8)
//   k_seg_group the same for short rows: a group of G <= 32 lanes per row
//   k_finalize  fold of P accumulator slots (cross-rank, or cross-chunk) + init, rounding to T (a6/a9)
#pragma once
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

__device__ __forceinline__ V8 ldv(const V8* p) {
  V8 v;
  asm("ld.global.nc.L1::no_allocate.L2::evict_first.L2::256B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]), "=r"(v.w[6]),
        "=r"(v.w[7])
      : "l"(p));
  return v;
}
__device__ __forceinline__ V4 ldv(const V4* p) {
  V4 v;
  asm("ld.global.nc.L1::no_allocate.L2::evict_first.L2::256B.v4.b64 {%0,%1,%2,%3}, [%4];"
      : "=l"(v.w[0]), "=l"(v.w[1]), "=l"(v.w[2]), "=l"(v.w[3])
      : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t lds(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint64_t lds(const uint64_t* p) { return (uint64_t)__ldg((const unsigned long long*)p); }

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
};
enum { MODE_RESULT = 0, MODE_PARTIAL = 1, MODE_ACCUM_FIRST = 2, MODE_ACCUM = 3 };

template <class R>
__device__ __forceinline__ void store_out(const FlatParams& p, int64_t row, typename R::A total) {
  using A = typename R::A;
  using B = typename R::B;
  switch (p.mode) {
    case MODE_RESULT: {
      A t = total;
      if (p.has_init) t = R::op(R::lift((B)p.init), total);  // var = var_original ⊕ fold (R1)
      ((B*)p.out)[row] = R::fin(t);
      break;
    }
    case MODE_PARTIAL: ((uint64_t*)p.out)[row] = pack(total); break;
    case MODE_ACCUM_FIRST: *(uint64_t*)p.out = pack(total); break;
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

// ------------------------------------------------------------------------------------------ flat
template <class R, int BLOCK, int U>
__global__ void __launch_bounds__(BLOCK) k_flat(FlatParams p) {
  using B = typename R::B;
  using A = typename R::A;
  using VT = typename Vec<B>::T;
  constexpr int VW = Vec<B>::W;
  constexpr int64_t TILE = (int64_t)BLOCK * U;
  __shared__ A sm[BLOCK / 32 > 0 ? BLOCK / 32 : 1];
  __shared__ int s_last;

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

  A acc[VW];
#pragma unroll
  for (int k = 0; k < VW; ++k) acc[k] = R::id();

  // a3: the hot loop — whole tiles of BLOCK*U vectors, U independent 256-bit loads in flight per thread
  const int64_t ntiles = nv / TILE;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const VT* base = vp + t * TILE + threadIdx.x;
    VT v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldv(base + u * BLOCK);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < VW; ++k) acc[k] = R::op(acc[k], R::lift(v[u].w[k]));
  }
  // ragged last tile
  for (int64_t i = ntiles * TILE + (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * BLOCK) {
    const VT v = ldv(vp + i);
#pragma unroll
    for (int k = 0; k < VW; ++k) acc[k] = R::op(acc[k], R::lift(v.w[k]));
  }
  // head and tail scalars (< VW each)
  const int64_t g = (int64_t)blockIdx.x * BLOCK + threadIdx.x;
  if (g < head) acc[0] = R::op(acc[0], R::lift(lds(a + g)));
  if (g < n - tail0) acc[VW - 1] = R::op(acc[VW - 1], R::lift(lds(a + tail0 + g)));

  // fold the private copies in a fixed tree
#pragma unroll
  for (int s = VW / 2; s > 0; s >>= 1)
#pragma unroll
    for (int k = 0; k < s; ++k) acc[k] = R::op(acc[k], acc[k + s]);

  // a4 + a5
  A cta = block_reduce<R, BLOCK>(acc[0], sm);

  if (gridDim.x == 1) {
    if (threadIdx.x == 0) store_out<R>(p, row, cta);
    return;
  }
  // a6: publish the CTA partial; the CTA that takes the last ticket finishes the row
  uint64_t* parts = p.partials + row * gridDim.x;
  if (threadIdx.x == 0) {
    __stcg(parts + blockIdx.x, pack(cta));
    __threadfence();
    const unsigned t = atomicAdd(p.tickets + row, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  A v = R::id();
  for (int i = threadIdx.x; i < (int)gridDim.x; i += BLOCK) v = R::op(v, unpack<A>(__ldcg(parts + i)));
  __syncthreads();  // sm reuse
  A total = block_reduce<R, BLOCK>(v, sm);
  if (threadIdx.x == 0) {
    store_out<R>(p, row, total);
    p.tickets[row] = 0u;  // ready for the next launch on this workspace
  }
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
template <class R, int WARPS, int U>
__global__ void __launch_bounds__(WARPS * 32) k_seg_warp(SegParams p) {
  using B = typename R::B;
  using A = typename R::A;
  using VT = typename Vec<B>::T;
  constexpr int VW = Vec<B>::W;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  for (int64_t r = gw; r < p.rows; r += nw) {
    const B* a = (const B*)p.a + r * p.row_stride;
    const int64_t n = p.cols;
    int64_t head = (int64_t)(((32u - ((uintptr_t)a & 31u)) & 31u) / sizeof(B));
    if (head > n) head = n;
    const int64_t nv = (n - head) / VW;
    const int64_t tail0 = head + nv * VW;
    const VT* vp = (const VT*)(a + head);
    A acc[VW];
#pragma unroll
    for (int k = 0; k < VW; ++k) acc[k] = R::id();
    int64_t i = lane;
    for (; i + (U - 1) * 32 < nv; i += U * 32) {
      VT v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ldv(vp + i + u * 32);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < VW; ++k) acc[k] = R::op(acc[k], R::lift(v[u].w[k]));
    }
    for (; i < nv; i += 32) {
      const VT v = ldv(vp + i);
#pragma unroll
      for (int k = 0; k < VW; ++k) acc[k] = R::op(acc[k], R::lift(v.w[k]));
    }
    if (lane < head) acc[0] = R::op(acc[0], R::lift(lds(a + lane)));
    if (lane < n - tail0) acc[VW - 1] = R::op(acc[VW - 1], R::lift(lds(a + tail0 + lane)));
#pragma unroll
    for (int s = VW / 2; s > 0; s >>= 1)
#pragma unroll
      for (int k = 0; k < s; ++k) acc[k] = R::op(acc[k], acc[k + s]);
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
