// ipm_fused.cuh — several reduction variables over ONE pass of the iteration space.
//
// A loop may carry more than one reduction variable ("reduction clauses carry ... >=1 scalar
// variable"; SPEC.md:253 a reduction list per kernel) and the loop body may fold an expression of the
// element rather than the element itself — SRAD's reduction region accumulates the sum and the sum of squares
// of the image. Each variable keeps its own private accumulator in every thread; the warp,
// CTA and cross-CTA levels run once per variable. Expressions are evaluated in the accumulator domain
// (R13 in DESIGN.md): x*x and x*y of float32 inputs are exact in float64, integer products wrap mod 2^w.
#pragma once
#include <type_traits>
#include "ipm_kernels.cuh"

namespace ipm {

enum { EX = 0, EXX = 1, EXY = 2 };

// one reduction variable: operator R applied to expression E of (x, y)
template <class R, int E>
struct Comp {
  using A = typename R::A;
  using B = typename R::B;
  __device__ static A id() { return R::id(); }
  __device__ static A val(B x, B y) {
    if constexpr (E == EX) {
      return R::lift(x);
    } else if constexpr (E == EXX) {
      const A v = R::lift(x);
      return v * v;
    } else {
      return R::lift(x) * R::lift(y);
    }
  }
  __device__ static A op(A a, A b) { return R::op(a, b); }
  __device__ static A warp(A a) { return R::warp(a); }
  __device__ static B fin(A a, uint64_t init, int has_init) {
    return R::fin(has_init ? R::op(R::lift((B)init), a) : a);
  }
};

struct NoComp {
  using A = uint32_t;
  using B = uint32_t;
  __device__ static A id() { return 0u; }
  __device__ static A val(B, B) { return 0u; }
  __device__ static A op(A a, A) { return a; }
  __device__ static A warp(A a) { return a; }
  __device__ static B fin(A a, uint64_t, int) { return a; }
};

template <class C0, class C1 = NoComp, class C2 = NoComp, class C3 = NoComp>
struct Sig {
  using B = typename C0::B;
  static constexpr int NV = 1 + !std::is_same<C1, NoComp>::value + !std::is_same<C2, NoComp>::value +
                            !std::is_same<C3, NoComp>::value;
  struct Acc {
    typename C0::A a0;
    typename C1::A a1;
    typename C2::A a2;
    typename C3::A a3;
  };
  __device__ static Acc id() { return {C0::id(), C1::id(), C2::id(), C3::id()}; }
  __device__ static Acc val(B x, B y) { return {C0::val(x, y), C1::val(x, y), C2::val(x, y), C3::val(x, y)}; }
  __device__ static Acc op(const Acc& a, const Acc& b) {
    return {C0::op(a.a0, b.a0), C1::op(a.a1, b.a1), C2::op(a.a2, b.a2), C3::op(a.a3, b.a3)};
  }
};

struct FusedParams {
  const void* x;
  const void* y;          // second stream (EXY), else nullptr
  int64_t n;
  uint64_t init[4];
  int has_init;
  void* out;              // NV elements of the element type
  uint64_t* partials;     // NV * gridDim.x slots, variable-major
  unsigned* ticket;
};

template <class C>
__device__ __forceinline__ typename C::A fused_block(typename C::A v, uint64_t* sm8) {
  using A = typename C::A;
  A* sm = (A*)sm8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = C::warp(v);
  __syncthreads();
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  A r = C::id();
  if (warp == 0) {
    r = lane < (int)(blockDim.x >> 5) ? sm[lane] : C::id();
    r = C::warp(r);
  }
  return r;
}

template <class C>
__device__ __forceinline__ void fused_finish(const FusedParams& p, int v, typename C::A cta, bool last,
                                             uint64_t* sm8) {
  using A = typename C::A;
  using B = typename C::B;
  if (!last) return;
  A t = C::id();
  const uint64_t* parts = p.partials + (size_t)v * gridDim.x;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) t = C::op(t, unpack<A>(__ldcg(parts + i)));
  t = fused_block<C>(t, sm8);
  if (threadIdx.x == 0) ((B*)p.out)[v] = C::fin(t, p.init[v], p.has_init);
}

// TWO: read y as a second stream. VEC: both streams share the same alignment mod 32 (256-bit loads); else
// element loads (coalesced across the warp).
// MINB: the launch-bounds minimum of resident CTAs per SM. 0 (the product) states none: ptxas then gives the
// float32 x*y kernel 48 registers (4 CTAs per SM resident, 7.03-7.12 TB/s); MINB = 4 made it 61 registers and
// 4 % slower, MINB = 1 left 1 resident CTA (profiles/r01_sweep_fused_pipe.txt)
template <class S, class C0, class C1, class C2, class C3, bool TWO, bool VEC, int BLOCK, int U, bool PIPE = false,
          int MINB = 0>
__global__ void __launch_bounds__(BLOCK, MINB) k_fused(FusedParams p) {
  using B = typename S::B;
  using Acc = typename S::Acc;
  using VT = typename Vec<B>::T;
  constexpr int VW = Vec<B>::W;
  constexpr int64_t TILE = (int64_t)BLOCK * U;
  __shared__ uint64_t sm8[32];
  __shared__ int s_last;
  const B* x = (const B*)p.x;
  const B* y = TWO ? (const B*)p.y : x;
  const int64_t n = p.n;
  Acc acc[2] = {S::id(), S::id()};
  const int64_t g = (int64_t)blockIdx.x * BLOCK + threadIdx.x;
  const int64_t gsz = (int64_t)gridDim.x * BLOCK;
  if (VEC) {
    int64_t head = (int64_t)(((32u - ((uintptr_t)x & 31u)) & 31u) / sizeof(B));
    if (head > n) head = n;
    const int64_t nv = (n - head) / VW;
    const int64_t tail0 = head + nv * VW;
    const VT* xv = (const VT*)(x + head);
    const VT* yv = (const VT*)(y + head);
    const int64_t ntiles = nv / TILE;
    // PIPE: the next tile's loads are issued before this one is folded (measured equal or slower than the plain
    // loop: the extra registers cost resident CTAs, profiles/r01_sweep_fused_pipe.txt; the product uses PIPE=false)
    if (PIPE && (int64_t)blockIdx.x < ntiles) {
      VT na[U], nb[TWO ? U : 1];
      auto issue = [&](int64_t t) {
        const int64_t base = t * TILE + threadIdx.x;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          na[u] = ldv(xv + base + u * BLOCK);
          if (TWO) nb[TWO ? u : 0] = ldv(yv + base + u * BLOCK);
        }
      };
      issue(blockIdx.x);
#pragma unroll 1
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        VT a[U], b[TWO ? U : 1];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          a[u] = na[u];
          if (TWO) b[TWO ? u : 0] = nb[TWO ? u : 0];
        }
        if (t + gridDim.x < ntiles) issue(t + gridDim.x);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int k = 0; k < VW; ++k)
            acc[k & 1] = S::op(acc[k & 1], S::val(a[u].w[k], TWO ? b[TWO ? u : 0].w[k] : a[u].w[k]));
      }
    }
    for (int64_t t = blockIdx.x; !PIPE && t < ntiles; t += gridDim.x) {
      const int64_t base = t * TILE + threadIdx.x;
      VT a[U], b[TWO ? U : 1];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a[u] = ldv(xv + base + u * BLOCK);
        if (TWO) b[TWO ? u : 0] = ldv(yv + base + u * BLOCK);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < VW; ++k)
          acc[k & 1] = S::op(acc[k & 1], S::val(a[u].w[k], TWO ? b[TWO ? u : 0].w[k] : a[u].w[k]));
    }
    for (int64_t i = ntiles * TILE + g; i < nv; i += gsz) {
      const VT a = ldv(xv + i);
      const VT b = TWO ? ldv(yv + i) : a;
#pragma unroll
      for (int k = 0; k < VW; ++k) acc[k & 1] = S::op(acc[k & 1], S::val(a.w[k], b.w[k]));
    }
    if (g < head) acc[0] = S::op(acc[0], S::val(lds(x + g), lds(y + g)));
    if (g < n - tail0) acc[1] = S::op(acc[1], S::val(lds(x + tail0 + g), lds(y + tail0 + g)));
  } else {
    for (int64_t i = g; i < n; i += gsz) acc[i & 1] = S::op(acc[i & 1], S::val(lds(x + i), lds(y + i)));
  }
  Acc t = S::op(acc[0], acc[1]);
  // per-variable CTA totals
  typename C0::A c0 = fused_block<C0>(t.a0, sm8);
  typename C1::A c1 = S::NV > 1 ? fused_block<C1>(t.a1, sm8) : C1::id();
  typename C2::A c2 = S::NV > 2 ? fused_block<C2>(t.a2, sm8) : C2::id();
  typename C3::A c3 = S::NV > 3 ? fused_block<C3>(t.a3, sm8) : C3::id();
  if (gridDim.x == 1) {
    if (threadIdx.x == 0) {
      using BB = typename C0::B;
      ((BB*)p.out)[0] = C0::fin(c0, p.init[0], p.has_init);
      if (S::NV > 1) ((BB*)p.out)[1] = C1::fin(c1, p.init[1], p.has_init);
      if (S::NV > 2) ((BB*)p.out)[2] = C2::fin(c2, p.init[2], p.has_init);
      if (S::NV > 3) ((BB*)p.out)[3] = C3::fin(c3, p.init[3], p.has_init);
    }
    return;
  }
  if (threadIdx.x == 0) {
    __stcg(p.partials + blockIdx.x, pack(c0));
    if (S::NV > 1) __stcg(p.partials + gridDim.x + blockIdx.x, pack(c1));
    if (S::NV > 2) __stcg(p.partials + 2 * gridDim.x + blockIdx.x, pack(c2));
    if (S::NV > 3) __stcg(p.partials + 3 * gridDim.x + blockIdx.x, pack(c3));
    s_last = ticket_acq_rel(p.ticket) == gridDim.x - 1;
  }
  __syncthreads();
  const bool last = s_last;
  if (!last) return;
  fused_finish<C0>(p, 0, c0, last, sm8);
  if (S::NV > 1) fused_finish<C1>(p, 1, c1, last, sm8);
  if (S::NV > 2) fused_finish<C2>(p, 2, c2, last, sm8);
  if (S::NV > 3) fused_finish<C3>(p, 3, c3, last, sm8);
  if (threadIdx.x == 0) *p.ticket = 0u;
}

}  // namespace ipm
