// ipm_ops.cuh — the nine reduction operators of the OpenACC `reduction(op:var)` clause on the four element
// types, as device-side accumulator algebras.
//
// Each Red<OP, DT> defines
//   B      raw element bits (uint32_t / uint64_t) — what the vector loads deliver
//   A      the accumulator: the private copy of `var` each thread holds ("per-thread private v
//          initialized to op's identity"); chosen so that ⊕ on A is associative and commutative, which makes
//          the result independent of how iterations are spread over lanes, warps and CTAs:
//            int + * & | ^  -> unsigned w-bit words (wrap mod 2^w, R3)
//            int max min    -> signed w-bit integers
//            && ||          -> unsigned words: && = unsigned min of the truth-relevant bits (0 iff some element
//                              is false), || = bitwise or (≠0 iff some element is true) — C truthiness (R5)
//            f32 + *        -> float64 (one rounding at the end, R6);  f64 + * -> float64
//            f32 max min    -> {max.NaN/min.NaN of the values, signed max/min of the raw bits}; the second
//                              component decides the sign of a zero result (IEEE 754-2019 maximum, R10)
//            f64 max min    -> a 64-bit totally-ordered integer key, NaN mapped to the absorbing end (R10)
//   id()   identity of ⊕ on A            lift(b)  element bits -> A
//   op()   ⊕ on A                        warp(a)  ⊕ over the 32 lanes (all lanes get the result)
//   fin(a) A -> result bits of the element type (canonical quiet NaN, 0/1 for && ||)
//
// Vector level = a warp ("vector ... warp"): redux.sync where the ISA has it (REDUX / CREDUX on
// sm_100a), a xor-butterfly of shuffles otherwise.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "ipm.h"

namespace ipm {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ float u2f(uint32_t b) { return __uint_as_float(b); }
__device__ __forceinline__ uint32_t f2u(float f) { return __float_as_uint(f); }
__device__ __forceinline__ double u2d(uint64_t b) { return __longlong_as_double((long long)b); }
__device__ __forceinline__ uint64_t d2u(double d) { return (uint64_t)__double_as_longlong(d); }

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fmin_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float redux_fmax_nan(float a) {
  float r;
  asm volatile("redux.sync.max.NaN.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(a));
  return r;
}
__device__ __forceinline__ float redux_fmin_nan(float a) {
  float r;
  asm volatile("redux.sync.min.NaN.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(a));
  return r;
}

template <class X, class F>
__device__ __forceinline__ X butterfly(X v, F f) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = f(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

template <int OP, int DT>
struct Red;

// ------------------------------------------------------------------------------------------ int32
template <>
struct Red<IPM_ADD, IPM_I32> {
  using B = uint32_t; using A = uint32_t;
  __device__ static A id() { return 0u; }
  __device__ static A lift(B b) { return b; }
  __device__ static A op(A a, A b) { return a + b; }
  __device__ static A warp(A a) { return __reduce_add_sync(FULL, a); }
  __device__ static B fin(A a) { return a; }
};
template <>
struct Red<IPM_MUL, IPM_I32> {
  using B = uint32_t; using A = uint32_t;
  __device__ static A id() { return 1u; }
  __device__ static A lift(B b) { return b; }
  __device__ static A op(A a, A b) { return a * b; }
  __device__ static A warp(A a) { return butterfly(a, [](A x, A y) { return x * y; }); }
  __device__ static B fin(A a) { return a; }
};
template <>
struct Red<IPM_MAX, IPM_I32> {
  using B = uint32_t; using A = int32_t;
  __device__ static A id() { return INT32_MIN; }
  __device__ static A lift(B b) { return (int32_t)b; }
  __device__ static A op(A a, A b) { return max(a, b); }
  __device__ static A warp(A a) { return __reduce_max_sync(FULL, a); }
  __device__ static B fin(A a) { return (uint32_t)a; }
};
template <>
struct Red<IPM_MIN, IPM_I32> {
  using B = uint32_t; using A = int32_t;
  __device__ static A id() { return INT32_MAX; }
  __device__ static A lift(B b) { return (int32_t)b; }
  __device__ static A op(A a, A b) { return min(a, b); }
  __device__ static A warp(A a) { return __reduce_min_sync(FULL, a); }
  __device__ static B fin(A a) { return (uint32_t)a; }
};
template <>
struct Red<IPM_BAND, IPM_I32> {
  using B = uint32_t; using A = uint32_t;
  __device__ static A id() { return ~0u; }
  __device__ static A lift(B b) { return b; }
  __device__ static A op(A a, A b) { return a & b; }
  __device__ static A warp(A a) { return __reduce_and_sync(FULL, a); }
  __device__ static B fin(A a) { return a; }
};
template <>
struct Red<IPM_BOR, IPM_I32> {
  using B = uint32_t; using A = uint32_t;
  __device__ static A id() { return 0u; }
  __device__ static A lift(B b) { return b; }
  __device__ static A op(A a, A b) { return a | b; }
  __device__ static A warp(A a) { return __reduce_or_sync(FULL, a); }
  __device__ static B fin(A a) { return a; }
};
template <>
struct Red<IPM_BXOR, IPM_I32> {
  using B = uint32_t; using A = uint32_t;
  __device__ static A id() { return 0u; }
  __device__ static A lift(B b) { return b; }
  __device__ static A op(A a, A b) { return a ^ b; }
  __device__ static A warp(A a) { return __reduce_xor_sync(FULL, a); }
  __device__ static B fin(A a) { return a; }
};
template <>
struct Red<IPM_LAND, IPM_I32> {  // unsigned min of the words: 0 iff some element is 0
  using B = uint32_t; using A = uint32_t;
  __device__ static A id() { return ~0u; }
  __device__ static A lift(B b) { return b; }
  __device__ static A op(A a, A b) { return min(a, b); }
  __device__ static A warp(A a) { return __reduce_min_sync(FULL, a); }
  __device__ static B fin(A a) { return a != 0u ? 1u : 0u; }
};
template <>
struct Red<IPM_LOR, IPM_I32> {  // or of the words: ≠0 iff some element is ≠0
  using B = uint32_t; using A = uint32_t;
  __device__ static A id() { return 0u; }
  __device__ static A lift(B b) { return b; }
  __device__ static A op(A a, A b) { return a | b; }
  __device__ static A warp(A a) { return __reduce_or_sync(FULL, a); }
  __device__ static B fin(A a) { return a != 0u ? 1u : 0u; }
};

// ------------------------------------------------------------------------------------------ int64
#define IPM_RED64(OPC, IDV, EXPR, FINEXPR)                                                     \
  template <>                                                                                  \
  struct Red<OPC, IPM_I64> {                                                                   \
    using B = uint64_t; using A = uint64_t;                                                    \
    __device__ static A id() { return IDV; }                                                   \
    __device__ static A lift(B b) { return b; }                                                \
    __device__ static A op(A a, A b) { return EXPR; }                                          \
    __device__ static A warp(A a) { return butterfly(a, [](A x, A y) { return op(x, y); }); } \
    __device__ static B fin(A a) { return FINEXPR; }                                           \
  };
IPM_RED64(IPM_ADD, 0ull, a + b, a)
IPM_RED64(IPM_MUL, 1ull, a * b, a)
IPM_RED64(IPM_BAND, ~0ull, a & b, a)
IPM_RED64(IPM_BOR, 0ull, a | b, a)
IPM_RED64(IPM_BXOR, 0ull, a ^ b, a)
IPM_RED64(IPM_LOR, 0ull, a | b, (a != 0ull ? 1ull : 0ull))
#undef IPM_RED64
template <>
struct Red<IPM_LAND, IPM_I64> {  // unsigned min of the words: 0 iff some element is 0
  using B = uint64_t; using A = uint64_t;
  __device__ static A id() { return ~0ull; }
  __device__ static A lift(B b) { return b; }
  __device__ static A op(A a, A b) { return a < b ? a : b; }
  __device__ static A warp(A a) { return butterfly(a, [](A x, A y) { return op(x, y); }); }
  __device__ static B fin(A a) { return a != 0ull ? 1ull : 0ull; }
  // lane-local: unsigned min of (low | high) words, 32 bits (0 iff some element is 0): 2 instructions per element
  using L = uint32_t;
  __device__ static L lid() { return ~0u; }
  __device__ static L lstep(L l, B b) { return min(l, (uint32_t)b | (uint32_t)(b >> 32)); }
  __device__ static L lcomb(L a, L b) { return min(a, b); }
  __device__ static A lout(L l) { return l; }
};

template <>
struct Red<IPM_MAX, IPM_I64> {
  using B = uint64_t; using A = int64_t;
  __device__ static A id() { return INT64_MIN; }
  __device__ static A lift(B b) { return (int64_t)b; }
  __device__ static A op(A a, A b) { return a > b ? a : b; }
  __device__ static A warp(A a) { return butterfly(a, [](A x, A y) { return op(x, y); }); }
  __device__ static B fin(A a) { return (uint64_t)a; }
};
template <>
struct Red<IPM_MIN, IPM_I64> {
  using B = uint64_t; using A = int64_t;
  __device__ static A id() { return INT64_MAX; }
  __device__ static A lift(B b) { return (int64_t)b; }
  __device__ static A op(A a, A b) { return a < b ? a : b; }
  __device__ static A warp(A a) { return butterfly(a, [](A x, A y) { return op(x, y); }); }
  __device__ static B fin(A a) { return (uint64_t)a; }
};

// ------------------------------------------------------------------------------------------ float32
template <>
struct Red<IPM_ADD, IPM_F32> {  // float64 accumulation, one rounding to float32 at the end (R6)
  using B = uint32_t; using A = double;
  __device__ static A id() { return 0.0; }
  __device__ static A lift(B b) { return (double)u2f(b); }
  __device__ static A op(A a, A b) { return a + b; }
  __device__ static A warp(A a) { return butterfly(a, [](A x, A y) { return x + y; }); }
  __device__ static B fin(A a) {
    const float f = __double2float_rn(a);
    return f != f ? 0x7FC00000u : f2u(f);
  }
};
template <>
struct Red<IPM_MUL, IPM_F32> {
  using B = uint32_t; using A = double;
  __device__ static A id() { return 1.0; }
  __device__ static A lift(B b) { return (double)u2f(b); }
  __device__ static A op(A a, A b) { return a * b; }
  __device__ static A warp(A a) { return butterfly(a, [](A x, A y) { return x * y; }); }
  __device__ static B fin(A a) {
    const float f = __double2float_rn(a);
    return f != f ? 0x7FC00000u : f2u(f);
  }
};

struct FPair {  // {NaN-propagating extreme of the values, signed extreme of the raw bits}
  float m;
  int32_t s;
};
template <>
struct Red<IPM_MAX, IPM_F32> {
  // m = max.NaN over the values: exact except for the sign of a zero result. s = signed max of the raw
  // bits: s >= 0 iff some element has its sign bit clear; if the maximum is ±0 that element is +0.
  using B = uint32_t; using A = FPair;
  __device__ static A id() { return {-__int_as_float(0x7f800000), INT32_MIN}; }
  __device__ static A lift(B b) { return {u2f(b), (int32_t)b}; }
  __device__ static A op(A a, A b) { return {fmax_nan(a.m, b.m), max(a.s, b.s)}; }
  __device__ static A warp(A a) { return {redux_fmax_nan(a.m), __reduce_max_sync(FULL, a.s)}; }
  __device__ static B fin(A a) {
    if (a.m != a.m) return 0x7FC00000u;
    if (a.m == 0.0f) return a.s >= 0 ? 0x00000000u : 0x80000000u;
    return f2u(a.m);
  }
};
template <>
struct Red<IPM_MIN, IPM_F32> {
  // s = signed min of the raw bits: s == INT32_MIN iff some element is -0.0 (its bits are 0x80000000).
  using B = uint32_t; using A = FPair;
  __device__ static A id() { return {__int_as_float(0x7f800000), INT32_MAX}; }
  __device__ static A lift(B b) { return {u2f(b), (int32_t)b}; }
  __device__ static A op(A a, A b) { return {fmin_nan(a.m, b.m), min(a.s, b.s)}; }
  __device__ static A warp(A a) { return {redux_fmin_nan(a.m), __reduce_min_sync(FULL, a.s)}; }
  __device__ static B fin(A a) {
    if (a.m != a.m) return 0x7FC00000u;
    if (a.m == 0.0f) return a.s == INT32_MIN ? 0x80000000u : 0x00000000u;
    return f2u(a.m);
  }
};
template <>
struct Red<IPM_LAND, IPM_F32> {  // truth = magnitude bits ≠ 0 (so -0.0 is false, NaN true)
  using B = uint32_t; using A = uint32_t;
  __device__ static A id() { return ~0u; }
  __device__ static A lift(B b) { return b & 0x7FFFFFFFu; }
  __device__ static A op(A a, A b) { return min(a, b); }
  __device__ static A warp(A a) { return __reduce_min_sync(FULL, a); }
  __device__ static B fin(A a) { return a != 0u ? 0x3F800000u : 0u; }
};
template <>
struct Red<IPM_LOR, IPM_F32> {  // or of the raw bits; the sign bit is masked off at the end
  using B = uint32_t; using A = uint32_t;
  __device__ static A id() { return 0u; }
  __device__ static A lift(B b) { return b; }
  __device__ static A op(A a, A b) { return a | b; }
  __device__ static A warp(A a) { return __reduce_or_sync(FULL, a); }
  __device__ static B fin(A a) { return (a & 0x7FFFFFFFu) != 0u ? 0x3F800000u : 0u; }
};

// ------------------------------------------------------------------------------------------ float64
template <>
struct Red<IPM_ADD, IPM_F64> {
  using B = uint64_t; using A = double;
  __device__ static A id() { return 0.0; }
  __device__ static A lift(B b) { return u2d(b); }
  __device__ static A op(A a, A b) { return a + b; }
  __device__ static A warp(A a) { return butterfly(a, [](A x, A y) { return x + y; }); }
  __device__ static B fin(A a) { return a != a ? 0x7FF8000000000000ull : d2u(a); }
};
template <>
struct Red<IPM_MUL, IPM_F64> {
  using B = uint64_t; using A = double;
  __device__ static A id() { return 1.0; }
  __device__ static A lift(B b) { return u2d(b); }
  __device__ static A op(A a, A b) { return a * b; }
  __device__ static A warp(A a) { return butterfly(a, [](A x, A y) { return x * y; }); }
  __device__ static B fin(A a) { return a != a ? 0x7FF8000000000000ull : d2u(a); }
};

// totally ordered key of a double: non-negative values keep their bits, negative values flip the magnitude
// bits, so that signed integer order = IEEE order with -0 < +0; NaN is mapped to SENT (absorbing for ⊕)
template <int64_t SENT>
__device__ __forceinline__ int64_t f64_key(uint64_t b) {
  const bool nan = (b & 0x7FFFFFFFFFFFFFFFull) > 0x7FF0000000000000ull;
  const int64_t k = (int64_t)(b ^ ((uint64_t)((int64_t)b >> 63) & 0x7FFFFFFFFFFFFFFFull));
  return nan ? SENT : k;
}
__device__ __forceinline__ uint64_t f64_unkey(int64_t k) {
  return (uint64_t)(k ^ ((k >> 63) & 0x7FFFFFFFFFFFFFFFll));
}
// any of four doubles is a NaN: `yes` if so, `no` otherwise (four chained unordered compares, one select)
__device__ __forceinline__ int32_t any_nan4(uint64_t a, uint64_t b, uint64_t c, uint64_t d, int32_t yes, int32_t no) {
  int32_t r;
  asm("{\n.reg .pred p;\n"
      "setp.nan.f64 p, %1, %1;\n"
      "setp.nan.or.f64 p, %2, %2, p;\n"
      "setp.nan.or.f64 p, %3, %3, p;\n"
      "setp.nan.or.f64 p, %4, %4, p;\n"
      "selp.s32 %0, %5, %6, p;\n}"
      : "=r"(r)
      : "d"(u2d(a)), "d"(u2d(b)), "d"(u2d(c)), "d"(u2d(d)), "r"(yes), "r"(no));
  return r;
}
// lane-local accumulator of float64 max / min (L): the extreme VALUE kept by a compare-select (a NaN operand is
// never selected) plus one 32-bit word s over the elements' high words: for max the signed maximum (>= 0 iff some
// element has its sign bit clear — if the maximum is ±0 that element is +0), for min the unsigned maximum
// (>= 2^31 iff some element has its sign bit set — if the minimum is ±0 that element is -0); s is forced to its
// absorbing value (INT32_MAX / 0xFFFFFFFF, itself only the high word of a NaN) when a NaN is seen. 4 instructions
// per element + 6 per 32-byte vector, against 15 per element for the order-preserving key; the key (A) is formed
// once, when the lane's value leaves the register (lout), so partial slots, warp and CTA combines are unchanged.
struct F64Ext {
  double m;
  int32_t s;
};
template <>
struct Red<IPM_MAX, IPM_F64> {
  using B = uint64_t; using A = int64_t;
  __device__ static A id() { return (int64_t)(0xFFF0000000000000ull ^ 0x7FFFFFFFFFFFFFFFull); }  // key(-inf)
  __device__ static A lift(B b) { return f64_key<INT64_MAX>(b); }
  __device__ static A op(A a, A b) { return a > b ? a : b; }
  __device__ static A warp(A a) { return butterfly(a, [](A x, A y) { return op(x, y); }); }
  __device__ static B fin(A a) { return a == INT64_MAX ? 0x7FF8000000000000ull : f64_unkey(a); }
  using L = F64Ext;
  __device__ static L lid() { return {-__longlong_as_double(0x7FF0000000000000ll), INT32_MIN}; }
  __device__ static L lstep(L l, B b) {
    const double x = u2d(b);
    return {x > l.m ? x : l.m, max(l.s, (int32_t)(b >> 32))};
  }
  __device__ static void lnan(L& l, B a, B b, B c, B d) { l.s = max(l.s, any_nan4(a, b, c, d, INT32_MAX, INT32_MIN)); }
  __device__ static L lcomb(L a, L b) { return {b.m > a.m ? b.m : a.m, max(a.s, b.s)}; }
  __device__ static A lout(L l) {
    if (l.s == INT32_MAX) return INT64_MAX;
    const uint64_t bits = l.m == 0.0 ? (l.s >= 0 ? 0ull : 0x8000000000000000ull) : d2u(l.m);
    return (int64_t)(bits ^ ((uint64_t)((int64_t)bits >> 63) & 0x7FFFFFFFFFFFFFFFull));
  }
};
template <>
struct Red<IPM_MIN, IPM_F64> {
  using B = uint64_t; using A = int64_t;
  __device__ static A id() { return (int64_t)0x7FF0000000000000ll; }  // key(+inf)
  __device__ static A lift(B b) { return f64_key<INT64_MIN>(b); }
  __device__ static A op(A a, A b) { return a < b ? a : b; }
  __device__ static A warp(A a) { return butterfly(a, [](A x, A y) { return op(x, y); }); }
  __device__ static B fin(A a) { return a == INT64_MIN ? 0x7FF8000000000000ull : f64_unkey(a); }
  using L = F64Ext;  // s: unsigned maximum of the high words, kept in an int32_t
  __device__ static L lid() { return {__longlong_as_double(0x7FF0000000000000ll), 0}; }
  __device__ static L lstep(L l, B b) {
    const double x = u2d(b);
    return {x < l.m ? x : l.m, (int32_t)max((uint32_t)l.s, (uint32_t)(b >> 32))};
  }
  __device__ static void lnan(L& l, B a, B b, B c, B d) {
    l.s = (int32_t)max((uint32_t)l.s, (uint32_t)any_nan4(a, b, c, d, -1, 0));
  }
  __device__ static L lcomb(L a, L b) { return {b.m < a.m ? b.m : a.m, (int32_t)max((uint32_t)a.s, (uint32_t)b.s)}; }
  __device__ static A lout(L l) {
    if ((uint32_t)l.s == 0xFFFFFFFFu) return INT64_MIN;
    const uint64_t bits = l.m == 0.0 ? ((uint32_t)l.s >= 0x80000000u ? 0x8000000000000000ull : 0ull) : d2u(l.m);
    return (int64_t)(bits ^ ((uint64_t)((int64_t)bits >> 63) & 0x7FFFFFFFFFFFFFFFull));
  }
};
template <>
struct Red<IPM_LAND, IPM_F64> {
  using B = uint64_t; using A = uint64_t;
  __device__ static A id() { return ~0ull; }
  __device__ static A lift(B b) { return b & 0x7FFFFFFFFFFFFFFFull; }
  __device__ static A op(A a, A b) { return a < b ? a : b; }
  __device__ static A warp(A a) { return butterfly(a, [](A x, A y) { return op(x, y); }); }
  __device__ static B fin(A a) { return a != 0ull ? 0x3FF0000000000000ull : 0ull; }
  // lane-local: unsigned min of (low | magnitude high) words, 32 bits (0 iff some element is ±0)
  using L = uint32_t;
  __device__ static L lid() { return ~0u; }
  __device__ static L lstep(L l, B b) { return min(l, (uint32_t)b | ((uint32_t)(b >> 32) & 0x7FFFFFFFu)); }
  __device__ static L lcomb(L a, L b) { return min(a, b); }
  __device__ static A lout(L l) { return l; }
};
template <>
struct Red<IPM_LOR, IPM_F64> {
  using B = uint64_t; using A = uint64_t;
  __device__ static A id() { return 0ull; }
  __device__ static A lift(B b) { return b; }
  __device__ static A op(A a, A b) { return a | b; }
  __device__ static A warp(A a) { return butterfly(a, [](A x, A y) { return op(x, y); }); }
  __device__ static B fin(A a) { return (a & 0x7FFFFFFFFFFFFFFFull) != 0ull ? 0x3FF0000000000000ull : 0ull; }
};

// Lane-local accumulation (the hot loops): a Red may define a cheaper per-thread accumulator L (lid, lstep,
// lcomb, lout -> A, and optionally lnan for a whole 32-byte vector of float64); otherwise L = A with
// step = op(l, lift(b)). Only the kernels' register loops use L; warp / CTA / slot combines stay on A.
template <class R, class = void>
struct Loc {
  using L = typename R::A;
  __device__ __forceinline__ static L id() { return R::id(); }
  __device__ __forceinline__ static L step(L l, typename R::B b) { return R::op(l, R::lift(b)); }
  __device__ __forceinline__ static L comb(L a, L b) { return R::op(a, b); }
  __device__ __forceinline__ static typename R::A out(L l) { return l; }
  template <class V>
  __device__ __forceinline__ static void vec(L* acc, const V& v) {
#pragma unroll
    for (int k = 0; k < (int)(sizeof(V) / sizeof(typename R::B)); ++k) acc[k] = step(acc[k], v.w[k]);
  }
};
template <class T>
struct VoidT {
  using type = void;
};
template <class R>
struct Loc<R, typename VoidT<typename R::L>::type> {
  using L = typename R::L;
  using B = typename R::B;
  __device__ __forceinline__ static L id() { return R::lid(); }
  __device__ __forceinline__ static L step(L l, B b) {  // one scalar element (head / tail / masked paths)
    l = R::lstep(l, b);
    nan4(l, b, b, b, b, 0);
    return l;
  }
  __device__ __forceinline__ static L comb(L a, L b) { return R::lcomb(a, b); }
  __device__ __forceinline__ static typename R::A out(L l) { return R::lout(l); }
  template <class V>
  __device__ __forceinline__ static void vec(L* acc, const V& v) {  // one 32-byte vector: per element, then one NaN check
    constexpr int W = (int)(sizeof(V) / sizeof(B));
#pragma unroll
    for (int k = 0; k < W; ++k) acc[k] = R::lstep(acc[k], v.w[k]);
    if (W == 4) nan4(acc[0], v.w[0], v.w[1 % W], v.w[2 % W], v.w[3 % W], 0);
  }
  // the NaN check, for Reds that define lnan (float64 max / min; SFINAE on it)
  template <class RR = R>
  __device__ __forceinline__ static auto nan4(L& l, B a, B b, B c, B d, int) -> decltype(RR::lnan(l, a, b, c, d), void()) {
    R::lnan(l, a, b, c, d);
  }
  __device__ __forceinline__ static void nan4(L&, B, B, B, B, long) {}
};

// pack/unpack an accumulator into the 8-byte partial slots of the workspace
template <class A>
__device__ __forceinline__ uint64_t pack(A a) {
  static_assert(sizeof(A) <= 8, "accumulator must fit a slot");
  uint64_t u = 0;
  memcpy(&u, &a, sizeof(A));
  return u;
}
template <class A>
__device__ __forceinline__ A unpack(uint64_t u) {
  A a;
  memcpy(&a, &u, sizeof(A));
  return a;
}

}  // namespace ipm
