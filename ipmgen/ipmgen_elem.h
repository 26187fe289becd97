/* ipmgen_elem.h — the per-element definition of the generator (see ipmgen.h), compiled for the host by
 * gen_host.c and for the device by gen_device.cu. Input definition only: no reduction arithmetic. */
#ifndef IPMGEN_ELEM_H
#define IPMGEN_ELEM_H
#include "ipmgen.h"

#ifdef __CUDACC__
#define IPMGEN_FN __host__ __device__ static inline
#else
#define IPMGEN_FN static inline
#endif

IPMGEN_FN uint64_t ipmgen_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

IPMGEN_FN uint64_t ipmgen_draw(uint64_t seed, uint64_t i) {
  return ipmgen_mix(seed * IPMGEN_GOLDEN + (i + 1) * IPMGEN_GOLDEN);
}

/* exact power-of-two scaling without libm (so host and device agree bit for bit) */
IPMGEN_FN float ipmgen_f32_scaled(int64_t k, int e) {
  /* k in (-2^24, 2^24): exactly representable; multiply by 2^e (e in [-30,0]) is exact */
  float f = (float)k;
  union { uint32_t u; float f; } s;
  s.u = (uint32_t)(127 + e) << 23;
  return f * s.f;
}
IPMGEN_FN double ipmgen_f64_scaled(int64_t k, int e) {
  double d = (double)k; /* |k| < 2^53: exact */
  union { uint64_t u; double d; } s;
  s.u = (uint64_t)(1023 + e) << 52;
  return d * s.d;
}

/* base value bits of element i (64-bit container; caller truncates to the element size) */
IPMGEN_FN uint64_t ipmgen_base_bits(const ipmgen_spec* sp, int64_t i) {
  const uint64_t h = ipmgen_draw(sp->seed, (uint64_t)i);
  const int dt = sp->dtype;
  int kind = sp->kind;
  union { float f; uint32_t u; } cf;
  union { double d; uint64_t u; } cd;
  if (kind == IPMGEN_ALLBITS && (dt == IPMGEN_I32 || dt == IPMGEN_I64)) return ~0ULL;
  if (kind == IPMGEN_ALLBITS) kind = IPMGEN_RANDOM;
  if (kind == IPMGEN_SIGNS && (dt == IPMGEN_I32 || dt == IPMGEN_I64)) kind = IPMGEN_ODD;
  if (kind == IPMGEN_ODD && (dt == IPMGEN_F32 || dt == IPMGEN_F64)) kind = IPMGEN_RANDOM;
  switch (kind) {
    case IPMGEN_IOTA:
    case IPMGEN_MOD:
    case IPMGEN_CONST: {
      int64_t v;
      if (kind == IPMGEN_IOTA) v = i + (int64_t)sp->param;
      else if (kind == IPMGEN_MOD) v = i % (int64_t)sp->param;
      else v = (int64_t)sp->param;
      if (dt == IPMGEN_I32 || dt == IPMGEN_I64) return (uint64_t)v;
      if (kind == IPMGEN_CONST) { /* floats: the parameter itself, rounded once to T */
        if (dt == IPMGEN_F32) { cf.f = (float)sp->param; return cf.u; }
        cd.d = sp->param; return cd.u;
      }
      if (dt == IPMGEN_F32) { cf.f = (float)v; return cf.u; }
      cd.d = (double)v; return cd.u;
    }
    case IPMGEN_SIGNS:
      if (dt == IPMGEN_F32) { cf.f = (h >> 63) ? -1.0f : 1.0f; return cf.u; }
      cd.d = (h >> 63) ? -1.0 : 1.0; return cd.u;
    case IPMGEN_SIGNED:
      if (dt == IPMGEN_F32) { cf.f = ipmgen_f32_scaled((int64_t)(h >> 40) - (1LL << 23), -13); return cf.u; }
      if (dt == IPMGEN_F64) { cd.d = ipmgen_f64_scaled((int64_t)(h >> 11) - (1LL << 52), -42); return cd.u; }
      break; /* ints: RANDOM */
    case IPMGEN_ODD:
      if (dt == IPMGEN_I32) return (h >> 32) | 1ULL;
      return h | 1ULL;
    case IPMGEN_NONZERO:
      if (dt == IPMGEN_I32) return (h >> 32) | 1ULL;
      if (dt == IPMGEN_I64) return h | 1ULL;
      if (dt == IPMGEN_F32) { cf.f = ipmgen_f32_scaled((int64_t)((h >> 40) | 1ULL), -14); return cf.u; }
      cd.d = ipmgen_f64_scaled((int64_t)((h >> 11) | 1ULL), -43); return cd.u;
    default: break;
  }
  /* RANDOM */
  if (dt == IPMGEN_I32) return h >> 32;
  if (dt == IPMGEN_I64) return h;
  if (dt == IPMGEN_F32) { cf.f = ipmgen_f32_scaled((int64_t)(h >> 40), -14); return cf.u; }
  cd.d = ipmgen_f64_scaled((int64_t)(h >> 11), -43); return cd.u;
}

IPMGEN_FN int64_t ipmgen_plant_position(const ipmgen_spec* sp, int32_t k) {
  return (int64_t)(ipmgen_draw(sp->seed ^ IPMGEN_TAG_POS, (uint64_t)k) % (uint64_t)sp->n);
}

IPMGEN_FN uint64_t ipmgen_plant_bits(const ipmgen_spec* sp, int32_t k) {
  const uint64_t v = ipmgen_draw(sp->seed ^ IPMGEN_TAG_VAL, (uint64_t)k);
  const int dt = sp->dtype;
  const int w = (dt == IPMGEN_I32 || dt == IPMGEN_F32) ? 32 : 64;
  union { float f; uint32_t u; } cf;
  union { double d; uint64_t u; } cd;
  switch (sp->plant_kind) {
    case IPMGEN_PLANT_VALUE:
      if (dt == IPMGEN_I32 || dt == IPMGEN_I64) return (uint64_t)(int64_t)sp->plant_param;
      if (dt == IPMGEN_F32) { cf.f = (float)sp->plant_param; return cf.u; }
      cd.d = sp->plant_param; return cd.u;
    case IPMGEN_PLANT_FACTOR: {
      const int64_t m = (1LL << 23) + (int64_t)(v >> 41);
      const int e = (v & 1ULL) ? -24 : -23;
      if (dt == IPMGEN_F32) { cf.f = ipmgen_f32_scaled(m, e); return cf.u; }
      if (dt == IPMGEN_F64) { cd.d = ipmgen_f64_scaled(m, e); return cd.u; }
      return (uint64_t)(m | 1); /* ints: an odd factor */
    }
    case IPMGEN_PLANT_CLEARBIT: return ~(1ULL << (v % (uint64_t)w));
    case IPMGEN_PLANT_SETBIT: return 1ULL << (v % (uint64_t)w);
    case IPMGEN_PLANT_RANDOM: {
      ipmgen_spec s2 = *sp;
      s2.kind = IPMGEN_RANDOM;
      s2.seed = sp->seed ^ IPMGEN_TAG_VAL;
      return ipmgen_base_bits(&s2, (int64_t)k);
    }
    default: return 0;
  }
}

IPMGEN_FN int ipmgen_elem_size(int dt) { return (dt == IPMGEN_I32 || dt == IPMGEN_F32) ? 4 : 8; }

#endif
