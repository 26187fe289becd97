/* ipmgen.h — seeded synthetic input generator (counter-based), shared by the oracle side and the CUDA side.
 *
 * This module holds NONE of the reduction arithmetic: it only defines what the i-th input element is.
 * It exists so that (a) multi-GiB inputs are generated on the device and never cross PCIe, and (b) the CPU
 * oracle can stream the same elements in chunks without materialising 64 GiB (SURVEY.md §8(c) "Input
 * generator"; the recipe and the workload each kind models are listed in DESIGN.md §"Input recipe").
 *
 * The generator is specified once here and implemented twice (gen_host.c for the CPU, gen_device.cu for the
 * GPU). tests/test_gen.py checks the host implementation against its own definition; tests/test_gpu_gen.py
 * checks device == host on sampled indices.
 *
 *   h(seed, i)  = splitmix64 output i of the stream whose state starts at seed*G (G = 0x9E3779B97F4A7C15):
 *                 mix(seed*G + (i+1)*G), mix(z) = the splitmix64 finaliser.  All arithmetic mod 2^64.
 *
 * Element i of a buffer of logical length n is base(kind, dtype, h(seed, i), i) unless i is one of the
 * nplant planted positions p_k = h(seed ^ TAG_POS, k) mod n (k = 0..nplant-1, applied in k order, a later
 * plant overwrites an earlier one), in which case it is plant(plant_kind, dtype, h(seed ^ TAG_VAL, k)).
 * All floating-point values are exact dyadic rationals, so host and device produce identical bits.
 */
#ifndef IPMGEN_H
#define IPMGEN_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* element types (same numbering as ipm_dtype, but this header is independent of ipm.h on purpose) */
enum { IPMGEN_I32 = 0, IPMGEN_I64 = 1, IPMGEN_F32 = 2, IPMGEN_F64 = 3 };

enum {
  IPMGEN_RANDOM = 0,  /* i32: (int32)(h>>32); i64: (int64)h; f32: (h>>40)*2^-14 in [0,1024); f64: (h>>11)*2^-43 */
  IPMGEN_SIGNED = 1,  /* ints: as RANDOM; f32: ((h>>40) - 2^23)*2^-13 in [-1024,1024); f64: ((h>>11)-2^52)*2^-42.
                         Never -0.0 (an integer 0 converts to +0.0). */
  IPMGEN_ODD = 2,     /* ints: RANDOM | 1 (units mod 2^w: products never collapse to 0); floats: as RANDOM */
  IPMGEN_IOTA = 3,    /* (T)(i + param) ; ints wrap mod 2^w */
  IPMGEN_MOD = 4,     /* (T)(i mod (int64)param) */
  IPMGEN_CONST = 5,   /* (T)param (ints: (int64)param then truncation) */
  IPMGEN_SIGNS = 6,   /* floats: (h>>63) ? -1.0 : +1.0 ; ints: as ODD */
  IPMGEN_ALLBITS = 7, /* every bit set: ints ~0 ; floats: not defined (returns RANDOM) */
  IPMGEN_NONZERO = 8  /* ints: RANDOM | 1 ; f32: ((h>>40)|1)*2^-14 ; f64: ((h>>11)|1)*2^-43 — never zero */
};

enum {
  IPMGEN_PLANT_NONE = 0,
  IPMGEN_PLANT_VALUE = 1,    /* (T)plant_param at each planted position */
  IPMGEN_PLANT_FACTOR = 2,   /* floats: (2^23 + (v>>41)) * 2^-23 * ((v & 1) ? 0.5 : 1.0) in [0.5, 2) */
  IPMGEN_PLANT_CLEARBIT = 3, /* ints: ~(1 << (v mod w)) */
  IPMGEN_PLANT_SETBIT = 4,   /* ints: (1 << (v mod w)) */
  IPMGEN_PLANT_RANDOM = 5    /* the RANDOM base value of a different stream: base(RANDOM, v) */
};

typedef struct {
  int32_t kind;       /* IPMGEN_* base kind */
  int32_t dtype;      /* IPMGEN_I32 .. IPMGEN_F64 */
  uint64_t seed;
  int64_t n;          /* logical length (plant positions are taken mod n) */
  double param;       /* base-kind parameter (IOTA offset, MOD modulus, CONST value) */
  int32_t plant_kind; /* IPMGEN_PLANT_* */
  int32_t nplant;     /* number of planted positions (0 = none) */
  double plant_param; /* PLANT_VALUE value */
} ipmgen_spec;

#define IPMGEN_GOLDEN 0x9E3779B97F4A7C15ULL
#define IPMGEN_TAG_POS 0x5DEECE66DA3B1F27ULL
#define IPMGEN_TAG_VAL 0xC2B2AE3D27D4EB4FULL

/* host implementation (gen_host.c): element bits of elements [lo, lo+count) into out (element-size each) */
int ipmgen_fill_host(const ipmgen_spec* spec, int64_t lo, int64_t count, void* out);
/* the raw counter-based draw, exported for the generator's own tests */
uint64_t ipmgen_h(uint64_t seed, uint64_t i);
/* planted position k (host), for tests that need to know where the plants are */
int64_t ipmgen_plant_pos(const ipmgen_spec* spec, int32_t k);

/* device implementation (gen_device.cu): same elements, written to device memory on `stream`
 * (a cudaStream_t passed as void*). Returns 0 on success, a CUDA error code otherwise. */
int ipmgen_fill_device(const ipmgen_spec* spec, int64_t lo, int64_t count, void* dev_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
