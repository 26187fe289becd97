/* gen_host.c — host implementation of the generator defined in ipmgen.h (input definition only). */
#include <string.h>
#include "ipmgen_elem.h"

uint64_t ipmgen_h(uint64_t seed, uint64_t i) { return ipmgen_draw(seed, i); }

int64_t ipmgen_plant_pos(const ipmgen_spec* sp, int32_t k) {
  if (sp->n <= 0) return -1;
  return ipmgen_plant_position(sp, k);
}

int ipmgen_fill_host(const ipmgen_spec* sp, int64_t lo, int64_t count, void* out) {
  if (!sp || (count > 0 && !out) || lo < 0 || count < 0) return 1;
  if (sp->dtype < IPMGEN_I32 || sp->dtype > IPMGEN_F64) return 2;
  const int es = ipmgen_elem_size(sp->dtype);
  if (es == 4) {
    uint32_t* o = (uint32_t*)out;
    for (int64_t j = 0; j < count; ++j) o[j] = (uint32_t)ipmgen_base_bits(sp, lo + j);
  } else {
    uint64_t* o = (uint64_t*)out;
    for (int64_t j = 0; j < count; ++j) o[j] = ipmgen_base_bits(sp, lo + j);
  }
  if (sp->plant_kind != IPMGEN_PLANT_NONE && sp->n > 0) {
    for (int32_t k = 0; k < sp->nplant; ++k) { /* k order: later plants overwrite earlier ones */
      const int64_t p = ipmgen_plant_position(sp, k);
      if (p < lo || p >= lo + count) continue;
      const uint64_t b = ipmgen_plant_bits(sp, k);
      if (es == 4) ((uint32_t*)out)[p - lo] = (uint32_t)b;
      else ((uint64_t*)out)[p - lo] = b;
    }
  }
  return 0;
}
