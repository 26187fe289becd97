// gen_device.cu — device implementation of the generator defined in ipmgen.h (input definition only).
// Used by tests and bench.py to create multi-GiB inputs in HBM without a host round trip.
#include <cuda_runtime.h>
#include "ipmgen_elem.h"

template <typename U>
__global__ void ipmgen_fill_kernel(ipmgen_spec sp, int64_t lo, int64_t count, U* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride)
    out[j] = (U)ipmgen_base_bits(&sp, lo + j);
}

// plants are applied by one thread in k order so that a later plant overwrites an earlier one
template <typename U>
__global__ void ipmgen_plant_kernel(ipmgen_spec sp, int64_t lo, int64_t count, U* __restrict__ out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (int32_t k = 0; k < sp.nplant; ++k) {
    const int64_t p = ipmgen_plant_position(&sp, k);
    if (p >= lo && p < lo + count) out[p - lo] = (U)ipmgen_plant_bits(&sp, k);
  }
}

extern "C" int ipmgen_fill_device(const ipmgen_spec* sp, int64_t lo, int64_t count, void* dev_out, void* stream) {
  if (!sp || lo < 0 || count < 0 || (count > 0 && !dev_out)) return (int)cudaErrorInvalidValue;
  if (count == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = 256;
  int64_t blocks = (count + threads - 1) / threads;
  if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
  const bool four = (sp->dtype == IPMGEN_I32 || sp->dtype == IPMGEN_F32);
  if (four) ipmgen_fill_kernel<uint32_t><<<(unsigned)blocks, threads, 0, st>>>(*sp, lo, count, (uint32_t*)dev_out);
  else ipmgen_fill_kernel<uint64_t><<<(unsigned)blocks, threads, 0, st>>>(*sp, lo, count, (uint64_t*)dev_out);
  if (sp->plant_kind != IPMGEN_PLANT_NONE && sp->nplant > 0 && sp->n > 0) {
    if (four) ipmgen_plant_kernel<uint32_t><<<1, 1, 0, st>>>(*sp, lo, count, (uint32_t*)dev_out);
    else ipmgen_plant_kernel<uint64_t><<<1, 1, 0, st>>>(*sp, lo, count, (uint64_t*)dev_out);
  }
  return (int)cudaGetLastError();
}
