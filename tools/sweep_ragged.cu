// sweep_ragged.cu — tuning experiment (not product): times k_ragged_vec variants (warps per CTA, CTAs per SM,
// vectors per lane) + k_ragged_fix on a CSR offsets file, with CUDA events.
// usage: sweep_ragged OFFSETS.bin   (int64 row offsets, rows+1 of them; written by tools/sweep_ragged.py)
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <functional>
#include <vector>
#include "ipm_kernels.cuh"

using namespace ipm;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

static float time_ms(std::function<void()> f, int reps) {
  for (int i = 0; i < 3; ++i) f();
  CK(cudaDeviceSynchronize());
  std::vector<float> v;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); v.push_back(ms);
  }
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

struct Data { void* a; int64_t* off; int64_t rows, nnz; void* out; void* ws; void* ref; int sms; };

template <class R, int WARPS, int MINB, int VPL, bool FF = true, int PFV = 0>
void run(const char* name, const Data& d) {
  using B = typename R::B;
  CK(cudaFuncSetAttribute(k_ragged_vec<R, WARPS, MINB, VPL, FF, PFV>, cudaFuncAttributePreferredSharedMemoryCarveout,
                          (int)cudaSharedmemCarveoutMaxShared));
  int maxb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, k_ragged_vec<R, WARPS, MINB, VPL, FF, PFV>, WARPS * 32, 0));
  const int blocks = d.sms * MINB;
  const int64_t nw = (int64_t)blocks * WARPS;
  RaggedParams p{};
  p.a = d.a; p.off = d.off; p.rows = d.rows; p.init = 0; p.has_init = 0; p.out = d.out;
  int64_t* base = (int64_t*)d.ws;
  p.head_row = base; p.head_part = (uint64_t*)(base + 8192); p.tail_row = base + 2 * 8192;
  p.tail_part = (uint64_t*)(base + 3 * 8192);
  auto f = [&] {
    k_ragged_vec<R, WARPS, MINB, VPL, FF, PFV><<<blocks, WARPS * 32>>>(p);
    k_ragged_fix<R><<<(unsigned)((nw + 7) / 8), 256>>>(p, nw);
  };
  float ms = time_ms(f, 20);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  // same bits as the first variant (all use the same fold order only within a lane chunk: compare loosely)
  std::vector<B> got(d.rows), ref(d.rows);
  CK(cudaMemcpy(got.data(), d.out, d.rows * sizeof(B), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ref.data(), d.ref, d.rows * sizeof(B), cudaMemcpyDeviceToHost));
  int64_t bad = 0;
  for (int64_t i = 0; i < d.rows; ++i) {
    const double g = (double)got[i], r = (double)ref[i];
    if (!(g == r || (g - r) * (g - r) <= 1e-20 * r * r + 1e-30)) ++bad;
  }
  const double bytes = d.nnz * sizeof(B) + (d.rows + 1) * 8.0 + d.rows * sizeof(B);
  printf("%-4s W=%d MINB=%d VPL=%d FF=%d PFV=%d occ=%d  %7.3f ms  %7.1f GB/s  mismatches=%lld\n", name, WARPS, MINB, VPL, (int)FF, PFV, maxb, ms,
         bytes / ms / 1e6, (long long)bad);
}

template <class R, int BLOCK, int VPT, int MINB, int PFD>
void run_tile(const char* name, const Data& d) {
  using B = typename R::B;
  auto kern = k_ragged_tile<R, BLOCK, VPT, MINB, PFD>;
  constexpr int smem = RaggedTile<R, BLOCK, VPT>::SMEM;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared));
  int maxb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, kern, BLOCK, smem));
  const int blocks = d.sms * std::min(MINB, maxb);
  RaggedParams p{};
  p.a = d.a; p.off = d.off; p.rows = d.rows; p.init = 0; p.has_init = 0; p.out = d.out;
  int64_t* base = (int64_t*)d.ws;
  p.head_row = base; p.head_part = (uint64_t*)(base + 8192); p.tail_row = base + 2 * 8192;
  p.tail_part = (uint64_t*)(base + 3 * 8192);
  auto f = [&] {
    kern<<<blocks, BLOCK, smem>>>(p);
    k_ragged_fix<R><<<(unsigned)((blocks + 7) / 8), 256>>>(p, blocks);
  };
  float ms = time_ms(f, 20);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<B> got(d.rows), ref(d.rows);
  CK(cudaMemcpy(got.data(), d.out, d.rows * sizeof(B), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ref.data(), d.ref, d.rows * sizeof(B), cudaMemcpyDeviceToHost));
  int64_t bad = 0;
  for (int64_t i = 0; i < d.rows; ++i) {
    const double g = (double)got[i], r = (double)ref[i];
    if (!(g == r || (g - r) * (g - r) <= 1e-20 * r * r + 1e-30)) ++bad;
  }
  const double bytes = d.nnz * sizeof(B) + (d.rows + 1) * 8.0 + d.rows * sizeof(B);
  printf("%-4s tile BLOCK=%d VPT=%d MINB=%d PFD=%d occ=%d  %7.3f ms  %7.1f GB/s  mismatches=%lld\n", name, BLOCK, VPT, MINB,
         PFD, maxb, ms, bytes / ms / 1e6, (long long)bad);
}

template <class R>
void all(const char* name, Data d) {
  using B = typename R::B;
  CK(cudaMalloc(&d.a, d.nnz * sizeof(B)));
  CK(cudaMemset(d.a, 0x3e, d.nnz * sizeof(B)));
  CK(cudaMalloc(&d.out, d.rows * sizeof(B)));
  CK(cudaMalloc(&d.ref, d.rows * sizeof(B)));
  {  // reference: the product configuration
    run<R, 4, 8, 2, false>(name, Data{d.a, d.off, d.rows, d.nnz, d.ref, d.ws, d.ref, d.sms});
  }
  constexpr int PFV = sizeof(typename R::A) > sizeof(typename R::B) ? -1 : 1;  // the product's warp kernel
  run<R, 4, 8, 2, true, PFV>(name, d);
  run_tile<R, 128, 4, 4, 2>(name, d);
  run_tile<R, 128, 4, 4, 3>(name, d);
  run_tile<R, 128, 2, 6, 2>(name, d);
  run_tile<R, 128, 2, 8, 2>(name, d);
  run_tile<R, 256, 2, 3, 2>(name, d);
  run_tile<R, 256, 2, 4, 2>(name, d);
  run_tile<R, 64, 4, 8, 2>(name, d);
  run_tile<R, 64, 2, 12, 2>(name, d);
  run<R, 4, 8, 2, true, PFV>(name, d);
  CK(cudaFree(d.a)); CK(cudaFree(d.out)); CK(cudaFree(d.ref));
}

int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  fseek(f, 0, SEEK_END);
  const int64_t cnt = ftell(f) / 8;
  fseek(f, 0, SEEK_SET);
  std::vector<int64_t> off(cnt);
  if (fread(off.data(), 8, cnt, f) != (size_t)cnt) return 1;
  fclose(f);
  Data d{};
  d.rows = cnt - 1;
  d.nnz = off.back() - off[0];
  CK(cudaMalloc(&d.off, cnt * 8));
  CK(cudaMemcpy(d.off, off.data(), cnt * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&d.ws, 4 * 8192 * 8));
  cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, 0);
  printf("%s: rows=%lld nnz=%lld\n", argv[1], (long long)d.rows, (long long)d.nnz);
  all<Red<IPM_ADD, IPM_F32>>("f32+", d);
  all<Red<IPM_ADD, IPM_F64>>("f64+", d);
  all<Red<IPM_BXOR, IPM_I32>>("i32^", d);
  return 0;
}
