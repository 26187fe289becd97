// sweep_flat.cu — tuning experiment (not product): times the product's k_flat / k_seg_warp templates over
// block size, loads in flight (U), cache hint and CTAs per SM, on large inputs, with CUDA events.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1412_1127_b200/csrc
//        -o build/sweep_flat tools/sweep_flat.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <functional>
#include <string>
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

template <class R, int BLOCK, int U, int HINT, int SCHED = 0>
void run_flat(const char* name, void* buf, size_t bytes, void* ws, int sms, int only_cps = 0) {
  int maxb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, k_flat<R, BLOCK, U, HINT, SCHED>, BLOCK, 0));
  const int64_t n = bytes / sizeof(typename R::B);
  for (int cps = 1; cps <= maxb; cps *= 2) {
    if (only_cps && cps != only_cps) continue;
    FlatParams p{};
    p.a = buf; p.n = n; p.row_stride = 0; p.init = 0; p.has_init = 0; p.mode = MODE_PARTIAL;
    p.out = (char*)ws + 4160; p.partials = (uint64_t*)((char*)ws + 8192); p.tickets = (unsigned*)ws;
    p.counter = (unsigned long long*)((char*)ws + 4096 + 512);
    const int grid = sms * cps;
    float ms = time_ms([&] { k_flat<R, BLOCK, U, HINT, SCHED><<<grid, BLOCK>>>(p); }, 10);
    CK(cudaGetLastError());
    printf("flat %-10s B=%4d U=%d H=%d S=%d cps=%d grid=%5d  %7.3f ms  %7.1f GB/s\n", name, BLOCK, U, HINT, SCHED, cps,
           grid, ms, bytes / ms / 1e6);
  }
}

template <class R, int WARPS, int U, int HINT, int PF = 0>
void run_seg(const char* name, void* buf, void* out, int sms) {
  int maxb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, k_seg_warp<R, WARPS, U, HINT, PF>, WARPS * 32, 0));
  const int64_t rows = 65536, cols = 4096;
  for (int cps = 1; cps <= maxb; cps *= 2) {
    SegParams p{buf, rows, cols, cols, 0, 0, out};
    const int grid = std::min<int64_t>(sms * cps, (rows + WARPS - 1) / WARPS);
    float ms = time_ms([&] { k_seg_warp<R, WARPS, U, HINT, PF><<<grid, WARPS * 32>>>(p); }, 10);
    CK(cudaGetLastError());
    printf("seg  %-10s W=%2d U=%d H=%d PF=%d cps=%d grid=%5d  %7.3f ms  %7.1f GB/s\n", name, WARPS, U, HINT, PF, cps, grid, ms,
           (rows * cols * 4.0 + rows * 4) / ms / 1e6);
  }
}

template <class R, int WARPS, int S, int CH>
void run_seg_tma(const char* name, void* buf, void* out, int sms, int64_t rows, int64_t cols) {
  constexpr int smem = SegTma<R, WARPS, S, CH>::SMEM;
  CK(cudaFuncSetAttribute(k_seg_tma<R, WARPS, S, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int maxb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, k_seg_tma<R, WARPS, S, CH>, WARPS * 32, smem));
  for (int cps = 1; cps <= maxb; cps *= 2) {
    SegParams p{buf, rows, cols, cols, 0, 0, out};
    const int grid = std::min<int64_t>(sms * cps, (rows + WARPS - 1) / WARPS);
    float ms = time_ms([&] { k_seg_tma<R, WARPS, S, CH><<<grid, WARPS * 32, smem>>>(p); }, 10);
    CK(cudaGetLastError());
    printf("tma  %-10s W=%2d S=%d CH=%5d cps=%d grid=%5d rows=%ld cols=%ld %7.3f ms  %7.1f GB/s\n", name, WARPS, S, CH, cps,
           grid, (long)rows, (long)cols, ms, (rows * cols * 4.0 + rows * 4) / ms / 1e6);
  }
}

template <class R, int U = 4, bool PIPE = false, int BLK = 256>
void run_guided(const char* name, void* buf, size_t bytes, void* ws, int sms, int64_t maxch = 0) {
  const int64_t n = bytes / sizeof(typename R::B);
  FlatParams p{};
  p.a = buf; p.n = n; p.row_stride = 0; p.init = 0; p.has_init = 0; p.mode = MODE_PARTIAL;
  p.out = (char*)ws + 4160; p.partials = (uint64_t*)((char*)ws + 8192); p.tickets = (unsigned*)ws;
  p.counter = (unsigned long long*)((char*)ws + 4096 + 512);
  const int grid = sms * (1024 / BLK);
  p.max_chunks = maxch ? maxch : 16384 - grid - 1;
  float ms = time_ms([&] { k_flat_guided<R, BLK, U, PIPE><<<grid, BLK>>>(p); }, 20);
  CK(cudaGetLastError());
  printf("guided %-8s B=%4d U=%d P=%d grid=%5d maxch=%6ld  %7.3f ms  %7.1f GB/s\n", name, BLK, U, (int)PIPE, grid,
         (long)p.max_chunks, ms, bytes / ms / 1e6);
}

// experiment: the flat clause fed by TMA bulk copies (1 persistent CTA per SM, S-stage ring of CHB bytes,
// one producer thread, all 256 threads consume from shared memory); full tiles only (the sweep sizes are
// multiples of the tile)
template <class R, int S, int CHB, int NT = 256, int MINB = 1, int WAIT = 0>
__global__ void __launch_bounds__(NT, MINB) k_flat_tma(const void* a, int64_t nbytes, uint64_t* out) {
  using B = typename R::B;
  using A = typename R::A;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = (uint64_t*)(smem + (size_t)S * CHB);
  __shared__ A sm[NT / 32];
  const int64_t ntiles = nbytes / CHB;
  if (threadIdx.x == 0)
    for (int i = 0; i < S; ++i) mbar_init(bar + i, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int64_t my = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;  // tiles b, b+G, ...
  auto issue = [&](int64_t i) {
    const int st = (int)(i % S);
    const int64_t t = blockIdx.x + i * gridDim.x;
    mbar_expect_tx(bar + st, CHB);
    bulk_g2s(smem + (size_t)st * CHB, (const char*)a + t * CHB, CHB, bar + st);
  };
  if (threadIdx.x == 0)
    for (int64_t i = 0; i < S && i < my; ++i) issue(i);
  constexpr int EPV = 16 / sizeof(B);
  A acc[EPV];
#pragma unroll
  for (int k = 0; k < EPV; ++k) acc[k] = R::id();
  for (int64_t i = 0; i < my; ++i) {
    const int st = (int)(i % S);
    if (WAIT == 0) {
      mbar_wait(bar + st, (uint32_t)((i / S) & 1));
    } else if (WAIT == 1) {
      if ((threadIdx.x & 31) == 0) mbar_wait(bar + st, (uint32_t)((i / S) & 1));
      __syncwarp();
    } else {
      if (threadIdx.x == 0) mbar_wait(bar + st, (uint32_t)((i / S) & 1));
      __syncthreads();
    }
    const unsigned char* c = smem + (size_t)st * CHB;
#pragma unroll 4
    for (int o = threadIdx.x * 16; o < CHB; o += NT * 16) {
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
    __syncthreads();
    if (threadIdx.x == 0 && i + S < my) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + S);
    }
  }
#pragma unroll
  for (int k = 1; k < EPV; ++k) acc[0] = R::op(acc[0], acc[k]);
  A t = block_reduce<R, NT>(acc[0], sm);
  if (threadIdx.x == 0) out[blockIdx.x] = pack(t);
}

template <class R, int S, int CHB, int NT = 256, int CPS = 1, int WAIT = 0>
void run_flat_tma(const char* name, void* buf, size_t bytes, void* ws, int sms) {
  constexpr int smem = S * CHB + S * 8;
  CK(cudaFuncSetAttribute(k_flat_tma<R, S, CHB, NT, CPS, WAIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  float ms = time_ms([&] { k_flat_tma<R, S, CHB, NT, CPS, WAIT><<<sms * CPS, NT, smem>>>(buf, (int64_t)bytes, (uint64_t*)((char*)ws + 8192)); }, 20);
  CK(cudaGetLastError());
  printf("tmaflat %-7s S=%2d CHB=%6d NT=%d cps=%d W=%d  %7.3f ms  %7.1f GB/s\n", name, S, CHB, NT, CPS, WAIT, ms, bytes / ms / 1e6);
}


template <class R, int U, int PF = 0>
void run_2d(const char* name, void* buf, void* ws, int sms, int64_t rows, int64_t cols, int64_t stride, int cps) {
  using B = typename R::B;
  Params2D q{};
  q.f.a = buf; q.f.mode = MODE_RESULT; q.f.out = (char*)ws + 4096; q.f.partials = (uint64_t*)((char*)ws + 8192);
  q.f.tickets = (unsigned*)ws; q.f.world = 1;
  q.rows = rows; q.cols = cols; q.row_stride = stride;
  const int grid = sms * cps;
  float ms = time_ms([&] { k_2d<R, 256, U, PF><<<grid, 256>>>(q); }, 20);
  CK(cudaGetLastError());
  B res;
  CK(cudaMemcpy(&res, q.f.out, sizeof(B), cudaMemcpyDeviceToHost));
  const double bytes = (double)rows * cols * sizeof(B);
  printf("2d %-6s %lldx%lld stride %lld U=%d PF=%d cps=%d  %7.3f ms  %7.1f GB/s  result=%.17g\n", name,
         (long long)rows, (long long)cols, (long long)stride, U, PF, cps, ms, bytes / ms / 1e6, (double)res);
}

int main(int argc, char** argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t big = (size_t)16 << 30;
  void* buf; void* ws; void* out;
  CK(cudaMalloc(&buf, big));
  CK(cudaMemset(buf, 1, big));
  CK(cudaMalloc(&ws, 1 << 20));
  CK(cudaMemset(ws, 0, 1 << 20));
  CK(cudaMalloc(&out, 1 << 20));
  const std::string mode = argc > 1 ? argv[1] : "all";
  for (size_t bytes : {(size_t)1 << 30, (size_t)4 << 30, (size_t)16 << 30}) {
    printf("== %zu GiB\n", bytes >> 30);
    if (mode == "all" || mode == "hint") {
      run_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 0>("f32+", buf, bytes, ws, sms);
      run_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 1>("f32+", buf, bytes, ws, sms);
      run_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 2>("f32+", buf, bytes, ws, sms);
      run_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 3>("f32+", buf, bytes, ws, sms);
      run_flat<Red<IPM_BXOR, IPM_I32>, 256, 4, 0>("i32^", buf, bytes, ws, sms);
      run_flat<Red<IPM_BXOR, IPM_I32>, 256, 4, 1>("i32^", buf, bytes, ws, sms);
      run_flat<Red<IPM_BXOR, IPM_I64>, 256, 4, 0>("i64^", buf, bytes, ws, sms);
      run_flat<Red<IPM_BXOR, IPM_I64>, 256, 4, 1>("i64^", buf, bytes, ws, sms);
    }
    if (mode == "all" || mode == "shape") {
      run_flat<Red<IPM_ADD, IPM_F32>, 256, 2, 0>("f32+", buf, bytes, ws, sms);
      run_flat<Red<IPM_ADD, IPM_F32>, 256, 8, 0>("f32+", buf, bytes, ws, sms);
      run_flat<Red<IPM_ADD, IPM_F32>, 512, 4, 0>("f32+", buf, bytes, ws, sms);
      run_flat<Red<IPM_ADD, IPM_F32>, 1024, 2, 0>("f32+", buf, bytes, ws, sms);
      run_flat<Red<IPM_ADD, IPM_F32>, 128, 8, 0>("f32+", buf, bytes, ws, sms);
      run_flat<Red<IPM_BXOR, IPM_I32>, 256, 8, 0>("i32^", buf, bytes, ws, sms);
      run_flat<Red<IPM_BXOR, IPM_I32>, 512, 4, 0>("i32^", buf, bytes, ws, sms);
      run_flat<Red<IPM_BXOR, IPM_I32>, 1024, 4, 0>("i32^", buf, bytes, ws, sms);
      run_flat<Red<IPM_ADD, IPM_F64>, 256, 4, 0>("f64+", buf, bytes, ws, sms);
      run_flat<Red<IPM_ADD, IPM_F64>, 256, 8, 0>("f64+", buf, bytes, ws, sms);
      run_flat<Red<IPM_MAX, IPM_F64>, 256, 4, 0>("f64max", buf, bytes, ws, sms);
    }
  }
  if (mode == "segdt") {  // old product grid (sms * 4) vs the balanced choice (ipm_api.cu seg_grid), per fold
    auto go = [&](auto red, const char* name, int64_t rows) {
      using R = decltype(red);
      using B = typename R::B;
      int occ = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_seg_warp<R, 8, 8, 0>, 256, 0));
      const int64_t cols = 4096;
      const int64_t gmax = (int64_t)sms * occ, glo = gmax * 3 / 4;
      int64_t best = gmax; double be = 0;
      for (int64_t g = glo; g <= gmax; ++g) {
        const int64_t nw = g * 8;
        const double e = (double)rows / (double)(((rows + nw - 1) / nw) * nw);
        if (e > be + 1e-9) { be = e; best = g; }
      }
      for (int rep = 0; rep < 2; ++rep)
        for (int64_t grid : {(int64_t)sms * 4, best}) {
          SegParams p{buf, rows, cols, cols, 0, 0, out};
          float ms = time_ms([&] { k_seg_warp<R, 8, 8, 0><<<(int)grid, 256>>>(p); }, 20);
          CK(cudaGetLastError());
          printf("segdt %-6s occ=%d rows=%lld grid=%5lld rows/warp=%.2f  %7.3f ms  %7.1f GB/s\n", name, occ,
                 (long long)rows, (long long)grid, rows / (grid * 8.0), ms, (rows * cols * (double)sizeof(B) + rows * sizeof(B)) / ms / 1e6);
        }
    };
    go(Red<IPM_ADD, IPM_F32>{}, "f32+", 65536);
    go(Red<IPM_MAX, IPM_F32>{}, "f32max", 65536);
    go(Red<IPM_ADD, IPM_F64>{}, "f64+", 65536);
    go(Red<IPM_MUL, IPM_F64>{}, "f64*", 65536);
    go(Red<IPM_BXOR, IPM_I32>{}, "i32^", 65536);
    go(Red<IPM_MIN, IPM_I64>{}, "i64min", 65536);
    go(Red<IPM_ADD, IPM_F32>{}, "f32+", 50000);
    go(Red<IPM_ADD, IPM_F32>{}, "f32+", 100003);
    return 0;
  }
  if (mode == "segtail") {  // C3: rows per warp exactly equal (grid 512 / 1024) vs the product's sms * 4
    for (int rep = 0; rep < 3; ++rep) {
      const int64_t rows = 65536, cols = 4096;
      for (int grid : {592, 512, 1024, 1184, 256 * 3}) {
        SegParams p{buf, rows, cols, cols, 0, 0, out};
        float ms = time_ms([&] { k_seg_warp<Red<IPM_ADD, IPM_F32>, 8, 8, 0><<<grid, 256>>>(p); }, 20);
        CK(cudaGetLastError());
        printf("segtail f32+ W=8 U=8 grid=%5d rows/warp=%.2f  %7.3f ms  %7.1f GB/s\n", grid, rows / (grid * 8.0), ms,
               (rows * cols * 4.0 + rows * 4) / ms / 1e6);
      }
    }
    return 0;
  }
  if (mode == "pf") {  // L2 bulk prefetch of the warp's next row / item (PF=1) against none
    for (int rep = 0; rep < 2; ++rep) {
      printf("== segmented 65536 x 4096 f32 / f64 (32768 x 4096)\n");
      run_seg<Red<IPM_ADD, IPM_F32>, 8, 8, 0, 0>("f32+", buf, out, sms);
      run_seg<Red<IPM_ADD, IPM_F32>, 8, 8, 0, 1>("f32+", buf, out, sms);
      run_seg<Red<IPM_ADD, IPM_F32>, 8, 4, 0, 1>("f32+", buf, out, sms);
      run_seg<Red<IPM_BXOR, IPM_I32>, 8, 8, 0, 0>("i32^", buf, out, sms);
      run_seg<Red<IPM_BXOR, IPM_I32>, 8, 8, 0, 1>("i32^", buf, out, sms);
      printf("== 2-D\n");
      for (int shape = 0; shape < 2; ++shape) {
        const int64_t rows = shape == 0 ? 16384 : 262144, cols = shape == 0 ? 16000 : 1000,
                      stride = shape == 0 ? 16384 : 1024;
        run_2d<Red<IPM_ADD, IPM_F32>, 4, 0>("f32+", buf, ws, sms, rows, cols, stride, 4);
        run_2d<Red<IPM_ADD, IPM_F32>, 4, 1>("f32+", buf, ws, sms, rows, cols, stride, 4);
        run_2d<Red<IPM_ADD, IPM_F64>, 4, 0>("f64+", buf, ws, sms, rows / 2, cols, stride, 4);
        run_2d<Red<IPM_ADD, IPM_F64>, 4, 1>("f64+", buf, ws, sms, rows / 2, cols, stride, 4);
        run_2d<Red<IPM_BXOR, IPM_I32>, 4, 0>("i32^", buf, ws, sms, rows, cols, stride, 4);
        run_2d<Red<IPM_BXOR, IPM_I32>, 4, 1>("i32^", buf, ws, sms, rows, cols, stride, 4);
      }
    }
    return 0;
  }
  if (mode == "2d") {
    for (int shape = 0; shape < 3; ++shape) {
      const int64_t rows = shape == 0 ? 16384 : shape == 1 ? 262144 : 4096, cols = shape == 0 ? 16000 : shape == 1 ? 1000 : 65000,
                    stride = shape == 0 ? 16384 : shape == 1 ? 1024 : 65536;
      for (int cps : {2, 4, 8}) {
        run_2d<Red<IPM_ADD, IPM_F32>, 4>("f32+", buf, ws, sms, rows, cols, stride, cps);
        run_2d<Red<IPM_ADD, IPM_F32>, 8>("f32+", buf, ws, sms, rows, cols, stride, cps);
        run_2d<Red<IPM_ADD, IPM_F64>, 4>("f64+", buf, ws, sms, rows / 2, cols, stride, cps);
        run_2d<Red<IPM_BXOR, IPM_I32>, 4>("i32^", buf, ws, sms, rows, cols, stride, cps);
      }
    }
    return 0;
  }
  if (mode == "all" || mode == "seg") {
    printf("== segmented 65536 x 4096 f32\n");
    run_seg<Red<IPM_ADD, IPM_F32>, 8, 4, 0>("f32+", buf, out, sms);
    run_seg<Red<IPM_ADD, IPM_F32>, 8, 2, 0>("f32+", buf, out, sms);
    run_seg<Red<IPM_ADD, IPM_F32>, 8, 8, 0>("f32+", buf, out, sms);
    run_seg<Red<IPM_ADD, IPM_F32>, 4, 4, 0>("f32+", buf, out, sms);
    run_seg<Red<IPM_ADD, IPM_F32>, 16, 4, 0>("f32+", buf, out, sms);
    run_seg<Red<IPM_ADD, IPM_F32>, 8, 4, 1>("f32+", buf, out, sms);
  }
  if (mode == "all" || mode == "seg" || mode == "tma") {
    printf("== TMA segmented\n");
    for (int64_t cols : {4096, 65536}) {
      const int64_t rows = (int64_t)65536 * 4096 / cols;
      run_seg_tma<Red<IPM_ADD, IPM_F32>, 8, 4, 4096>("f32+", buf, out, sms, rows, cols);
      run_seg_tma<Red<IPM_ADD, IPM_F32>, 8, 2, 8192>("f32+", buf, out, sms, rows, cols);
      run_seg_tma<Red<IPM_ADD, IPM_F32>, 4, 4, 8192>("f32+", buf, out, sms, rows, cols);
      run_seg_tma<Red<IPM_ADD, IPM_F32>, 8, 8, 2048>("f32+", buf, out, sms, rows, cols);
      run_seg_tma<Red<IPM_ADD, IPM_F32>, 4, 8, 4096>("f32+", buf, out, sms, rows, cols);
      run_seg_tma<Red<IPM_ADD, IPM_F32>, 2, 8, 8192>("f32+", buf, out, sms, rows, cols);
    }
  }
  if (mode == "sched") {
    for (size_t bytes : {(size_t)1 << 30, (size_t)4 << 30, (size_t)16 << 30}) {
      printf("== sched %zu GiB\n", bytes >> 30);
      run_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 0, 0>("f32+", buf, bytes, ws, sms, 4);
      run_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 0, 1>("f32+", buf, bytes, ws, sms, 4);
      run_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 0, 2>("f32+", buf, bytes, ws, sms, 4);
      run_flat<Red<IPM_ADD, IPM_F32>, 1024, 2, 0, 0>("f32+", buf, bytes, ws, sms, 1);
      run_flat<Red<IPM_ADD, IPM_F32>, 1024, 2, 0, 1>("f32+", buf, bytes, ws, sms, 1);
      run_flat<Red<IPM_ADD, IPM_F32>, 1024, 2, 0, 2>("f32+", buf, bytes, ws, sms, 1);
      run_flat<Red<IPM_ADD, IPM_F32>, 512, 4, 0, 0>("f32+", buf, bytes, ws, sms, 0);
      run_flat<Red<IPM_ADD, IPM_F32>, 512, 4, 0, 2>("f32+", buf, bytes, ws, sms, 0);
      run_flat<Red<IPM_BXOR, IPM_I32>, 256, 4, 0, 0>("i32^", buf, bytes, ws, sms, 4);
      run_flat<Red<IPM_BXOR, IPM_I32>, 256, 4, 0, 2>("i32^", buf, bytes, ws, sms, 4);
      run_flat<Red<IPM_BXOR, IPM_I32>, 1024, 2, 0, 0>("i32^", buf, bytes, ws, sms, 1);
      run_flat<Red<IPM_BXOR, IPM_I32>, 1024, 2, 0, 2>("i32^", buf, bytes, ws, sms, 1);
      run_flat<Red<IPM_BXOR, IPM_I32>, 1024, 4, 0, 0>("i32^", buf, bytes, ws, sms, 1);
      run_flat<Red<IPM_BXOR, IPM_I32>, 1024, 4, 0, 2>("i32^", buf, bytes, ws, sms, 1);
      run_flat<Red<IPM_ADD, IPM_F64>, 256, 4, 0, 0>("f64+", buf, bytes, ws, sms, 4);
      run_flat<Red<IPM_ADD, IPM_F64>, 256, 4, 0, 2>("f64+", buf, bytes, ws, sms, 4);
      run_flat<Red<IPM_ADD, IPM_F64>, 1024, 2, 0, 0>("f64+", buf, bytes, ws, sms, 1);
      run_flat<Red<IPM_ADD, IPM_F64>, 1024, 2, 0, 2>("f64+", buf, bytes, ws, sms, 1);
      run_flat<Red<IPM_MAX, IPM_F64>, 1024, 2, 0, 0>("f64max", buf, bytes, ws, sms, 1);
      run_flat<Red<IPM_MAX, IPM_F64>, 256, 4, 0, 0>("f64max", buf, bytes, ws, sms, 4);
      run_flat<Red<IPM_MUL, IPM_I64>, 1024, 2, 0, 0>("i64*", buf, bytes, ws, sms, 1);
      run_flat<Red<IPM_MUL, IPM_I64>, 1024, 2, 0, 2>("i64*", buf, bytes, ws, sms, 1);
    }
  }
  if (mode == "guided") {
    // spin the clocks up first
    for (int i = 0; i < 30; ++i) k_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 0, 0><<<sms * 4, 256>>>(FlatParams{buf, (int64_t)(big / 4), 0, 0, 0, MODE_PARTIAL, (char*)ws + 4160, (uint64_t*)((char*)ws + 8192), (unsigned*)ws, nullptr, 0});
    CK(cudaDeviceSynchronize());
    for (size_t bytes : {(size_t)1 << 30, (size_t)4 << 30, (size_t)16 << 30}) {
      printf("== guided %zu GiB\n", bytes >> 30);
      for (int rep = 0; rep < 2; ++rep) {
        run_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 0, 0>("f32+", buf, bytes, ws, sms, 4);
        run_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 0, 2>("f32+", buf, bytes, ws, sms, 4);
        run_guided<Red<IPM_ADD, IPM_F32>>("f32+", buf, bytes, ws, sms);
        run_flat<Red<IPM_ADD, IPM_F64>, 256, 4, 0, 0>("f64+", buf, bytes, ws, sms, 4);
        run_flat<Red<IPM_ADD, IPM_F64>, 256, 4, 0, 2>("f64+", buf, bytes, ws, sms, 4);
        run_guided<Red<IPM_ADD, IPM_F64>>("f64+", buf, bytes, ws, sms);
        run_flat<Red<IPM_BXOR, IPM_I32>, 256, 4, 0, 0>("i32^", buf, bytes, ws, sms, 4);
        run_flat<Red<IPM_BXOR, IPM_I32>, 256, 4, 0, 2>("i32^", buf, bytes, ws, sms, 4);
        run_guided<Red<IPM_BXOR, IPM_I32>>("i32^", buf, bytes, ws, sms);
        run_guided<Red<IPM_MAX, IPM_F32>>("f32max", buf, bytes, ws, sms);
        run_guided<Red<IPM_MUL, IPM_I64>>("i64*", buf, bytes, ws, sms);
        run_guided<Red<IPM_MAX, IPM_F64>>("f64max", buf, bytes, ws, sms);
      }
    }
  }
  if (mode == "gshape") {
    for (int i = 0; i < 30; ++i) k_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 0, 0><<<sms * 4, 256>>>(FlatParams{buf, (int64_t)(big / 4), 0, 0, 0, MODE_PARTIAL, (char*)ws + 4160, (uint64_t*)((char*)ws + 8192), (unsigned*)ws, nullptr, 0});
    CK(cudaDeviceSynchronize());
    for (size_t bytes : {(size_t)1 << 30, (size_t)16 << 30}) {
      printf("== gshape %zu GiB\n", bytes >> 30);
      for (int rep = 0; rep < 2; ++rep) {
        run_guided<Red<IPM_ADD, IPM_F32>, 2, true, 256>("f32+", buf, bytes, ws, sms);
        run_guided<Red<IPM_ADD, IPM_F32>, 2, true, 128>("f32+", buf, bytes, ws, sms);
        run_guided<Red<IPM_ADD, IPM_F32>, 2, true, 512>("f32+", buf, bytes, ws, sms);
        run_guided<Red<IPM_ADD, IPM_F32>, 1, true, 256>("f32+", buf, bytes, ws, sms);
        run_guided<Red<IPM_ADD, IPM_F32>, 1, true, 512>("f32+", buf, bytes, ws, sms);
        run_guided<Red<IPM_ADD, IPM_F32>, 3, true, 256>("f32+", buf, bytes, ws, sms);
        run_guided<Red<IPM_BXOR, IPM_I32>, 2, true, 256>("i32^", buf, bytes, ws, sms);
        run_guided<Red<IPM_BXOR, IPM_I32>, 2, true, 128>("i32^", buf, bytes, ws, sms);
        run_guided<Red<IPM_BXOR, IPM_I32>, 4, true, 128>("i32^", buf, bytes, ws, sms);
        run_guided<Red<IPM_BXOR, IPM_I32>, 1, true, 512>("i32^", buf, bytes, ws, sms);
      }
    }
  }
  if (mode == "chunks") {
    for (int i = 0; i < 30; ++i) k_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 0, 0><<<sms * 4, 256>>>(FlatParams{buf, (int64_t)(big / 4), 0, 0, 0, MODE_PARTIAL, (char*)ws + 4160, (uint64_t*)((char*)ws + 8192), (unsigned*)ws, nullptr, 0});
    CK(cudaDeviceSynchronize());
    for (size_t bytes : {(size_t)1 << 30, (size_t)4 << 30, (size_t)16 << 30}) {
      printf("== chunks %zu GiB\n", bytes >> 30);
      for (int rep = 0; rep < 2; ++rep) {
        run_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 0, 2>("f32+", buf, bytes, ws, sms, 4);
        for (int64_t mc : {0, 4096, 2048, 1024, 512, 256})
          run_guided<Red<IPM_ADD, IPM_F32>, 2, true>("f32+", buf, bytes, ws, sms, mc);
      }
    }
  }
  if (mode == "pipe") {
    for (int i = 0; i < 30; ++i) k_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 0, 0><<<sms * 4, 256>>>(FlatParams{buf, (int64_t)(big / 4), 0, 0, 0, MODE_PARTIAL, (char*)ws + 4160, (uint64_t*)((char*)ws + 8192), (unsigned*)ws, nullptr, 0});
    CK(cudaDeviceSynchronize());
    for (size_t bytes : {(size_t)1 << 30, (size_t)16 << 30}) {
      printf("== pipe %zu GiB\n", bytes >> 30);
      for (int rep = 0; rep < 2; ++rep) {
        run_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 0, 0>("f32+", buf, bytes, ws, sms, 4);
        run_guided<Red<IPM_ADD, IPM_F32>>("f32+", buf, bytes, ws, sms);
        run_flat<Red<IPM_ADD, IPM_F32>, 256, 2, 0, 3>("f32+", buf, bytes, ws, sms, 4);
        run_guided<Red<IPM_ADD, IPM_F32>, 2, true>("f32+", buf, bytes, ws, sms);
        run_guided<Red<IPM_ADD, IPM_F32>, 3, true>("f32+", buf, bytes, ws, sms);
        run_guided<Red<IPM_BXOR, IPM_I32>, 2, true>("i32^", buf, bytes, ws, sms);
        run_guided<Red<IPM_ADD, IPM_F64>, 2, true>("f64+", buf, bytes, ws, sms);
        run_guided<Red<IPM_MAX, IPM_F64>, 2, true>("f64max", buf, bytes, ws, sms);
        run_guided<Red<IPM_MAX, IPM_F32>, 2, true>("f32max", buf, bytes, ws, sms);
        run_guided<Red<IPM_MUL, IPM_I64>, 2, true>("i64*", buf, bytes, ws, sms);
        run_flat<Red<IPM_BXOR, IPM_I32>, 256, 4, 0, 0>("i32^", buf, bytes, ws, sms, 4);
        run_flat<Red<IPM_BXOR, IPM_I32>, 256, 2, 0, 3>("i32^", buf, bytes, ws, sms, 4);
        run_guided<Red<IPM_BXOR, IPM_I32>, 4, false>("i32^", buf, bytes, ws, sms);
      }
    }
  }
  if (mode == "tmaflat") {
    for (int i = 0; i < 30; ++i) k_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 0, 0><<<sms * 4, 256>>>(FlatParams{buf, (int64_t)(big / 4), 0, 0, 0, MODE_PARTIAL, (char*)ws + 4160, (uint64_t*)((char*)ws + 8192), (unsigned*)ws, nullptr, 0});
    CK(cudaDeviceSynchronize());
    for (size_t bytes : {(size_t)1 << 30, (size_t)16 << 30}) {
      printf("== tmaflat %zu GiB\n", bytes >> 30);
      for (int rep = 0; rep < 2; ++rep) {
        run_flat<Red<IPM_ADD, IPM_F32>, 256, 4, 0, 0>("f32+", buf, bytes, ws, sms, 4);
        run_guided<Red<IPM_ADD, IPM_F32>>("f32+", buf, bytes, ws, sms);
#define TMAV(RED, NAME)                                                           \
        run_flat_tma<RED, 8, 16384, 256, 1, 0>(NAME, buf, bytes, ws, sms);            \
        run_flat_tma<RED, 8, 16384, 256, 1, 1>(NAME, buf, bytes, ws, sms);            \
        run_flat_tma<RED, 8, 16384, 256, 1, 2>(NAME, buf, bytes, ws, sms);            \
        run_flat_tma<RED, 12, 16384, 256, 1, 1>(NAME, buf, bytes, ws, sms);           \
        run_flat_tma<RED, 6, 32768, 256, 1, 1>(NAME, buf, bytes, ws, sms);
        using Rf32 = Red<IPM_ADD, IPM_F32>;
        using Rf64 = Red<IPM_ADD, IPM_F64>;
        using Ri32 = Red<IPM_BXOR, IPM_I32>;
        using Rmax = Red<IPM_MAX, IPM_F64>;
        TMAV(Rf32, "f32+")
        TMAV(Rf64, "f64+")
        TMAV(Ri32, "i32^")
        TMAV(Rmax, "f64max")
        run_flat<Red<IPM_BXOR, IPM_I32>, 256, 4, 0, 0>("i32^", buf, bytes, ws, sms, 4);
      }
    }
  }
  if (mode == "all" || mode == "big") {
    printf("== flat variants at 16 GiB\n");
    const size_t bytes = (size_t)16 << 30;
    run_flat<Red<IPM_ADD, IPM_F32>, 1024, 4, 0>("f32+", buf, bytes, ws, sms);
    run_flat<Red<IPM_ADD, IPM_F32>, 512, 8, 0>("f32+", buf, bytes, ws, sms);
    run_flat<Red<IPM_ADD, IPM_F64>, 1024, 4, 0>("f64+", buf, bytes, ws, sms);
    run_flat<Red<IPM_MAX, IPM_F32>, 1024, 4, 0>("f32max", buf, bytes, ws, sms);
    run_flat<Red<IPM_MAX, IPM_F32>, 256, 4, 0>("f32max", buf, bytes, ws, sms);
    run_flat<Red<IPM_MUL, IPM_I64>, 256, 4, 0>("i64*", buf, bytes, ws, sms);
    run_flat<Red<IPM_MUL, IPM_I64>, 1024, 4, 0>("i64*", buf, bytes, ws, sms);
  }
  return 0;
}
