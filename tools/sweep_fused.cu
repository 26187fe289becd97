// sweep_fused.cu — tuning experiment (not product): k_fused (several variables / x·y in one pass) with and
// without software pipelining of the tile loop, on 2^28-element arrays, CUDA events.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <functional>
#include <vector>
#include "ipm_fused.cuh"

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

template <class S, class C0, class C1, class C2, class C3, bool TWO, int U, bool PIPE, int MINB = 4>
void run(const char* name, void* x, void* y, int64_t n, void* ws, int sms, int cps) {
  using B = typename S::B;
  FusedParams p{};
  p.x = x; p.y = TWO ? y : nullptr; p.n = n; p.has_init = 0; p.out = (char*)ws + 4096;
  p.partials = (uint64_t*)((char*)ws + 8192); p.ticket = (unsigned*)ws;
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused<S, C0, C1, C2, C3, TWO, true, 256, U, PIPE, MINB>, 256, 0));
  const int grid = sms * cps;
  float ms = time_ms([&] { k_fused<S, C0, C1, C2, C3, TWO, true, 256, U, PIPE, MINB><<<grid, 256>>>(p); }, 20);
  CK(cudaGetLastError());
  B out[4];
  CK(cudaMemcpy(out, p.out, sizeof out, cudaMemcpyDeviceToHost));
  const double bytes = (double)n * sizeof(B) * (TWO ? 2 : 1);
  printf("fused %-8s U=%d PIPE=%d MINB=%d occ=%d cps=%d  %7.3f ms  %7.1f GB/s  out0=%.17g\n", name, U, (int)PIPE, MINB, occ, cps, ms,
         bytes / ms / 1e6, (double)out[0]);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t n = (int64_t)1 << 28;
  void *x, *y, *ws;
  CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&y, n * 8)); CK(cudaMalloc(&ws, 1 << 20));
  CK(cudaMemset(x, 0x3c, n * 8)); CK(cudaMemset(y, 0x3c, n * 8)); CK(cudaMemset(ws, 0, 1 << 20));
  using ADDX = Comp<Red<IPM_ADD, IPM_F32>, EX>;
  using ADDXX = Comp<Red<IPM_ADD, IPM_F32>, EXX>;
  using ADDXY = Comp<Red<IPM_ADD, IPM_F32>, EXY>;
  using MINX = Comp<Red<IPM_MIN, IPM_F32>, EX>;
  using MAXX = Comp<Red<IPM_MAX, IPM_F32>, EX>;
  using STATS = Sig<ADDX, ADDXX, MINX, MAXX>;
  using DOT = Sig<ADDXY>;
  using SS = Sig<ADDX, ADDXX>;
  using D_ADDX = Comp<Red<IPM_ADD, IPM_F64>, EX>;
  using D_ADDXX = Comp<Red<IPM_ADD, IPM_F64>, EXX>;
  using DSS = Sig<D_ADDX, D_ADDXX>;
  for (int rep = 0; rep < 3; ++rep) {
    run<DOT, ADDXY, NoComp, NoComp, NoComp, true, 2, false, 0>("dot", x, y, n, ws, sms, 4);
    run<DOT, ADDXY, NoComp, NoComp, NoComp, true, 2, false, 4>("dot", x, y, n, ws, sms, 4);
    run<DOT, ADDXY, NoComp, NoComp, NoComp, true, 2, false, 5>("dot", x, y, n, ws, sms, 5);
    run<STATS, ADDX, ADDXX, MINX, MAXX, false, 2, false, 0>("stats", x, y, n, ws, sms, 4);
    run<STATS, ADDX, ADDXX, MINX, MAXX, false, 2, false, 4>("stats", x, y, n, ws, sms, 4);
    run<STATS, ADDX, ADDXX, MINX, MAXX, false, 2, false, 5>("stats", x, y, n, ws, sms, 5);
  }
  return 0;
}
