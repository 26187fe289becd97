// cub_context.cu — library context (not product): CUB DeviceReduce on the same sizes as bench.py's suite,
// CUDA-event timed, inputs larger than L2. Prints one JSON object per line.
#include <cub/cub.cuh>
#include <cuda/std/functional>
#include <cstdio>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <class F>
static float time_ms(F f, int reps) {
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

template <class T, class O, class Op>
void run(const char* name, int64_t n, Op op, O init) {
  T* in; O* out; void* tmp = nullptr; size_t tb = 0;
  CK(cudaMalloc(&in, n * sizeof(T)));
  CK(cudaMemset(in, 0x3c, n * sizeof(T)));
  CK(cudaMalloc(&out, sizeof(O)));
  CK(cub::DeviceReduce::Reduce(tmp, tb, in, out, n, op, init));
  CK(cudaMalloc(&tmp, tb));
  const float ms = time_ms([&] { cub::DeviceReduce::Reduce(tmp, tb, in, out, n, op, init); }, 20);
  CK(cudaGetLastError());
  printf("{\"lib\": \"cub::DeviceReduce::Reduce\", \"case\": \"%s\", \"n\": %lld, \"ms\": %.5f, \"GB/s\": %.1f}\n", name,
         (long long)n, ms, n * sizeof(T) / ms / 1e6);
  fflush(stdout);
  CK(cudaFree(in)); CK(cudaFree(out)); CK(cudaFree(tmp));
}

int main() {
  run<float, float>("sum_float32_acc_float32_2^28", (int64_t)1 << 28, cuda::std::plus<>{}, 0.0f);
  run<float, double>("sum_float32_acc_float64_2^28", (int64_t)1 << 28, cuda::std::plus<>{}, 0.0);
  run<float, float>("max_float32_2^28", (int64_t)1 << 28, cuda::maximum<>{}, -INFINITY);
  run<double, double>("sum_float64_2^28", (int64_t)1 << 28, cuda::std::plus<>{}, 0.0);
  run<int, int>("sum_int32_2^30", (int64_t)1 << 30, cuda::std::plus<>{}, 0);
  run<float, double>("sum_float32_acc_float64_2^32", (int64_t)1 << 32, cuda::std::plus<>{}, 0.0);
  return 0;
}
