// cub_context.cu — library context (not product): CUB DeviceReduce on the same sizes as bench.py's suite,
// CUDA-event timed, inputs larger than L2. Prints one JSON object per line.
// usage: cub_context [ragged_offsets.bin]   (int64 CSR offsets, rows + 1 of them)
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

// CSR segmented reduce (float32 values, float64 accumulation, float32 out like the clause) over row offsets
// read from a file of int64 (rows + 1 entries)
static void run_segmented(const char* name, const std::vector<int64_t>& off) {
  const int64_t rows = (int64_t)off.size() - 1, nnz = off.back() - off.front();
  float* in; double* out; int64_t* d_off; void* tmp = nullptr; size_t tb = 0;
  CK(cudaMalloc(&in, nnz * sizeof(float)));
  CK(cudaMemset(in, 0x3c, nnz * sizeof(float)));
  CK(cudaMalloc(&out, rows * sizeof(double)));
  CK(cudaMalloc(&d_off, off.size() * sizeof(int64_t)));
  CK(cudaMemcpy(d_off, off.data(), off.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  CK(cub::DeviceSegmentedReduce::Reduce(tmp, tb, in, out, rows, d_off, d_off + 1, cuda::std::plus<>{}, 0.0));
  CK(cudaMalloc(&tmp, tb));
  const float ms = time_ms([&] {
    cub::DeviceSegmentedReduce::Reduce(tmp, tb, in, out, rows, d_off, d_off + 1, cuda::std::plus<>{}, 0.0);
  }, 20);
  CK(cudaGetLastError());
  const double bytes = nnz * 4.0 + (rows + 1) * 8.0 + rows * 8.0;
  printf("{\"lib\": \"cub::DeviceSegmentedReduce::Reduce\", \"case\": \"%s\", \"rows\": %lld, \"nnz\": %lld, "
         "\"ms\": %.5f, \"GB/s\": %.1f}\n", name, (long long)rows, (long long)nnz, ms, bytes / ms / 1e6);
  fflush(stdout);
  CK(cudaFree(in)); CK(cudaFree(out)); CK(cudaFree(d_off)); CK(cudaFree(tmp));
}

int main(int argc, char** argv) {
  {  // C3 as CSR: 65536 rows x 4096
    std::vector<int64_t> off(65537);
    for (int64_t r = 0; r <= 65536; ++r) off[r] = r * 4096;
    run_segmented("segmented_float32_acc_float64_65536x4096", off);
  }
  if (argc > 1) {  // the ragged suite's power-law offsets
    FILE* f = fopen(argv[1], "rb");
    if (f) {
      fseek(f, 0, SEEK_END);
      const long cnt = ftell(f) / 8;
      fseek(f, 0, SEEK_SET);
      std::vector<int64_t> off(cnt);
      if (fread(off.data(), 8, cnt, f) == (size_t)cnt) run_segmented("ragged_float32_acc_float64_csr", off);
      fclose(f);
    }
  }
  run<float, float>("sum_float32_acc_float32_2^28", (int64_t)1 << 28, cuda::std::plus<>{}, 0.0f);
  run<float, double>("sum_float32_acc_float64_2^28", (int64_t)1 << 28, cuda::std::plus<>{}, 0.0);
  run<float, float>("max_float32_2^28", (int64_t)1 << 28, cuda::maximum<>{}, -INFINITY);
  run<double, double>("sum_float64_2^28", (int64_t)1 << 28, cuda::std::plus<>{}, 0.0);
  run<int, int>("sum_int32_2^30", (int64_t)1 << 30, cuda::std::plus<>{}, 0);
  run<float, double>("sum_float32_acc_float64_2^32", (int64_t)1 << 32, cuda::std::plus<>{}, 0.0);
  return 0;
}
