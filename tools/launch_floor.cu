// launch_floor.cu — context for C1: CUDA-event time of empty / trivial kernels on the box (not product).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/lat tools/launch_floor.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <algorithm>
__global__ void k_empty() {}
__global__ void k_one(int* o) { if (threadIdx.x == 0) *o = 1; }
__global__ void k_read(const int* a, int n, int* o) {
  int s = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += a[i];
  s = __reduce_add_sync(0xffffffffu, s);
  if ((threadIdx.x & 31) == 0) atomicAdd(o, s);
}
template <class F> float med(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  std::vector<float> v;
  for (int i = 0; i < 200; ++i) f();
  cudaDeviceSynchronize();
  for (int i = 0; i < 500; ++i) { cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); v.push_back(ms * 1000); }
  std::sort(v.begin(), v.end()); return v[v.size() / 2];
}
int main() {
  int *o, *a; cudaMalloc(&o, 4); cudaMalloc(&a, 4 << 20); cudaMemset(a, 0, 4 << 20);
  printf("empty kernel<<<1,32>>>     %.2f us\n", med([&] { k_empty<<<1, 32>>>(); }));
  printf("empty kernel<<<592,256>>>  %.2f us\n", med([&] { k_empty<<<592, 256>>>(); }));
  printf("one store <<<1,256>>>      %.2f us\n", med([&] { k_one<<<1, 256>>>(o); }));
  printf("read 4 KiB <<<1,256>>>     %.2f us\n", med([&] { k_read<<<1, 256>>>(a, 1024, o); }));
  printf("nothing (events only)      %.2f us\n", med([&] {}));
  return 0;
}
