/* acc_reduce.c — calling libipm from plain C (no Python, no torch): the boundary is a C ABI.
 *
 *   #pragma acc data copyin(a[0:n])
 *   #pragma acc parallel loop reduction(+:sum) reduction(max:m)
 *   for (i = 0; i < n; ++i) { sum += a[i]; m = max(m, a[i]); }
 *
 * Build (tests/test_capi.py does this):
 *   gcc -std=c99 -O2 -Wall -Werror -pedantic -I include -isystem /usr/local/cuda/include examples/acc_reduce.c \
 *       -L paper_1412_1127_b200 -lipm -Wl,-rpath,$PWD/paper_1412_1127_b200 -L/usr/local/cuda/lib64 -lcudart
 * Exit status 0 iff every result matches its closed form. */
#define _POSIX_C_SOURCE 199309L
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <time.h>

#include <cuda_runtime_api.h>

#include "ipm.h"

#define CHECK(call)                                                                            \
  do {                                                                                         \
    ipm_status s_ = (call);                                                                    \
    if (s_ != IPM_OK) {                                                                        \
      fprintf(stderr, "%s: %s (%s)\n", #call, ipm_status_str(s_), ipm_last_error_message()); \
      return 2;                                                                                \
    }                                                                                          \
  } while (0)

int main(void) {
  const int64_t n = (int64_t)1 << 24;
  int32_t* a = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  int64_t i;
  void *dev = NULL, *ws = NULL;
  int32_t sum = 0, mx = INT32_MIN, x = 0;
  int failures = 0;
  if (!a) return 2;
  for (i = 0; i < n; ++i) a[i] = (int32_t)(i + 1);

  /* the data clause: copyin(a[0:n]) through the present table */
  CHECK(ipm_copyin(a, (size_t)n * sizeof(int32_t), &dev, NULL));
  if (cudaMalloc(&ws, ipm_workspace_bytes()) != cudaSuccess) return 2;
  CHECK(ipm_workspace_init(ws, NULL));

  /* reduction(+:sum): n(n+1)/2 mod 2^32 (two's-complement wrap) */
  CHECK(ipm_reduce(IPM_ADD, IPM_I32, dev, n, &sum, ws, NULL));
  if ((uint32_t)sum != (uint32_t)(((uint64_t)n * (uint64_t)(n + 1) / 2) & 0xFFFFFFFFu)) {
    fprintf(stderr, "sum: got %d\n", sum);
    failures++;
  }
  /* reduction(max:m) */
  CHECK(ipm_reduce(IPM_MAX, IPM_I32, dev, n, &mx, ws, NULL));
  if (mx != (int32_t)n) {
    fprintf(stderr, "max: got %d\n", mx);
    failures++;
  }
  /* reduction(^:x): XOR of 1..n, closed form for n = 2^24 (n mod 4 == 0) -> n */
  CHECK(ipm_reduce(IPM_BXOR, IPM_I32, dev, n, &x, ws, NULL));
  if (x != (int32_t)n) {
    fprintf(stderr, "xor: got %d\n", x);
    failures++;
  }
  /* & on a float is rejected at the boundary */
  {
    float f = 0.0f;
    if (ipm_reduce(IPM_BAND, IPM_F32, dev, 1, &f, ws, NULL) != IPM_E_REDOP) failures++;
  }
  /* present lookup of a sub-range, then the end of the data region */
  {
    void* sub = NULL;
    CHECK(ipm_present(a + 100, 4 * sizeof(int32_t), &sub));
    if ((char*)sub != (char*)dev + 100 * sizeof(int32_t)) failures++;
  }
  /* host-side latency of the synchronous clause on BASELINE config 1 (2^20 int32): launch + kernel + 4-byte D2H */
  {
    const int64_t n1 = (int64_t)1 << 20;
    struct timespec t0, t1;
    int r, reps = 2000;
    for (r = 0; r < 100; ++r) CHECK(ipm_reduce(IPM_ADD, IPM_I32, dev, n1, &x, ws, NULL));
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (r = 0; r < reps; ++r) {
      x = 0;
      CHECK(ipm_reduce(IPM_ADD, IPM_I32, dev, n1, &x, ws, NULL));
    }
    clock_gettime(CLOCK_MONOTONIC, &t1);
    printf("ipm_reduce(+, 2^20 int32) synchronous call: %.2f us (L2-warm)\n",
           ((t1.tv_sec - t0.tv_sec) * 1e9 + (t1.tv_nsec - t0.tv_nsec)) / 1e3 / reps);
    if (x != (int32_t)(((uint64_t)n1 * (uint64_t)(n1 + 1) / 2) & 0xFFFFFFFFu)) failures++;
  }
  CHECK(ipm_delete(a, NULL));
  if (ipm_present_count() != 0) failures++;
  cudaFree(ws);
  free(a);
  printf("acc_reduce: %s\n", failures ? "FAILED" : "ok");
  return failures ? 1 : 0;
}
