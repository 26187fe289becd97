/* cpu_omp.c — the CPU analogue of the clause as a BASELINE (BASELINE.md "CPU native baseline"): OpenMP
 * `parallel for reduction(+:sum)` in the input's native precision on all host cores. Not the oracle (oracle/ is
 * the reference for correctness); bench.py times it next to the GPU numbers at N = 1. Built by tools/build.py
 * (gcc -O3 -march=x86-64-v2 -fopenmp) into tools/bin/libcpu_omp.so; optional. */
#include <omp.h>
#include <stdint.h>

int cpu_omp_threads(void) { return omp_get_max_threads(); }

/* reduction(+:s) over float32 with a float32 accumulator per thread, as `float s; #pragma acc loop reduction(+:s)`
 * would be compiled for a CPU target */
float cpu_omp_sum_f32(const float* a, int64_t n) {
  float s = 0.0f;
#pragma omp parallel for simd reduction(+ : s) schedule(static)
  for (int64_t i = 0; i < n; ++i) s += a[i];
  return s;
}

/* the same with a float64 accumulator (the precision the GPU path uses for float32 +) */
double cpu_omp_sum_f32_f64(const float* a, int64_t n) {
  double s = 0.0;
#pragma omp parallel for simd reduction(+ : s) schedule(static)
  for (int64_t i = 0; i < n; ++i) s += a[i];
  return s;
}
