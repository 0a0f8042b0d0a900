// alu_peak.cu — issue-rate microbenchmarks that give the ALU roofline its
// measured denominators (VERDICT r01 "missing 6"; SURVEY.md §8(d) "Roof:
// R_int ... take these from MEASURED_PEAKS.json or a microbenchmark of the
// IADD3 / ISETP.EX / SEL mix").  Not part of the product; built by
// __graft_entry__.build() into tools/alu_peak, run on the B200 by
// tools/alu_peak.py, which writes profiles/alu_peak_r02.json.
//
// Every kernel runs NCH independent dependency chains per thread (enough ILP
// to cover the 4-cycle ALU / fp64 latency) over a persistent grid of
// 148 x 8 x 256 threads, so the measured rate is the pipe's throughput, not
// its latency.  Each kernel reports "units" (the semantic operation it
// repeats) per second; tools/alu_peak.py converts to SASS instructions with
// the per-unit instruction counts read from cuobjdump of this binary.
//
//   iadd   : a = a + b + c (IADD3), alu pipe only
//   mix    : IADD3 + IMAD alternating chains (alu + fma pipes): the issue ceiling
//   imax64 : int64 x = max(x, y) + d  -- the 1F1B cell in int64 (SURVEY: 8 int32 ops)
//   dcell  : double x = (x > y ? x : y) + d -- the 1F1B cell as the product runs it (fp64)
//   dadd   : double a = a + b, fp64 pipe only
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NCH = 8;
constexpr int ITERS = 4096;

__global__ void __launch_bounds__(256) k_iadd(uint32_t* out, uint32_t b, uint32_t c) {
  uint32_t a[NCH];
#pragma unroll
  for (int k = 0; k < NCH; ++k) a[k] = threadIdx.x + k;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < NCH; ++k) asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a[k]) : "r"(b), "r"(c + it));
  }
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < NCH; ++k) s ^= a[k];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void __launch_bounds__(256) k_mix(uint32_t* out, uint32_t b, uint32_t c) {
  uint32_t a[NCH];
#pragma unroll
  for (int k = 0; k < NCH; ++k) a[k] = threadIdx.x + k;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      if (k & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b | 1), "r"(c + it));
      else asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a[k]) : "r"(b), "r"(c + it));
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < NCH; ++k) s ^= a[k];
  if (s == 0x12345678u) out[0] = s;
}

// int64 max-plus cell: x_k = max(x_k, x_{k+1}) + d (chains coupled pairwise
// like neighbouring pipeline stages; still NCH-way parallel per step)
__global__ void __launch_bounds__(256) k_imax64(long long* out, long long d) {
  long long x[NCH];
#pragma unroll
  for (int k = 0; k < NCH; ++k) x[k] = threadIdx.x * 7 + k;
  for (int it = 0; it < ITERS; ++it) {
    long long o[NCH];
#pragma unroll
    for (int k = 0; k < NCH; ++k) o[k] = x[k];
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const long long y = o[(k + 1) % NCH] + (long long)it;
      x[k] = (o[k] > y ? o[k] : y) + d;
    }
  }
  long long s = 0;
#pragma unroll
  for (int k = 0; k < NCH; ++k) s ^= x[k];
  if (s == 0x12345678) out[0] = s;
}

// the fp64 cell of Pipe<P> (hsim_core.cuh): X[s] = dmax(old[s], old[s-1]) + f[s]
__global__ void __launch_bounds__(256) k_dcell(double* out, double d) {
  double x[NCH];
#pragma unroll
  for (int k = 0; k < NCH; ++k) x[k] = (double)(threadIdx.x * 7 + k);
  const double dd = d + (double)threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
    double o[NCH];
#pragma unroll
    for (int k = 0; k < NCH; ++k) o[k] = x[k];
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const double y = o[(k + 1) % NCH];
      x[k] = (o[k] > y ? o[k] : y) + dd;
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < NCH; ++k) s += x[k];
  if (s == 1.2345) out[0] = s;
}

__global__ void __launch_bounds__(256) k_dadd(double* out, double b) {
  double a[NCH];
#pragma unroll
  for (int k = 0; k < NCH; ++k) a[k] = (double)(threadIdx.x + k);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < NCH; ++k) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(a[k]) : "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < NCH; ++k) s += a[k];
  if (s == 1.2345) out[0] = s;
}

template <typename F>
static float time_kernel(F launch, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  const int blocks = sms * 8, threads = 256;
  const double thr = (double)blocks * threads;
  void* buf = nullptr;
  cudaMalloc(&buf, 64);
  const int reps = argc > 1 ? atoi(argv[1]) : 20;
  struct R { const char* name; const char* unit; double per_thread_iter; float ms; };
  R r[5] = {
      {"iadd", "IADD3", 2.0 * NCH, time_kernel([&] { k_iadd<<<blocks, threads>>>((uint32_t*)buf, 3u, 5u); }, reps)},
      {"mix", "IADD3|IMAD", 1.5 * NCH, time_kernel([&] { k_mix<<<blocks, threads>>>((uint32_t*)buf, 3u, 5u); }, reps)},
      {"imax64", "int64 cell", 1.0 * NCH, time_kernel([&] { k_imax64<<<blocks, threads>>>((long long*)buf, 3); }, reps)},
      {"dcell", "fp64 cell", 1.0 * NCH, time_kernel([&] { k_dcell<<<blocks, threads>>>((double*)buf, 3.0); }, reps)},
      {"dadd", "DADD", 1.0 * NCH, time_kernel([&] { k_dadd<<<blocks, threads>>>((double*)buf, 1.0); }, reps)},
  };
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "CUDA error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  printf("{\"sms\": %d, \"clock_attr_mhz\": %.0f, \"grid\": [%d, %d], \"iters\": %d, \"kernels\": {", sms, clk_khz / 1e3,
         blocks, threads, ITERS);
  for (int k = 0; k < 5; ++k) {
    const double units = thr * ITERS * r[k].per_thread_iter;
    printf("%s\"%s\": {\"unit\": \"%s\", \"units_per_thread_iter\": %.1f, \"ms\": %.4f, \"units_per_s\": %.6e}",
           k ? ", " : "", r[k].name, r[k].unit, r[k].per_thread_iter, r[k].ms, units / (r[k].ms * 1e-3));
  }
  printf("}}\n");
  cudaFree(buf);
  return 0;
}
