// FP32 / FP64 CUDA-core peak microbenchmark for the LANN roofline denominator.
// MEASURED_PEAKS.json (driver-written) carries only HBM and bf16 tensor peaks; the
// LANN trainer is bound by the FP32 FMA pipe, so this measures FFMA, FFMA2 (the
// sm_100 packed f32x2 FMA), DFMA / DADD / DMUL throughput and dependent latencies.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int kChains = 8;

__global__ void ffma_tput(float* out, float a, float b, int iters) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-7f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) x[c] = fmaf(x[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5f) out[0] = s;
}

__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }

__global__ void ffma2_tput(float* out, float a, float b, int iters) {
  unsigned long long x[kChains];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  unsigned long long ar = f2u(av), br = f2u(bv);
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = f2u(make_float2(threadIdx.x * 1e-7f + c, c + 0.5f));
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c)
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(ar), "l"(br));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) { float2 v = *reinterpret_cast<float2*>(&x[c]); s += v.x + v.y; }
  if (s == 1234.5f) out[0] = s;
}

__global__ void dfma_tput(double* out, double a, double b, int iters) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-7 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;
}

__global__ void dadd_tput(double* out, double b, int iters) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-7 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) x[c] = __dadd_rn(x[c], b);
  }
  double s = 0.;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;
}

// dependent-chain latency, one warp
__global__ void dadd_lat(double* out, double b, int iters, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = __dadd_rn(x, b);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = x; cyc[0] = t1 - t0; }
}
__global__ void ffma_lat(float* out, float a, float b, int iters, long long* cyc) {
  float x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = fmaf(x, a, b);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = x; cyc[0] = t1 - t0; }
}

template <typename F>
float time_ms(F f) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  float* fo; double* dof; long long* cyc;
  CK(cudaMalloc(&fo, 64)); CK(cudaMalloc(&dof, 64)); CK(cudaMalloc(&cyc, 64));
  const int threads = 512, blocks = sms * 4, iters = 4096;
  const double flops_f = 2.0 * kChains * 16.0 * iters * threads * (double)blocks;
  float t = time_ms([&] { ffma_tput<<<blocks, threads>>>(fo, 0.999f, 1e-3f, iters); });
  printf("{\"sms\": %d, \"ffma_tflops\": %.2f, ", sms, flops_f / t / 1e9);
  t = time_ms([&] { ffma2_tput<<<blocks, threads>>>(fo, 0.999f, 1e-3f, iters); });
  printf("\"ffma2_tflops\": %.2f, ", 2 * flops_f / t / 1e9);
  t = time_ms([&] { dfma_tput<<<blocks, threads>>>(dof, 0.999, 1e-3, iters / 4); });
  printf("\"dfma_tflops\": %.2f, ", flops_f / 4 / t / 1e9);
  t = time_ms([&] { dadd_tput<<<blocks, threads>>>(dof, 1e-3, iters / 4); });
  printf("\"dadd_gops\": %.1f, ", flops_f / 2 / 4 / t / 1e6);
  long long hc[2];
  dadd_lat<<<1, 32>>>(dof, 1e-3, 1024, cyc); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(hc, cyc, 8, cudaMemcpyDeviceToHost));
  printf("\"dadd_latency_cyc\": %.2f, ", hc[0] / (1024.0 * 16));
  ffma_lat<<<1, 32>>>(fo, 0.999f, 1e-3f, 1024, cyc); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(hc, cyc, 8, cudaMemcpyDeviceToHost));
  printf("\"ffma_latency_cyc\": %.2f, ", hc[0] / (1024.0 * 16));
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("\"clock_khz_attr\": %d}\n", clk);
  return 0;
}
