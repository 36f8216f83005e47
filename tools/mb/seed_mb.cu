// Microbenchmark (developer tool): dependent latency of FP64 reciprocal / rsqrt seeds on B200.
#include <cstdio>
#include <cuda_runtime.h>
template <int V>
__global__ void k(double* out, long long* cyc, int iters) {
  double x = 1.2345 + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double y;
    if (V == 0) asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    else if (V == 1) asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    else if (V == 2) { float f = __double2float_rn(x); y = (double)__frcp_rn(f); }
    else if (V == 3) { float f; asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f) : "d"(x)); float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f)); asm volatile("cvt.f64.f32 %0, %1;" : "=d"(y) : "f"(r)); }
    else if (V == 4) { y = __longlong_as_double(0x7fde5d0f4e8e7b1fLL - __double_as_longlong(x)); }
    else { y = __dadd_rn(x, 1e-300); }
    x = __dadd_rn(y, 1.2345);  // keep the chain dependent and x in range
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 12); cudaMallocManaged(&cyc, 64);
  const char* n[6] = {"MUFU.RCP64H (rcp.approx.ftz.f64)", "MUFU.RSQ64H (rsqrt.approx.ftz.f64)", "f64->f32, __frcp_rn, ->f64",
                      "cvt.f32.f64 + rcp.approx.f32 + cvt.f64.f32", "integer magic seed", "DADD only (baseline)"};
  auto run = [&](auto kern, int v) {
    for (int r = 0; r < 2; ++r) kern<<<1, 32>>>(out, cyc, 4096);
    cudaDeviceSynchronize();
    printf("%-44s %.1f cycles per step (incl. one DADD)\n", n[v], cyc[0] / 4096.0);
  };
  run(k<0>, 0); run(k<1>, 1); run(k<2>, 2); run(k<3>, 3); run(k<4>, 4); run(k<5>, 5);
}
