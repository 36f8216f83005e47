// Microbenchmark (developer tool): FP64 issue rate per warp and per SM sub-partition on the
// B200: K independent DADD (or DMUL) chains per thread, W warps per CTA on one SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o fp64_issue_mb fp64_issue_mb.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int K, bool MUL>
__global__ void issue(double* out, long long* cyc, int iters) {
  double a[K];
#pragma unroll
  for (int k = 0; k < K; ++k) a[k] = threadIdx.x * 1e-3 + k;
  const double b = 1.0000001;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < K; ++k) a[k] = MUL ? __dmul_rn(a[k], b) : __dadd_rn(a[k], b);
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if ((threadIdx.x & 31) == 0) cyc[threadIdx.x >> 5] = t1 - t0;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 64 * 8);
  const int iters = 4096;
  auto run = [&](auto k, const char* name, int K, int warps) {
    for (int r = 0; r < 2; ++r) k<<<1, 32 * warps>>>(out, cyc, iters);
    cudaDeviceSynchronize();
    double mx = 0; for (int w = 0; w < warps; ++w) mx = cyc[w] > mx ? cyc[w] : mx;
    printf("%-6s K=%d warps=%2d: cycles per instr per warp %.2f  (SM-wide warp-instr/cycle %.3f)\n", name, K, warps,
           mx / (double(iters) * K), warps * double(iters) * K / mx);
  };
  for (int w : {1, 2, 4, 8, 16}) {
    run(issue<1, false>, "DADD", 1, w);
    run(issue<2, false>, "DADD", 2, w);
    run(issue<4, false>, "DADD", 4, w);
    run(issue<8, false>, "DADD", 8, w);
    run(issue<8, true>, "DMUL", 8, w);
  }
  return 0;
}
