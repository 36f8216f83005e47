// Microbenchmark (developer tool): FP64 issue cost of a warp instruction by number of active
// lanes (32 / 16 / 8): K independent DMUL streams per thread, W warps on one SM sub-partition.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o fp64_lanes_mb fp64_lanes_mb.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void issue(double* out, long long* cyc, int iters, int active) {
  const int l = threadIdx.x & 31;
  long long t0 = clock64();
  if (l < active) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = l * 1e-3 + k;
    const double b = 1.0000001;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = __dmul_rn(a[k], b);
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  }
  __syncwarp();
  long long t1 = clock64();
  if (l == 0) cyc[threadIdx.x >> 5] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 64 * 8);
  const int iters = 4096;
  for (int warps : {1, 4}) {  // 4 warps: one per sub-partition
    for (int act : {32, 16, 8, 4}) {
      for (int r = 0; r < 2; ++r) issue<<<1, 32 * warps>>>(out, cyc, iters, act);
      cudaDeviceSynchronize();
      printf("warps=%d active lanes=%2d: cycles per DMUL warp-instruction %.2f\n", warps, act,
             cyc[0] / (8.0 * iters));
    }
  }
  return 0;
}
