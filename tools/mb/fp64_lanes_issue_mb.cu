// Microbenchmark (developer tool): FP64 issue cost per warp instruction on the B200 as a function
// of active lanes (K = 8 independent DADD chains per thread, one warp, or one warp on each of the
// four SM sub-partitions). Does a partially active warp finish its FP64 instructions sooner?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o fp64_lanes_issue_mb fp64_lanes_issue_mb.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void issue(double* out, long long* cyc, int iters, int act) {
  double a[K];
#pragma unroll
  for (int k = 0; k < K; ++k) a[k] = threadIdx.x * 1e-3 + k;
  const double b = 1.0000001;
  __syncthreads();
  long long t0 = clock64();
  if ((threadIdx.x & 31) < act) {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int k = 0; k < K; ++k) a[k] = __dadd_rn(a[k], b);
  }
  __syncwarp();
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
  for (int warps : {1, 4, 8})
    for (int act : {32, 16, 8, 4, 1}) {
      for (int r = 0; r < 2; ++r) issue<8><<<1, 32 * warps>>>(out, cyc, iters, act);
      cudaDeviceSynchronize();
      double mx = 0; for (int w = 0; w < warps; ++w) mx = cyc[w] > mx ? cyc[w] : mx;
      printf("DADD K=8 warps=%d active lanes=%2d: cycles per warp-instr %.2f\n", warps, act, mx / (double(iters) * 8));
    }
  return 0;
}
