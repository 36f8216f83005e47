// Microbenchmark (developer tool): does a dependent DADD chain slow down when its addend comes
// from a different register every link (register-bank pairing) rather than from a shared-memory
// load? One warp, cycles per link.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o dadd_bank_mb dadd_bank_mb.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096, R = 512;
#ifndef WARPS
#define WARPS 1
#endif  // links timed; ring of links in shared memory

template <int V>
__global__ void k(double* out, long long* cyc, const double* src) {
  const int l = threadIdx.x & 31;  // lane; warps w > 0 use their own rows below
  double g = 0.0;
  double c[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) c[u] = src[u * 32 + l];
  const double h = src[l];
  long long t0 = clock64();
  if (V == 0) {  // one addend register
#pragma unroll 16
    for (int j = 0; j < N; ++j) g = __dadd_rn(g, h);
  } else if (V == 1) {  // sixteen addend registers in turn
    for (int j = 0; j < N / 16; ++j) {
#pragma unroll
      for (int u = 0; u < 16; ++u) g = __dadd_rn(g, c[u]);
    }
  } else if (V == 2) {  // the accumulator alternates between two registers
    double g2 = 0.0;
    for (int j = 0; j < N / 16; ++j) {
#pragma unroll
      for (int u = 0; u < 16; u += 2) {
        g2 = __dadd_rn(g, c[u]);
        g = __dadd_rn(g2, c[u + 1]);
      }
    }
  } else if (V == 3) {  // addend as the first operand
    for (int j = 0; j < N / 16; ++j) {
#pragma unroll
      for (int u = 0; u < 16; ++u) g = __dadd_rn(c[u], g);
    }
  }
  if (V == 4 || V == 5) {  // addends streamed from shared memory, loads a 16-link block ahead
    extern __shared__ double row_all[];  // per warp [R][32]: link j of lane l at row[j * 32 + l]
    double* row = row_all + (threadIdx.x >> 5) * (R / 3) * 32 * 0;
    if (V == 4) {  // 16-byte loads (two links per load) as in the pipelined trainer
      const double2* r2 = reinterpret_cast<const double2*>(row);
      double2 a[8], b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = r2[u * 32 + l];
      for (int j = 0; j < N / 16; j += 2) {
#pragma unroll
        for (int u = 0; u < 8; ++u) b[u] = r2[((j + 1) * 8 + u) % (R / 2) * 32 + l];
#pragma unroll
        for (int u = 0; u < 8; ++u) { g = __dadd_rn(g, a[u].x); g = __dadd_rn(g, a[u].y); }
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = r2[((j + 2) * 8 + u) % (R / 2) * 32 + l];
#pragma unroll
        for (int u = 0; u < 8; ++u) { g = __dadd_rn(g, b[u].x); g = __dadd_rn(g, b[u].y); }
      }
    } else {  // 8-byte loads (one link per load)
      double a[16], b[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) a[u] = row[u * 32 + l];
      for (int j = 0; j < N / 16; j += 2) {
#pragma unroll
        for (int u = 0; u < 16; ++u) b[u] = row[(((j + 1) * 16 + u) % R) * 32 + l];
#pragma unroll
        for (int u = 0; u < 16; ++u) g = __dadd_rn(g, a[u]);
#pragma unroll
        for (int u = 0; u < 16; ++u) a[u] = row[(((j + 2) * 16 + u) % R) * 32 + l];
#pragma unroll
        for (int u = 0; u < 16; ++u) g = __dadd_rn(g, b[u]);
      }
    }
  }
  long long t1 = clock64();
  out[l] = g;
  if (threadIdx.x == 0) cyc[V] = t1 - t0;
  if (threadIdx.x == 32) cyc[8 + V] = t1 - t0;
}

int main() {
  double *out, *src;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMalloc(&src, 4096 * 8);
  cudaMemset(src, 0, 4096 * 8);
  cudaMallocManaged(&cyc, 64 * 8);
  for (int it = 0; it < 3; ++it) {
    k<0><<<1, 32>>>(out, cyc, src);
    k<1><<<1, 32>>>(out, cyc, src);
    k<2><<<1, 32>>>(out, cyc, src);
    k<3><<<1, 32>>>(out, cyc, src);
    cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, R * 32 * 8);
    cudaFuncSetAttribute(k<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, R * 32 * 8);
    k<4><<<1, 32 * WARPS, R * 32 * 8>>>(out, cyc, src);
    k<5><<<1, 32 * WARPS, R * 32 * 8>>>(out, cyc, src);
    cudaDeviceSynchronize();
  }
  printf("one addend register      %.2f cycles/link\n", cyc[0] / double(N));
  printf("16 addend registers      %.2f\n", cyc[1] / double(N));
  printf("alternating accumulator  %.2f\n", cyc[2] / double(N));
  printf("addend first operand     %.2f\n", cyc[3] / double(N));
  printf("16-byte shared loads     %.2f\n", cyc[4] / double(N));
  printf("8-byte shared loads      %.2f\n", cyc[5] / double(N));
  printf("(%d warps; warp 1: %.2f %.2f)\n", WARPS, cyc[12] / double(N), cyc[13] / double(N));
  return 0;
}
