// Microbenchmark (developer tool): cycles per link of one dependent DADD chain per lane,
// with the second operand (a) a constant, (b) registers loaded before the timed loop, (c) a
// shared-memory row read two samples per 16-B load with the next block prefetched, as
// train_fp64_pipe's chain lanes do. W chain warps on one SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o dadd_chain_mb dadd_chain_mb.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int LD = 258, N = 256;

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ bool mb_test(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mb_wait(unsigned long long* bar, unsigned parity) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
               "@!p bra W_%=;\n\t}" ::"r"(su32(bar)), "r"(parity) : "memory");
}

template <int V>
__global__ void chain(double* out, long long* cyc) {
  extern __shared__ __align__(16) double sm[];
  __shared__ unsigned long long bars[8];
  for (int i = threadIdx.x; i < 96 * LD; i += blockDim.x) sm[i] = 1e-3 * (i % 97);
  if (threadIdx.x < 8) {  // completed phase 0: waits on parity 0 succeed at once
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[threadIdx.x])) : "memory");
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(su32(&bars[threadIdx.x])) : "memory");
  }
  __syncthreads();
  const int w = threadIdx.x >> 5;
  const double2* T = reinterpret_cast<const double2*>(sm + (threadIdx.x % 96) * LD);
  double g = 0.0;
  double2 A[16], B[16];
  for (int j = 0; j < 16; ++j) A[j] = T[j];
  long long t0 = clock64();
  for (int rep = 0; rep < 16; ++rep) {
    if (V == 0) {
#pragma unroll
      for (int j = 0; j < N; ++j) g = __dadd_rn(g, 1.0000001);
    } else if (V == 1) {
      for (int b = 0; b < 8; ++b) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          g = __dadd_rn(g, A[j].x);
          g = __dadd_rn(g, A[j].y);
        }
      }
    } else if (V == 5) {  // g += t[s] * a[s]: two 16-B loads per sample pair, the DMUL off the chain
      const double2* T2 = reinterpret_cast<const double2*>(sm + ((threadIdx.x / 6) % 96) * LD);
      const double2* A2 = reinterpret_cast<const double2*>(sm + (threadIdx.x % 6 + 40) * LD);
      for (int b = 0; b < 8; b += 2) {
        double2 tb[16], ab[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) { tb[j] = T2[(b + 1) * 16 + j]; ab[j] = A2[(b + 1) * 16 + j]; }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          g = __dadd_rn(g, __dmul_rn(A[j].x, B[j].x));
          g = __dadd_rn(g, __dmul_rn(A[j].y, B[j].y));
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) { A[j] = T2[((b + 2) & 7) * 16 + j]; B[j] = A2[((b + 2) & 7) * 16 + j]; }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          g = __dadd_rn(g, __dmul_rn(tb[j].x, ab[j].x));
          g = __dadd_rn(g, __dmul_rn(tb[j].y, ab[j].y));
        }
      }
    } else if (V == 3 || V == 4) {  // + a barrier test (3) / blocking wait (4) per block
      for (int b = 0; b < 8; ++b) {
        bool pre = true;
        if (V == 3) pre = mb_test(&bars[(b + 1) & 7], 0);
        else mb_wait(&bars[(b + 1) & 7], 0);
#pragma unroll
        for (int j = 0; j < 16; ++j) B[j] = T[((b + 1) & 7) * 16 + j];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          g = __dadd_rn(g, A[j].x);
          g = __dadd_rn(g, A[j].y);
        }
        if (!pre) {
          mb_wait(&bars[(b + 1) & 7], 0);
#pragma unroll
          for (int j = 0; j < 16; ++j) B[j] = T[((b + 1) & 7) * 16 + j];
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) A[j] = B[j];
      }
    } else {
      for (int b = 0; b < 8; b += 2) {
#pragma unroll
        for (int j = 0; j < 16; ++j) B[j] = T[(b + 1) * 16 + j];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          g = __dadd_rn(g, A[j].x);
          g = __dadd_rn(g, A[j].y);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) A[j] = T[((b + 2) & 7) * 16 + j];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          g = __dadd_rn(g, B[j].x);
          g = __dadd_rn(g, B[j].y);
        }
      }
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = g;
  if ((threadIdx.x & 31) == 0) cyc[w] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 64 * 8);
  const int smem = 96 * LD * 8;
  auto run = [&](auto k, const char* name, int warps) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int r = 0; r < 2; ++r) k<<<1, 32 * warps, smem>>>(out, cyc);
    cudaDeviceSynchronize();
    double mx = 0;
    for (int w = 0; w < warps; ++w) mx = cyc[w] > mx ? cyc[w] : mx;
    printf("%-28s warps=%d: cycles/link %.2f\n", name, warps, mx / (16.0 * N));
  };
  for (int w : {1, 3}) {
    run(chain<0>, "const operand", w);
    run(chain<1>, "register operands", w);
    run(chain<2>, "smem rows, block prefetch", w);
    run(chain<3>, "  + mbarrier test per block", w);
    run(chain<4>, "  + mbarrier wait per block", w);
    run(chain<5>, "t*a products in the chain lane", w);
  }
  return 0;
}
