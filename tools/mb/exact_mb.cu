// Test + microbenchmark (developer tool) for csrc/exact_fp64.cuh: (1) the verified fast division
// and sqrt against CUDA's correctly rounded __ddiv_rn / __dsqrt_rn on billions of random operands
// (mixed exponent ranges, Adam-like ranges, random bit patterns); (2) the latency of one Adam step.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -I../../paper_2003_07497_b200/csrc -o exact_mb exact_mb.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "exact_fp64.cuh"

using namespace lann;

__device__ unsigned long long sm64(unsigned long long& s) {
  unsigned long long z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// a double with a random mantissa and an exponent uniform in [lo, hi] (unbiased), random sign
__device__ double rnd(unsigned long long& s, int lo, int hi, bool sign) {
  const unsigned long long r = sm64(s);
  const int ex = lo + int((r >> 52) % (unsigned)(hi - lo + 1));
  unsigned long long bits = (r & 0xfffffffffffffull) | ((unsigned long long)(ex + 1023) << 52);
  if (sign && ((r >> 63) & 1)) bits |= 1ull << 63;
  return __longlong_as_double(bits);
}

__global__ void check(unsigned long long seed, int iters, int mode, unsigned long long* cnt) {
  unsigned long long s = seed ^ (blockIdx.x * 1315423911ull + threadIdx.x * 2654435761ull);
  unsigned long long n_ok = 0, n_bad = 0, n_fb = 0;
  for (int it = 0; it < iters; ++it) {
    double a, b;
    if (mode == 0) { a = rnd(s, -200, 200, true); b = rnd(s, -200, 200, true); }
    else if (mode == 1) { a = rnd(s, -60, 0, true); b = rnd(s, -20, 0, false); }      // Adam-like
    else if (mode == 2) { a = __longlong_as_double(sm64(s)); b = __longlong_as_double(sm64(s)); }
    else { a = rnd(s, -1000, 1000, true); b = rnd(s, -1000, 1000, true); }
    bool ok = true;
    const double q = div_checked(a, b, rcp_refined(b), ok);
    const double e = __ddiv_rn(a, b);
    if (ok) { if (__double_as_longlong(q) == __double_as_longlong(e)) ++n_ok; else ++n_bad; } else ++n_fb;
    const double v = fabs(a);
    bool ok2 = true;
    const double r = sqrt_checked(v, ok2);
    const double f = __dsqrt_rn(v);
    if (ok2) { if (__double_as_longlong(r) == __double_as_longlong(f)) ++n_ok; else ++n_bad; } else ++n_fb;
  }
  atomicAdd(&cnt[0], n_ok);
  atomicAdd(&cnt[1], n_bad);
  atomicAdd(&cnt[2], n_fb);
}

template <int V>
__global__ void adam(double* out, long long* cyc, const double2* bc, int iters) {
  double w = 0.1 + threadIdx.x * 1e-3, m = 0, v = 0, g = 1e-3;
  const double lr = 1e-2, b1 = 0.9, b2 = 0.999, c1 = 1.0 - b1, c2 = 1.0 - b2, eps = 1e-8;
  long long t0 = clock64();
  for (int e = 0; e < iters; ++e) {
    const double2 c = bc[e & 1023];
    const double y1 = rcp_refined(c.x), y2 = rcp_refined(c.y);  // per epoch, off the chain
    const double mk = __dadd_rn(__dmul_rn(b1, m), __dmul_rn(c1, g));
    const double vk = __dadd_rn(__dmul_rn(b2, v), __dmul_rn(__dmul_rn(c2, g), g));
    m = mk;
    v = vk;
    double step;
    if (V == 0) {
      step = __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mk, c.x)), __dadd_rn(__dsqrt_rn(__ddiv_rn(vk, c.y)), eps));
    } else {
      bool ok = true;
      const double mhat = div_checked(mk, c.x, y1, ok);
      const double vhat = div_checked(vk, c.y, y2, ok);
      const double den = __dadd_rn(sqrt_checked(vhat, ok), eps);
      const double num = __dmul_rn(lr, mhat);
      step = div_checked(num, den, rcp_refined(den), ok);
      if (__any_sync(0xffffffffu, !ok) && !ok)
        step = __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mk, c.x)), __dadd_rn(__dsqrt_rn(__ddiv_rn(vk, c.y)), eps));
    }
    w = __dsub_rn(w, step);
    g = __dmul_rn(w, 1e-3);
  }
  long long t1 = clock64();
  out[threadIdx.x] = w;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  unsigned long long* cnt;
  cudaMallocManaged(&cnt, 3 * sizeof(unsigned long long));
  const char* names[4] = {"exp [-200,200]", "Adam-like", "random bits", "exp [-1000,1000]"};
  for (int mode = 0; mode < 4; ++mode) {
    cnt[0] = cnt[1] = cnt[2] = 0;
    check<<<148 * 8, 256>>>(12345 + mode, 4096, mode, cnt);  // 2 x 1.24 G operations per mode
    cudaDeviceSynchronize();
    printf("%-18s verified-equal %llu  MISMATCH %llu  fallback %llu\n", names[mode], cnt[0], cnt[1], cnt[2]);
  }
  double* out; long long* cyc; double2* bc;
  cudaMalloc(&out, 1 << 16); cudaMallocManaged(&cyc, 64); cudaMallocManaged(&bc, 1024 * sizeof(double2));
  for (int i = 0; i < 1024; ++i) bc[i] = make_double2(1.0 - 0.5 / (i + 2), 1.0 - 0.9 / (i + 2));
  for (int r = 0; r < 2; ++r) adam<0><<<1, 96>>>(out, cyc, bc, 4000);
  cudaDeviceSynchronize();
  printf("Adam step, __ddiv_rn/__dsqrt_rn:  %.1f cycles\n", cyc[0] / 4000.0);
  for (int r = 0; r < 2; ++r) adam<1><<<1, 96>>>(out, cyc, bc, 4000);
  cudaDeviceSynchronize();
  printf("Adam step, verified fast path:    %.1f cycles\n", cyc[0] / 4000.0);
  return 0;
}
