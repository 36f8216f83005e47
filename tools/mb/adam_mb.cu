// Microbenchmark (developer tool): latency of one exact-order FP64 Adam step
// (mlp.cpp:142-154 with __ddiv_rn / __dsqrt_rn), iterations made dependent through g.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o adam_mb adam_mb.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__global__ void adam(double* out, long long* cyc, const double2* bc, int iters) {
  double w = 0.1 + threadIdx.x * 1e-3, m = 0, v = 0, g = 1e-3;
  const double lr = 1e-2, b1 = 0.9, b2 = 0.999, c1 = 1.0 - b1, c2 = 1.0 - b2, eps = 1e-8;
  long long t0 = clock64();
  for (int e = 0; e < iters; ++e) {
    const double2 c = bc[e & 1023];
    const double mk = __dadd_rn(__dmul_rn(b1, m), __dmul_rn(c1, g));
    const double vk = __dadd_rn(__dmul_rn(b2, v), __dmul_rn(__dmul_rn(c2, g), g));
    m = mk;
    v = vk;
    if (V == 0) {
      const double mhat = __ddiv_rn(mk, c.x);
      const double vhat = __ddiv_rn(vk, c.y);
      w = __dsub_rn(w, __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps)));
    } else if (V == 1) {  // sqrt only on the path (timing split)
      w = __dsub_rn(w, __dsqrt_rn(vk));
    } else if (V == 2) {  // one division only
      w = __dsub_rn(w, __ddiv_rn(mk, vk + 1.0));
    } else {  // no div/sqrt
      w = __dsub_rn(w, __dmul_rn(mk, vk));
    }
    g = __dmul_rn(w, 1e-3);
  }
  long long t1 = clock64();
  out[threadIdx.x] = w;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* out; long long* cyc; double2* bc;
  cudaMalloc(&out, 1 << 16); cudaMallocManaged(&cyc, 64); cudaMallocManaged(&bc, 1024 * sizeof(double2));
  for (int i = 0; i < 1024; ++i) bc[i] = make_double2(1.0 - 0.5 / (i + 2), 1.0 - 0.9 / (i + 2));
  const int iters = 4000;
  auto run = [&](auto k, const char* name) {
    for (int r = 0; r < 2; ++r) k<<<1, 96>>>(out, cyc, bc, iters);
    cudaDeviceSynchronize();
    printf("%-28s %.1f cycles per dependent step\n", name, cyc[0] / double(iters));
  };
  run(adam<0>, "full Adam step");
  run(adam<1>, "m,v + sqrt");
  run(adam<2>, "m,v + one division");
  run(adam<3>, "m,v only");
  return 0;
}
