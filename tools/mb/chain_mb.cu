// Microbenchmark (developer tool): cycles per link of an exact-order FP64 chain
// g = g + t[s]*a[s] over shared-memory rows, as the pipelined FP64 trainer runs it.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o chain_mb chain_mb.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int LD = 258, N = 256;

template <int V>
__global__ void chain(double* out, long long* cyc, int busy_warps) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 40 * LD; i += blockDim.x) sm[i] = 1.0 + 1e-3 * (i % 97);
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (w >= 3) {  // busy producers: independent DMUL/DADD streams
    if (w - 3 >= busy_warps) return;
    double a = l, b = 1.0000001, c = 0.5;
    for (int k = 0; k < 4000; ++k) { a = __dadd_rn(__dmul_rn(a, b), c); c = __dmul_rn(c, b); }
    out[threadIdx.x] = a + c;
    return;
  }
  const int trow = (w * 8 + l / 6) % 8, arow = 16 + l % 6;
  const double2* T = reinterpret_cast<const double2*>(sm + trow * LD);
  const double2* A = reinterpret_cast<const double2*>(sm + arow * LD);
  const bool has_a = l < 30;
  double g = 0.0;
  long long t0 = clock64();
  for (int rep = 0; rep < 8; ++rep) {
    if (V == 0) {  // as in train_fp64_pipe: 4-pair unrolled, loads at the top
#pragma unroll 4
      for (int j = 0; j < N / 2; ++j) {
        const double2 t = T[j];
        const double2 x = has_a ? A[j] : make_double2(1.0, 1.0);
        g = __dadd_rn(g, __dmul_rn(t.x, x.x));
        g = __dadd_rn(g, __dmul_rn(t.y, x.y));
      }
    } else if (V == 1) {  // software pipelined: products of the next 4 pairs formed ahead
      double p[8], q[8];
      double2 t[4], x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { t[u] = T[u]; x[u] = has_a ? A[u] : make_double2(1.0, 1.0); }
#pragma unroll
      for (int u = 0; u < 4; ++u) { p[2*u] = __dmul_rn(t[u].x, x[u].x); p[2*u+1] = __dmul_rn(t[u].y, x[u].y); }
      for (int j = 4; j < N / 2; j += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) { t[u] = T[j + u]; x[u] = has_a ? A[j + u] : make_double2(1.0, 1.0); }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          q[2*u] = __dmul_rn(t[u].x, x[u].x); q[2*u+1] = __dmul_rn(t[u].y, x[u].y);
          g = __dadd_rn(g, p[2*u]); g = __dadd_rn(g, p[2*u+1]);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) p[u] = q[u];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) g = __dadd_rn(g, p[u]);
    } else if (V == 4 || V == 5 || V == 7) {  // loads two groups ahead, products one group ahead
      const bool ha = V == 5 ? true : has_a;
      double2 ta[4], xa[4], tb[4], xb[4];
      double p[8];
      auto ld = [&](int j, double2* t, double2* x) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          t[u] = T[j + u];
          if (V == 7) { const double2 v = A[j + u]; x[u] = make_double2(ha ? v.x : 1.0, ha ? v.y : 1.0); }
          else x[u] = ha ? A[j + u] : make_double2(1.0, 1.0);
        }
      };
      auto mul = [&](const double2* t, const double2* x) {
#pragma unroll
        for (int u = 0; u < 4; ++u) { p[2*u] = __dmul_rn(t[u].x, x[u].x); p[2*u+1] = __dmul_rn(t[u].y, x[u].y); }
      };
      ld(0, ta, xa);
      ld(4, tb, xb);
      mul(ta, xa);
      for (int j = 8; j < N / 2; j += 8) {
        ld(j, ta, xa);
        double q[8];
#pragma unroll
        for (int u = 0; u < 4; ++u) { q[2*u] = __dmul_rn(tb[u].x, xb[u].x); q[2*u+1] = __dmul_rn(tb[u].y, xb[u].y); }
#pragma unroll
        for (int u = 0; u < 8; ++u) g = __dadd_rn(g, p[u]);
        ld(j + 4, tb, xb);
        mul(ta, xa);
#pragma unroll
        for (int u = 0; u < 8; ++u) g = __dadd_rn(g, q[u]);
      }
      double q[8];
#pragma unroll
      for (int u = 0; u < 4; ++u) { q[2*u] = __dmul_rn(tb[u].x, xb[u].x); q[2*u+1] = __dmul_rn(tb[u].y, xb[u].y); }
#pragma unroll
      for (int u = 0; u < 8; ++u) g = __dadd_rn(g, p[u]);
#pragma unroll
      for (int u = 0; u < 8; ++u) g = __dadd_rn(g, q[u]);
    } else if (V == 6) {  // products of a whole 16-pair block first, then its 32 DADDs
#pragma unroll 1
      for (int j = 0; j < N / 2; j += 16) {
        double p[32];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const double2 t = T[j + u];
          const double2 x = has_a ? A[j + u] : make_double2(1.0, 1.0);
          p[2*u] = __dmul_rn(t.x, x.x); p[2*u+1] = __dmul_rn(t.y, x.y);
        }
#pragma unroll
        for (int u = 0; u < 32; ++u) g = __dadd_rn(g, p[u]);
      }
    } else if (V == 8) {  // train_fp64_pipe's structure: 16-pair blocks, next block loaded before the links
      double2 a[16], b[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) a[u] = T[u];
#pragma unroll
      for (int blk = 0; blk < N / 32; ++blk) {
        double2(&cur)[16] = (blk & 1) ? b : a;
        double2(&nxt)[16] = (blk & 1) ? a : b;
        const int nb = blk + 1 < N / 32 ? blk + 1 : blk;
#pragma unroll
        for (int u = 0; u < 16; ++u) nxt[u] = T[nb * 16 + u];
#pragma unroll
        for (int u = 0; u < 16; ++u) { g = __dadd_rn(g, cur[u].x); g = __dadd_rn(g, cur[u].y); }
      }
    } else if (V == 9 || V == 10) {  // 8-pair units: loads of u + 2, a fixed-latency staging copy of u + 1
      // (x * one or x + (-0), both exact), the DADD links of u over staged registers only
      const double one = cyc[63] == 12345 ? 2.0 : 1.0, nz = cyc[63] == 12345 ? 1.0 : -0.0;
      double2 la[8], lb[8];
      double sa[16], sb[16];
      auto stage = [&](double(&s_)[16], const double2(&l)[8]) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          s_[2 * u] = V == 9 ? __dmul_rn(l[u].x, one) : __dadd_rn(l[u].x, nz);
          s_[2 * u + 1] = V == 9 ? __dmul_rn(l[u].y, one) : __dadd_rn(l[u].y, nz);
        }
      };
#pragma unroll
      for (int u = 0; u < 8; ++u) { la[u] = T[u]; lb[u] = T[8 + u]; }
      stage(sa, la);
      constexpr int NU = N / 16;
#pragma unroll
      for (int un = 0; un < NU; ++un) {
        double2(&l2)[8] = (un & 1) ? lb : la;   // loads of un + 2 reuse the buffer of un
        double2(&l1)[8] = (un & 1) ? la : lb;   // raw loads of un + 1
        double(&sc)[16] = (un & 1) ? sb : sa;
        double(&sn)[16] = (un & 1) ? sa : sb;
        if (un + 2 < NU) {
#pragma unroll
          for (int u = 0; u < 8; ++u) l2[u] = T[(un + 2) * 8 + u];
        }
        if (un + 1 < NU) stage(sn, l1);
#pragma unroll
        for (int u = 0; u < 16; ++u) g = __dadd_rn(g, sc[u]);
      }
    } else if (V == 2) {  // pure DADD chain over one row (phased kernel's product rows)
#pragma unroll 8
      for (int j = 0; j < N / 2; ++j) {
        const double2 t = T[j];
        g = __dadd_rn(g, t.x);
        g = __dadd_rn(g, t.y);
      }
    } else {  // register-only dependent DADD chain (latency floor)
      double h = 1e-3 * l;
#pragma unroll 16
      for (int j = 0; j < N; ++j) g = __dadd_rn(g, h);
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = g;
  if (l == 0) cyc[w] = t1 - t0;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 64 * 8); cyc[63] = 0;
  const int smem = 40 * LD * 8;
  auto run = [&](auto k, const char* name, int busy) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int it = 0; it < 2; ++it) k<<<1, 32 * (3 + busy), smem>>>(out, cyc, busy);
    cudaDeviceSynchronize();
    printf("%-34s busy=%d  cycles/link: %.2f %.2f %.2f\n", name, busy, cyc[0] / (8.0 * N), cyc[1] / (8.0 * N), cyc[2] / (8.0 * N));
  };
  for (int busy : {0, 4, 8}) {
    run(chain<0>, "V0 loads-at-top (pipe kernel)", busy);
    run(chain<1>, "V1 products one group ahead", busy);
    run(chain<4>, "V4 loads 2 ahead, products 1 ahead", busy);
    run(chain<5>, "V5 = V4 without predication", busy);
    run(chain<7>, "V7 = V4, unpredicated load + select", busy);
    run(chain<6>, "V6 16-pair block: products then DADDs", busy);
    run(chain<2>, "V2 DADD over product row", busy);
    run(chain<8>, "V8 pipe kernel's 16-pair blocks", busy);
    run(chain<9>, "V9 8-pair units, staged by x*one", busy);
    run(chain<10>, "V10 8-pair units, staged by x+(-0)", busy);
    run(chain<3>, "V3 register DADD chain", busy);
  }
  return 0;
}
