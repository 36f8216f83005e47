// measure.cu — real runtime measurement of GPU-class kernel variants on the B200 (SURVEY.md
// 8(f) row 3: "the step before the path"). The reference measures its CPU kernels with
// datagen::measure (datagen.cpp:118-160: warm-ups, then the median of `reps` timed runs) or an
// external black box (external.cpp); the paper's GPU variants (section IV-A) are exactly such
// black boxes without n_thd. This file provides them for the B200: every variant runs the
// reference kernel's mathematics (reference.cpp:14-66) on device-resident operands and is timed
// with CUDA events on the engine stream (median of reps after warm-ups).
//
//   mm   (A m x n, density d1) x (B n x k, density d2) -> C m x k
//        gemm_tiled   64x64 shared-memory tiled FP32 GEMM, 4x4 outputs per thread
//        cublas_sgemm cuBLAS SGEMM (library black box, loaded with dlopen)
//        spmm_csr     CSR(A) x dense B, one warp per row of A
//   mv   (A m x n, density d) x (x n)
//        gemv_dense   one warp per row, coalesced row reads
//        spmv_csr     CSR(A) x x, one warp per row
//   mc   direct r x r convolution (valid), A m x n density d
//        conv_direct  one thread per output, filter in shared memory
//   mp   s x s max pooling with stride s (partial windows start from 0, reference.cpp:38-52)
//        maxpool      one thread per output
//   blur 3-point horizontal then vertical mean on an n x n image (reference.cpp:54-66)
//        blur_sched   the GPU-style schedule (s1, s2, s3): CTA of s2 x min(s3, 1024/s2) threads,
//                     s1 outputs per thread along x, a tile of s2*s1 x s3 outputs per CTA
//
// Operands come from a counter hash of (seed, operand, index): value in [0, 1), kept non-zero
// with probability d (so nnz ~ d * rows * cols; the reference's exact-count sampler only changes
// which positions are zero). tests/test_gpu_measure.py rebuilds them in numpy and checks every
// variant's output checksum against the reference mathematics.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include "../../include/lann_engine.h"
#include "kernels.cuh"

namespace lann {
namespace {

__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
// operand element: value (top 24 bits -> [0,1)) and keep flag (an independent hash < d * 2^53)
__host__ __device__ inline float gen_value(uint64_t seed, uint32_t op, uint64_t i) {
  return float(mix64(seed ^ (uint64_t(op) << 56) ^ (i * 2 + 0)) >> 40) * (1.0f / 16777216.0f);
}
__host__ __device__ inline bool gen_keep(uint64_t seed, uint32_t op, uint64_t i, double d) {
  if (d >= 1.0) return true;
  return double(mix64(seed ^ (uint64_t(op) << 56) ^ (i * 2 + 1)) >> 11) * 0x1.0p-53 < d;
}

__global__ void fill_kernel(float* out, uint64_t n, uint64_t seed, uint32_t op, double d) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = gen_keep(seed, op, i, d) ? gen_value(seed, op, i) : 0.f;
}

__global__ void row_nnz_kernel(const float* a, int rows, int cols, int* cnt) {
  const int r = blockIdx.x;
  int c = 0;
  for (int j = threadIdx.x; j < cols; j += blockDim.x) c += a[size_t(r) * cols + j] != 0.f;
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ int part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += part[w];
    cnt[r] = t;
  }
}

__global__ void csr_fill_kernel(const float* a, int rows, int cols, const int* rowptr, int* colidx, float* vals) {
  const int r = blockIdx.x;
  if (threadIdx.x != 0) return;
  int o = rowptr[r];
  for (int j = 0; j < cols; ++j) {
    const float v = a[size_t(r) * cols + j];
    if (v != 0.f) {
      colidx[o] = j;
      vals[o] = v;
      ++o;
    }
  }
}

// ---- variants ----------------------------------------------------------------------------------
constexpr int GT = 64;  // GEMM tile
__global__ void __launch_bounds__(256) gemm_tiled_kernel(const float* A, const float* B, float* C, int M, int K,
                                                         int N) {
  // C[M x N] = A[M x K] B[K x N] (row-major); 16x16 threads, 4x4 outputs each
  __shared__ float As[16][GT + 4];
  __shared__ float Bs[16][GT + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int row0 = blockIdx.y * GT, col0 = blockIdx.x * GT;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * GT; e += 256) {
      const int r = e / 16, kk = e % 16;  // A tile: GT rows x 16 k
      const int gr = row0 + r, gk = k0 + kk;
      As[kk][r] = (gr < M && gk < K) ? A[size_t(gr) * K + gk] : 0.f;
      const int kb = e / GT, c = e % GT;  // B tile: 16 k x GT cols
      const int gkb = k0 + kb, gc = col0 + c;
      Bs[kb][c] = (gkb < K && gc < N) ? B[size_t(gkb) * N + gc] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = row0 + ty * 4 + i, c = col0 + tx * 4 + j;
      if (r < M && c < N) C[size_t(r) * N + c] = acc[i][j];
    }
}

__global__ void spmm_csr_kernel(const int* rowptr, const int* colidx, const float* vals, const float* B, float* C,
                                int M, int N) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= M) return;
  const int p0 = rowptr[warp], p1 = rowptr[warp + 1];
  for (int c = lane; c < N; c += 32) {
    float acc = 0.f;
    for (int p = p0; p < p1; ++p) acc = fmaf(vals[p], B[size_t(colidx[p]) * N + c], acc);
    C[size_t(warp) * N + c] = acc;
  }
}

__global__ void gemv_kernel(const float* A, const float* x, float* y, int M, int N) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= M) return;
  const float* row = A + size_t(warp) * N;
  float acc = 0.f;
  for (int j = lane; j < N; j += 32) acc = fmaf(row[j], x[j], acc);
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) y[warp] = acc;
}

__global__ void spmv_csr_kernel(const int* rowptr, const int* colidx, const float* vals, const float* x, float* y,
                                int M) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= M) return;
  float acc = 0.f;
  for (int p = rowptr[warp] + lane; p < rowptr[warp + 1]; p += 32) acc = fmaf(vals[p], x[colidx[p]], acc);
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) y[warp] = acc;
}

__global__ void conv_kernel(const float* A, const float* F, float* O, int M, int N, int r) {
  __shared__ float f[64];
  if (threadIdx.x < r * r) f[threadIdx.x] = F[threadIdx.x];
  __syncthreads();
  const int om = M - r + 1, on = N - r + 1;
  const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
  if (j >= on || i >= om) return;
  float acc = 0.f;
  for (int u = 0; u < r; ++u)
    for (int v = 0; v < r; ++v) acc = fmaf(A[size_t(i + u) * N + j + v], f[u * r + v], acc);
  O[size_t(i) * on + j] = acc;
}

__global__ void pool_kernel(const float* A, float* O, int M, int N, int s) {
  const int om = (M + s - 1) / s, on = (N + s - 1) / s;
  const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
  if (j >= on || i >= om) return;
  const int r0 = i * s, r1 = min(M, r0 + s), c0 = j * s, c1 = min(N, c0 + s);
  const bool partial = (r1 - r0) * (c1 - c0) < s * s;
  float best = partial ? 0.f : A[size_t(r0) * N + c0];
  for (int p = r0; p < r1; ++p)
    for (int q = c0; q < c1; ++q) best = fmaxf(best, A[size_t(p) * N + q]);
  O[size_t(i) * on + j] = best;
}

// blur, pass 1: bx[y][x] = (img[y][x] + img[y][x+1] + img[y][x+2]) / 3, x < n-2; pass 2 vertical.
// CTA (s2, ty) threads; thread handles s1 consecutive x outputs and rows y, y+ty, ... of its tile.
__global__ void blur_h_kernel(const float* img, float* bx, int n, int s1, int s3) {
  const int w = n - 2;
  const int x0 = (blockIdx.x * blockDim.x + threadIdx.x) * s1;
  for (int yy = threadIdx.y; yy < s3; yy += blockDim.y) {
    const int y = blockIdx.y * s3 + yy;
    if (y >= n) break;
    const float* row = img + size_t(y) * n;
    for (int k = 0; k < s1 && x0 + k < w; ++k)
      bx[size_t(y) * w + x0 + k] = (row[x0 + k] + row[x0 + k + 1] + row[x0 + k + 2]) / 3.f;
  }
}
__global__ void blur_v_kernel(const float* bx, float* out, int n, int s1, int s3) {
  const int w = n - 2;
  const int x0 = (blockIdx.x * blockDim.x + threadIdx.x) * s1;
  for (int yy = threadIdx.y; yy < s3; yy += blockDim.y) {
    const int y = blockIdx.y * s3 + yy;
    if (y >= w) break;
    for (int k = 0; k < s1 && x0 + k < w; ++k)
      out[size_t(y) * w + x0 + k] =
          (bx[size_t(y) * w + x0 + k] + bx[size_t(y + 1) * w + x0 + k] + bx[size_t(y + 2) * w + x0 + k]) / 3.f;
  }
}

__global__ void checksum_kernel(const float* v, uint64_t n, double* out) {
  double acc = 0.0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    acc += double(v[i]);
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

// ---- cuBLAS, loaded at first use (a library black box; the engine does not link it) ----------
struct Cublas {
  void* lib = nullptr;
  int (*create)(void**) = nullptr;
  int (*set_stream)(void*, cudaStream_t) = nullptr;
  int (*sgemm)(void*, int, int, int, int, int, const float*, const float*, int, const float*, int, const float*,
               float*, int) = nullptr;
  std::mutex mu;
  std::map<int, void*> handles;  // one cuBLAS handle per device (a handle is bound to its device)
  static Cublas& get() {
    static Cublas c;
    std::lock_guard<std::mutex> lk(c.mu);
    if (!c.lib) {
      c.lib = dlopen("libcublas.so.12", RTLD_NOW | RTLD_LOCAL);
      if (!c.lib) c.lib = dlopen("/usr/local/cuda/lib64/libcublas.so.12", RTLD_NOW | RTLD_LOCAL);
      if (c.lib) {
        c.create = reinterpret_cast<decltype(c.create)>(dlsym(c.lib, "cublasCreate_v2"));
        c.set_stream = reinterpret_cast<decltype(c.set_stream)>(dlsym(c.lib, "cublasSetStream_v2"));
        c.sgemm = reinterpret_cast<decltype(c.sgemm)>(dlsym(c.lib, "cublasSgemm_v2"));
      }
    }
    return c;
  }
  void* handle_for_current_device() {
    std::lock_guard<std::mutex> lk(mu);
    if (!create || !set_stream || !sgemm) return nullptr;
    int dev = 0;
    cudaGetDevice(&dev);
    auto it = handles.find(dev);
    if (it != handles.end()) return it->second;
    void* h = nullptr;
    if (create(&h) != 0) return nullptr;
    handles[dev] = h;
    return h;
  }
};

struct Variant {
  int kind;
  const char* name;
};
const Variant kVariants[] = {
    {LANN_MM, "gemm_tiled"}, {LANN_MM, "cublas_sgemm"}, {LANN_MM, "spmm_csr"}, {LANN_MV, "gemv_dense"},
    {LANN_MV, "spmv_csr"},   {LANN_MC, "conv_direct"},  {LANN_MP, "maxpool"},  {LANN_BLUR, "blur_sched"},
};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t b) {
    if (b <= bytes) return;
    if (p) cudaFree(p);
    bytes = std::max(b, bytes * 2);
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      p = nullptr;
      bytes = 0;
    }
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

unsigned grid_for(uint64_t n) { return unsigned(std::min<uint64_t>((n + 255) / 256, 148ull * 16)); }

}  // namespace

int measure_variant_count(int kind) {
  int n = 0;
  for (const auto& v : kVariants) n += v.kind == kind;
  return n;
}

const char* measure_variant_name(int kind, int idx) {
  for (const auto& v : kVariants)
    if (v.kind == kind && idx-- == 0) return v.name;
  return nullptr;
}

int measure_instances(int kind, const char* variant, int n, const double* feats, int warmups, int reps,
                      uint64_t seed, double* runtime_s, double* checksum, cudaStream_t s, std::string& err) {
  bool known = false;
  for (const auto& v : kVariants) known |= v.kind == kind && variant && std::strcmp(v.name, variant) == 0;
  if (!known) {
    err = std::string("no B200 variant '") + (variant ? variant : "") + "' for this kernel kind";
    return LANN_PARAM_ERROR;
  }
  if (reps < 1 || warmups < 0) {
    err = "timing policy needs reps >= 1 and warmups >= 0";
    return LANN_PARAM_ERROR;
  }
  const std::string v = variant;
  DevBuf A, B, C, S, rowptr, colidx, vals, csum;  // per call: no state shared between engines / devices
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int status = LANN_OK;
  for (int i = 0; i < n && status == LANN_OK; ++i) {
    const double* f = feats + size_t(i) * LANN_ROW;
    const uint64_t iseed = mix64(seed ^ (0x3C6EF372FE94F82BULL * uint64_t(i + 1)));
    auto fill = [&](DevBuf& b, uint64_t count, uint32_t op, double d) {
      b.ensure(count * sizeof(float));
      fill_kernel<<<grid_for(count), 256, 0, s>>>(static_cast<float*>(b.p), count, iseed, op, d);
    };
    auto build_csr = [&](int rows, int cols) {
      rowptr.ensure(size_t(rows + 1) * sizeof(int));
      int* rp = static_cast<int*>(rowptr.p);
      cudaMemsetAsync(rp, 0, size_t(rows + 1) * sizeof(int), s);
      row_nnz_kernel<<<rows, 256, 0, s>>>(static_cast<float*>(A.p), rows, cols, rp);
      size_t tmp = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, tmp, rp, rp, rows + 1, s);
      S.ensure(tmp);
      cub::DeviceScan::ExclusiveSum(S.p, tmp, rp, rp, rows + 1, s);
      int nnz = 0;
      cudaMemcpyAsync(&nnz, rp + rows, sizeof(int), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      colidx.ensure(size_t(std::max(nnz, 1)) * sizeof(int));
      vals.ensure(size_t(std::max(nnz, 1)) * sizeof(float));
      csr_fill_kernel<<<rows, 32, 0, s>>>(static_cast<float*>(A.p), rows, cols, rp, static_cast<int*>(colidx.p),
                                          static_cast<float*>(vals.p));
    };
    uint64_t out_n = 0;
    std::function<void()> run;
    if (kind == LANN_MM) {
      const int m = int(f[0]), nn = int(f[1]), k = int(f[2]);
      const double d1 = f[3], d2 = f[4];
      if (m < 1 || nn < 1 || k < 1 || !(d1 > 0 && d1 <= 1) || !(d2 > 0 && d2 <= 1)) status = LANN_PARAM_ERROR;
      fill(A, uint64_t(m) * nn, 0, d1);
      fill(B, uint64_t(nn) * k, 1, d2);
      C.ensure(size_t(m) * k * sizeof(float));
      out_n = uint64_t(m) * k;
      float *a = static_cast<float*>(A.p), *b = static_cast<float*>(B.p), *c = static_cast<float*>(C.p);
      if (v == "gemm_tiled") {
        run = [=] { gemm_tiled_kernel<<<dim3((k + GT - 1) / GT, (m + GT - 1) / GT), 256, 0, s>>>(a, b, c, m, nn, k); };
      } else if (v == "cublas_sgemm") {
        Cublas& cb = Cublas::get();
        void* handle = cb.handle_for_current_device();
        if (!handle) {
          err = "cuBLAS could not be loaded";
          status = LANN_PARAM_ERROR;
          break;
        }
        cb.set_stream(handle, s);
        run = [=, &cb] {
          const float one = 1.f, zero = 0.f;
          // row-major C = A B  ==  column-major C^T = B^T A^T
          cb.sgemm(handle, 0, 0, k, m, nn, &one, b, k, a, nn, &zero, c, k);
        };
      } else {
        build_csr(m, nn);
        const int *rp = static_cast<int*>(rowptr.p), *ci = static_cast<int*>(colidx.p);
        const float* va = static_cast<float*>(vals.p);
        run = [=] { spmm_csr_kernel<<<(m * 32 + 255) / 256, 256, 0, s>>>(rp, ci, va, b, c, m, k); };
      }
    } else if (kind == LANN_MV) {
      const int m = int(f[0]), nn = int(f[1]);
      const double d = f[2];
      if (m < 1 || nn < 1 || !(d > 0 && d <= 1)) status = LANN_PARAM_ERROR;
      fill(A, uint64_t(m) * nn, 0, d);
      fill(B, uint64_t(nn), 1, 1.0);
      C.ensure(size_t(m) * sizeof(float));
      out_n = uint64_t(m);
      float *a = static_cast<float*>(A.p), *x = static_cast<float*>(B.p), *y = static_cast<float*>(C.p);
      if (v == "gemv_dense") {
        run = [=] { gemv_kernel<<<(m * 32 + 255) / 256, 256, 0, s>>>(a, x, y, m, nn); };
      } else {
        build_csr(m, nn);
        const int *rp = static_cast<int*>(rowptr.p), *ci = static_cast<int*>(colidx.p);
        const float* va = static_cast<float*>(vals.p);
        run = [=] { spmv_csr_kernel<<<(m * 32 + 255) / 256, 256, 0, s>>>(rp, ci, va, x, y, m); };
      }
    } else if (kind == LANN_MC) {
      const int m = int(f[0]), nn = int(f[1]), r = int(f[2]);
      const double d = f[3];
      if (r < 1 || r > 8 || m < r || nn < r || !(d > 0 && d <= 1)) status = LANN_PARAM_ERROR;
      fill(A, uint64_t(m) * nn, 0, d);
      fill(B, uint64_t(r) * r, 1, 1.0);
      const int om = m - r + 1, on = nn - r + 1;
      C.ensure(size_t(om) * on * sizeof(float));
      out_n = uint64_t(om) * on;
      float *a = static_cast<float*>(A.p), *fl = static_cast<float*>(B.p), *o = static_cast<float*>(C.p);
      run = [=] { conv_kernel<<<dim3((on + 127) / 128, om), 128, 0, s>>>(a, fl, o, m, nn, r); };
    } else if (kind == LANN_MP) {
      const int m = int(f[0]), nn = int(f[1]), st = int(f[3]);
      const double d = f[4];
      if (m < 1 || nn < 1 || st < 1 || !(d > 0 && d <= 1)) status = LANN_PARAM_ERROR;
      fill(A, uint64_t(m) * nn, 0, d);
      const int om = (m + st - 1) / st, on = (nn + st - 1) / st;
      C.ensure(size_t(om) * on * sizeof(float));
      out_n = uint64_t(om) * on;
      float *a = static_cast<float*>(A.p), *o = static_cast<float*>(C.p);
      run = [=] { pool_kernel<<<dim3((on + 127) / 128, om), 128, 0, s>>>(a, o, m, nn, st); };
    } else {  // blur
      const int nn = int(f[0]), s1 = int(f[1]), s2 = int(f[2]), s3 = int(f[3]);
      if (nn < 3 || s1 < 1 || s2 < 1 || s3 < 1 || s2 > 1024) status = LANN_PARAM_ERROR;
      fill(A, uint64_t(nn) * nn, 0, 1.0);
      B.ensure(size_t(nn) * (nn - 2) * sizeof(float));
      C.ensure(size_t(nn - 2) * (nn - 2) * sizeof(float));
      out_n = uint64_t(nn - 2) * (nn - 2);
      float *img = static_cast<float*>(A.p), *bx = static_cast<float*>(B.p), *o = static_cast<float*>(C.p);
      const int ty = std::max(1, std::min(s3, 1024 / s2));
      const dim3 blk(s2, ty);
      const int tile_w = s2 * s1;
      const dim3 gh((nn - 2 + tile_w - 1) / tile_w, (nn + s3 - 1) / s3);
      const dim3 gv((nn - 2 + tile_w - 1) / tile_w, (nn - 2 + s3 - 1) / s3);
      run = [=] {
        blur_h_kernel<<<gh, blk, 0, s>>>(img, bx, nn, s1, s3);
        blur_v_kernel<<<gv, blk, 0, s>>>(bx, o, nn, s1, s3);
      };
    }
    if (status != LANN_OK) {
      if (err.empty()) err = "invalid instance parameters for measurement";
      break;
    }
    if (cudaGetLastError() != cudaSuccess || !A.p || !C.p) {
      err = "device allocation or operand generation failed";
      status = LANN_CUDA_ERROR;
      break;
    }
    for (int w = 0; w < warmups; ++w) run();
    std::vector<float> t(static_cast<std::size_t>(reps), 0.f);
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(e0, s);
      run();
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&t[size_t(r)], e0, e1);
    }
    if (cudaGetLastError() != cudaSuccess) {
      err = "variant launch failed";
      status = LANN_CUDA_ERROR;
      break;
    }
    std::sort(t.begin(), t.end());  // datagen.cpp median_of
    const double med = reps % 2 ? t[size_t(reps / 2)] : 0.5 * (double(t[size_t(reps / 2 - 1)]) + t[size_t(reps / 2)]);
    runtime_s[i] = med * 1e-3;
    if (checksum) {
      csum.ensure(sizeof(double));
      cudaMemsetAsync(csum.p, 0, sizeof(double), s);
      checksum_kernel<<<grid_for(out_n), 256, 0, s>>>(static_cast<float*>(C.p), out_n, static_cast<double*>(csum.p));
      cudaMemcpyAsync(&checksum[i], csum.p, sizeof(double), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return status;
}

}  // namespace lann
