// Microbenchmark (developer tool): what a thread-block-cluster split of ONE LANN model would pay
// per epoch on the B200 (the FP32 CTA trainer's critical path, train_fp32.cu):
//   (a) __syncthreads() of a 128-thread CTA (today's two barriers per epoch),
//   (b) a cluster barrier (barrier.cluster.arrive.release + wait.acquire) for 2 and 4 CTAs,
//   (c) one epoch's cross-CTA exchange: every CTA writes its 72 partial gradient sums into
//       CTA 0's shared memory (st.shared::cluster), cluster barrier, CTA 0 sums and writes the
//       72 updated weights back into every CTA (st.shared::cluster), cluster barrier,
//   (d) dependent DSMEM load latency (ld.shared::cluster chain into the peer CTA).
// Cycles per iteration from clock64 on CTA 0, thread 0 (median of the clusters launched).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_mb cluster_mb.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;
constexpr int kIters = 4096, kP = 72;

__device__ __forceinline__ void cluster_sync_ra() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void cta_barrier(long long* out) {
  const long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / kIters;
}

__global__ void cluster_barrier(long long* out) {
  const long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) cluster_sync_ra();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / kIters;
}

__global__ void cluster_exchange(long long* out) {
  __shared__ float part[4][kP];  // on CTA 0: every CTA's partial sums
  __shared__ float w[kP];        // every CTA: the model's weights
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank(), n = cl.num_blocks();
  const int t = threadIdx.x;
  if (t < kP) w[t] = 1.0f;
  cl.sync();
  float* part0 = cl.map_shared_rank(&part[0][0], 0);
  float g = 0.001f * t;
  const long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) {
    if (t < kP) part0[rank * kP + t] = g + w[t];  // partials -> CTA 0
    cluster_sync_ra();
    if (rank == 0 && t < kP) {
      float s = 0.f;
      for (unsigned q = 0; q < n; ++q) s += part[q][t];
      const float nw = w[t] - 1e-6f * s;
      for (unsigned q = 0; q < n; ++q) cl.map_shared_rank(w, q)[t] = nw;  // weights -> every CTA
    }
    cluster_sync_ra();
    g = w[t < kP ? t : 0] * 1e-3f;
  }
  const long long t1 = clock64();
  if (t == 0) out[blockIdx.x] = (t1 - t0) / kIters;
}

__global__ void dsmem_latency(long long* out) {
  __shared__ unsigned ring[256];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) ring[i] = (i * 17 + 1) & 255;
  cl.sync();
  const unsigned peer = (cl.block_rank() + 1) % cl.num_blocks();
  unsigned* remote = cl.map_shared_rank(ring, peer);
  unsigned j = 0;
  const long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) j = remote[j];
  const long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / kIters + (j == 12345 ? 1 : 0);
}

template <class K>
long long run(K kern, int cluster, int grid) {
  long long* d = nullptr;
  cudaMalloc(&d, grid * sizeof(long long));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, d);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  long long best = h[0];
  for (int i = 0; i < grid; i += cluster) best = h[i] < best ? h[i] : best;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) std::printf("error: %s\n", cudaGetErrorString(e));
  return best;
}

int main() {
  std::printf("__syncthreads (128 threads): %lld cycles\n", run(cta_barrier, 1, 8));
  for (int c : {2, 4}) {
    std::printf("cluster %d: barrier %lld cycles, epoch exchange (72 partials in, 72 weights out, 2 barriers) "
                "%lld cycles, dependent DSMEM load %lld cycles\n",
                c, run(cluster_barrier, c, 8 * c), run(cluster_exchange, c, 8 * c), run(dsmem_latency, c, 8 * c));
  }
  return 0;
}
