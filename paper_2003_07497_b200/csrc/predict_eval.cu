// predict_eval.cu — K2 (batched prediction) and K3 (metrics) kernels.
//
// K2 predict: one thread per (row, model) pair, models::predict semantics
//   (models.cpp:346-363): min-max normalise (models.cpp:118-127), forward
//   (mlp.cpp:36-52), de-normalise (+exp for log targets, models.cpp:135-139),
//   clamp to >= 1e-9. The FP64 variant keeps the reference operation order
//   with no contraction, so predictions are bit-identical for identical
//   weights (exp goes through the CUDA libm, <= 1 ulp from glibc, for
//   log-target models only). The FP32 variant runs the forward pass in FP32
//   with FMA and de-normalises in FP64.
// K3 eval: one CTA per (truth, pred) set: MAPE (eval.cpp:26-32), thresholded
//   MAPE with the truth-only drop order (eval.cpp:34-57), Spearman with
//   average ranks (eval.cpp:59-90). Ranks come from O(n^2) counting in
//   parallel; every floating-point sum runs sequentially in the reference's
//   order, so the metrics are bit-identical.
#include <cmath>

#include "kernels.cuh"

namespace lann {
namespace {

constexpr int kMaxWidth = 64;

template <bool kExact>
__global__ void predict_kernel(PredictArgs a) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= a.n_rows) return;
  const int m = a.row_model[row];
  const int I = a.n_inputs[m], H1 = a.h1[m], H2 = a.h2[m];
  const double* nrm = a.norm + 18 * (int64_t)m;
  const double* x = a.rows + row * 8;
  const double* w = a.params + a.param_offset[m];
  double v;
  if (kExact) {
    double a0[8], a1[kMaxWidth], a2[kMaxWidth];
    for (int j = 0; j < I; ++j) {
      const double range = __dsub_rn(nrm[8 + j], nrm[j]);
      a0[j] = range > 0.0 ? __ddiv_rn(__dsub_rn(x[j], nrm[j]), range) : 0.0;
    }
    int off = 0;
    for (int o = 0; o < H1; ++o) {
      double z = w[I * H1 + o];
      for (int i = 0; i < I; ++i) z = __dadd_rn(z, __dmul_rn(w[o * I + i], a0[i]));
      a1[o] = z > 0.0 ? z : 0.0;
    }
    off = (I + 1) * H1;
    const double* last_in = a1;
    int nin = H1;
    if (H2 > 0) {
      for (int o = 0; o < H2; ++o) {
        double z = w[off + H1 * H2 + o];
        for (int i = 0; i < H1; ++i) z = __dadd_rn(z, __dmul_rn(w[off + o * H1 + i], a1[i]));
        a2[o] = z > 0.0 ? z : 0.0;
      }
      off += (H1 + 1) * H2;
      last_in = a2;
      nin = H2;
    }
    double z = w[off + nin];
    for (int i = 0; i < nin; ++i) z = __dadd_rn(z, __dmul_rn(w[off + i], last_in[i]));
    v = z;
  } else {
    float a0[8], a1[kMaxWidth], a2[kMaxWidth];
    for (int j = 0; j < I; ++j) {
      const double range = nrm[8 + j] - nrm[j];
      a0[j] = range > 0.0 ? (float)((x[j] - nrm[j]) / range) : 0.f;
    }
    int off = 0;
    for (int o = 0; o < H1; ++o) {
      float z = (float)w[I * H1 + o];
      for (int i = 0; i < I; ++i) z = fmaf((float)w[o * I + i], a0[i], z);
      a1[o] = fmaxf(z, 0.f);
    }
    off = (I + 1) * H1;
    const float* last_in = a1;
    int nin = H1;
    if (H2 > 0) {
      for (int o = 0; o < H2; ++o) {
        float z = (float)w[off + H1 * H2 + o];
        for (int i = 0; i < H1; ++i) z = fmaf((float)w[off + o * H1 + i], a1[i], z);
        a2[o] = fmaxf(z, 0.f);
      }
      off += (H1 + 1) * H2;
      last_in = a2;
      nin = H2;
    }
    float z = (float)w[off + nin];
    for (int i = 0; i < nin; ++i) z = fmaf((float)w[off + i], last_in[i], z);
    v = (double)z;
  }
  const double trange = __dsub_rn(nrm[17], nrm[16]);
  double t = trange > 0.0 ? __dadd_rn(nrm[16], __dmul_rn(v, trange)) : nrm[16];
  if (a.log_target[m]) t = exp(t);
  a.out[row] = t < 1e-9 ? 1e-9 : t;  // std::max(value, 1e-9)
}

// K3: one CTA per set; n <= blockDim * kPerThread handled through shared memory.
__global__ void __launch_bounds__(256) eval_kernel(EvalArgs a) {
  extern __shared__ double sm[];
  const int set = blockIdx.x;
  const int n = a.len[set];
  const double* t = a.truth + a.offset[set];
  const double* p = a.pred + a.offset[set];
  double* st = sm;            // truth
  double* sp = st + n;        // pred
  double* rt = sp + n;        // truth ranks
  double* rp = rt + n;        // pred ranks
  int* pos = (int*)(rp + n);  // sorted position of each sample by (truth, index)
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    st[i] = t[i];
    sp[i] = p[i];
    if (!(t[i] > 0.0)) atomicOr(&bad, 1);  // eval.cpp:16-22 check_pair
  }
  __syncthreads();
  if (n < 2 || bad) {
    if (threadIdx.x == 0) {
      a.status[set] = 4;  // LANN_DOMAIN_ERROR
      a.mape[set] = a.mape_thr[set] = a.rho[set] = 0.0;
      a.n_kept[set] = 0;
    }
    return;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double ti = st[i], pi = sp[i];
    int lt = 0, et = 0, lp = 0, ep = 0, before = 0;
    for (int j = 0; j < n; ++j) {
      const double tj = st[j], pj = sp[j];
      lt += tj < ti;
      et += tj == ti;
      lp += pj < pi;
      ep += pj == pi;
      before += (tj < ti) || (tj == ti && j < i);
    }
    // average 1-based rank of the tie group at positions [less, less+eq-1] (eval.cpp:59-75)
    rt[i] = ((double)lt + (double)(lt + et - 1)) / 2.0 + 1.0;
    rp[i] = ((double)lp + (double)(lp + ep - 1)) / 2.0 + 1.0;
    pos[before] = i;
  }
  __syncthreads();
  const int n_drop = (int)floor(__dadd_rn(__dmul_rn(a.drop_fraction, (double)n), 1e-12));
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i)
      acc = __dadd_rn(acc, __ddiv_rn(fabs(__dsub_rn(st[i], sp[i])), st[i]));
    a.mape[set] = __ddiv_rn(__dmul_rn(100.0, acc), (double)n);
  } else if (threadIdx.x == 32) {
    if (n_drop >= n) {
      a.status[set] = 4;
    } else {
      double acc = 0.0;
      for (int k = n_drop; k < n; ++k) {
        const int j = pos[k];
        acc = __dadd_rn(acc, __ddiv_rn(fabs(__dsub_rn(st[j], sp[j])), st[j]));
      }
      a.mape_thr[set] = __ddiv_rn(__dmul_rn(100.0, acc), (double)(n - n_drop));
      a.n_kept[set] = n - n_drop;
      a.status[set] = 0;
    }
  } else if (threadIdx.x == 64) {
    const double nn = (double)n;
    double d2 = 0.0;
    for (int i = 0; i < n; ++i) {
      const double d = __dsub_rn(rt[i], rp[i]);
      d2 = __dadd_rn(d2, __dmul_rn(d, d));
    }
    a.rho[set] = __dsub_rn(1.0, __ddiv_rn(__dmul_rn(6.0, d2), __dmul_rn(nn, __dsub_rn(__dmul_rn(nn, nn), 1.0))));
  }
}

// K3 for sets too large for one CTA's shared memory (the reference handles any size,
// eval.cpp:26-108): ranks and sorted positions counted by a grid over (sample block, set), the
// other samples streamed through shared memory in tiles; the sequential sums then run in a
// second kernel from global memory, in the same order as eval_kernel.
constexpr int kRankTile = 1024;

__global__ void __launch_bounds__(256) eval_rank_global(EvalArgs a, double* rt_g, double* rp_g, int* pos_g) {
  __shared__ double tt[kRankTile], tp[kRankTile];
  const int set = blockIdx.y;
  const int n = a.len[set];
  const int64_t o = a.offset[set];
  const double* t = a.truth + o;
  const double* p = a.pred + o;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if ((int)(blockIdx.x * blockDim.x) >= n) return;  // uniform per CTA
  const double ti = i < n ? t[i] : 0.0, pi = i < n ? p[i] : 0.0;
  int lt = 0, et = 0, lp = 0, ep = 0, before = 0;
  for (int j0 = 0; j0 < n; j0 += kRankTile) {
    const int m = min(kRankTile, n - j0);
    __syncthreads();
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
      tt[j] = t[j0 + j];
      tp[j] = p[j0 + j];
    }
    __syncthreads();
    for (int j = 0; j < m; ++j) {
      const double tj = tt[j], pj = tp[j];
      lt += tj < ti;
      et += tj == ti;
      lp += pj < pi;
      ep += pj == pi;
      before += (tj < ti) || (tj == ti && j0 + j < i);
    }
  }
  if (i < n) {
    rt_g[o + i] = ((double)lt + (double)(lt + et - 1)) / 2.0 + 1.0;
    rp_g[o + i] = ((double)lp + (double)(lp + ep - 1)) / 2.0 + 1.0;
    pos_g[o + before] = i;
  }
}

__global__ void __launch_bounds__(96) eval_sums_global(EvalArgs a, const double* rt_g, const double* rp_g,
                                                       const int* pos_g) {
  const int set = blockIdx.x;
  const int n = a.len[set];
  const int64_t o = a.offset[set];
  const double* st = a.truth + o;
  const double* sp = a.pred + o;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (!(st[i] > 0.0)) atomicOr(&bad, 1);  // eval.cpp:16-22 check_pair
  __syncthreads();
  if (n < 2 || bad) {
    if (threadIdx.x == 0) {
      a.status[set] = 4;  // LANN_DOMAIN_ERROR
      a.mape[set] = a.mape_thr[set] = a.rho[set] = 0.0;
      a.n_kept[set] = 0;
    }
    return;
  }
  const int n_drop = (int)floor(__dadd_rn(__dmul_rn(a.drop_fraction, (double)n), 1e-12));
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, __ddiv_rn(fabs(__dsub_rn(st[i], sp[i])), st[i]));
    a.mape[set] = __ddiv_rn(__dmul_rn(100.0, acc), (double)n);
  } else if (threadIdx.x == 32) {
    if (n_drop >= n) {
      a.status[set] = 4;
    } else {
      double acc = 0.0;
      for (int k = n_drop; k < n; ++k) {
        const int j = pos_g[o + k];
        acc = __dadd_rn(acc, __ddiv_rn(fabs(__dsub_rn(st[j], sp[j])), st[j]));
      }
      a.mape_thr[set] = __ddiv_rn(__dmul_rn(100.0, acc), (double)(n - n_drop));
      a.n_kept[set] = n - n_drop;
      a.status[set] = 0;
    }
  } else if (threadIdx.x == 64) {
    const double nn = (double)n;
    double d2 = 0.0;
    for (int i = 0; i < n; ++i) {
      const double d = __dsub_rn(rt_g[o + i], rp_g[o + i]);
      d2 = __dadd_rn(d2, __dmul_rn(d, d));
    }
    a.rho[set] = __dsub_rn(1.0, __ddiv_rn(__dmul_rn(6.0, d2), __dmul_rn(nn, __dsub_rn(__dmul_rn(nn, nn), 1.0))));
  }
}

}  // namespace

void launch_predict_fp64(const PredictArgs& a, cudaStream_t s) {
  if (a.n_rows <= 0) return;
  predict_kernel<true><<<(unsigned)((a.n_rows + 127) / 128), 128, 0, s>>>(a);
}

void launch_predict_fp32(const PredictArgs& a, cudaStream_t s) {
  if (a.n_rows <= 0) return;
  predict_kernel<false><<<(unsigned)((a.n_rows + 127) / 128), 128, 0, s>>>(a);
}

// max_len bounds the shared-memory footprint: 4 doubles + 1 int per sample. Sets that do not
// fit one CTA's shared memory take the two-kernel global-memory path (scratch: rank and position
// arrays over the whole [0, total) index range, stream-ordered allocation).
int eval_launch_count(int max_len, int max_smem) {
  return size_t(max_len) * 36 + 16 <= size_t(max_smem) ? 1 : 2;
}

void launch_eval(const EvalArgs& a, int max_len, int max_smem, int64_t total, cudaStream_t s) {
  if (a.n_sets <= 0) return;
  if (eval_launch_count(max_len, max_smem) == 1) {
    const int bytes = max_len * (4 * 8 + 4) + 16;
    cudaFuncSetAttribute(eval_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    eval_kernel<<<a.n_sets, 256, bytes, s>>>(a);
    return;
  }
  void* scratch = nullptr;
  const size_t nt = size_t(total);
  if (cudaMallocAsync(&scratch, nt * (8 + 8 + 4) + 16, s) != cudaSuccess) return;
  double* rt = static_cast<double*>(scratch);
  double* rp = rt + nt;
  int* pos = reinterpret_cast<int*>(rp + nt);
  const dim3 grid((unsigned)((max_len + 255) / 256), (unsigned)a.n_sets);
  eval_rank_global<<<grid, 256, 0, s>>>(a, rt, rp, pos);
  eval_sums_global<<<a.n_sets, 96, 0, s>>>(a, rt, rp, pos);
  cudaFreeAsync(scratch, s);
}

}  // namespace lann
