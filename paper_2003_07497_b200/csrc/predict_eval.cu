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
#include <algorithm>
#include <cmath>
#include <type_traits>

#include "exact_fp64.cuh"
#include "kernels.cuh"

namespace lann {
namespace {

constexpr int kMaxWidth = 64;

// Generic shapes (any widths up to 64, one or two hidden layers): local-memory activations.
// Out of line, the row passed by value: the compiled-shape path keeps its row in registers.
struct Row8 {
  double v[8];
};
template <bool kExact>
__device__ __noinline__ double forward_generic(const Row8 xr, const double* nrm, const double* w, int I, int H1,
                                               int H2) {
  const double* x = xr.v;
  if (kExact) {
    double a0[8], a1[kMaxWidth], a2[kMaxWidth];
    for (int j = 0; j < I; ++j) {
      const double range = __dsub_rn(nrm[8 + j], nrm[j]);
      a0[j] = range > 0.0 ? __ddiv_rn(__dsub_rn(x[j], nrm[j]), range) : 0.0;
    }
    for (int o = 0; o < H1; ++o) {
      double z = w[I * H1 + o];
      for (int i = 0; i < I; ++i) z = __dadd_rn(z, __dmul_rn(w[o * I + i], a0[i]));
      a1[o] = gate(z, z);
    }
    int off = (I + 1) * H1;
    const double* last_in = a1;
    int nin = H1;
    if (H2 > 0) {
      for (int o = 0; o < H2; ++o) {
        double z = w[off + H1 * H2 + o];
        for (int i = 0; i < H1; ++i) z = __dadd_rn(z, __dmul_rn(w[off + o * H1 + i], a1[i]));
        a2[o] = gate(z, z);
      }
      off += (H1 + 1) * H2;
      last_in = a2;
      nin = H2;
    }
    double z = w[off + nin];
    for (int i = 0; i < nin; ++i) z = __dadd_rn(z, __dmul_rn(w[off + i], last_in[i]));
    return z;
  } else {
    float a0[8], a1[kMaxWidth], a2[kMaxWidth];
    for (int j = 0; j < I; ++j) {
      const double range = nrm[8 + j] - nrm[j];
      a0[j] = range > 0.0 ? (float)((x[j] - nrm[j]) / range) : 0.f;
    }
    for (int o = 0; o < H1; ++o) {
      float z = (float)w[I * H1 + o];
      for (int i = 0; i < I; ++i) z = fmaf((float)w[o * I + i], a0[i], z);
      a1[o] = fmaxf(z, 0.f);
    }
    int off = (I + 1) * H1;
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
    return (double)z;
  }
}

// Compiled shapes (the LANN nets: I-8-1 and I-5-5-1): fully unrolled, activations in registers,
// R rows of the SAME model per call so every weight is loaded once for R rows (the predictor is
// load-instruction bound otherwise: ~100 weight loads per row).
// FP64 exact: the reference order (mlp.cpp:36-52) after NormStats::normalize's division
// (models.cpp:118-127). FP32: inputs normalised in FP64 by the model's precomputed reciprocal
// ranges (one rounding), the forward pass on FFMA with the model's FP32 weight copy.
template <bool kExact, int I, int H1, int H2, int R>
__device__ __forceinline__ void forward_shape(const double (&x)[R][8], const double* nrm, const double* rinv,
                                              const double* __restrict__ w, const float* __restrict__ wf,
                                              double (&v)[R]) {
  constexpr int B1 = I * H1, W2 = B1 + H1, B2 = W2 + H1 * H2;
  constexpr int WO = H2 > 0 ? B2 + H2 : B1 + H1;
  constexpr int BO = WO + (H2 > 0 ? H2 : H1);
  using T = std::conditional_t<kExact, double, float>;
  T a0[R][I], a1[R][H1], a2[R][H2 > 0 ? H2 : 1];
  auto wt = [&](int k) -> T {
    if constexpr (kExact) return __ldg(w + k);
    else return __ldg(wf + k);
  };
  auto madd = [](T z, T ww, T a) -> T {
    if constexpr (kExact) return __dadd_rn(z, __dmul_rn(ww, a));
    else return fmaf(ww, a, z);
  };
  auto relu = [](T z) -> T {
    if constexpr (kExact) return gate(z, z);
    else return fmaxf(z, 0.f);
  };
#pragma unroll
  for (int j = 0; j < I; ++j) {
    const double lo = __ldg(nrm + j);
    if constexpr (kExact) {
      const double range = __dsub_rn(__ldg(nrm + 8 + j), lo);
#pragma unroll
      for (int r = 0; r < R; ++r) a0[r][j] = range > 0.0 ? __ddiv_rn(__dsub_rn(x[r][j], lo), range) : 0.0;
    } else {
      const double ri = __ldg(rinv + j);
#pragma unroll
      for (int r = 0; r < R; ++r) a0[r][j] = (float)((x[r][j] - lo) * ri);
    }
  }
#pragma unroll
  for (int o = 0; o < H1; ++o) {
    const T b = wt(B1 + o);
    T z[R];
#pragma unroll
    for (int r = 0; r < R; ++r) z[r] = b;
#pragma unroll
    for (int i = 0; i < I; ++i) {
      const T ww = wt(o * I + i);
#pragma unroll
      for (int r = 0; r < R; ++r) z[r] = madd(z[r], ww, a0[r][i]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) a1[r][o] = relu(z[r]);
  }
  T z[R];
  const T bo = wt(BO);
#pragma unroll
  for (int r = 0; r < R; ++r) z[r] = bo;
  if constexpr (H2 > 0) {
#pragma unroll
    for (int o = 0; o < H2; ++o) {
      const T b = wt(B2 + o);
      T q[R];
#pragma unroll
      for (int r = 0; r < R; ++r) q[r] = b;
#pragma unroll
      for (int i = 0; i < H1; ++i) {
        const T ww = wt(W2 + o * H1 + i);
#pragma unroll
        for (int r = 0; r < R; ++r) q[r] = madd(q[r], ww, a1[r][i]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) a2[r][o] = relu(q[r]);
    }
#pragma unroll
    for (int i = 0; i < H2; ++i) {
      const T ww = wt(WO + i);
#pragma unroll
      for (int r = 0; r < R; ++r) z[r] = madd(z[r], ww, a2[r][i]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < H1; ++i) {
      const T ww = wt(WO + i);
#pragma unroll
      for (int r = 0; r < R; ++r) z[r] = madd(z[r], ww, a1[r][i]);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = (double)z[r];
}

// models.cpp:135-139 + the clamp of predict (models.cpp:362)
__device__ __forceinline__ double denorm(double v, const double* nrm, int logt) {
  const double tmin = __ldg(nrm + 16), trange = __dsub_rn(__ldg(nrm + 17), tmin);
  double t = trange > 0.0 ? __dadd_rn(tmin, __dmul_rn(v, trange)) : tmin;
  if (logt) t = exp(t);
  return t < 1e-9 ? 1e-9 : t;  // std::max(value, 1e-9)
}

// R rows of one model: compiled shapes unrolled, others through the generic forward row by row
template <bool kExact, int R>
__device__ __forceinline__ void predict_rows(const PredictArgs& a, const double* rinv, const float* wf, int m,
                                             const double (&x)[R][8], double (&out)[R]) {
  const int I = __ldg(a.n_inputs + m), H1 = __ldg(a.h1 + m), H2 = __ldg(a.h2 + m);
  const double* nrm = a.norm + 18 * (int64_t)m;
  const double* ri = rinv ? rinv + 8 * (int64_t)m : nullptr;
  const int64_t po = __ldg(a.param_offset + m);
  const double* w = a.params + po;
  const float* f = wf ? wf + po : nullptr;
  double v[R];
  const int key = (I << 8) | (H1 << 4) | H2;
#define LANN_SHAPE(II, A, B) \
  case ((II) << 8) | ((A) << 4) | (B): forward_shape<kExact, II, A, B, R>(x, nrm, ri, w, f, v); break;
  switch (key) {
    LANN_SHAPE(1, 8, 0) LANN_SHAPE(2, 8, 0) LANN_SHAPE(3, 8, 0) LANN_SHAPE(4, 8, 0)
    LANN_SHAPE(5, 8, 0) LANN_SHAPE(6, 8, 0) LANN_SHAPE(7, 8, 0)
    LANN_SHAPE(4, 5, 5) LANN_SHAPE(5, 5, 5) LANN_SHAPE(6, 5, 5)
    default:
#pragma unroll
      for (int r = 0; r < R; ++r) {
        Row8 row;
#pragma unroll
        for (int k = 0; k < 8; ++k) row.v[k] = x[r][k];
        v[r] = forward_generic<kExact>(row, nrm, w, I, H1, H2);
      }
  }
#undef LANN_SHAPE
  const int logt = __ldg(a.log_target + m);
#pragma unroll
  for (int r = 0; r < R; ++r) out[r] = denorm(v[r], nrm, logt);
}

// K2 predict (models.cpp:346-363): grid-stride over QUADS of consecutive rows. A quad whose four
// rows share a model (rows are grouped by model in predict_dataset order, so nearly all do) runs
// as one 4-row call: its model indices in one 16-B load, its 256 B of inputs in 16-B
// non-coherent loads, every weight loaded once for the four rows. Mixed quads and the ragged
// tail go row by row.
template <bool kExact, int R>
__global__ void __launch_bounds__(256) predict_kernel(PredictArgs a, const double* rinv, const float* wf) {
  static_assert(R == 1 || R == 2 || R == 4, "rows per thread");
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n_quads = a.n_rows / R;
  auto load = [&](int64_t row, double(&x)[8]) {
    const double2* xr = reinterpret_cast<const double2*>(a.rows + row * 8);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double2 v = __ldg(xr + k);
      x[2 * k] = v.x;
      x[2 * k + 1] = v.y;
    }
  };
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t q = t0; q < n_quads; q += stride) {
    const int64_t row = q * R;
    int ms[R];
    if constexpr (R == 4) {
      const int4 mm = __ldg(reinterpret_cast<const int4*>(a.row_model + row));
      ms[0] = mm.x, ms[1] = mm.y, ms[2] = mm.z, ms[3] = mm.w;
    } else if constexpr (R == 2) {
      const int2 mm = __ldg(reinterpret_cast<const int2*>(a.row_model + row));
      ms[0] = mm.x, ms[1] = mm.y;
    } else {
      ms[0] = __ldg(a.row_model + row);
    }
    double x[R][8];
#pragma unroll
    for (int r = 0; r < R; ++r) load(row + r, x[r]);
    bool same = true;
#pragma unroll
    for (int r = 1; r < R; ++r) same = same && ms[r] == ms[0];
    if (same) {
      double out[R];
      predict_rows<kExact, R>(a, rinv, wf, ms[0], x, out);
#pragma unroll
      for (int r = 0; r + 1 < R; r += 2) reinterpret_cast<double2*>(a.out + row)[r / 2] = make_double2(out[r], out[r + 1]);
      if constexpr (R == 1) a.out[row] = out[0];
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double xo[1][8], o[1];
#pragma unroll
        for (int k = 0; k < 8; ++k) xo[0][k] = x[r][k];
        predict_rows<kExact, 1>(a, rinv, wf, ms[r], xo, o);
        a.out[row + r] = o[0];
      }
    }
  }
  for (int64_t row = n_quads * R + t0; row < a.n_rows; row += stride) {  // the tail
    double xo[1][8], o[1];
    load(row, xo[0]);
    predict_rows<kExact, 1>(a, rinv, wf, __ldg(a.row_model + row), xo, o);
    a.out[row] = o[0];
  }
}

// FP32 path preparation: per-model reciprocal ranges (0 where the range is 0) and an FP32
// copy of every weight (one thread per parameter / per model).
__global__ void predict_prep_kernel(PredictArgs a, int n_models, int64_t n_params, double* rinv, float* wf) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n_params) wf[t] = (float)a.params[t];
  if (t < n_models) {
    const double* nrm = a.norm + 18 * t;
    for (int j = 0; j < 8; ++j) {
      const double range = nrm[8 + j] - nrm[j];
      rinv[8 * t + j] = range > 0.0 ? 1.0 / range : 0.0;
    }
  }
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

// Fold-mean model of a cross-validation ensemble (lann_engine.h): grid (row blocks, ensemble),
// one thread per test row; the k fold models predict the row one after another (a warp's rows
// share every model, so weight loads are uniform) and the predictions are summed in fold order,
// then divided by k. The ensemble's truth is written beside the predictions so the pair is an
// ordinary eval set. Block (0, e) also records whether every member trained and evaluated OK.
template <bool kExact>
__global__ void __launch_bounds__(128) fold_mean_kernel(PredictArgs pa, FoldMeanArgs f, const double* rinv,
                                                        const float* wf) {
  const int e = blockIdx.y;
  const int k = __ldg(f.ens_k + e);
  const int* members = f.ens_models + (int64_t)e * f.kmax;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int bad = -1;
    for (int i = 0; i < k && bad < 0; ++i) {
      const int m = __ldg(members + i);
      if (__ldg(f.model_bad + m) >= 0) bad = 2 * i;                // TrainingError
      else if (__ldg(f.model_status + m) != 0) bad = 2 * i + 1;  // no held-out metrics (DomainError)
    }
    f.ens_bad[e] = bad;
  }
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = __ldg(f.ens_len + e);
  if (r >= n) return;
  const int64_t row = __ldg(f.ens_rows + e) + r;
  double x[1][8];
  const double2* xr = reinterpret_cast<const double2*>(f.rows + row * 8);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double2 v = __ldg(xr + q);
    x[0][2 * q] = v.x;
    x[0][2 * q + 1] = v.y;
  }
  double sum = 0.0;
  for (int i = 0; i < k; ++i) {
    double o[1];
    predict_rows<kExact, 1>(pa, rinv, wf, __ldg(members + i), x, o);
    sum = i == 0 ? o[0] : __dadd_rn(sum, o[0]);
  }
  const int64_t out = __ldg(f.ens_out + e) + r;
  f.pred[out] = __ddiv_rn(sum, (double)k);
  f.truth_out[out] = __ldg(f.truth + row);
}

// Group statistics, one CTA per group: the OK items are compacted in order (block scan), then
// per metric the mean is the sequential sum / count (one thread, item order) and the median the
// value(s) at sorted positions (n-1)/2 and n/2, found by counting ranks (ties broken by order)
// over tiles of the compacted values staged in shared memory.
constexpr int kStatTile = 1024;

__global__ void __launch_bounds__(256) cv_stats_kernel(CvStatsArgs a) {
  __shared__ double tile[kStatTile];
  __shared__ int warp_sum[8];
  __shared__ int base;
  __shared__ double mid[2];
  const int g = blockIdx.x;
  const int len = a.item_len[g];
  const int64_t off = a.item_off[g];
  const int* items = a.items + off;
  double* vals = a.scratch + off;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  // ordered compaction: each thread keeps the (id, position) of its OK items of the first 8 chunks
  // in registers; groups longer than 8 chunks are gathered sequentially by thread 0 instead
  int my_id[8], my_pos[8], n_mine = 0;
  int n_ok = 0;
  for (int c0 = 0; c0 < len; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    int id = -1;
    bool ok = false;
    if (i < len) {
      id = items[i];
      ok = a.status[id] == 0 && a.bad[id] < 0;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, ok);
    if (lane == 0) warp_sum[warp] = __popc(mask);
    __syncthreads();
    int before = base;
    for (int w = 0; w < warp; ++w) before += warp_sum[w];
    before += __popc(mask & ((1u << lane) - 1u));
    int total = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) total += warp_sum[w];
    __syncthreads();
    if (threadIdx.x == 0) base += total;
    if (ok && len <= 8 * (int)blockDim.x) {
      my_id[n_mine] = id;
      my_pos[n_mine] = before;
      ++n_mine;
    }
    n_ok += total;
  }
  __syncthreads();
  const int n = n_ok;
  const double* ms[3] = {a.m0, a.m1, a.m2};
  for (int q = 0; q < 3; ++q) {
    // gather this metric's values in compacted order
    for (int t = 0; t < n_mine; ++t) vals[my_pos[t]] = ms[q][my_id[t]];
    if (len > 8 * (int)blockDim.x) {
      __syncthreads();
      if (threadIdx.x == 0) {
        int p = 0;
        for (int i = 0; i < len; ++i) {
          const int id = items[i];
          if (a.status[id] == 0 && a.bad[id] < 0) vals[p++] = ms[q][id];
        }
      }
    }
    __syncthreads();
    // ranks: each thread owns values i = threadIdx.x, + blockDim.x, ...
    for (int i0 = 0; i0 < n; i0 += blockDim.x) {
      const int i = i0 + threadIdx.x;
      const double vi = i < n ? vals[i] : 0.0;
      int rank = 0;
      for (int j0 = 0; j0 < n; j0 += kStatTile) {
        const int m = min(kStatTile, n - j0);
        __syncthreads();
        for (int j = threadIdx.x; j < m; j += blockDim.x) tile[j] = vals[j0 + j];
        __syncthreads();
        for (int j = 0; j < m; ++j) {
          const double vj = tile[j];
          rank += (vj < vi) || (vj == vi && j0 + j < i);
        }
      }
      if (i < n) {
        if (rank == (n - 1) / 2) mid[0] = vi;
        if (rank == n / 2) mid[1] = vi;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double mean = 0.0, median = 0.0;
      if (n > 0) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, vals[i]);
        mean = __ddiv_rn(acc, (double)n);
        median = (n & 1) ? mid[1] : __ddiv_rn(__dadd_rn(mid[0], mid[1]), 2.0);
      }
      a.out[(int64_t)g * 6 + 2 * q] = mean;
      a.out[(int64_t)g * 6 + 2 * q + 1] = median;
      if (q == 0) a.n_ok[g] = n;
    }
    __syncthreads();
  }
}

}  // namespace

namespace {
// rows per thread: 4 for FP32 (weights loaded once per quad; 61% of HBM); the FP64-exact path
// is FP64-issue heavy (a correctly rounded division per input) and register-bound at 4 rows
#ifndef LANN_EXACT_ROWS
#define LANN_EXACT_ROWS 1
#endif
constexpr int kExactRows = LANN_EXACT_ROWS;
unsigned predict_grid(int64_t n_rows) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n_rows + 255) / 256, cap = int64_t(sms) * 8;  // 8 CTAs of 256 per SM
  return (unsigned)std::max<int64_t>(1, std::min(want, cap));
}
}  // namespace

void launch_predict_fp64(const PredictArgs& a, cudaStream_t s) {
  if (a.n_rows <= 0) return;
  predict_kernel<true, kExactRows><<<predict_grid(a.n_rows), 256, 0, s>>>(a, nullptr, nullptr);
}

// n_models / n_params size the FP32 preparation (reciprocal ranges, FP32 weight copy); the
// scratch lives for the launch only (stream-ordered allocation)
void launch_predict_fp32(const PredictArgs& a, int n_models, int64_t n_params, cudaStream_t s) {
  if (a.n_rows <= 0) return;
  void* scratch = nullptr;
  const size_t bytes = size_t(n_models) * 8 * sizeof(double) + size_t(n_params) * sizeof(float) + 16;
  if (cudaMallocAsync(&scratch, bytes, s) != cudaSuccess) return;
  double* rinv = static_cast<double*>(scratch);
  float* wf = reinterpret_cast<float*>(rinv + size_t(n_models) * 8);
  const int64_t n_prep = std::max<int64_t>(n_models, n_params);
  predict_prep_kernel<<<(unsigned)((n_prep + 255) / 256), 256, 0, s>>>(a, n_models, n_params, rinv, wf);
  predict_kernel<false, 4><<<predict_grid(a.n_rows), 256, 0, s>>>(a, rinv, wf);
  cudaFreeAsync(scratch, s);
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

void launch_fold_mean(const PredictArgs& pa, const FoldMeanArgs& f, int max_len, bool exact, int n_models,
                      int64_t n_params, cudaStream_t s) {
  if (f.n_ens <= 0 || max_len <= 0) return;
  const dim3 grid((unsigned)((max_len + 127) / 128), (unsigned)f.n_ens);
  if (exact) {
    fold_mean_kernel<true><<<grid, 128, 0, s>>>(pa, f, nullptr, nullptr);
    return;
  }
  void* scratch = nullptr;
  const size_t bytes = size_t(n_models) * 8 * sizeof(double) + size_t(n_params) * sizeof(float) + 16;
  if (cudaMallocAsync(&scratch, bytes, s) != cudaSuccess) return;
  double* rinv = static_cast<double*>(scratch);
  float* wf = reinterpret_cast<float*>(rinv + size_t(n_models) * 8);
  const int64_t n_prep = std::max<int64_t>(n_models, n_params);
  predict_prep_kernel<<<(unsigned)((n_prep + 255) / 256), 256, 0, s>>>(pa, n_models, n_params, rinv, wf);
  fold_mean_kernel<false><<<grid, 128, 0, s>>>(pa, f, rinv, wf);
  cudaFreeAsync(scratch, s);
}

void launch_cv_stats(const CvStatsArgs& a, cudaStream_t s) {
  if (a.n_groups <= 0) return;
  cv_stats_kernel<<<a.n_groups, 256, 0, s>>>(a);
}

}  // namespace lann
