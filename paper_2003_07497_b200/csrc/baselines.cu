// baselines.cu — the non-LANN model families of the reference's five-family comparison
// (models.cpp:184-333, forest.cpp), batched over a population on the GPU:
//
//   const (C) and lrc (LR+C): least squares by the normal equations (models.cpp:220-265):
//     columns equilibrated by their max |x|, Gram matrix + right-hand side accumulated sample by
//     sample, Gaussian elimination with partial pivoting and a 1e-13 relative pivot floor
//     (solve_linear, models.cpp:186-218), a 1e-8 ridge retry on singular designs. One CTA per
//     model: one thread per Gram entry walks the samples in the reference's order; one thread
//     solves. Compiled with -fmad=false: bit-identical to the reference.
//   nlrc (NLR+C): bagged CART regression forest (forest.cpp): per tree a bootstrap of n draws
//     (host: Rng(derive_seed(seed, t)).bounded(n), sorted), exhaustive SSE-reduction splits over
//     every feature, depth-limited. One CTA per (model, tree), level-synchronous: every node of
//     a level is split at once from per-feature sorted slot lists that are stably partitioned
//     into the children (the classic GPU CART layout), node means summed in the reference's
//     sample order. Nodes come out breadth-first; the host renumbers them to the reference's
//     depth-first preorder. Ties between equal feature values can be ordered differently from
//     std::sort, so split sums may differ in the last bits (parity within tolerance).
//   prediction: intercept + sum w_j x_j (models.cpp:357-360); mean of the trees' leaf values
//     (forest.cpp:13-27); both clamped at 1e-9.
#include <cmath>
#include <cstddef>
#include <cstdint>

#include "../../include/lann_engine.h"
#include "kernels.cuh"

namespace lann {
namespace {

// ---- least squares ---------------------------------------------------------------------------
constexpr int kMaxLin = LANN_ROW + 1;  // features + intercept

__device__ bool solve_linear(double* a, double* b, int n, double* x) {  // models.cpp:186-218
  double diag_scale = 0.0;
  for (int i = 0; i < n; ++i) diag_scale = fmax(diag_scale, fabs(a[i * n + i]));
  const double pivot_floor = fmax(diag_scale, 1.0) * 1e-13;
  for (int col = 0; col < n; ++col) {
    int pivot = col;
    for (int row = col + 1; row < n; ++row)
      if (fabs(a[row * n + col]) > fabs(a[pivot * n + col])) pivot = row;
    if (fabs(a[pivot * n + col]) < pivot_floor) return false;
    if (pivot != col) {
      for (int j = 0; j < n; ++j) {
        const double t = a[pivot * n + j];
        a[pivot * n + j] = a[col * n + j];
        a[col * n + j] = t;
      }
      const double t = b[pivot];
      b[pivot] = b[col];
      b[col] = t;
    }
    const double inv = 1.0 / a[col * n + col];
    for (int row = col + 1; row < n; ++row) {
      const double f = a[row * n + col] * inv;
      if (f == 0.0) continue;
      for (int j = col; j < n; ++j) a[row * n + j] -= f * a[col * n + j];
      b[row] -= f * b[col];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double acc = b[i];
    for (int j = i + 1; j < n; ++j) acc -= a[i * n + j] * x[j];
    x[i] = acc / a[i * n + i];
  }
  return true;
}

__global__ void fit_linear_kernel(LinearArgs a) {
  const int m = blockIdx.x;
  const int p = a.n_feats[m], n = p + 1, rows = a.n_rows[m];
  const double* X = a.X + a.row_offset[m] * LANN_ROW;
  const double* y = a.y + a.row_offset[m];
  __shared__ double scale[LANN_ROW];
  __shared__ double gram[kMaxLin * kMaxLin], rhs[kMaxLin], sol[kMaxLin], g2[kMaxLin * kMaxLin], r2[kMaxLin];
  const int t = threadIdx.x;
  if (t < p) {
    double s = 0.0;
    for (int r = 0; r < rows; ++r) s = fmax(s, fabs(X[r * LANN_ROW + t]));
    scale[t] = s == 0.0 ? 1.0 : s;
  }
  __syncthreads();
  // thread (i, j), j >= i: gram[i][j] += xi * xj over samples in order; thread n*n + i: rhs[i]
  if (t < n * n) {
    const int i = t / n, j = t % n;
    if (j >= i) {
      double acc = 0.0;
      for (int r = 0; r < rows; ++r) {
        const double xi = i < p ? X[r * LANN_ROW + i] / scale[i] : 1.0;
        const double xj = j < p ? X[r * LANN_ROW + j] / scale[j] : 1.0;
        acc += xi * xj;
      }
      gram[i * n + j] = acc;
    }
  } else if (t < n * n + n) {
    const int i = t - n * n;
    double acc = 0.0;
    for (int r = 0; r < rows; ++r) {
      const double xi = i < p ? X[r * LANN_ROW + i] / scale[i] : 1.0;
      acc += xi * y[r];
    }
    rhs[i] = acc;
  }
  __syncthreads();
  if (t == 0) {
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < i; ++j) gram[i * n + j] = gram[j * n + i];
    for (int k = 0; k < n * n; ++k) g2[k] = gram[k];
    for (int k = 0; k < n; ++k) r2[k] = rhs[k];
    bool ok = solve_linear(gram, rhs, n, sol);
    if (!ok) {
      for (int i = 0; i < p; ++i) g2[i * n + i] += a.ridge;
      ok = solve_linear(g2, r2, n, sol);
    }
    a.status[m] = ok ? 0 : 1;
    for (int j = 0; j < LANN_ROW; ++j) a.weights[m * LANN_ROW + j] = (ok && j < p) ? sol[j] / scale[j] : 0.0;
    a.intercept[m] = ok ? sol[n - 1] : 0.0;
  }
}

__global__ void predict_linear_kernel(PredictLinearArgs a) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r >= a.n_rows) return;
  const int m = a.row_model[r];
  const double* w = a.weights + m * LANN_ROW;
  double v = a.intercept[m];
  for (int j = 0; j < a.n_feats[m]; ++j) v += w[j] * a.rows[r * LANN_ROW + j];
  a.out[r] = fmax(v, 1e-9);
}

// ---- forest ----------------------------------------------------------------------------------
// shared memory: X [n][LANN_ROW] (double), y [n], sample of slot [n] (u16), lists 2 x (p+1) x n
// (u16), level tables 2 x {start, count, node} x n (i32)
// kGlobal: the same working set in a per-CTA slice of a global scratch buffer, for training sets
// too large for shared memory (the reference forest takes any size, forest.cpp:13-143)
template <bool kGlobal>
__global__ void fit_forest_kernel(ForestArgs a) {
  extern __shared__ __align__(16) unsigned char dsmem[];
  const int m = blockIdx.y, tree = blockIdx.x;
  unsigned char* smem =
      kGlobal ? a.scratch_ws + (size_t(m) * a.trees + tree) * a.ws_stride : dsmem;
  const int n = a.n_rows[m], p = a.n_feats[m], L = p + 1;
  const int tid = threadIdx.x, T = blockDim.x;
  double* X = reinterpret_cast<double*>(smem);
  double* y = X + size_t(a.max_rows) * LANN_ROW;
  uint16_t* samp = reinterpret_cast<uint16_t*>(y + a.max_rows);
  uint16_t* lists0 = samp + a.max_rows;
  uint16_t* lists1 = lists0 + size_t(LANN_ROW + 1) * a.max_rows;
  int* tab0 = reinterpret_cast<int*>(lists1 + size_t(LANN_ROW + 1) * a.max_rows + 8);
  tab0 = reinterpret_cast<int*>((reinterpret_cast<uintptr_t>(tab0) + 15) & ~uintptr_t(15));
  int* tab1 = tab0 + 3 * a.max_rows;
  __shared__ int n_level, n_next, n_nodes;
  // per (node, feature) best split of the current level
  const double* gX = a.X + a.row_offset[m] * LANN_ROW;
  const double* gy = a.y + a.row_offset[m];
  for (int k = tid; k < n * LANN_ROW; k += T) X[k] = gX[k];
  for (int k = tid; k < n; k += T) y[k] = gy[k];
  const uint16_t* boot = a.bootstrap + (size_t(m) * a.trees + tree) * a.max_rows;
  for (int k = tid; k < n; k += T) samp[k] = boot[k];
  __syncthreads();
  // root lists: list p = natural slot order; list f = slots stably sorted by X[sample][f]
  for (int k = tid; k < n; k += T) {
    lists0[size_t(p) * a.max_rows + k] = uint16_t(k);
    for (int f = 0; f < p; ++f) {
      const double v = X[samp[k] * LANN_ROW + f];
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        const double u = X[samp[j] * LANN_ROW + f];
        rank += (u < v) || (u == v && j < k);
      }
      lists0[size_t(f) * a.max_rows + rank] = uint16_t(k);
    }
  }
  if (tid == 0) {
    tab0[0] = 0;      // start
    tab0[1] = n;      // count
    tab0[2] = 0;      // node id (breadth-first)
    n_level = 1;
    n_nodes = 1;
  }
  __syncthreads();
  const size_t nbase = (size_t(m) * a.trees + tree) * size_t(2 * a.max_rows);
  int* out_feat = a.node_feature + nbase;
  double* out_thr = a.node_threshold + nbase;
  int* out_left = a.node_left + nbase;
  int* out_right = a.node_right + nbase;
  double* out_val = a.node_value + nbase;
  double* best_sse = a.scratch_sse + (size_t(m) * a.trees + tree) * size_t(a.max_rows) * LANN_ROW;
  double* best_thr = a.scratch_thr + (size_t(m) * a.trees + tree) * size_t(a.max_rows) * LANN_ROW;
  uint16_t* cur = lists0;
  uint16_t* nxt = lists1;
  int* ct = tab0;
  int* nt = tab1;
  for (int depth = 0;; ++depth) {
    const int nl = n_level;
    if (nl == 0) break;
    // node values (mean of y in the reference's sample order) and per-(node, feature) best cuts
    for (int task = tid; task < nl * L; task += T) {
      const int node = task / L, f = task % L;
      const int start = ct[3 * node], cnt = ct[3 * node + 1];
      const uint16_t* lst = cur + size_t(f) * a.max_rows + start;
      if (f == p) {
        double acc = 0.0;
        for (int k = 0; k < cnt; ++k) acc += y[samp[lst[k]]];
        out_val[ct[3 * node + 2]] = acc / double(cnt);
        out_feat[ct[3 * node + 2]] = -1;
        out_left[ct[3 * node + 2]] = -1;
        out_right[ct[3 * node + 2]] = -1;
        out_thr[ct[3 * node + 2]] = 0.0;
        continue;
      }
      double sse_best = INFINITY, thr = 0.0;
      if (depth < a.max_depth && cnt >= a.min_samples_split) {
        double sum_total = 0.0, sq_total = 0.0;
        for (int k = 0; k < cnt; ++k) {
          const double yv = y[samp[lst[k]]];
          sum_total += yv;
          sq_total += yv * yv;
        }
        double sum_left = 0.0, sq_left = 0.0;
        for (int cut = 1; cut < cnt; ++cut) {
          const double yv = y[samp[lst[cut - 1]]];
          sum_left += yv;
          sq_left += yv * yv;
          const double lo = X[samp[lst[cut - 1]] * LANN_ROW + f];
          const double hi = X[samp[lst[cut]] * LANN_ROW + f];
          if (lo == hi) continue;
          const double nlf = double(cut), nrf = double(cnt - cut);
          const double sum_right = sum_total - sum_left, sq_right = sq_total - sq_left;
          const double sse = (sq_left - sum_left * sum_left / nlf) + (sq_right - sum_right * sum_right / nrf);
          if (sse < sse_best) {
            sse_best = sse;
            thr = lo + (hi - lo) / 2.0;
          }
        }
      }
      best_sse[node * LANN_ROW + f] = sse_best;
      best_thr[node * LANN_ROW + f] = thr;
    }
    __syncthreads();
    // choose the split per node (first feature with the strictly smallest SSE), count children
    if (tid == 0) {
      int next = 0, offset = 0;
      for (int node = 0; node < nl; ++node) {
        int bf = -1;
        double bs = INFINITY, bt = 0.0;
        for (int f = 0; f < p; ++f)
          if (best_sse[node * LANN_ROW + f] < bs) {
            bs = best_sse[node * LANN_ROW + f];
            bf = f;
            bt = best_thr[node * LANN_ROW + f];
          }
        const int start = ct[3 * node], cnt = ct[3 * node + 1], id = ct[3 * node + 2];
        int nleft = 0;
        if (bf >= 0) {
          const uint16_t* lst = cur + size_t(p) * a.max_rows + start;
          for (int k = 0; k < cnt; ++k) nleft += X[samp[lst[k]] * LANN_ROW + bf] <= bt;
        }
        if (bf < 0 || nleft == 0 || nleft == cnt) {
          best_sse[node * LANN_ROW] = -1.0;  // leaf marker for the partition pass
          continue;
        }
        out_feat[id] = bf;
        out_thr[id] = bt;
        out_left[id] = n_nodes;
        out_right[id] = n_nodes + 1;
        nt[3 * next] = offset;
        nt[3 * next + 1] = nleft;
        nt[3 * next + 2] = n_nodes;
        nt[3 * (next + 1)] = offset + nleft;
        nt[3 * (next + 1) + 1] = cnt - nleft;
        nt[3 * (next + 1) + 2] = n_nodes + 1;
        // remember where this node's children go and its split for the partition pass
        best_sse[node * LANN_ROW] = double(next);
        best_thr[node * LANN_ROW] = bt;
        best_thr[node * LANN_ROW + 1] = double(bf);
        n_nodes += 2;
        next += 2;
        offset += cnt;
      }
      n_next = next;
    }
    __syncthreads();
    // stable partition of every list of every split node into the next level's segments
    for (int task = tid; task < nl * L; task += T) {
      const int node = task / L, f = task % L;
      if (best_sse[node * LANN_ROW] < 0.0) continue;
      const int ch = int(best_sse[node * LANN_ROW]);
      const double bt = best_thr[node * LANN_ROW];
      const int bf = int(best_thr[node * LANN_ROW + 1]);
      const int start = ct[3 * node], cnt = ct[3 * node + 1];
      const uint16_t* src = cur + size_t(f) * a.max_rows + start;
      uint16_t* dl = nxt + size_t(f) * a.max_rows + nt[3 * ch];
      uint16_t* dr = nxt + size_t(f) * a.max_rows + nt[3 * (ch + 1)];
      int il = 0, ir = 0;
      for (int k = 0; k < cnt; ++k) {
        const uint16_t s = src[k];
        if (X[samp[s] * LANN_ROW + bf] <= bt) dl[il++] = s;
        else dr[ir++] = s;
      }
    }
    __syncthreads();
    if (tid == 0) n_level = n_next;
    uint16_t* tl = cur;
    cur = nxt;
    nxt = tl;
    int* tt = ct;
    ct = nt;
    nt = tt;
    __syncthreads();
  }
  if (tid == 0) a.node_count[size_t(m) * a.trees + tree] = n_nodes;
}

__global__ void predict_forest_kernel(PredictForestArgs a) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r >= a.n_rows) return;
  const int m = a.row_model[r];
  const double* x = a.rows + r * LANN_ROW;
  double acc = 0.0;
  for (int t = 0; t < a.trees; ++t) {
    const size_t base = (size_t(m) * a.trees + t) * size_t(a.nodes_per_tree);
    int node = 0;
    while (a.node_feature[base + node] >= 0)
      node = x[a.node_feature[base + node]] <= a.node_threshold[base + node] ? a.node_left[base + node]
                                                                             : a.node_right[base + node];
    acc += a.node_value[base + node];
  }
  a.out[r] = fmax(acc / double(a.trees), 1e-9);
}

}  // namespace

void launch_fit_linear(const LinearArgs& a, cudaStream_t s) {
  fit_linear_kernel<<<a.n_models, 128, 0, s>>>(a);
}
void launch_predict_linear(const PredictLinearArgs& a, cudaStream_t s) {
  if (a.n_rows > 0) predict_linear_kernel<<<unsigned((a.n_rows + 127) / 128), 128, 0, s>>>(a);
}
size_t forest_smem_bytes(int max_rows) {
  return size_t(max_rows) * LANN_ROW * 8 + size_t(max_rows) * 8 + size_t(max_rows) * 2 +
         2 * size_t(LANN_ROW + 1) * max_rows * 2 + 16 + 16 + 2 * 3 * size_t(max_rows) * 4;
}
void launch_fit_forest(const ForestArgs& a, cudaStream_t s) {
  if (a.scratch_ws) {
    fit_forest_kernel<true><<<dim3(a.trees, a.n_models), 128, 0, s>>>(a);
    return;
  }
  const size_t smem = forest_smem_bytes(a.max_rows);
  cudaFuncSetAttribute(fit_forest_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  fit_forest_kernel<false><<<dim3(a.trees, a.n_models), 128, smem, s>>>(a);
}
void launch_predict_forest(const PredictForestArgs& a, cudaStream_t s) {
  if (a.n_rows > 0) predict_forest_kernel<<<unsigned((a.n_rows + 127) / 128), 128, 0, s>>>(a);
}

}  // namespace lann
