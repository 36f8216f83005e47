// mlp_ops.cu — the per-net building blocks of mlp.hpp on the GPU, batched over nets:
//   Mlp::forward       (mlp.cpp:36-62)   one thread per (row, net)
//   mse_loss           (mlp.cpp:64-73)   forward per row, then the sequential sum per net
//   mse_gradient       (mlp.cpp:75-122)  one CTA per net: sample threads store per-parameter
//                                        terms, parameter threads sum them in sample order
//   AdamState::update  (mlp.cpp:142-154) one thread per parameter
// Nets of any depth (up to kMaxLayers layers) and widths up to kMaxW, the reference's generic
// Mlp (the population trainers compile the LANN shapes instead). Exact operation order, no
// contraction (-fmad=false and explicit __d*_rn), so every result is bit-identical to the
// reference's for the same inputs.
#include <cmath>

#include "kernels.cuh"

namespace lann {
namespace {

constexpr int kMaxW = kMaxMlpWidth;

struct NetView {
  int L;             // layers
  const int* dims;   // L + 1 dims
  const double* p;   // flat parameters, mlp.cpp:124-131 layout
};

__device__ __forceinline__ NetView net_of(const MlpArgs& a, int n) {
  NetView v;
  v.L = a.n_dims[n] - 1;
  v.dims = a.dims + a.dims_offset[n];
  v.p = a.params + a.param_offset[n];
  return v;
}

// forward_cached (mlp.cpp:36-52) keeping every layer's activations: acts[l][i], l = 0..L.
// Only output unit 0 of the last layer is computed (Mlp::forward returns acts.back()[0]).
__device__ double forward_acts(const NetView& v, const double* x, double (*acts)[kMaxW], bool all_out) {
  for (int i = 0; i < v.dims[0]; ++i) acts[0][i] = x[i];
  const double* w = v.p;
  for (int l = 0; l < v.L; ++l) {
    const int in = v.dims[l], out = v.dims[l + 1];
    const double* b = w + in * out;
    const bool hidden = l + 1 < v.L;
    const int n_out = hidden || all_out ? out : 1;
    for (int o = 0; o < n_out; ++o) {
      double z = b[o];
      for (int i = 0; i < in; ++i) z = __dadd_rn(z, __dmul_rn(w[o * in + i], acts[l][i]));
      acts[l + 1][o] = hidden ? (z > 0.0 ? z : 0.0) : z;
    }
    w = b + out;
  }
  return acts[v.L][0];
}

__global__ void mlp_forward_kernel(MlpArgs a, double* out) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= a.total_rows) return;
  const int n = a.row_net[r];
  const NetView v = net_of(a, n);
  double acts[kMaxLayers + 1][kMaxW];
  out[r] = forward_acts(v, a.X + a.x_offset[n] + (r - a.row_offset[n]) * v.dims[0], acts, false);
}

// mse_loss: acc += e*e over rows in order, then acc / N (mlp.cpp:67-72)
__global__ void mlp_loss_kernel(MlpArgs a, const double* fwd, double* loss) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= a.n_nets) return;
  const int64_t r0 = a.row_offset[n];
  const int N = a.n_rows[n];
  double acc = 0.0;
  for (int s = 0; s < N; ++s) {
    const double e = __dsub_rn(fwd[r0 + s], a.y[r0 + s]);
    acc = __dadd_rn(acc, __dmul_rn(e, e));
  }
  loss[n] = __ddiv_rn(acc, (double)N);
}

// mse_gradient: phase 1 (threads over samples) stores each sample's term per parameter,
// (inv_n*delta[o])*a_prev[i] for a weight (mlp.cpp:113), inv_n*delta[o] for a bias (:117), and
// err^2; phase 2 (threads over parameters) sums each row in sample order from 0.0; the loss is
// the err^2 row's sum times inv_n (:120). Scratch: (P + 1) x N doubles per net.
__global__ void __launch_bounds__(128) mlp_grad_kernel(MlpArgs a, double* scratch, const int64_t* scratch_offset,
                                                       double* loss, double* grad) {
  const int n = blockIdx.x;
  const NetView v = net_of(a, n);
  const int N = a.n_rows[n];
  const int P = a.n_params[n];
  double* T = scratch + scratch_offset[n];  // [P + 1][N]
  const double inv_n = 1.0 / (double)N;      // mlp.cpp:84
  const double* X = a.X + a.x_offset[n];
  const double* Y = a.y + a.row_offset[n];
  for (int s = threadIdx.x; s < N; s += blockDim.x) {
    double acts[kMaxLayers + 1][kMaxW];
    double delta[2][kMaxW];
    forward_acts(v, X + (int64_t)s * v.dims[0], acts, true);
    const double err = __dsub_rn(acts[v.L][0], Y[s]);  // mlp.cpp:90
    T[(int64_t)P * N + s] = __dmul_rn(err, err);
    // walk the layers backwards: the delta of layer l (mlp.cpp:92-104), then its terms
    int cur = 0;
    delta[cur][0] = __dmul_rn(2.0, err);
    // offsets of each layer's weights in the flat layout
    int off[kMaxLayers + 1];
    off[0] = 0;
    for (int l = 0; l < v.L; ++l) off[l + 1] = off[l] + (v.dims[l] + 1) * v.dims[l + 1];
    for (int l = v.L - 1; l >= 0; --l) {
      const int in = v.dims[l], out = v.dims[l + 1];
      const double* d = delta[cur];
      for (int o = 0; o < out; ++o) {
        const double t = __dmul_rn(inv_n, d[o]);
        for (int i = 0; i < in; ++i) T[(int64_t)(off[l] + o * in + i) * N + s] = __dmul_rn(t, acts[l][i]);
        T[(int64_t)(off[l] + in * out + o) * N + s] = t;
      }
      if (l > 0) {  // delta of the layer below: acc = 0.0 + sum_o w[o,i]*delta[o], ReLU gate
        const double* w = v.p + off[l];
        double* dn = delta[cur ^ 1];
        for (int i = 0; i < in; ++i) {
          double acc = 0.0;
          for (int o = 0; o < out; ++o) acc = __dadd_rn(acc, __dmul_rn(w[o * in + i], d[o]));
          dn[i] = acts[l][i] > 0.0 ? acc : 0.0;
        }
        cur ^= 1;
      }
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j <= P; j += blockDim.x) {
    const double* row = T + (int64_t)j * N;
    double g = 0.0;
    for (int s = 0; s < N; ++s) g = __dadd_rn(g, row[s]);
    if (j < P) grad[a.param_offset[n] + j] = g;
    else loss[n] = __dmul_rn(g, inv_n);  // result.loss *= inv_n
  }
}

// AdamState::update (mlp.cpp:142-154) in the reference's expression order; bc1 / bc2 are
// 1 - pow(beta, step) from the host libm (the reference's std::pow).
__global__ void adam_kernel(AdamArgs a) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const double g = a.grad[i];
  const double m = __dadd_rn(__dmul_rn(a.beta1, a.m[i]), __dmul_rn(__dsub_rn(1.0, a.beta1), g));
  const double v = __dadd_rn(__dmul_rn(a.beta2, a.v[i]), __dmul_rn(__dmul_rn(__dsub_rn(1.0, a.beta2), g), g));
  a.m[i] = m;
  a.v[i] = v;
  const double mhat = __ddiv_rn(m, a.bc1);
  const double vhat = __ddiv_rn(v, a.bc2);
  a.params[i] = __dsub_rn(a.params[i], __ddiv_rn(__dmul_rn(a.lr, mhat), __dadd_rn(__dsqrt_rn(vhat), a.eps)));
}

}  // namespace

void launch_mlp_forward(const MlpArgs& a, double* out, cudaStream_t s) {
  if (a.total_rows > 0)
    mlp_forward_kernel<<<unsigned((a.total_rows + 127) / 128), 128, 0, s>>>(a, out);
}

void launch_mlp_loss(const MlpArgs& a, const double* fwd, double* loss, cudaStream_t s) {
  launch_mlp_forward(a, const_cast<double*>(fwd), s);
  mlp_loss_kernel<<<unsigned((a.n_nets + 127) / 128), 128, 0, s>>>(a, fwd, loss);
}

void launch_mlp_grad(const MlpArgs& a, double* scratch, const int64_t* scratch_offset, double* loss, double* grad,
                     cudaStream_t s) {
  mlp_grad_kernel<<<unsigned(a.n_nets), 128, 0, s>>>(a, scratch, scratch_offset, loss, grad);
}

void launch_adam(const AdamArgs& a, cudaStream_t s) {
  if (a.n > 0) adam_kernel<<<unsigned((a.n + 255) / 256), 256, 0, s>>>(a);
}

}  // namespace lann
