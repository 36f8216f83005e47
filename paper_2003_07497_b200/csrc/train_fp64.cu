// train_fp64.cu — K1a: the FP64 exact-order LANN trainer ("parity mode").
//
// Reproduces models::train_full_batch (mlp.cpp:156-175) bit for bit: the same
// forward order (mlp.cpp:36-52), the same per-sample delta recursion
// (mlp.cpp:93-104), the same SEQUENTIAL per-parameter gradient accumulation
// over samples (mlp.cpp:106-118), the same Adam expression order
// (mlp.cpp:142-154) and the pre-update loss trace / non-finite check.
// Built with -fmad=false and written with explicit __d*_rn intrinsics so no
// multiply-add is ever contracted (the reference object code has no FMA).
//
// Mapping (one CTA per model, models ordered longest-first):
//   phase A  threads own SAMPLES: forward + backward for their samples, writing a
//            per-sample record {x, hidden activations, inv_n*delta, err^2};
//   phase B  threads own PARAMETERS: each sums its N per-sample terms in sample
//            order (the only order-sensitive reduction), then applies Adam;
//            one thread sums the loss terms in sample order.
// Two __syncthreads per epoch. The N-long dependent DADD chain (8 cycles each)
// bounds the epoch latency; several CTAs per SM overlap their chains.
// Phase A is compiled per network shape for the default topologies (all loops
// unrolled, shared-memory offsets immediate); other shapes use a generic path.
#include <cmath>

#include "kernels.cuh"

namespace lann {
namespace {

constexpr int kMaxKB = 8;  // parameters owned per thread in phase B (P <= 8 * blockDim)

struct Shape {
  int I, H1, H2, nl, P, R;
  int dims[4];
  int woff[3], boff[3];
  int inoff[3];  // record offset of each layer's input vector
  int toff[3];   // record offset of each layer's (scaled) deltas
  int e2;        // record offset of err^2
};

__host__ __device__ constexpr int rec_stride(int H1, int H2) {
  return (8 + 2 * (H1 + (H2 > 0 ? H2 : 0)) + 2) | 1;  // odd: minimal bank pattern for 8-byte accesses
}

__device__ Shape make_shape(int I, int H1, int H2) {
  Shape s;
  s.I = I;
  s.H1 = H1;
  s.H2 = H2;
  s.nl = H2 > 0 ? 3 : 2;
  s.dims[0] = I;
  s.dims[1] = H1;
  s.dims[2] = H2 > 0 ? H2 : 1;
  s.dims[3] = 1;
  int off = 0;
  for (int l = 0; l < s.nl; ++l) {
    s.woff[l] = off;
    off += s.dims[l] * s.dims[l + 1];
    s.boff[l] = off;
    off += s.dims[l + 1];
  }
  s.P = off;
  const int hidden = H1 + (H2 > 0 ? H2 : 0);
  s.inoff[0] = 0;
  s.inoff[1] = 8;
  s.inoff[2] = 8 + H1;
  const int t0 = 8 + hidden;
  s.toff[0] = t0;
  s.toff[1] = t0 + s.dims[1];
  s.toff[2] = t0 + s.dims[1] + s.dims[2];
  s.e2 = t0 + hidden + 1;
  s.R = rec_stride(H1, H2);
  return s;
}

// ---- phase A, compiled shape ------------------------------------------------------
// Record layout (doubles): [0,8) x | [8, 8+H1) a1 | [.., +H2) a2 | t1[H1] | t2[H2] | tout | e2
template <int I, int H1, int H2>
struct Fixed {
  static constexpr int HS = H1 + H2;
  static constexpr int A1 = 8, A2 = 8 + H1;
  static constexpr int T1 = 8 + HS, T2 = T1 + H1, TO = T1 + HS, E2 = TO + 1;
  static constexpr int R = rec_stride(H1, H2);
  static constexpr int W1 = 0, B1 = I * H1;
  static constexpr int W2 = B1 + H1, B2 = W2 + H1 * H2;          // 2 hidden layers
  static constexpr int WO = H2 > 0 ? B2 + H2 : B1 + H1;          // output weights
  static constexpr int BO = WO + (H2 > 0 ? H2 : H1);
  static constexpr int P = BO + 1;

  __device__ static void sample(const double* __restrict__ w, double* __restrict__ r, double y,
                                double inv_n) {
    double x[I];
#pragma unroll
    for (int i = 0; i < I; ++i) x[i] = r[i];
    // layer 1 in groups of 4 neurons (4 DADD chains in flight) — the group loop is
    // not unrolled so the weights are not all hoisted into registers at once
    constexpr int G1 = (H1 + 3) / 4;
#pragma unroll 1
    for (int gi = 0; gi < G1; ++gi) {
      double z[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) z[k] = (gi * 4 + k < H1) ? w[B1 + gi * 4 + k] : 0.0;
#pragma unroll
      for (int i = 0; i < I; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (gi * 4 + k < H1) z[k] = __dadd_rn(z[k], __dmul_rn(w[W1 + (gi * 4 + k) * I + i], x[i]));
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (gi * 4 + k < H1) r[A1 + gi * 4 + k] = z[k] > 0.0 ? z[k] : 0.0;
    }
    double a1[H1];
#pragma unroll
    for (int o = 0; o < H1; ++o) a1[o] = r[A1 + o];
    double a2[H2 > 0 ? H2 : 1];
    double z;
    if constexpr (H2 > 0) {
#pragma unroll
      for (int o = 0; o < H2; ++o) a2[o] = w[B2 + o];
#pragma unroll
      for (int i = 0; i < H1; ++i)
#pragma unroll
        for (int o = 0; o < H2; ++o) a2[o] = __dadd_rn(a2[o], __dmul_rn(w[W2 + o * H1 + i], a1[i]));
#pragma unroll
      for (int o = 0; o < H2; ++o) {
        a2[o] = a2[o] > 0.0 ? a2[o] : 0.0;
        r[A2 + o] = a2[o];
      }
      z = w[BO];
#pragma unroll
      for (int i = 0; i < H2; ++i) z = __dadd_rn(z, __dmul_rn(w[WO + i], a2[i]));
    } else {
      z = w[BO];
#pragma unroll
      for (int i = 0; i < H1; ++i) z = __dadd_rn(z, __dmul_rn(w[WO + i], a1[i]));
    }
    const double err = __dsub_rn(z, y);
    r[E2] = __dmul_rn(err, err);
    const double dout = __dmul_rn(2.0, err);
    r[TO] = __dmul_rn(inv_n, dout);
    if constexpr (H2 > 0) {
      double d2[H2];
#pragma unroll
      for (int i = 0; i < H2; ++i) {
        const double acc = __dadd_rn(0.0, __dmul_rn(w[WO + i], dout));
        d2[i] = a2[i] > 0.0 ? acc : 0.0;
        r[T2 + i] = __dmul_rn(inv_n, d2[i]);
      }
      double acc[H1];
#pragma unroll
      for (int i = 0; i < H1; ++i) acc[i] = 0.0;
#pragma unroll
      for (int o = 0; o < H2; ++o)
#pragma unroll
        for (int i = 0; i < H1; ++i) acc[i] = __dadd_rn(acc[i], __dmul_rn(w[W2 + o * H1 + i], d2[o]));
#pragma unroll
      for (int i = 0; i < H1; ++i) r[T1 + i] = __dmul_rn(inv_n, a1[i] > 0.0 ? acc[i] : 0.0);
    } else {
#pragma unroll
      for (int i = 0; i < H1; ++i) {
        const double acc = __dadd_rn(0.0, __dmul_rn(w[WO + i], dout));
        r[T1 + i] = __dmul_rn(inv_n, a1[i] > 0.0 ? acc : 0.0);
      }
    }
  }
};

// ---- phase A, generic shape (runtime loops) ------------------------------------------
__device__ void sample_generic(const Shape& sh, const double* __restrict__ w, double* __restrict__ r,
                               double y, double inv_n) {
  for (int l = 0; l < sh.nl; ++l) {
    const int in = sh.dims[l], out = sh.dims[l + 1];
    const double* wl = w + sh.woff[l];
    const double* bl = w + sh.boff[l];
    const double* ain = r + sh.inoff[l];
    if (l + 1 < sh.nl) {
      double* aout = r + sh.inoff[l + 1];
      for (int o = 0; o < out; o += 4) {  // four independent DADD chains in flight
        const int n4 = out - o < 4 ? out - o : 4;
        double z[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) z[k] = k < n4 ? bl[o + k] : 0.0;
        for (int i = 0; i < in; ++i) {
          const double ai = ain[i];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (k < n4) z[k] = __dadd_rn(z[k], __dmul_rn(wl[(o + k) * in + i], ai));
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k < n4) aout[o + k] = z[k] > 0.0 ? z[k] : 0.0;
      }
    } else {
      double z = bl[0];
      for (int i = 0; i < in; ++i) z = __dadd_rn(z, __dmul_rn(wl[i], ain[i]));
      const double err = __dsub_rn(z, y);
      r[sh.e2] = __dmul_rn(err, err);
      r[sh.toff[l]] = __dmul_rn(2.0, err);  // unscaled output delta (mlp.cpp:92)
    }
  }
  for (int l = sh.nl - 2; l >= 0; --l) {  // hidden deltas from the next layer's, unscaled
    const int nin = sh.dims[l + 1], nout = sh.dims[l + 2];
    const double* wn = w + sh.woff[l + 1];
    const double* dn = r + sh.toff[l + 1];
    const double* act = r + sh.inoff[l + 1];
    double* d = r + sh.toff[l];
    for (int i = 0; i < nin; i += 4) {
      const int n4 = nin - i < 4 ? nin - i : 4;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int o = 0; o < nout; ++o) {
        const double dno = dn[o];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k < n4) acc[k] = __dadd_rn(acc[k], __dmul_rn(wn[o * nin + i + k], dno));
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < n4) d[i + k] = act[i + k] > 0.0 ? acc[k] : 0.0;
    }
  }
  // scale in place: t = inv_n * delta (the left factor of mlp.cpp:113,117)
  const int nd = sh.e2 - sh.toff[0];
  for (int j = 0; j < nd; ++j) r[sh.toff[0] + j] = __dmul_rn(inv_n, r[sh.toff[0] + j]);
}

// Sequential sum over samples of t[s] * a[s] (or t[s] alone when ap is null), in sample
// order, with the shared-memory loads of batch b+1 issued before the DADD chain of
// batch b so only the 8-cycle DADD latency is exposed.
// Two alternating register buffers (A, B) of U samples each: while one batch's DADD
// chain runs, the other batch's loads are in flight; no register copies.
template <int U, bool kMul>
__device__ __forceinline__ double chain_sum_impl(const double* __restrict__ tp,
                                                 const double* __restrict__ ap, int N, int R) {
  double g = 0.0;
  double ta[U], xa[U], tb[U], xb[U];
  auto load = [&](int s0, double* t, double* x) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      t[u] = tp[(s0 + u) * R];
      if (kMul) x[u] = ap[(s0 + u) * R];
    }
  };
  auto consume = [&](const double* t, const double* x) {
#pragma unroll
    for (int u = 0; u < U; ++u) g = __dadd_rn(g, kMul ? __dmul_rn(t[u], x[u]) : t[u]);
  };
  int s = 0;
  if (N >= U) load(0, ta, xa);
  for (; s + 2 * U <= N; s += 2 * U) {
    load(s + U, tb, xb);
    consume(ta, xa);
    if (s + 3 * U <= N) load(s + 2 * U, ta, xa);
    consume(tb, xb);
  }
  if (s + U <= N) {
    consume(ta, xa);
    s += U;
  }
  for (; s < N; ++s) g = __dadd_rn(g, kMul ? __dmul_rn(tp[s * R], ap[s * R]) : tp[s * R]);
  return g;
}

template <int U>
__device__ __forceinline__ double chain_sum(const double* __restrict__ tp, const double* __restrict__ ap,
                                            int N, int R) {
  return ap ? chain_sum_impl<U, true>(tp, ap, N, R) : chain_sum_impl<U, false>(tp, nullptr, N, R);
}

template <int KB, int I, int H1, int H2, bool SMEM>
__global__ void __launch_bounds__(256) train_fp64_exact(TrainArgs a) {
  constexpr bool kFixed = I > 0;
  using F = Fixed<(I > 0 ? I : 1), (H1 > 0 ? H1 : 1), H2>;
  extern __shared__ double smem[];
  const int m = a.order[blockIdx.x];
  const int tile = a.model_tile[m];
  const int N = a.tile_rows[tile];
  const int E = a.epochs[m];
  const double lr = a.lr[m];
  const Shape sh = make_shape(a.tile_inputs[tile], a.h1[m], a.h2[m]);
  const int P = sh.P;
  const int R = kFixed ? F::R : sh.R;
  const int tid = threadIdx.x, nt = blockDim.x;

  double* w = smem;           // [P]
  double* mom = w + P;        // [P] Adam m
  double* vel = mom + P;      // [P] Adam v
  double* Ls = vel + P;       // [1] epoch loss
  // SMEM: records follow the model state in shared memory (a pointer the compiler can
  // prove is shared, so every record access is an LDS/STS); else per-model global scratch
  double* rec;
  if constexpr (SMEM) rec = Ls + 2;
  else rec = a.scratch + a.scratch_offset[m];

  const double* gp = a.params + a.param_offset[m];
  for (int p = tid; p < P; p += nt) {
    w[p] = gp[p];
    mom[p] = 0.0;
    vel[p] = 0.0;
  }
  const double* X = a.X + a.tile_offset[tile] * 8;
  const double* Y = a.y + a.tile_offset[tile];
  for (int s = tid; s < N; s += nt) {
    for (int i = 0; i < 7; ++i) rec[(size_t)s * R + i] = X[(size_t)s * 8 + i];
    rec[(size_t)s * R + 7] = Y[s];  // inputs use slots 0..I-1 (I <= 7): slot 7 holds the target
    rec[(size_t)s * R + R - 1] = 1.0;  // padding slot: bias terms are t * 1.0 (exact)
  }

  // phase-B ownership: parameter p -> (record offset of its delta, of its input or -1)
  int tix[KB], aix[KB];
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    const int p = tid + k * nt;
    tix[k] = -1;
    aix[k] = -1;
    if (p < P) {
      for (int l = 0; l < sh.nl; ++l) {
        const int in = sh.dims[l], out = sh.dims[l + 1];
        if (p >= sh.woff[l] && p < sh.boff[l]) {
          const int q = p - sh.woff[l];
          tix[k] = sh.toff[l] + q / in;
          aix[k] = sh.inoff[l] + q % in;
        } else if (p >= sh.boff[l] && p < sh.boff[l] + out) {
          tix[k] = sh.toff[l] + (p - sh.boff[l]);
          aix[k] = sh.R - 1;  // x 1.0: every lane of a warp runs the same multiply-add chain
        }
      }
    }
  }
  const int e2off = sh.e2;
  const int loss_tid = nt - 1;
  const double inv_n = 1.0 / (double)N;  // mlp.cpp:84
  const double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
  const double c1 = 1.0 - beta1, c2 = 1.0 - beta2;
  double* trace = a.loss_trace ? a.loss_trace + a.trace_offset[m] : nullptr;
  int bad = -1;
  double last = 0.0;
  __syncthreads();

  const bool prof = a.phase_cycles && blockIdx.x == 0 && tid == 0;
  long long pc[4] = {0, 0, 0, 0};
  for (int e = 0; e < E; ++e) {
    const long long clk0 = prof ? clock64() : 0;
    const double2 bc = a.bias_corr[e];  // issued early: its latency hides behind phase A
    // ---- phase A: per-sample forward / backward (mlp.cpp:86-104) ----
    for (int s = tid; s < N; s += nt) {
      double* r = rec + (size_t)s * R;
      if constexpr (kFixed) F::sample(w, r, r[7], inv_n);  // y cached in record slot 7
      else sample_generic(sh, w, r, Y[s], inv_n);
    }
    __syncthreads();
    const long long clk1 = prof ? clock64() : 0;

    // ---- phase B: sequential per-parameter sums + Adam (mlp.cpp:106-118, 142-154) ----
    double g[KB];
#pragma unroll
    for (int k = 0; k < KB; ++k) g[k] = 0.0;
    long long clk2 = 0;
    if (tix[0] >= 0) {
      if (KB == 1) {
        g[0] = chain_sum<8>(rec + tix[0], aix[0] >= 0 ? rec + aix[0] : nullptr, N, R);
        if (prof) clk2 = clock64();
      } else {
        for (int s = 0; s < N; ++s) {
          const double* r = rec + (size_t)s * R;
#pragma unroll
          for (int k = 0; k < KB; ++k) {
            if (tix[k] >= 0) {
              const double t = r[tix[k]];
              g[k] = __dadd_rn(g[k], aix[k] >= 0 ? __dmul_rn(t, r[aix[k]]) : t);
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        const int p = tid + k * nt;
        if (tix[k] >= 0) {
          const double mk = __dadd_rn(__dmul_rn(beta1, mom[p]), __dmul_rn(c1, g[k]));
          const double vk = __dadd_rn(__dmul_rn(beta2, vel[p]), __dmul_rn(__dmul_rn(c2, g[k]), g[k]));
          mom[p] = mk;
          vel[p] = vk;
          const double mhat = __ddiv_rn(mk, bc.x);
          const double vhat = __ddiv_rn(vk, bc.y);
          w[p] = __dsub_rn(w[p], __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps)));
        }
      }
    }
    if (tid == loss_tid) {
      double L = chain_sum<8>(rec + e2off, nullptr, N, R);
      L = __dmul_rn(L, inv_n);  // mlp.cpp:120
      Ls[0] = L;
      if (trace && (e % a.trace_stride) == 0) trace[e / a.trace_stride] = L;
    }
    const long long clk3 = prof ? clock64() : 0;
    __syncthreads();
    if (prof) {
      const long long clk4 = clock64();
      pc[0] += clk1 - clk0;  // phase A + barrier
      pc[1] += clk2 - clk1;  // parameter-0 chain
      pc[2] += clk3 - clk2;  // its Adam step
      pc[3] += clk4 - clk3;  // waiting for the slowest chain / loss
    }
    last = Ls[0];
    if (!isfinite(last)) {  // mlp.cpp:166-169: TrainingError(epoch) before the update
      bad = e;
      break;
    }
  }
  if (prof)
    for (int k = 0; k < 4; ++k) a.phase_cycles[k] = pc[k];

  double* outp = a.params + a.param_offset[m];
  for (int p = tid; p < P; p += nt) outp[p] = w[p];
  if (tid == 0) {
    a.final_loss[m] = last;
    a.nonfinite_epoch[m] = bad;
  }
}

}  // namespace

int fp64_record_doubles(int in, int h1, int h2) {
  (void)in;
  return rec_stride(h1, h2);
}

bool fp64_shape_compiled(int in, int h1, int h2) {
  if (h1 == 8 && h2 == 0) return in >= 1 && in <= 7;
  if (h1 == 5 && h2 == 5) return in >= 4 && in <= 6;
  return false;
}

// Dynamic shared memory = (3P + 2) doubles of model state, plus the per-sample
// records when a.smem_records is set; the host sizes dyn_bytes for the largest model.
// shape = {I, H1, H2} when every model of the launch has that compiled shape, else {0,0,0}.
void launch_train_fp64(const TrainArgs& a, int max_p, int dyn_bytes, const int* shape,
                       cudaStream_t s) {
  const int block = 256;
  const int kb = (max_p + block - 1) / block;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_bytes);
    kern<<<a.n_models, block, dyn_bytes, s>>>(a);
  };
  if (shape && shape[0] > 0 && kb <= 1 && a.smem_records) {
    const int I = shape[0], H1 = shape[1], H2 = shape[2];
    if (H1 == 8 && H2 == 0) {
      switch (I) {
        case 1: return go(train_fp64_exact<1, 1, 8, 0, true>);
        case 2: return go(train_fp64_exact<1, 2, 8, 0, true>);
        case 3: return go(train_fp64_exact<1, 3, 8, 0, true>);
        case 4: return go(train_fp64_exact<1, 4, 8, 0, true>);
        case 5: return go(train_fp64_exact<1, 5, 8, 0, true>);
        case 6: return go(train_fp64_exact<1, 6, 8, 0, true>);
        case 7: return go(train_fp64_exact<1, 7, 8, 0, true>);
      }
    } else if (H1 == 5 && H2 == 5) {
      switch (I) {
        case 4: return go(train_fp64_exact<1, 4, 5, 5, true>);
        case 5: return go(train_fp64_exact<1, 5, 5, 5, true>);
        case 6: return go(train_fp64_exact<1, 6, 5, 5, true>);
      }
    }
  }
  if (a.smem_records) {
    if (kb <= 1) go(train_fp64_exact<1, 0, 0, 0, true>);
    else if (kb <= 2) go(train_fp64_exact<2, 0, 0, 0, true>);
    else if (kb <= 4) go(train_fp64_exact<4, 0, 0, 0, true>);
    else go(train_fp64_exact<kMaxKB, 0, 0, 0, true>);
  } else {
    if (kb <= 1) go(train_fp64_exact<1, 0, 0, 0, false>);
    else if (kb <= 2) go(train_fp64_exact<2, 0, 0, 0, false>);
    else if (kb <= 4) go(train_fp64_exact<4, 0, 0, 0, false>);
    else go(train_fp64_exact<kMaxKB, 0, 0, 0, false>);
  }
}

}  // namespace lann
