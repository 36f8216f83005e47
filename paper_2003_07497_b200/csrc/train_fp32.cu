// train_fp32.cu — K1b: the FP32 throughput LANN trainer.
//
// Same algorithm as models::train_full_batch (mlp.cpp:156-175): full-batch
// MSE gradient (mlp.cpp:75-122) + Adam(0.9, 0.999, 1e-8) (mlp.cpp:142-154),
// loss recorded before each update, training stopped at the first non-finite
// loss. Differences from the FP64 parity kernel: FP32 FMA arithmetic and tree
// reductions over samples, so traces agree with the reference only up to FP32
// rounding.
//
// Two mappings, chosen by population size (engine.cpp build_plan):
//  * train_fp32_kernel<K> — MANY models (sweeps): one warp per CTA trains 32/K
//    models that share one training tile (same combination and fold, different
//    init seeds); each model spreads over K lanes that split its samples.
//    Weights and gradient accumulators live in registers (fully unrolled for the
//    compile-time shape); with K = 1 all 32 lanes read the same row (shared-
//    memory broadcast); with K > 1 the per-lane partials are summed by a shuffle
//    butterfly, after which every lane applies the identical Adam step.
//  * train_fp32_h8_kernel<K> — the same mapping for the one-hidden-layer-of-8
//    prediction nets with hidden units paired on the packed FP32 FMA (FFMA2).
//  * train_fp32_h55_kernel<K> — the same for the 5-5 selection nets (two FFMA2 pairs and
//    one scalar unit per layer).
//  * train_fp32_cta_kernel<W> — FEW models (the 48-combo population): one model
//    per CTA of W warps so the per-epoch LATENCY is minimised; threads own
//    samples (two per thread, interleaved in one basic block); gradients are
//    reduced inside each warp by a register-only recursive-halving reduce-scatter
//    without power-of-two padding (LeanRS; a shared-memory transpose variant is
//    kept for comparison) and then across warps through shared memory; owner
//    threads apply Adam; new weights are broadcast back through shared memory
//    (two __syncthreads per epoch).
// In both, the tile (N rows x 8 floats, target y in column 7) is staged ONCE into
// shared memory by a TMA bulk copy (cp.async.bulk + mbarrier) and re-read from
// there every epoch, so HBM traffic per model-epoch is ~0.
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"

namespace lann {
namespace {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// mbarrier init by one thread; the caller syncs before anyone waits on it.
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  const uint32_t b = smem_addr(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// TMA 1-D bulk copy global -> shared, completion tracked by an (initialised) mbarrier.
__device__ __forceinline__ void tma_load_tile(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar) {
  const uint32_t b = smem_addr(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t b = smem_addr(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(b),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Flat parameter layout of the reference (mlp.cpp:124-131): L0.w [H1][I], L0.b,
// then (2 hidden) L1.w [H2][H1], L1.b, then output w, b.
template <int I, int H1, int H2>
struct Net {
  static constexpr int L1W = 0;
  static constexpr int L1B = I * H1;
  static constexpr int L2W = L1B + H1;
  static constexpr int L2B = H2 > 0 ? L2W + H1 * H2 : L2W + H1;
  static constexpr int L3W = L2B + (H2 > 0 ? H2 : 1);
  static constexpr int L3B = H2 > 0 ? L3W + H2 : L3W;
  static constexpr int P = H2 > 0 ? L3B + 1 : L2B + 1;
};

// Forward + backward of ONE sample, accumulating its gradient contribution into gr
// and err^2 into loss. scale = 2/N folds the 1/N of the mean and the 2 of d(err^2).
// kFirst: gr and loss are ASSIGNED this sample's terms (no zeroing pass, FMUL for FFMA).
template <int I, int H1, int H2, bool kFirst = false>
__device__ __forceinline__ void accumulate_sample(const float* w, const float* xv, float* gr,
                                                  float& loss, float scale, bool valid = true) {
  auto acc = [](float& g, float v) { g = kFirst ? v : g + v; };
  auto fma_acc = [](float& g, float x, float y) { g = kFirst ? x * y : fmaf(x, y, g); };
  using N = Net<I, H1, H2>;
  float z1[H1];
#pragma unroll
  for (int h = 0; h < H1; ++h) {
    float z = w[N::L1B + h];
#pragma unroll
    for (int i = 0; i < I; ++i) z = fmaf(w[N::L1W + h * I + i], xv[i], z);
    z1[h] = fmaxf(z, 0.f);
  }
  float out;
  float z2[H2 > 0 ? H2 : 1];
  if constexpr (H2 > 0) {
#pragma unroll
    for (int o = 0; o < H2; ++o) {
      float z = w[N::L2B + o];
#pragma unroll
      for (int h = 0; h < H1; ++h) z = fmaf(w[N::L2W + o * H1 + h], z1[h], z);
      z2[o] = fmaxf(z, 0.f);
    }
    float acc0 = w[N::L3B], acc1 = 0.f;
#pragma unroll
    for (int o = 0; o < H2; ++o) {
      if (o & 1) acc1 = fmaf(w[N::L3W + o], z2[o], acc1);
      else acc0 = fmaf(w[N::L3W + o], z2[o], acc0);
    }
    out = acc0 + acc1;
  } else {
    float acc0 = w[N::L2B], acc1 = 0.f;
#pragma unroll
    for (int h = 0; h < H1; ++h) {
      if (h & 1) acc1 = fmaf(w[N::L2W + h], z1[h], acc1);
      else acc0 = fmaf(w[N::L2W + h], z1[h], acc0);
    }
    out = acc0 + acc1;
  }
  const float err = valid ? out - xv[7] : 0.f;
  fma_acc(loss, err, err);
  const float d = err * scale;
  if constexpr (H2 > 0) {
    acc(gr[N::L3B], d);
    float d2[H2];
#pragma unroll
    for (int o = 0; o < H2; ++o) {
      fma_acc(gr[N::L3W + o], d, z2[o]);
      d2[o] = z2[o] > 0.f ? w[N::L3W + o] * d : 0.f;
      acc(gr[N::L2B + o], d2[o]);
    }
#pragma unroll
    for (int h = 0; h < H1; ++h) {
      float bd = 0.f;
#pragma unroll
      for (int o = 0; o < H2; ++o) {
        fma_acc(gr[N::L2W + o * H1 + h], d2[o], z1[h]);
        bd = o == 0 ? w[N::L2W + h] * d2[0] : fmaf(w[N::L2W + o * H1 + h], d2[o], bd);
      }
      const float d1 = z1[h] > 0.f ? bd : 0.f;
      acc(gr[N::L1B + h], d1);
#pragma unroll
      for (int i = 0; i < I; ++i) fma_acc(gr[N::L1W + h * I + i], d1, xv[i]);
    }
  } else {
    acc(gr[N::L2B], d);
#pragma unroll
    for (int h = 0; h < H1; ++h) {
      fma_acc(gr[N::L2W + h], d, z1[h]);
      const float d1 = z1[h] > 0.f ? w[N::L2W + h] * d : 0.f;
      acc(gr[N::L1B + h], d1);
#pragma unroll
      for (int i = 0; i < I; ++i) fma_acc(gr[N::L1W + h * I + i], d1, xv[i]);
    }
  }
}

__device__ __forceinline__ void load_row(const float* trow, int s, float* xv) {
  const float4 lo = *reinterpret_cast<const float4*>(trow + s * 8);
  const float4 hi = *reinterpret_cast<const float4*>(trow + s * 8 + 4);
  xv[0] = lo.x; xv[1] = lo.y; xv[2] = lo.z; xv[3] = lo.w;
  xv[4] = hi.x; xv[5] = hi.y; xv[6] = hi.z; xv[7] = hi.w;
}

// One Adam step in FP32 (mlp.cpp:142-154): m = 0.9m + 0.1g, v = 0.999v + 0.001g^2,
// w -= lr/bc1 * m / (sqrt(v/bc2) + 1e-8), with step = lr/bc1 and rb2 = 1/bc2.
__device__ __forceinline__ float adam_step(float& mo, float& ve, float g, float step, float rb2) {
  mo = fmaf(0.1f, g, 0.9f * mo);
  ve = fmaf(0.001f * g, g, 0.999f * ve);
  return step * mo * rcp_approx(sqrt_approx(ve * rb2) + 1e-8f);
}

// ---------------------------------------------------------------------------------
template <int I, int H1, int H2, int K>
__global__ void __launch_bounds__(32) train_fp32_kernel(TrainF32Args a) {
  constexpr int P = Net<I, H1, H2>::P;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bar;
  const int lane = threadIdx.x;
  const int g = blockIdx.x;
  const int first = a.group_first[g];
  const int count = a.group_count[g];
  const int slot = lane / K, sub = lane % K;
  const bool active = slot < count;
  const int m = a.sorted_model[first + (active ? slot : 0)];
  const int tile = a.model_tile[m];
  const int rows = a.tile_rows[tile];
  const int E = a.epochs[m];

  float* trow = reinterpret_cast<float*>(smem_raw);  // [rows][8]
  float* adam = trow + (size_t)rows * 8;            // [2][P][32]
  if (lane == 0) mbar_init(&bar);
  __syncwarp();
  if (lane == 0) tma_load_tile(trow, a.rows + a.tile_offset[tile] * 8, (uint32_t)rows * 32u, &bar);

  float w[P], gr[P];
  const double* gp = a.params + a.param_offset[m];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    w[p] = (float)gp[p];
    adam[p * 32 + lane] = 0.f;
    adam[(P + p) * 32 + lane] = 0.f;
  }
  const float lr = (float)a.lr[m];
  const float scale = 2.0f / (float)rows;
  const float inv_n = 1.0f / (float)rows;
  double* trace = (a.loss_trace && active) ? a.loss_trace + a.trace_offset[m] : nullptr;
  int bad = -1;
  float last = 0.f, pw1 = 1.f, pw2 = 1.f;
  mbar_wait(&bar, 0);
  __syncwarp();

  for (int e = 0; e < E; ++e) {
#pragma unroll
    for (int p = 0; p < P; ++p) gr[p] = 0.f;
    float loss = 0.f;
    for (int s = sub; s < rows; s += K) {
      float xv[8];
      load_row(trow, s, xv);
      accumulate_sample<I, H1, H2>(w, xv, gr, loss, scale);
    }
    // sum the K per-lane partials of each model (lanes slot*K .. slot*K+K-1)
#pragma unroll
    for (int off = 1; off < K; off <<= 1) {
#pragma unroll
      for (int p = 0; p < P; ++p) gr[p] += __shfl_xor_sync(0xffffffffu, gr[p], off);
      loss += __shfl_xor_sync(0xffffffffu, loss, off);
    }
    loss *= inv_n;
    pw1 *= 0.9f;
    pw2 *= 0.999f;
    if (bad < 0) {
      last = loss;
      if (trace && sub == 0 && (e % a.trace_stride) == 0) trace[e / a.trace_stride] = (double)loss;
      if (!isfinite(loss)) {
        bad = e;  // TrainingError(epoch): freeze, keep the warp converged
      } else {
        const float step = lr / (1.f - pw1), rb2 = 1.f / (1.f - pw2);
#pragma unroll
        for (int p = 0; p < P; ++p)
          w[p] -= adam_step(adam[p * 32 + lane], adam[(P + p) * 32 + lane], gr[p], step, rb2);
      }
    }
  }
  if (active && sub == 0) {
    double* outp = a.params + a.param_offset[m];
#pragma unroll
    for (int p = 0; p < P; ++p) outp[p] = (double)w[p];
    a.final_loss[m] = (double)last;
    a.nonfinite_epoch[m] = bad;
  }
}

// ---------------------------------------------------------------------------------
// Packed variant of train_fp32_kernel for the prediction nets (one hidden layer of 8):
// hidden units are paired and every pair runs on sm_100's packed FP32 FMA
// (fma.rn.f32x2 -> FFMA2, two FMAs per issue slot; the sample feature is a broadcast
// scalar operand). The unpacked kernel is issue-bound (179 instructions per sample, 149
// on the FMA pipe; profiles/r01_*); this one issues ~110 for the same 277 FLOP.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk(f32x2 p, float& a, float& b) {
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(p));
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

template <int I, int K>
__global__ void __launch_bounds__(32) train_fp32_h8_kernel(TrainF32Args a) {
  constexpr int HP = 4;  // hidden pairs (h = 2q, 2q+1)
  using N = Net<I, 8, 0>;
  constexpr int P = N::P;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bar;
  const int lane = threadIdx.x;
  const int first = a.group_first[blockIdx.x];
  const int count = a.group_count[blockIdx.x];
  const int slot = lane / K, sub = lane % K;
  const bool active = slot < count;
  const int m = a.sorted_model[first + (active ? slot : 0)];
  const int tile = a.model_tile[m];
  const int rows = a.tile_rows[tile];
  const int E = a.epochs[m];
  float* trow = reinterpret_cast<float*>(smem_raw);  // [rows][8]
  float* adam = trow + (size_t)rows * 8;            // [2][P][32], canonical parameter order
  if (lane == 0) mbar_init(&bar);
  __syncwarp();
  if (lane == 0) tma_load_tile(trow, a.rows + a.tile_offset[tile] * 8, (uint32_t)rows * 32u, &bar);

  const double* gp = a.params + a.param_offset[m];
  f32x2 w1[I][HP], b1[HP], w2[HP];
  float b2 = (float)gp[N::L2B];
#pragma unroll
  for (int q = 0; q < HP; ++q) {
#pragma unroll
    for (int i = 0; i < I; ++i)
      w1[i][q] = pk((float)gp[N::L1W + (2 * q) * I + i], (float)gp[N::L1W + (2 * q + 1) * I + i]);
    b1[q] = pk((float)gp[N::L1B + 2 * q], (float)gp[N::L1B + 2 * q + 1]);
    w2[q] = pk((float)gp[N::L2W + 2 * q], (float)gp[N::L2W + 2 * q + 1]);
  }
  for (int p = 0; p < P; ++p) {
    adam[p * 32 + lane] = 0.f;
    adam[(P + p) * 32 + lane] = 0.f;
  }
  const float lr = (float)a.lr[m];
  const float scale = 2.0f / (float)rows;
  const float inv_n = 1.0f / (float)rows;
  double* trace = (a.loss_trace && active) ? a.loss_trace + a.trace_offset[m] : nullptr;
  int bad = -1;
  float last = 0.f, pw1 = 1.f, pw2 = 1.f;
  mbar_wait(&bar, 0);
  __syncwarp();

  for (int e = 0; e < E; ++e) {
    f32x2 g1[I][HP], gb1[HP], gw2[HP];
    const f32x2 zero2 = pk(0.f, 0.f);
#pragma unroll
    for (int q = 0; q < HP; ++q) {
#pragma unroll
      for (int i = 0; i < I; ++i) g1[i][q] = zero2;
      gb1[q] = zero2;
      gw2[q] = zero2;
    }
    float gb2 = 0.f, loss = 0.f;
    auto step = [&](int s, bool valid) {  // valid = false: a padding sample, no contribution
      float xv[8];
      load_row(trow, s, xv);
      f32x2 xx[I];
#pragma unroll
      for (int i = 0; i < I; ++i) xx[i] = pk(xv[i], xv[i]);
      f32x2 z[HP];
#pragma unroll
      for (int q = 0; q < HP; ++q) {
        z[q] = b1[q];
#pragma unroll
        for (int i = 0; i < I; ++i) z[q] = fma2(w1[i][q], xx[i], z[q]);
      }
      f32x2 act[HP];
      float za[HP], zb[HP];
#pragma unroll
      for (int q = 0; q < HP; ++q) {
        upk(z[q], za[q], zb[q]);
        act[q] = pk(fmaxf(za[q], 0.f), fmaxf(zb[q], 0.f));
      }
      // two partial accumulators halve the output chain
      f32x2 acc0 = fma2(w2[0], act[0], pk(b2, 0.f)), acc1 = mul2(w2[1], act[1]);
#pragma unroll
      for (int q = 2; q < HP; ++q) {
        if (q & 1) acc1 = fma2(w2[q], act[q], acc1);
        else acc0 = fma2(w2[q], act[q], acc0);
      }
      float o0, o1;
      upk(add2(acc0, acc1), o0, o1);
      const float err = valid ? (o0 + o1) - xv[7] : 0.f;
      loss = fmaf(err, err, loss);
      const float d = err * scale;
      const f32x2 dd = pk(d, d);
      gb2 += d;
#pragma unroll
      for (int q = 0; q < HP; ++q) {
        gw2[q] = fma2(dd, act[q], gw2[q]);
        float ta, tb;
        upk(mul2(w2[q], dd), ta, tb);
        const f32x2 dq = pk(za[q] > 0.f ? ta : 0.f, zb[q] > 0.f ? tb : 0.f);
        gb1[q] = add2(gb1[q], dq);
#pragma unroll
        for (int i = 0; i < I; ++i) g1[i][q] = fma2(dq, xx[i], g1[i][q]);
      }
    };
    // (two samples per trip was measured slower here: 254 registers, 574 vs 528 ms on the sweep)
    for (int s = sub; s < rows; s += K) step(s, true);
    // sum the K per-lane partials of each model
#pragma unroll
    for (int off = 1; off < K; off <<= 1) {
      auto red = [&](f32x2& v) {
        float lo, hi;
        upk(v, lo, hi);
        lo += __shfl_xor_sync(0xffffffffu, lo, off);
        hi += __shfl_xor_sync(0xffffffffu, hi, off);
        v = pk(lo, hi);
      };
#pragma unroll
      for (int q = 0; q < HP; ++q) {
#pragma unroll
        for (int i = 0; i < I; ++i) red(g1[i][q]);
        red(gb1[q]);
        red(gw2[q]);
      }
      gb2 += __shfl_xor_sync(0xffffffffu, gb2, off);
      loss += __shfl_xor_sync(0xffffffffu, loss, off);
    }
    loss *= inv_n;
    pw1 *= 0.9f;
    pw2 *= 0.999f;
    if (bad < 0) {
      last = loss;
      if (trace && sub == 0 && (e % a.trace_stride) == 0) trace[e / a.trace_stride] = (double)loss;
      if (!isfinite(loss)) {
        bad = e;
      } else {
        const float step = lr / (1.f - pw1), rb2 = 1.f / (1.f - pw2);
        auto upd = [&](f32x2& wv, f32x2 gv, int p0, int p1) {
          float w0, w1v, g0, g1v;
          upk(wv, w0, w1v);
          upk(gv, g0, g1v);
          w0 -= adam_step(adam[p0 * 32 + lane], adam[(P + p0) * 32 + lane], g0, step, rb2);
          w1v -= adam_step(adam[p1 * 32 + lane], adam[(P + p1) * 32 + lane], g1v, step, rb2);
          wv = pk(w0, w1v);
        };
#pragma unroll
        for (int q = 0; q < HP; ++q) {
#pragma unroll
          for (int i = 0; i < I; ++i) upd(w1[i][q], g1[i][q], N::L1W + 2 * q * I + i, N::L1W + (2 * q + 1) * I + i);
          upd(b1[q], gb1[q], N::L1B + 2 * q, N::L1B + 2 * q + 1);
          upd(w2[q], gw2[q], N::L2W + 2 * q, N::L2W + 2 * q + 1);
        }
        b2 -= adam_step(adam[N::L2B * 32 + lane], adam[(P + N::L2B) * 32 + lane], gb2, step, rb2);
      }
    }
  }
  if (active && sub == 0) {
    double* outp = a.params + a.param_offset[m];
#pragma unroll
    for (int q = 0; q < HP; ++q) {
      float x0, x1;
#pragma unroll
      for (int i = 0; i < I; ++i) {
        upk(w1[i][q], x0, x1);
        outp[N::L1W + 2 * q * I + i] = x0;
        outp[N::L1W + (2 * q + 1) * I + i] = x1;
      }
      upk(b1[q], x0, x1);
      outp[N::L1B + 2 * q] = x0;
      outp[N::L1B + 2 * q + 1] = x1;
      upk(w2[q], x0, x1);
      outp[N::L2W + 2 * q] = x0;
      outp[N::L2W + 2 * q + 1] = x1;
    }
    outp[N::L2B] = b2;
    a.final_loss[m] = (double)last;
    a.nonfinite_epoch[m] = bad;
  }
}

// ---------------------------------------------------------------------------------
// Lean warp reduce-scatter of N values per lane (no power-of-two padding): at offset O
// every lane keeps ceil(n/2) values (the lower half if its O-bit is clear, else the
// upper half, zero-padded when n is odd), sends the other half to lane ^ O and adds what
// it receives. 72 values take 36+18+9+5+3 = 71 shuffles (93 with padding to 96).
// rs_map() gives the span of the original vector lane L finally holds: elements
// base + k for k < valid.
template <int N, int O>
struct LeanRS {
  static constexpr int H = (N + 1) / 2;
  template <int M>
  __device__ __forceinline__ static void run(float (&v)[M], int lane) {
    const bool up = (lane & O) != 0;
    auto half = [&](int j, float& keep, float& send) {
      const float lo = v[j];
      const float hi = (H + j < N) ? v[(H + j < N) ? H + j : 0] : 0.f;
      send = up ? lo : hi;
      keep = up ? hi : lo;
    };
    // pairs of kept values add on one FADD2 (packed f32x2)
#pragma unroll
    for (int j = 0; j + 1 < H; j += 2) {
      float k0, s0, k1, s1;
      half(j, k0, s0);
      half(j + 1, k1, s1);
      const float r0 = __shfl_xor_sync(0xffffffffu, s0, O);
      const float r1 = __shfl_xor_sync(0xffffffffu, s1, O);
      upk(add2(pk(k0, k1), pk(r0, r1)), v[j], v[j + 1]);
    }
    if constexpr (H & 1) {
      float k0, s0;
      half(H - 1, k0, s0);
      v[H - 1] = k0 + __shfl_xor_sync(0xffffffffu, s0, O);
    }
    if constexpr (O > 1) LeanRS<H, O / 2>::run(v, lane);
  }
};
__host__ __device__ constexpr int lean_rs_final(int n) {
  for (int o = 16; o >= 1; o >>= 1) n = (n + 1) / 2;
  return n;
}
__device__ __forceinline__ void lean_rs_map(int n, int lane, int& base, int& valid) {
  base = 0;
  valid = n;
  for (int o = 16; o >= 1; o >>= 1) {
    const int h = (n + 1) / 2;
    if (lane & o) {
      base += h;
      valid = valid > h ? valid - h : 0;
    } else {
      valid = valid < h ? valid : h;
    }
    n = h;
  }
}

// ---------------------------------------------------------------------------------
// Packed variant of train_fp32_kernel for the two-hidden-layer 5-5 selection nets (the sweep's
// blur part): units 0-3 of each layer run as two FFMA2 pairs, unit 4 as a scalar FFMA (no zero
// padding, so no pad moves), the broadcast operand being the input / layer-1 activation. Same
// mapping as train_fp32_kernel<K> (K lanes per model split the samples, butterfly over K,
// identical Adam in every lane); moments in shared memory in the canonical parameter order.
template <int I, int K>
__global__ void __launch_bounds__(32) train_fp32_h55_kernel(TrainF32Args a) {
  using N = Net<I, 5, 5>;
  constexpr int P = N::P;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bar;
  const int lane = threadIdx.x;
  const int first = a.group_first[blockIdx.x];
  const int count = a.group_count[blockIdx.x];
  const int slot = lane / K, sub = lane % K;
  const bool active = slot < count;
  const int m = a.sorted_model[first + (active ? slot : 0)];
  const int tile = a.model_tile[m];
  const int rows = a.tile_rows[tile];
  const int E = a.epochs[m];
  float* trow = reinterpret_cast<float*>(smem_raw);  // [rows][8]
  float* adam = trow + (size_t)rows * 8;            // [2][P][32]
  if (lane == 0) mbar_init(&bar);
  __syncwarp();
  if (lane == 0) tma_load_tile(trow, a.rows + a.tile_offset[tile] * 8, (uint32_t)rows * 32u, &bar);

  const double* gp = a.params + a.param_offset[m];
  auto W = [&](int p) { return (float)gp[p]; };
  // layer 1: pairs (0,1), (2,3) + scalar unit 4; likewise layer 2 and the output weights
  f32x2 w1p[I][2], b1p[2], w2p[5][2], b2p[2], w3p[2];
  float w1s[I], b1s, w2s[5], b2s, w3s, b3;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
#pragma unroll
    for (int i = 0; i < I; ++i) w1p[i][q] = pk(W(N::L1W + (2 * q) * I + i), W(N::L1W + (2 * q + 1) * I + i));
    b1p[q] = pk(W(N::L1B + 2 * q), W(N::L1B + 2 * q + 1));
#pragma unroll
    for (int h = 0; h < 5; ++h) w2p[h][q] = pk(W(N::L2W + (2 * q) * 5 + h), W(N::L2W + (2 * q + 1) * 5 + h));
    b2p[q] = pk(W(N::L2B + 2 * q), W(N::L2B + 2 * q + 1));
    w3p[q] = pk(W(N::L3W + 2 * q), W(N::L3W + 2 * q + 1));
  }
#pragma unroll
  for (int i = 0; i < I; ++i) w1s[i] = W(N::L1W + 4 * I + i);
  b1s = W(N::L1B + 4);
#pragma unroll
  for (int h = 0; h < 5; ++h) w2s[h] = W(N::L2W + 4 * 5 + h);
  b2s = W(N::L2B + 4);
  w3s = W(N::L3W + 4);
  b3 = W(N::L3B);
  for (int p = 0; p < P; ++p) {
    adam[p * 32 + lane] = 0.f;
    adam[(P + p) * 32 + lane] = 0.f;
  }
  const float lr = (float)a.lr[m];
  const float scale = 2.0f / (float)rows;
  const float inv_n = 1.0f / (float)rows;
  double* trace = (a.loss_trace && active) ? a.loss_trace + a.trace_offset[m] : nullptr;
  int bad = -1;
  float last = 0.f, pw1 = 1.f, pw2 = 1.f;
  mbar_wait(&bar, 0);
  __syncwarp();

  for (int e = 0; e < E; ++e) {
    const f32x2 zero2 = pk(0.f, 0.f);
    f32x2 g1p[I][2], gb1p[2], g2p[5][2], gb2p[2], g3p[2];
    float g1s[I], gb1s = 0.f, g2s[5], gb2s = 0.f, g3s = 0.f, gb3 = 0.f, loss = 0.f;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int i = 0; i < I; ++i) g1p[i][q] = zero2;
#pragma unroll
      for (int h = 0; h < 5; ++h) g2p[h][q] = zero2;
      gb1p[q] = gb2p[q] = g3p[q] = zero2;
    }
#pragma unroll
    for (int i = 0; i < I; ++i) g1s[i] = 0.f;
#pragma unroll
    for (int h = 0; h < 5; ++h) g2s[h] = 0.f;
    for (int s = sub; s < rows; s += K) {
      float xv[8];
      load_row(trow, s, xv);
      // layer 1
      f32x2 z1p[2];
      float z1s = b1s;
#pragma unroll
      for (int q = 0; q < 2; ++q) z1p[q] = b1p[q];
#pragma unroll
      for (int i = 0; i < I; ++i) {
        z1p[0] = fma2(w1p[i][0], pk(xv[i], xv[i]), z1p[0]);
        z1p[1] = fma2(w1p[i][1], pk(xv[i], xv[i]), z1p[1]);
        z1s = fmaf(w1s[i], xv[i], z1s);
      }
      float a1[5];
      upk(z1p[0], a1[0], a1[1]);
      upk(z1p[1], a1[2], a1[3]);
      a1[4] = z1s;
#pragma unroll
      for (int h = 0; h < 5; ++h) a1[h] = fmaxf(a1[h], 0.f);
      // layer 2
      f32x2 z2p[2] = {b2p[0], b2p[1]};
      float z2s = b2s;
#pragma unroll
      for (int h = 0; h < 5; ++h) {
        z2p[0] = fma2(w2p[h][0], pk(a1[h], a1[h]), z2p[0]);
        z2p[1] = fma2(w2p[h][1], pk(a1[h], a1[h]), z2p[1]);
        z2s = fmaf(w2s[h], a1[h], z2s);
      }
      float a2[5];
      upk(z2p[0], a2[0], a2[1]);
      upk(z2p[1], a2[2], a2[3]);
      a2[4] = z2s;
#pragma unroll
      for (int o = 0; o < 5; ++o) a2[o] = fmaxf(a2[o], 0.f);
      const f32x2 a2p0 = pk(a2[0], a2[1]), a2p1 = pk(a2[2], a2[3]);
      // output
      float o0, o1;
      upk(fma2(w3p[1], a2p1, mul2(w3p[0], a2p0)), o0, o1);
      const float out = (o0 + o1) + fmaf(w3s, a2[4], b3);
      const float err = out - xv[7];
      loss = fmaf(err, err, loss);
      const float d = err * scale;
      // backward
      gb3 += d;
      g3p[0] = fma2(a2p0, pk(d, d), g3p[0]);
      g3p[1] = fma2(a2p1, pk(d, d), g3p[1]);
      g3s = fmaf(a2[4], d, g3s);
      float d2[5];
      upk(mul2(w3p[0], pk(d, d)), d2[0], d2[1]);
      upk(mul2(w3p[1], pk(d, d)), d2[2], d2[3]);
      d2[4] = w3s * d;
#pragma unroll
      for (int o = 0; o < 5; ++o) d2[o] = a2[o] > 0.f ? d2[o] : 0.f;
      const f32x2 d2p0 = pk(d2[0], d2[1]), d2p1 = pk(d2[2], d2[3]);
      gb2p[0] = add2(gb2p[0], d2p0);
      gb2p[1] = add2(gb2p[1], d2p1);
      gb2s += d2[4];
      float d1[5];
#pragma unroll
      for (int h = 0; h < 5; ++h) {
        g2p[h][0] = fma2(d2p0, pk(a1[h], a1[h]), g2p[h][0]);
        g2p[h][1] = fma2(d2p1, pk(a1[h], a1[h]), g2p[h][1]);
        g2s[h] = fmaf(d2[4], a1[h], g2s[h]);
        float t0, t1;
        upk(fma2(w2p[h][1], d2p1, mul2(w2p[h][0], d2p0)), t0, t1);
        const float acc = (t0 + t1) + w2s[h] * d2[4];
        d1[h] = a1[h] > 0.f ? acc : 0.f;
      }
      const f32x2 d1p0 = pk(d1[0], d1[1]), d1p1 = pk(d1[2], d1[3]);
      gb1p[0] = add2(gb1p[0], d1p0);
      gb1p[1] = add2(gb1p[1], d1p1);
      gb1s += d1[4];
#pragma unroll
      for (int i = 0; i < I; ++i) {
        g1p[i][0] = fma2(d1p0, pk(xv[i], xv[i]), g1p[i][0]);
        g1p[i][1] = fma2(d1p1, pk(xv[i], xv[i]), g1p[i][1]);
        g1s[i] = fmaf(d1[4], xv[i], g1s[i]);
      }
    }
    // sum the K per-lane partials of each model
#pragma unroll
    for (int off = 1; off < K; off <<= 1) {
      auto red2 = [&](f32x2& v) {
        float lo, hi;
        upk(v, lo, hi);
        lo += __shfl_xor_sync(0xffffffffu, lo, off);
        hi += __shfl_xor_sync(0xffffffffu, hi, off);
        v = pk(lo, hi);
      };
      auto red1 = [&](float& v) { v += __shfl_xor_sync(0xffffffffu, v, off); };
#pragma unroll
      for (int q = 0; q < 2; ++q) {
#pragma unroll
        for (int i = 0; i < I; ++i) red2(g1p[i][q]);
#pragma unroll
        for (int h = 0; h < 5; ++h) red2(g2p[h][q]);
        red2(gb1p[q]);
        red2(gb2p[q]);
        red2(g3p[q]);
      }
#pragma unroll
      for (int i = 0; i < I; ++i) red1(g1s[i]);
#pragma unroll
      for (int h = 0; h < 5; ++h) red1(g2s[h]);
      red1(gb1s);
      red1(gb2s);
      red1(g3s);
      red1(gb3);
      red1(loss);
    }
    loss *= inv_n;
    pw1 *= 0.9f;
    pw2 *= 0.999f;
    if (bad < 0) {
      last = loss;
      if (trace && sub == 0 && (e % a.trace_stride) == 0) trace[e / a.trace_stride] = (double)loss;
      if (!isfinite(loss)) {
        bad = e;
      } else {
        const float step = lr / (1.f - pw1), rb2 = 1.f / (1.f - pw2);
        auto upd1 = [&](float& w, float g, int p) {
          w -= adam_step(adam[p * 32 + lane], adam[(P + p) * 32 + lane], g, step, rb2);
        };
        auto upd2 = [&](f32x2& wv, f32x2 gv, int p0, int p1) {
          float w0, w1v, g0, g1v;
          upk(wv, w0, w1v);
          upk(gv, g0, g1v);
          upd1(w0, g0, p0);
          upd1(w1v, g1v, p1);
          wv = pk(w0, w1v);
        };
#pragma unroll
        for (int q = 0; q < 2; ++q) {
#pragma unroll
          for (int i = 0; i < I; ++i) upd2(w1p[i][q], g1p[i][q], N::L1W + 2 * q * I + i, N::L1W + (2 * q + 1) * I + i);
          upd2(b1p[q], gb1p[q], N::L1B + 2 * q, N::L1B + 2 * q + 1);
#pragma unroll
          for (int h = 0; h < 5; ++h) upd2(w2p[h][q], g2p[h][q], N::L2W + 2 * q * 5 + h, N::L2W + (2 * q + 1) * 5 + h);
          upd2(b2p[q], gb2p[q], N::L2B + 2 * q, N::L2B + 2 * q + 1);
          upd2(w3p[q], g3p[q], N::L3W + 2 * q, N::L3W + 2 * q + 1);
        }
#pragma unroll
        for (int i = 0; i < I; ++i) upd1(w1s[i], g1s[i], N::L1W + 4 * I + i);
        upd1(b1s, gb1s, N::L1B + 4);
#pragma unroll
        for (int h = 0; h < 5; ++h) upd1(w2s[h], g2s[h], N::L2W + 20 + h);
        upd1(b2s, gb2s, N::L2B + 4);
        upd1(w3s, g3s, N::L3W + 4);
        upd1(b3, gb3, N::L3B);
      }
    }
  }
  if (active && sub == 0) {
    double* outp = a.params + a.param_offset[m];
    auto put2 = [&](f32x2 v, int p0, int p1) {
      float x0, x1;
      upk(v, x0, x1);
      outp[p0] = x0;
      outp[p1] = x1;
    };
#pragma unroll
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int i = 0; i < I; ++i) put2(w1p[i][q], N::L1W + 2 * q * I + i, N::L1W + (2 * q + 1) * I + i);
      put2(b1p[q], N::L1B + 2 * q, N::L1B + 2 * q + 1);
#pragma unroll
      for (int h = 0; h < 5; ++h) put2(w2p[h][q], N::L2W + 2 * q * 5 + h, N::L2W + (2 * q + 1) * 5 + h);
      put2(b2p[q], N::L2B + 2 * q, N::L2B + 2 * q + 1);
      put2(w3p[q], N::L3W + 2 * q, N::L3W + 2 * q + 1);
    }
#pragma unroll
    for (int i = 0; i < I; ++i) outp[N::L1W + 4 * I + i] = w1s[i];
    outp[N::L1B + 4] = b1s;
#pragma unroll
    for (int h = 0; h < 5; ++h) outp[N::L2W + 20 + h] = w2s[h];
    outp[N::L2B + 4] = b2s;
    outp[N::L3W + 4] = w3s;
    outp[N::L3B] = b3;
    a.final_loss[m] = (double)last;
    a.nonfinite_epoch[m] = bad;
  }
}

// ---------------------------------------------------------------------------------
template <int P>
struct CtaLayout {
  static constexpr int PT = (P + 3) & ~3;  // transpose row stride (float4 writes, 4-wavefront STS.128)
};

template <int I, int H1, int H2, int W, bool kShuffleReduce, bool kPair, bool kProf = false, bool kTrace = true>
__global__ void __launch_bounds__(32 * W, 1) train_fp32_cta_kernel(TrainF32Args a) {
  constexpr int P = Net<I, H1, H2>::P;
  constexpr int PT = CtaLayout<P>::PT;
  constexpr int T = 32 * W;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bar;
  __shared__ __align__(16) float wsh[PT];
  __shared__ float part[W][P + 1];  // per-warp partial gradients (+ loss)
  __shared__ float loss_sh[2];  // double-buffered: epoch e is checked at the top of e + 1
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = a.sorted_model[a.group_first[blockIdx.x]];
  const int tile = a.model_tile[m];
  const int rows = a.tile_rows[tile];
  const int E = a.epochs[m];
  float* trow = reinterpret_cast<float*>(smem_raw);                 // [rows][8]
  float* tbuf = trow + (size_t)rows * 8 + (size_t)warp * 32 * PT;  // [32][PT] per warp
  if (tid == 0) mbar_init(&bar);
  __syncthreads();
  if (tid == 0) tma_load_tile(trow, a.rows + a.tile_offset[tile] * 8, (uint32_t)rows * 32u, &bar);
  const double* gp = a.params + a.param_offset[m];
  for (int p = tid; p < PT; p += T) wsh[p] = p < P ? (float)gp[p] : 0.f;
  // owner thread of parameters tid, tid + T, ... (and of the loss slot P): Adam state
  constexpr int OWN = (P + 1 + T - 1) / T;
  float mo[OWN], ve[OWN];
#pragma unroll
  for (int k = 0; k < OWN; ++k) mo[k] = ve[k] = 0.f;
  const float lr = (float)a.lr[m];
  const float scale = 2.0f / (float)rows, inv_n = 1.0f / (float)rows;
  // kTrace = false (launches without a loss trace): the per-epoch trace store compiled out
  double* trace = (kTrace && a.loss_trace) ? a.loss_trace + a.trace_offset[m] : nullptr;
  int bad = -1;
  float last = 0.f;
  int rs_base, rs_valid;
  lean_rs_map(P + 1, lane, rs_base, rs_valid);
  mbar_wait(&bar, 0);
  __syncthreads();

  // kProf (LANN_PHASE_PROFILE launches only): the clock64 phase split; compiled out otherwise
  const bool prof = kProf && a.phase_cycles && blockIdx.x == 0 && tid == 0;
  long long pc[4] = {0, 0, 0, 0};
  // kPair: each thread's two samples are the same every epoch, so their rows stay in registers
  float xa[8], xb[8];
  if constexpr (kPair) {
    load_row(trow, tid < rows ? tid : 0, xa);
    load_row(trow, tid + T < rows ? tid + T : 0, xb);
  }
  const long long clk_begin = prof ? clock64() : 0;
  for (int e = 0; e < E; ++e) {
    const long long clk0 = prof ? clock64() : 0;
    // this epoch's Adam factors (host bias-correction reciprocals), loaded while the samples run
    const float2 br = a.bias_rcp[e];
    const float step = lr * br.x, rb2 = br.y;
    float w[PT];
#pragma unroll
    for (int p = 0; p < PT; p += 4) {
      const float4 v = *reinterpret_cast<const float4*>(wsh + p);
      w[p] = v.x;
      w[p + 1] = v.y;
      w[p + 2] = v.z;
      w[p + 3] = v.w;
    }
    // the previous epoch's loss (pre-update, mlp.cpp:165-172), read here so its shared-memory
    // latency hides behind the weight loads instead of stalling the loop back-edge
    if (e > 0) {
      const float L = loss_sh[(e - 1) & 1];
      last = L;
      if (trace && tid == 0 && ((e - 1) % a.trace_stride) == 0) trace[(e - 1) / a.trace_stride] = (double)L;
      if (!isfinite(L)) {
        bad = e - 1;
        break;  // uniform across the CTA (everyone read the same loss)
      }
    }
    float gr[PT];
    float loss = 0.f;
    if constexpr (kPair) {
      // two samples per thread in one basic block: independent chains interleave; the first
      // sample assigns the accumulators (no zeroing pass)
      if (rows <= 2 * T && tid < rows) {
        accumulate_sample<I, H1, H2, true>(w, xa, gr, loss, scale);
        accumulate_sample<I, H1, H2>(w, xb, gr, loss, scale, tid + T < rows);
#pragma unroll
        for (int p = P; p < PT; ++p) gr[p] = 0.f;
      } else if (rows <= 2 * T) {
#pragma unroll
        for (int p = 0; p < PT; ++p) gr[p] = 0.f;
      } else {
#pragma unroll
        for (int p = 0; p < PT; ++p) gr[p] = 0.f;
        for (int s0 = tid; s0 < rows; s0 += 2 * T) {
          const int s1 = s0 + T;
          float ya[8], yb[8];
          load_row(trow, s0, ya);
          load_row(trow, s1 < rows ? s1 : s0, yb);
          accumulate_sample<I, H1, H2>(w, ya, gr, loss, scale);
          accumulate_sample<I, H1, H2>(w, yb, gr, loss, scale, s1 < rows);
        }
      }
    } else {
#pragma unroll
      for (int p = 0; p < PT; ++p) gr[p] = 0.f;
      for (int s = tid; s < rows; s += T) {
        float xv[8];
        load_row(trow, s, xv);
        accumulate_sample<I, H1, H2>(w, xv, gr, loss, scale);
      }
    }
    const long long clk1 = prof ? clock64() : 0;
    if constexpr (kShuffleReduce) {
      // level 1: lean recursive-halving reduce-scatter in registers (LeanRS): lane L ends
      // with the warp sums of elements rs_base .. rs_base + rs_valid - 1 (loss = element P)
      float v[P + 1];
#pragma unroll
      for (int p = 0; p < P; ++p) v[p] = gr[p];
      v[P] = loss;
      LeanRS<P + 1, 16>::run(v, lane);
#pragma unroll
      for (int k = 0; k < lean_rs_final(P + 1); ++k)
        if (k < rs_valid) part[warp][rs_base + k] = v[k];
    } else {
      // level 1: warp transpose-sum through shared memory (lane j -> params j, j+32, ...)
      float* myrow = tbuf + lane * PT;
#pragma unroll
      for (int p = 0; p < PT; p += 4)
        *reinterpret_cast<float4*>(myrow + p) = make_float4(gr[p], gr[p + 1], gr[p + 2], gr[p + 3]);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) loss += __shfl_xor_sync(0xffffffffu, loss, off);
      __syncwarp();
#pragma unroll
      for (int k = 0; k < (P + 31) / 32; ++k) {
        const int p = lane + 32 * k;
        if (p < P) {
          float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
          for (int r = 0; r < 32; r += 4) {
            s0 += tbuf[(r + 0) * PT + p];
            s1 += tbuf[(r + 1) * PT + p];
            s2 += tbuf[(r + 2) * PT + p];
            s3 += tbuf[(r + 3) * PT + p];
          }
          part[warp][p] = (s0 + s1) + (s2 + s3);
        }
      }
      if (lane == 0) part[warp][P] = loss;
    }
    __syncthreads();
    const long long clk2 = prof ? clock64() : 0;
    // level 2: owners sum the W warp partials and apply Adam
    {
#pragma unroll
      for (int k = 0; k < OWN; ++k) {
        const int p = tid + k * T;
        if (p <= P) {
          float gsum = 0.f;
#pragma unroll
          for (int q = 0; q < W; ++q) gsum += part[q][p];
          if (p == P) loss_sh[e & 1] = gsum * inv_n;
          else wsh[p] -= adam_step(mo[k], ve[k], gsum, step, rb2);
        }
      }
    }
    __syncthreads();
    if (prof) {
      const long long clk3 = clock64();
      pc[0] += clk1 - clk0;  // weight reload + per-sample forward/backward
      pc[1] += clk2 - clk1;  // reduce-scatter + barrier
      pc[2] += clk3 - clk2;  // owner sums + Adam + barrier
    }
  }
  if (bad < 0 && E > 0) {  // the last epoch's loss (every thread passed its final barrier)
    const float L = loss_sh[(E - 1) & 1];
    last = L;
    if (trace && tid == 0 && ((E - 1) % a.trace_stride) == 0) trace[(E - 1) / a.trace_stride] = (double)L;
    if (!isfinite(L)) bad = E - 1;
  }
  if (prof) {
    pc[3] = clock64() - clk_begin;  // the whole epoch loop
    for (int k = 0; k < 4; ++k) a.phase_cycles[k] = pc[k];
  }
  // on a non-finite loss the reference discards the model (TrainingError); so do we
  double* outp = a.params + a.param_offset[m];
  for (int p = tid; p < P; p += T) outp[p] = (double)wsh[p];
  if (tid == 0) {
    a.final_loss[m] = (double)last;
    a.nonfinite_epoch[m] = bad;
  }
}

template <int I, int H1, int H2, int W>
void launch_cta(const TrainF32Args& a, int tile_bytes, cudaStream_t s) {
  constexpr int P = Net<I, H1, H2>::P;
  const char* pe = std::getenv("LANN_CTA_PAIR");
  const bool pair = pe == nullptr || pe[0] != '0';
  if (std::getenv("LANN_CTA_SMEM_REDUCE") == nullptr) {
    const int dyn = tile_bytes;
    if (pair && a.phase_cycles) {
      auto kern = train_fp32_cta_kernel<I, H1, H2, W, true, true, true>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
      kern<<<a.n_groups, 32 * W, dyn, s>>>(a);
    } else if (pair && a.loss_trace) {
      auto kern = train_fp32_cta_kernel<I, H1, H2, W, true, true>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
      kern<<<a.n_groups, 32 * W, dyn, s>>>(a);
    } else if (pair) {
      auto kern = train_fp32_cta_kernel<I, H1, H2, W, true, true, false, false>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
      kern<<<a.n_groups, 32 * W, dyn, s>>>(a);
    } else {
      auto kern = train_fp32_cta_kernel<I, H1, H2, W, true, false>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
      kern<<<a.n_groups, 32 * W, dyn, s>>>(a);
    }
  } else {
    auto kern = train_fp32_cta_kernel<I, H1, H2, W, false, false>;
    const int dyn = tile_bytes + W * 32 * CtaLayout<P>::PT * 4;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    kern<<<a.n_groups, 32 * W, dyn, s>>>(a);
  }
}

// dynamic smem = the largest tile of the launch (rows x 32 B) + Adam moments
template <int I, int H1, int H2, int K>
void launch_k(const TrainF32Args& a, int tile_bytes, cudaStream_t s) {
  constexpr int P = Net<I, H1, H2>::P;
  const int dyn = tile_bytes + 2 * P * 32 * 4;
  if constexpr (H1 == 8 && H2 == 0) {
    static const bool packed = std::getenv("LANN_FP32_UNPACKED") == nullptr;
    if (packed) {
      auto kern = train_fp32_h8_kernel<I, K>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
      kern<<<a.n_groups, 32, dyn, s>>>(a);
      return;
    }
  }
  if constexpr (H1 == 5 && H2 == 5) {
    if (std::getenv("LANN_FP32_UNPACKED") == nullptr) {
      auto kern = train_fp32_h55_kernel<I, K>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
      kern<<<a.n_groups, 32, dyn, s>>>(a);
      return;
    }
  }
  auto kern = train_fp32_kernel<I, H1, H2, K>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
  kern<<<a.n_groups, 32, dyn, s>>>(a);
}

// lanes: 1/2/4/8/32 = lanes per model in the warp kernel; 64/128/256 = threads per
// model in the CTA kernel.
template <int I, int H1, int H2>
bool dispatch_lanes(const TrainF32Args& a, int lanes, int tile_bytes, cudaStream_t s) {
  switch (lanes) {
    case 1: launch_k<I, H1, H2, 1>(a, tile_bytes, s); return true;
    case 2: launch_k<I, H1, H2, 2>(a, tile_bytes, s); return true;
    case 4: launch_k<I, H1, H2, 4>(a, tile_bytes, s); return true;
    case 8: launch_k<I, H1, H2, 8>(a, tile_bytes, s); return true;
    case 32: launch_k<I, H1, H2, 32>(a, tile_bytes, s); return true;
    case 64: launch_cta<I, H1, H2, 2>(a, tile_bytes, s); return true;
    case 128: launch_cta<I, H1, H2, 4>(a, tile_bytes, s); return true;
    case 256: launch_cta<I, H1, H2, 8>(a, tile_bytes, s); return true;
    default: return false;
  }
}

__global__ void pack_rows_kernel(const double* X, const double* y, int64_t n, float* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * 8) return;
  const int64_t r = i / 8;
  const int c = (int)(i % 8);
  out[i] = c == 7 ? (float)y[r] : (float)X[i];
}


// ---------------------------------------------------------------------------------
// FP32 for every other shape (unconstrained widths: 7-64-1, 6-40-40-1, ...; any I <= 7 and 1-2
// hidden layers of <= 64 units): one model per CTA of 256 threads. Weights and Adam moments in
// shared memory; per epoch the samples go through in chunks whose records (inputs, activations,
// deltas, one row per quantity, samples contiguous) fit shared memory: phase A threads own
// samples (forward and backward with FMA, the 2/N scale folded into the output delta), phase B
// threads own parameters and accumulate their sums over the chunk (carried across chunks); the
// loss is a block reduction of the per-thread err^2 sums; Adam as the other FP32 kernels
// (host bias-correction reciprocals).
constexpr int kWideT = 256;
constexpr int kWideKB = 20;  // parameters per thread: P <= 5120

__host__ __device__ constexpr int wide_rows(int h1, int h2) { return 8 + 2 * (h1 + h2) + 1; }

__global__ void __launch_bounds__(kWideT) train_fp32_wide_kernel(TrainWideArgs a) {
  extern __shared__ __align__(16) float wsm[];
  const int m = a.order[blockIdx.x];
  const int tile = a.model_tile[m];
  const int N = a.tile_rows[tile];
  const int I = a.tile_inputs[tile], H1 = a.h1[m], H2 = a.h2[m];
  const int E = a.epochs[m];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nl = H2 > 0 ? 3 : 2;
  int dims[4] = {I, H1, H2 > 0 ? H2 : 1, 1};
  int woff[3], boff[3], P = 0;
  for (int l = 0; l < nl; ++l) {
    woff[l] = P;
    P += dims[l] * dims[l + 1];
    boff[l] = P;
    P += dims[l + 1];
  }
  // record rows: x 0..6 | y 7 | a1 | a2 | t1 | t2 | tout (one row per quantity, samples contiguous)
  const int hid = H1 + (H2 > 0 ? H2 : 0);
  const int inoff[3] = {0, 8, 8 + H1};
  const int toff[3] = {8 + hid, 8 + hid + H1, 8 + hid + H1 + (H2 > 0 ? H2 : 0)};
  const int PP = (a.max_p + 3) & ~3;
  float* w = wsm;
  float* mo = w + PP;
  float* ve = mo + PP;
  float* red = ve + PP;  // [32] block reduction
  float* rec = red + 32;
  const int CH = a.chunk, ld = CH + 4;  // ld = 4 mod 32: a quarter-warp's float4 rows hit distinct banks
  const float* rows = a.rows + a.tile_offset[tile] * 8;
  const double* gp = a.params + a.param_offset[m];
  for (int p = tid; p < P; p += kWideT) {
    w[p] = (float)gp[p];
    mo[p] = 0.f;
    ve[p] = 0.f;
  }
  // phase-B ownership: parameter p -> record row of its delta and of its input (-1: a bias)
  // packed (delta row << 16) | (input row + 1); -1: no parameter
  int pix[kWideKB];
#pragma unroll
  for (int k = 0; k < kWideKB; ++k) {
    const int p = tid + k * kWideT;
    pix[k] = -1;
    for (int l = 0; l < nl && p < P; ++l) {
      const int in = dims[l], out = dims[l + 1];
      if (p >= woff[l] && p < boff[l])
        pix[k] = ((toff[l] + (p - woff[l]) / in) << 16) | (inoff[l] + (p - woff[l]) % in + 1);
      else if (p >= boff[l] && p < boff[l] + out)
        pix[k] = (toff[l] + (p - boff[l])) << 16;
    }
  }
  const float lr = (float)a.lr[m];
  const float scale = 2.0f / (float)N, inv_n = 1.0f / (float)N;
  double* trace = a.loss_trace ? a.loss_trace + a.trace_offset[m] : nullptr;
  int bad = -1;
  float last = 0.f;
  __syncthreads();
  for (int e = 0; e < E; ++e) {
    const float2 br = a.bias_rcp[e];
    const float step = lr * br.x, rb2 = br.y;
    float g[kWideKB];
#pragma unroll
    for (int k = 0; k < kWideKB; ++k) g[k] = 0.f;
    float lsum = 0.f;
    for (int c0 = 0; c0 < N; c0 += CH) {
      const int nc = N - c0 < CH ? N - c0 : CH;
      for (int sl = tid; sl < nc; sl += kWideT) {  // this chunk's inputs and targets
        const float* rw = rows + (size_t)(c0 + sl) * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) rec[i * ld + sl] = rw[i];
      }
      __syncthreads();
      // ---- phase A: forward / backward per sample (mlp.cpp:86-104) ----
      for (int sl = tid; sl < nc; sl += kWideT) {
        float* r = rec + sl;
        for (int l = 0; l < nl; ++l) {
          const int in = dims[l], out = dims[l + 1];
          const float* wl = w + woff[l];
          const float* bl = w + boff[l];
          const float* ain = r + inoff[l] * ld;
          if (l + 1 < nl) {
            float* aout = r + inoff[l + 1] * ld;
            for (int o = 0; o < out; o += 4) {  // four independent FMA chains in flight
              float z[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) z[q] = o + q < out ? bl[o + q] : 0.f;
              for (int i = 0; i < in; ++i) {
                const float ai = ain[i * ld];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  if (o + q < out) z[q] = fmaf(wl[(o + q) * in + i], ai, z[q]);
              }
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (o + q < out) aout[(o + q) * ld] = fmaxf(z[q], 0.f);
            }
          } else {
            float z = bl[0];
            for (int i = 0; i < in; ++i) z = fmaf(wl[i], ain[i * ld], z);
            const float err = z - r[7 * ld];
            lsum = fmaf(err, err, lsum);
            r[toff[l] * ld] = err * scale;  // d loss / d out, with the 1/N of the mean
          }
        }
        for (int l = nl - 2; l >= 0; --l) {  // hidden deltas from the next layer's
          const int nin = dims[l + 1], nout = dims[l + 2];
          const float* wn = w + woff[l + 1];
          const float* dn = r + toff[l + 1] * ld;
          const float* act = r + inoff[l + 1] * ld;
          float* d = r + toff[l] * ld;
          for (int i = 0; i < nin; i += 4) {
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            for (int o = 0; o < nout; ++o) {
              const float dno = dn[o * ld];
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (i + q < nin) acc[q] = fmaf(wn[o * nin + i + q], dno, acc[q]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (i + q < nin) d[(i + q) * ld] = act[(i + q) * ld] > 0.f ? acc[q] : 0.f;
          }
        }
      }
      __syncthreads();
      // ---- phase B: gradient sums over this chunk, carried across chunks ----
#pragma unroll
      for (int k = 0; k < kWideKB; ++k) {
        if (pix[k] >= 0) {  // float4 record reads, eight partial sums: eight FMA chains in flight
          const float* tr = rec + (pix[k] >> 16) * ld;
          const int ai = (pix[k] & 0xffff) - 1;
          if (ai >= 0) {
            const float* ar = rec + ai * ld;
            float4 u = make_float4(g[k], 0.f, 0.f, 0.f), v = make_float4(0.f, 0.f, 0.f, 0.f);
            int sl = 0;
            for (; sl + 8 <= nc; sl += 8) {
              const float4 t0 = *reinterpret_cast<const float4*>(tr + sl);
              const float4 a0 = *reinterpret_cast<const float4*>(ar + sl);
              const float4 t1 = *reinterpret_cast<const float4*>(tr + sl + 4);
              const float4 a1 = *reinterpret_cast<const float4*>(ar + sl + 4);
              u.x = fmaf(t0.x, a0.x, u.x); u.y = fmaf(t0.y, a0.y, u.y);
              u.z = fmaf(t0.z, a0.z, u.z); u.w = fmaf(t0.w, a0.w, u.w);
              v.x = fmaf(t1.x, a1.x, v.x); v.y = fmaf(t1.y, a1.y, v.y);
              v.z = fmaf(t1.z, a1.z, v.z); v.w = fmaf(t1.w, a1.w, v.w);
            }
            for (; sl < nc; ++sl) u.x = fmaf(tr[sl], ar[sl], u.x);
            g[k] = ((u.x + u.y) + (u.z + u.w)) + ((v.x + v.y) + (v.z + v.w));
          } else {
            float4 u = make_float4(g[k], 0.f, 0.f, 0.f), v = make_float4(0.f, 0.f, 0.f, 0.f);
            int sl = 0;
            for (; sl + 8 <= nc; sl += 8) {
              const float4 t0 = *reinterpret_cast<const float4*>(tr + sl);
              const float4 t1 = *reinterpret_cast<const float4*>(tr + sl + 4);
              u.x += t0.x; u.y += t0.y; u.z += t0.z; u.w += t0.w;
              v.x += t1.x; v.y += t1.y; v.z += t1.z; v.w += t1.w;
            }
            for (; sl < nc; ++sl) u.x += tr[sl];
            g[k] = ((u.x + u.y) + (u.z + u.w)) + ((v.x + v.y) + (v.z + v.w));
          }
        }
      }
      __syncthreads();  // the next chunk overwrites the records
    }
    // the pre-update loss (mlp.cpp:165-172): block reduction of the per-thread err^2 sums
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, off);
    if (lane == 0) red[warp] = lsum;
    __syncthreads();
    float L = 0.f;
#pragma unroll
    for (int q = 0; q < kWideT / 32; ++q) L += red[q];
    L *= inv_n;
    last = L;
    if (trace && tid == 0 && (e % a.trace_stride) == 0) trace[e / a.trace_stride] = (double)L;
    if (!isfinite(L)) {
      bad = e;
      break;  // uniform: every thread read the same sums
    }
#pragma unroll
    for (int k = 0; k < kWideKB; ++k) {
      const int p = tid + k * kWideT;
      if (pix[k] >= 0) w[p] -= adam_step(mo[p], ve[p], g[k], step, rb2);
    }
    __syncthreads();
  }
  double* outp = a.params + a.param_offset[m];
  for (int p = tid; p < P; p += kWideT) outp[p] = (double)w[p];
  if (tid == 0) {
    a.final_loss[m] = (double)last;
    a.nonfinite_epoch[m] = bad;
  }
}
}  // namespace

// Resident one-warp CTAs per SM of the warp kernel for (shape, lanes): the wave size the
// host uses to pick lanes per model without a long last wave.
template <int I, int H1, int H2, int K>
int slots_k(int tile_bytes) {
  constexpr int P = Net<I, H1, H2>::P;
  const int dyn = tile_bytes + 2 * P * 32 * 4;
  int n = 0;
  if constexpr (H1 == 8 && H2 == 0) {
    cudaFuncSetAttribute(train_fp32_h8_kernel<I, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, train_fp32_h8_kernel<I, K>, 32, dyn);
  } else if constexpr (H1 == 5 && H2 == 5) {
    cudaFuncSetAttribute(train_fp32_h55_kernel<I, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, train_fp32_h55_kernel<I, K>, 32, dyn);
  } else {
    cudaFuncSetAttribute(train_fp32_kernel<I, H1, H2, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, train_fp32_kernel<I, H1, H2, K>, 32, dyn);
  }
  return n;
}

template <int I, int H1, int H2>
int slots_shape(int lanes, int tile_bytes) {
  switch (lanes) {
    case 1: return slots_k<I, H1, H2, 1>(tile_bytes);
    case 2: return slots_k<I, H1, H2, 2>(tile_bytes);
    case 4: return slots_k<I, H1, H2, 4>(tile_bytes);
    case 8: return slots_k<I, H1, H2, 8>(tile_bytes);
    default: return slots_k<I, H1, H2, 32>(tile_bytes);
  }
}

int fp32_warp_slots_per_sm(int in, int h1, int h2, int lanes, int tile_bytes) {
  if (h1 == 8 && h2 == 0) {
    switch (in) {
      case 1: return slots_shape<1, 8, 0>(lanes, tile_bytes);
      case 2: return slots_shape<2, 8, 0>(lanes, tile_bytes);
      case 3: return slots_shape<3, 8, 0>(lanes, tile_bytes);
      case 4: return slots_shape<4, 8, 0>(lanes, tile_bytes);
      case 5: return slots_shape<5, 8, 0>(lanes, tile_bytes);
      case 6: return slots_shape<6, 8, 0>(lanes, tile_bytes);
      default: return slots_shape<7, 8, 0>(lanes, tile_bytes);
    }
  }
  switch (in) {
    case 4: return slots_shape<4, 5, 5>(lanes, tile_bytes);
    case 5: return slots_shape<5, 5, 5>(lanes, tile_bytes);
    default: return slots_shape<6, 5, 5>(lanes, tile_bytes);
  }
}

bool fp32_shape_supported(int in, int h1, int h2) {
  if (h1 == 8 && h2 == 0) return in >= 1 && in <= 7;
  if (h1 == 5 && h2 == 5) return in >= 4 && in <= 6;
  return false;
}

bool launch_train_fp32(const TrainF32Args& a, int in, int h1, int h2, int lanes, int tile_bytes,
                       cudaStream_t s) {
  if (h1 == 8 && h2 == 0) {
    switch (in) {
      case 1: return dispatch_lanes<1, 8, 0>(a, lanes, tile_bytes, s);
      case 2: return dispatch_lanes<2, 8, 0>(a, lanes, tile_bytes, s);
      case 3: return dispatch_lanes<3, 8, 0>(a, lanes, tile_bytes, s);
      case 4: return dispatch_lanes<4, 8, 0>(a, lanes, tile_bytes, s);
      case 5: return dispatch_lanes<5, 8, 0>(a, lanes, tile_bytes, s);
      case 6: return dispatch_lanes<6, 8, 0>(a, lanes, tile_bytes, s);
      case 7: return dispatch_lanes<7, 8, 0>(a, lanes, tile_bytes, s);
    }
  } else if (h1 == 5 && h2 == 5) {
    switch (in) {
      case 4: return dispatch_lanes<4, 5, 5>(a, lanes, tile_bytes, s);
      case 5: return dispatch_lanes<5, 5, 5>(a, lanes, tile_bytes, s);
      case 6: return dispatch_lanes<6, 5, 5>(a, lanes, tile_bytes, s);
    }
  }
  return false;
}

// FP32 rows [n][8] = normalised inputs x0..x6 with the target in column 7.
void launch_pack_rows(const double* X, const double* y, int64_t n, float* out, cudaStream_t s) {
  if (n <= 0) return;
  pack_rows_kernel<<<(unsigned)((n * 8 + 255) / 256), 256, 0, s>>>(X, y, n, out);
}

bool fp32_wide_supported(int in, int h1, int h2) {
  return in >= 1 && in <= 7 && h1 >= 1 && h1 <= 64 && h2 >= 0 && h2 <= 64 &&
         (in + 1) * h1 + (h2 > 0 ? (h1 + 1) * h2 + h2 + 1 : h1 + 1) <= kWideT * kWideKB;
}
int fp32_wide_rows(int h1, int h2) { return wide_rows(h1, h2); }
size_t fp32_wide_smem_bytes(int max_p, int rows, int chunk) {
  return (3 * size_t((max_p + 3) & ~3) + 32 + size_t(rows) * size_t(chunk + 4)) * sizeof(float);
}
void launch_train_fp32_wide(const TrainWideArgs& a, int dyn_bytes, cudaStream_t s) {
  if (a.n_models <= 0) return;
  cudaFuncSetAttribute(train_fp32_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_bytes);
  train_fp32_wide_kernel<<<a.n_models, kWideT, dyn_bytes, s>>>(a);
}

}  // namespace lann
