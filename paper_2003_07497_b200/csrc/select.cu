// select.cu — K2 selection kernels.
//
// select_schedule: selector::select(TrainedModel, n, candidates)
//   (selector.cpp:26-53): every candidate schedule scored by the blur model
//   (features {n, s1..s4, c = n^2}, features.cpp:40-45), argmin with strict <
//   and ties to the lexicographically smaller schedule. One thread per
//   candidate, a CTA-level (score, schedule) min-reduction, then a one-CTA
//   pass over the per-CTA winners.
// select_variants: for each of n_cands counter-generated candidate shapes, the
//   score of every variant model of the set and the argmin (ties -> lower
//   variant index, the strict-< rule of selector.cpp:38-39 over variant order).
//   Candidate i draws from splitmix64 seeded with derive_seed(seed, first+i)
//   (rng.hpp:10-22) with Rng::bounded's rejection rule (rng.hpp:34-40) in
//   sample_params' draw order (datagen.cpp:60-110) — generated in registers,
//   never stored. Model weights and normalisation live in shared memory.
#include <cmath>
#include <type_traits>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "kernels.cuh"

namespace lann {
namespace {

__device__ __forceinline__ uint64_t sm64(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t derive(uint64_t root, uint64_t stream) {
  uint64_t s = root ^ (0x9e3779b97f4a7c15ULL * (stream + 1));
  sm64(s);
  return sm64(s);
}
// Exact 64-bit remainder by a small divisor without the emulated 64-bit modulo:
// M = floor((2^64 - 1) / n) (table g_fastmod, built once per device), q = mulhi(r, M) is
// floor(r / n) minus at most 2, so r - q n lies in [0, 3n) and two conditional subtractions
// give r % n exactly.
constexpr uint32_t kFastModMax = 4096;
__device__ uint64_t g_fastmod[kFastModMax + 1];
__global__ void fastmod_init_kernel() {
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x + 1; n <= kFastModMax; n += gridDim.x * blockDim.x)
    g_fastmod[n] = ~0ULL / n;
}
__device__ __forceinline__ uint64_t fastmod(uint64_t r, uint64_t n, uint64_t M) {
  uint64_t rem = r - __umul64hi(r, M) * n;
  if (rem >= n) rem -= n;
  if (rem >= n) rem -= n;
  return rem;
}
__device__ __forceinline__ uint64_t bounded(uint64_t& s, uint64_t n) {
  // power of two: (2^64 - n) % n == 0, so the first draw is always accepted and
  // r % n == r & (n - 1) — the same value Rng::bounded returns, without a 64-bit modulo
  if ((n & (n - 1)) == 0) return sm64(s) & (n - 1);
  if (n <= kFastModMax) {
    const uint64_t M = g_fastmod[n];
    const uint64_t thr = fastmod(0 - n, n, M);
    for (;;) {
      const uint64_t r = sm64(s);
      if (r >= thr) return fastmod(r, n, M);
    }
  }
  const uint64_t thr = (0 - n) % n;
  for (;;) {
    const uint64_t r = sm64(s);
    if (r >= thr) return r % n;
  }
}
__device__ __forceinline__ uint32_t dim(uint64_t& s, uint32_t lo, uint32_t hi) {
  return lo + (uint32_t)bounded(s, (uint64_t)(hi - lo) + 1);
}
__device__ __forceinline__ double density(uint64_t& s, uint64_t cells, bool inc_one) {
  const int depth = 63 - __clzll((long long)cells);  // floor(log2 cells), cells >= 1
  const int first = inc_one ? 0 : 1;
  const int len = depth >= first ? depth - first + 1 : 0;
  if (len == 0) {
    (void)bounded(s, 1);
    return 1.0;
  }
  return ldexp(1.0, -(first + (int)bounded(s, (uint64_t)len)));
}

// Candidate shape i: base features (n_thd last) and complexity c.
__device__ int gen_candidate(int kind, int max_threads, uint64_t seed, int64_t idx, double* f,
                             uint64_t& c) {
  uint64_t s = derive(seed, (uint64_t)idx);
  const bool inc_one = kind != 1;
  uint32_t m, n, k, r, ps;
  double d1, d2;
  int nthd;
  switch (kind) {
    case 0:  // MM
      m = dim(s, 1, 1024);
      n = dim(s, 1, 1024);
      k = dim(s, 1, 1024);
      d1 = density(s, (uint64_t)m * n, inc_one);
      d2 = density(s, (uint64_t)n * k, inc_one);
      nthd = (int)dim(s, 1, (uint32_t)max_threads);
      f[0] = m; f[1] = n; f[2] = k; f[3] = d1; f[4] = d2; f[5] = nthd;
      c = (uint64_t)m * n * k;
      return 5;
    case 1:  // MV
      m = dim(s, 1, 1024);
      n = dim(s, 1, 1024);
      d1 = density(s, (uint64_t)m * n, inc_one);
      nthd = (int)dim(s, 1, (uint32_t)max_threads);
      f[0] = m; f[1] = n; f[2] = d1; f[3] = nthd;
      c = (uint64_t)m * n;
      return 3;
    case 2: {  // MC
      const uint32_t rs[3] = {3, 5, 7};
      r = rs[bounded(s, 3)];
      m = dim(s, r, 1024);
      n = dim(s, r, 1024);
      d1 = density(s, (uint64_t)m * n, inc_one);
      nthd = (int)dim(s, 1, (uint32_t)max_threads);
      f[0] = m; f[1] = n; f[2] = r; f[3] = d1; f[4] = nthd;
      c = (uint64_t)(m - r + 1) * (n - r + 1) * r * r;
      return 4;
    }
    default: {  // MP
      r = 2 + (uint32_t)bounded(s, 4);
      ps = 1 + (uint32_t)bounded(s, 2);
      m = dim(s, r, 1024);
      n = dim(s, r, 1024);
      d1 = density(s, (uint64_t)m * n, inc_one);
      nthd = (int)dim(s, 1, (uint32_t)max_threads);
      f[0] = m; f[1] = n; f[2] = r; f[3] = ps; f[4] = d1; f[5] = nthd;
      const uint64_t S = ps;
      c = ((n + S - 1) / S) * ((m + S - 1) / S) * S * S;
      return 5;
    }
  }
}

// Exact-order FP64 score (models.cpp:346-363) of model-input x under w / nrm.
__device__ double score_fp64(const double* w, const double* nrm, int I, int H1, int H2, int logt,
                             const double* x) {
  double a0[8], a1[64], a2[64];
  for (int j = 0; j < I; ++j) {
    const double range = __dsub_rn(nrm[8 + j], nrm[j]);
    a0[j] = range > 0.0 ? __ddiv_rn(__dsub_rn(x[j], nrm[j]), range) : 0.0;
  }
  for (int o = 0; o < H1; ++o) {
    double z = w[I * H1 + o];
    for (int i = 0; i < I; ++i) z = __dadd_rn(z, __dmul_rn(w[o * I + i], a0[i]));
    a1[o] = z > 0.0 ? z : 0.0;
  }
  int off = (I + 1) * H1;
  const double* in = a1;
  int nin = H1;
  if (H2 > 0) {
    for (int o = 0; o < H2; ++o) {
      double z = w[off + H1 * H2 + o];
      for (int i = 0; i < H1; ++i) z = __dadd_rn(z, __dmul_rn(w[off + o * H1 + i], a1[i]));
      a2[o] = z > 0.0 ? z : 0.0;
    }
    off += (H1 + 1) * H2;
    in = a2;
    nin = H2;
  }
  double z = w[off + nin];
  for (int i = 0; i < nin; ++i) z = __dadd_rn(z, __dmul_rn(w[off + i], in[i]));
  const double tr = __dsub_rn(nrm[17], nrm[16]);
  double t = tr > 0.0 ? __dadd_rn(nrm[16], __dmul_rn(z, tr)) : nrm[16];
  if (logt) t = exp(t);
  return t < 1e-9 ? 1e-9 : t;
}

// FP32 score: normalise with precomputed (min, 1/range) in FP32, FMA forward.
__device__ float score_fp32(const float* w, const float* nf, int I, int H1, int H2, int logt,
                            const double* x) {
  float a0[8], a1[64], a2[64];
  for (int j = 0; j < I; ++j) a0[j] = ((float)x[j] - nf[j]) * nf[8 + j];
  for (int o = 0; o < H1; ++o) {
    float z = w[I * H1 + o];
    for (int i = 0; i < I; ++i) z = fmaf(w[o * I + i], a0[i], z);
    a1[o] = fmaxf(z, 0.f);
  }
  int off = (I + 1) * H1;
  const float* in = a1;
  int nin = H1;
  if (H2 > 0) {
    for (int o = 0; o < H2; ++o) {
      float z = w[off + H1 * H2 + o];
      for (int i = 0; i < H1; ++i) z = fmaf(w[off + o * H1 + i], a1[i], z);
      a2[o] = fmaxf(z, 0.f);
    }
    off += (H1 + 1) * H2;
    in = a2;
    nin = H2;
  }
  float z = w[off + nin];
  for (int i = 0; i < nin; ++i) z = fmaf(w[off + i], in[i], z);
  float t = fmaf(z, nf[17], nf[16]);  // t_min + y * range (range 0 -> t_min)
  if (logt) t = __expf(t);
  return fmaxf(t, 1e-9f);
}

__device__ __forceinline__ bool sched_less(const uint32_t* a, const uint32_t* b) {
  for (int j = 0; j < 4; ++j)
    if (a[j] != b[j]) return a[j] < b[j];
  return false;
}

struct SchedArgs {
  int64_t n;
  const uint32_t* cands;
  uint32_t n_img;
  int I, H1, H2, logt;
  const double* w;
  const double* nrm;
  double* blk_score;
  int64_t* blk_idx;
};

// (score, schedule) argmin: strict < on score, ties to the smaller schedule.
__device__ __forceinline__ bool better(double s, int64_t i, double bs, int64_t bi, const uint32_t* c) {
  if (bi < 0) return i >= 0;
  if (i < 0) return false;
  if (s < bs) return true;
  if (s == bs) return sched_less(c + 4 * i, c + 4 * bi);
  return false;
}

__global__ void select_schedule_kernel(SchedArgs a, int pass) {
  __shared__ double ss[256];
  __shared__ int64_t si[256];
  double best = 0.0;
  int64_t bi = -1;
  if (pass == 0) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < a.n) {
      double x[8];
      x[0] = (double)a.n_img;
      for (int j = 0; j < 4; ++j) x[1 + j] = (double)a.cands[4 * i + j];
      x[5] = (double)((uint64_t)a.n_img * a.n_img);
      best = score_fp64(a.w, a.nrm, a.I, a.H1, a.H2, a.logt, x);
      bi = i;
    }
  } else {
    for (int64_t k = threadIdx.x; k < a.n; k += blockDim.x) {
      const double s = a.blk_score[k];
      const int64_t i = a.blk_idx[k];
      if (better(s, i, best, bi, a.cands)) {
        best = s;
        bi = i;
      }
    }
  }
  ss[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      const int o = threadIdx.x + st;
      if (better(ss[o], si[o], ss[threadIdx.x], si[threadIdx.x], a.cands)) {
        ss[threadIdx.x] = ss[o];
        si[threadIdx.x] = si[o];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.blk_score[pass == 0 ? blockIdx.x : 0] = ss[0];
    a.blk_idx[pass == 0 ? blockIdx.x : 0] = si[0];
  }
}

constexpr int kMaxModels = 32;
constexpr int kMaxParams = 96;  // lightweight nets (<= 75 parameters)
constexpr int kFastMaxV = 16;   // variant models in the constant-parameter fast path

struct VariantArgs {
  int n_models, precision, kind, max_threads;
  uint64_t seed;
  int64_t first, n;
  const int* n_inputs;
  const int* h1;
  const int* h2;
  const int* logt;
  const int* with_n_thd;
  const int64_t* param_offset;
  const double* params;
  const double* norm;
  void* out_idx;    // IdxT[n] or null
  void* out_score;  // ScoreT[n] or null
  unsigned long long* hist;  // [n_models] wins, or null
};

template <typename IdxT, typename ScoreT>
__global__ void __launch_bounds__(256) select_variants_kernel(VariantArgs a) {
  __shared__ double wd[kMaxModels][kMaxParams];
  __shared__ float wf[kMaxModels][kMaxParams];
  __shared__ double nd[kMaxModels][18];
  __shared__ float nf[kMaxModels][18];
  __shared__ int shp[kMaxModels][5];
  __shared__ unsigned wins[kMaxModels];
  if (threadIdx.x < kMaxModels) wins[threadIdx.x] = 0;
  for (int t = threadIdx.x; t < a.n_models * kMaxParams; t += blockDim.x) {
    const int m = t / kMaxParams, p = t % kMaxParams;
    const int I = a.n_inputs[m], H1 = a.h1[m], H2 = a.h2[m];
    const int P = H2 > 0 ? (I + 1) * H1 + (H1 + 1) * H2 + H2 + 1 : (I + 1) * H1 + H1 + 1;
    const double v = p < P ? a.params[a.param_offset[m] + p] : 0.0;
    wd[m][p] = v;
    wf[m][p] = (float)v;
  }
  for (int t = threadIdx.x; t < a.n_models; t += blockDim.x) {
    const double* n = a.norm + 18 * t;
    for (int j = 0; j < 18; ++j) nd[t][j] = n[j];
    for (int j = 0; j < 8; ++j) {
      const double range = n[8 + j] - n[j];
      nf[t][j] = (float)n[j];
      nf[t][8 + j] = range > 0.0 ? (float)(1.0 / range) : 0.f;
    }
    const double tr = n[17] - n[16];
    nf[t][16] = (float)n[16];
    nf[t][17] = tr > 0.0 ? (float)tr : 0.f;
    shp[t][0] = a.n_inputs[t];
    shp[t][1] = a.h1[t];
    shp[t][2] = a.h2[t];
    shp[t][3] = a.logt[t];
    shp[t][4] = a.with_n_thd[t];
  }
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
    double base[8];
    uint64_t c;
    const int nb = gen_candidate(a.kind, a.max_threads, a.seed, a.first + i, base, c);
    int best = -1;
    double best_s = 0.0;
    for (int v = 0; v < a.n_models; ++v) {
      double x[8];
      int I = 0;
      for (int j = 0; j < nb; ++j) x[I++] = base[j];
      if (shp[v][4]) x[I++] = base[nb];
      if (I < shp[v][0]) x[I++] = (double)c;  // the augmented family appends c
      const double s = a.precision == 0
                           ? score_fp64(wd[v], nd[v], shp[v][0], shp[v][1], shp[v][2], shp[v][3], x)
                           : (double)score_fp32(wf[v], nf[v], shp[v][0], shp[v][1], shp[v][2], shp[v][3], x);
      if (best < 0 || s < best_s) {
        best = v;
        best_s = s;
      }
    }
    if (a.out_idx) static_cast<IdxT*>(a.out_idx)[i] = (IdxT)best;
    if (a.out_score) static_cast<ScoreT*>(a.out_score)[i] = (ScoreT)best_s;
    if (a.hist) atomicAdd(&wins[best], 1u);
  }
  if (a.hist) {
    __syncthreads();
    if (threadIdx.x < a.n_models && wins[threadIdx.x])
      atomicAdd(&a.hist[threadIdx.x], (unsigned long long)wins[threadIdx.x]);
  }
}

// ---- fast path: prediction nets (one hidden layer of 8), FP32, <= 16 variant models -------
// Weights travel as a __grid_constant__ kernel parameter (constant bank), so every FFMA
// takes its weight as a constant-cache operand; min-max normalisation is folded into
// layer 1 on the host: W'[h][j] = W[h][j] / range_j, B'[h] = B[h] - sum_j W[h][j] min_j / range_j.
// Input columns are the kind's base features, then n_thd, then c (a model without n_thd
// or without c has zero weights there).
struct FastModels {
  int nv;
  float w1[kFastMaxV][8][8];  // [v][h][column]
  float b1[kFastMaxV][8];
  float w2[kFastMaxV][8];
  float b2[kFastMaxV];
  float tmin[kFastMaxV], trange[kFastMaxV];
  int logt[kFastMaxV];
};

template <int NB>
__global__ void __launch_bounds__(256) select_variants_fast(const __grid_constant__ FastModels fm,
                                                            int kind, int max_threads, uint64_t seed,
                                                            int64_t first, int64_t n, int* out_idx,
                                                            double* out_score) {
  constexpr int NC = NB + 2;  // columns: base features, n_thd, c
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double base[8];
    uint64_t c;
    gen_candidate(kind, max_threads, seed, first + i, base, c);
    float x[NC];
#pragma unroll
    for (int j = 0; j < NB; ++j) x[j] = (float)base[j];
    x[NB] = (float)base[NB];
    x[NB + 1] = (float)(double)c;
    int best = -1;
    float best_s = 0.f;
#pragma unroll
    for (int v = 0; v < kFastMaxV; ++v) {
      if (v < fm.nv) {
        float out = fm.b2[v];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          float z = fm.b1[v][h];
#pragma unroll
          for (int j = 0; j < NC; ++j) z = fmaf(fm.w1[v][h][j], x[j], z);
          out = fmaf(fm.w2[v][h], fmaxf(z, 0.f), out);
        }
        float t = fmaf(out, fm.trange[v], fm.tmin[v]);
        if (fm.logt[v]) t = __expf(t);
        t = fmaxf(t, 1e-9f);
        if (best < 0 || t < best_s) {
          best = v;
          best_s = t;
        }
      }
    }
    out_idx[i] = best;
    out_score[i] = (double)best_s;
  }
}

// Packed variant of select_variants_fast: hidden units in pairs on FFMA2 (sm_100 fma.rn.f32x2)
// with the candidate feature as the broadcast operand and the weight pairs as 64-bit uniform
// operands — the scorer is issue-bound (ncu: 81% issue slots), and this halves the FMA issue.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(f32x2 p, float& a, float& b) {
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(p));
}
__device__ __forceinline__ f32x2 ffma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

struct FastModels2 {
  int nv;
  f32x2 w1[kFastMaxV][8][4];  // [v][column][hidden pair]
  f32x2 b1[kFastMaxV][4];
  f32x2 w2[kFastMaxV][4];
  float b2[kFastMaxV];
  float tmin[kFastMaxV], trange[kFastMaxV];
  int logt[kFastMaxV];
};

// Outputs: IdxT / ScoreT per candidate (int32 + double, or the compact uint8 + float), either
// pointer may be null; hist (optional) counts each variant's wins (shared-memory tallies, one
// global atomic per variant per CTA).
template <int NB, typename IdxT, typename ScoreT>
__global__ void __launch_bounds__(256) select_variants_fast2(const __grid_constant__ FastModels2 fm,
                                                             int kind, int max_threads, uint64_t seed,
                                                             int64_t first, int64_t n, IdxT* out_idx,
                                                             ScoreT* out_score, unsigned long long* hist) {
  constexpr int NC = NB + 2;  // columns: base features, n_thd, c
  __shared__ unsigned wins[kFastMaxV];
  if (hist) {
    if (threadIdx.x < kFastMaxV) wins[threadIdx.x] = 0;
    __syncthreads();
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double base[8];
    uint64_t c;
    gen_candidate(kind, max_threads, seed, first + i, base, c);
    float x[NC];
#pragma unroll
    for (int j = 0; j < NB; ++j) x[j] = (float)base[j];
    x[NB] = (float)base[NB];
    x[NB + 1] = (float)(double)c;
    int best = -1;
    float best_s = 0.f;
#pragma unroll
    for (int v = 0; v < kFastMaxV; ++v) {
      if (v < fm.nv) {
        f32x2 z[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) z[q] = fm.b1[v][q];
#pragma unroll
        for (int j = 0; j < NC; ++j)
#pragma unroll
          for (int q = 0; q < 4; ++q) z[q] = ffma2(fm.w1[v][j][q], pk2(x[j], x[j]), z[q]);
        f32x2 acc = pk2(fm.b2[v], 0.f);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float za, zb;
          upk2(z[q], za, zb);
          acc = ffma2(fm.w2[v][q], pk2(fmaxf(za, 0.f), fmaxf(zb, 0.f)), acc);
        }
        float o0, o1;
        upk2(acc, o0, o1);
        float t = fmaf(o0 + o1, fm.trange[v], fm.tmin[v]);
        if (fm.logt[v]) t = __expf(t);
        t = fmaxf(t, 1e-9f);
        if (best < 0 || t < best_s) {
          best = v;
          best_s = t;
        }
      }
    }
    if (out_idx) out_idx[i] = (IdxT)best;
    if (out_score) out_score[i] = (ScoreT)best_s;
    if (hist) atomicAdd(&wins[best], 1u);
  }
  if (hist) {
    __syncthreads();
    if (threadIdx.x < fm.nv && wins[threadIdx.x]) atomicAdd(&hist[threadIdx.x], (unsigned long long)wins[threadIdx.x]);
  }
}

}  // namespace

// the fastmod table, filled once per device (stream-ordered before the first scorer launch)
void ensure_fastmod_table(cudaStream_t s) {
  static bool done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || done[dev]) return;
  fastmod_init_kernel<<<16, 256, 0, s>>>();
  done[dev] = true;
}

// Host side of the fast path: fold normalisation into layer 1 (in FP64, then round).
bool select_variants_fast_launch(int n_models, int kind, int max_threads, uint64_t seed, int64_t first,
                                 int64_t n, const int* n_inputs, const int* h1, const int* h2,
                                 const int* logt, const int* with_thd, const int64_t* param_offset,
                                 const double* params, const double* norm, void* d_idx, void* d_score,
                                 bool compact, unsigned long long* d_hist, int sms, cudaStream_t s) {
  if (n_models < 1 || n_models > kFastMaxV || kind < 0 || kind > 3) return false;
  ensure_fastmod_table(s);
  static const int nb_of[4] = {5, 3, 4, 5};
  const int nb = nb_of[kind];
  FastModels fm{};
  fm.nv = n_models;
  for (int v = 0; v < n_models; ++v) {
    if (h1[v] != 8 || h2[v] != 0) return false;
    const int I = n_inputs[v];
    const bool thd = with_thd[v] != 0;
    if (I != nb + (thd ? 1 : 0) && I != nb + (thd ? 1 : 0) + 1) return false;
    const bool aug = I == nb + (thd ? 1 : 0) + 1;
    int col[8];  // model input j -> column
    for (int j = 0; j < nb; ++j) col[j] = j;
    int k = nb;
    if (thd) col[k++] = nb;
    if (aug) col[k++] = nb + 1;
    const double* w = params + param_offset[v];
    const double* nr = norm + 18 * v;
    for (int h = 0; h < 8; ++h) {
      double b = w[I * 8 + h];
      for (int j = 0; j < I; ++j) {
        const double range = nr[8 + j] - nr[j];
        const double wj = w[h * I + j];
        if (range > 0.0) {
          fm.w1[v][h][col[j]] = (float)(wj / range);
          b -= wj * nr[j] / range;
        }
      }
      fm.b1[v][h] = (float)b;
      fm.w2[v][h] = (float)w[(I + 1) * 8 + h];
    }
    fm.b2[v] = (float)w[(I + 1) * 8 + 8];
    const double tr = nr[17] - nr[16];
    fm.tmin[v] = (float)nr[16];
    fm.trange[v] = tr > 0.0 ? (float)tr : 0.f;
    fm.logt[v] = logt[v];
  }
  int64_t blocks = (n + 255) / 256;
  const int64_t cap = (int64_t)sms * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (std::getenv("LANN_SELECT_UNPACKED") == nullptr) {
    FastModels2 f2{};
    f2.nv = fm.nv;
    for (int v = 0; v < fm.nv; ++v) {
      for (int q = 0; q < 4; ++q) {
        for (int j = 0; j < 8; ++j) {
          float pair[2] = {fm.w1[v][2 * q][j], fm.w1[v][2 * q + 1][j]};
          std::memcpy(&f2.w1[v][j][q], pair, 8);
        }
        float b[2] = {fm.b1[v][2 * q], fm.b1[v][2 * q + 1]};
        std::memcpy(&f2.b1[v][q], b, 8);
        float w[2] = {fm.w2[v][2 * q], fm.w2[v][2 * q + 1]};
        std::memcpy(&f2.w2[v][q], w, 8);
      }
      f2.b2[v] = fm.b2[v];
      f2.tmin[v] = fm.tmin[v];
      f2.trange[v] = fm.trange[v];
      f2.logt[v] = fm.logt[v];
    }
    auto go = [&](auto nbc) {
      constexpr int NB = decltype(nbc)::value;
      if (compact)
        select_variants_fast2<NB, unsigned char, float><<<(unsigned)blocks, 256, 0, s>>>(
            f2, kind, max_threads, seed, first, n, static_cast<unsigned char*>(d_idx), static_cast<float*>(d_score),
            d_hist);
      else
        select_variants_fast2<NB, int, double><<<(unsigned)blocks, 256, 0, s>>>(
            f2, kind, max_threads, seed, first, n, static_cast<int*>(d_idx), static_cast<double*>(d_score), d_hist);
    };
    switch (nb) {
      case 3: go(std::integral_constant<int, 3>{}); break;
      case 4: go(std::integral_constant<int, 4>{}); break;
      default: go(std::integral_constant<int, 5>{}); break;
    }
    return true;
  }
  if (compact || d_hist) return false;  // the unpacked developer path writes int32 + double only
  switch (nb) {
    case 3: select_variants_fast<3><<<(unsigned)blocks, 256, 0, s>>>(fm, kind, max_threads, seed, first, n, static_cast<int*>(d_idx), static_cast<double*>(d_score)); break;
    case 4: select_variants_fast<4><<<(unsigned)blocks, 256, 0, s>>>(fm, kind, max_threads, seed, first, n, static_cast<int*>(d_idx), static_cast<double*>(d_score)); break;
    default: select_variants_fast<5><<<(unsigned)blocks, 256, 0, s>>>(fm, kind, max_threads, seed, first, n, static_cast<int*>(d_idx), static_cast<double*>(d_score)); break;
  }
  return true;
}

int select_schedule_launch(int64_t n, const uint32_t* d_cands, uint32_t n_img, int I, int H1,
                           int H2, int logt, const double* d_w, const double* d_nrm,
                           double* d_blk_score, int64_t* d_blk_idx, cudaStream_t s) {
  SchedArgs a{n, d_cands, n_img, I, H1, H2, logt, d_w, d_nrm, d_blk_score, d_blk_idx};
  const int blocks = (int)((n + 255) / 256);
  select_schedule_kernel<<<blocks, 256, 0, s>>>(a, 0);
  a.n = blocks;
  select_schedule_kernel<<<1, 256, 0, s>>>(a, 1);
  return 2;
}

bool select_variants_supported(int n_models, int max_params) {
  return n_models >= 1 && n_models <= kMaxModels && max_params <= kMaxParams;
}

int select_variants_launch(int n_models, int precision, int kind, int max_threads, uint64_t seed,
                           int64_t first, int64_t n, const int* d_in, const int* d_h1,
                           const int* d_h2, const int* d_logt, const int* d_thd,
                           const int64_t* d_poff, const double* d_params, const double* d_norm,
                           void* d_idx, void* d_score, bool compact, unsigned long long* d_hist, int sms,
                           cudaStream_t s) {
  ensure_fastmod_table(s);
  VariantArgs a{n_models, precision, kind, max_threads, seed, first, n, d_in, d_h1, d_h2,
                d_logt, d_thd, d_poff, d_params, d_norm, d_idx, d_score, d_hist};
  int64_t blocks = (n + 255) / 256;
  const int64_t cap = (int64_t)sms * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (compact) select_variants_kernel<unsigned char, float><<<(unsigned)blocks, 256, 0, s>>>(a);
  else select_variants_kernel<int, double><<<(unsigned)blocks, 256, 0, s>>>(a);
  return 1;
}

}  // namespace lann
