/*
 * oracle/lann_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker, see
 * lann_oracle.h). A plain-C restatement of the reference LANN path in FP64 with
 * the reference's operation order; compiled with -ffp-contract=off like the
 * reference (generic x86-64, no FMA). Each function cites the reference line
 * range it restates (paths relative to /root/reference/proj/core/).
 */
#include "lann_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- rng.hpp ----------------------------------------------------------------- */

/* rng.hpp:10-15 */
uint64_t or_splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* rng.hpp:18-22 */
uint64_t or_derive_seed(uint64_t root, uint64_t stream) {
  uint64_t s = root ^ (0x9e3779b97f4a7c15ULL * (stream + 1));
  or_splitmix64(&s);
  return or_splitmix64(&s);
}

/* std::mt19937_64 (the engine of rng.hpp:66; fully specified by the C++ standard) */
typedef struct {
  uint64_t mt[312];
  int idx;
} rng_t;

static void rng_seed(rng_t* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

static uint64_t rng_next(rng_t* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:34-40 */
static uint64_t rng_bounded(rng_t* r, uint64_t n) {
  const uint64_t threshold = (0 - n) % n;
  for (;;) {
    uint64_t x = rng_next(r);
    if (x >= threshold) return x % n;
  }
}
/* rng.hpp:43-46 */
static int64_t rng_uniform_int(rng_t* r, int64_t lo, int64_t hi) {
  return lo + (int64_t)rng_bounded(r, (uint64_t)(hi - lo) + 1);
}
/* rng.hpp:49-55 */
static double rng_uniform(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
static double rng_uniform_range(rng_t* r, double lo, double hi) {
  return lo + (hi - lo) * rng_uniform(r);
}

/* ---- kernels / features ------------------------------------------------------ */

typedef struct {
  int kind;
  uint32_t m, n, k, r, s;
  double d1, d2, d;
  int n_thd;
  uint32_t sched[4];
} params_t;

static int bit_width(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }

/* datagen.cpp:38-45: dyadic ladder, returns its length, fills out */
static int density_ladder(uint64_t cells, int include_one, double* out) {
  const int depth = bit_width(cells) - 1;
  int n = 0;
  for (int j = include_one ? 0 : 1; j <= depth; ++j) out[n++] = ldexp(1.0, -j);
  if (n == 0) out[n++] = 1.0;
  return n;
}

static uint32_t bit_ceil32(uint32_t v) {
  uint32_t x = 1;
  while (x < v) x <<= 1;
  return x;
}

/* kernels.cpp:52-60 ScheduleSpace::{cpu_default,gpu_style} + kernels.cpp:77-87
 * enumerate_all (lexicographic). Returns count; out may be NULL. */
static int enumerate_lattice(int gpu_style, uint32_t* out) {
  uint32_t s1lo = 2, s1hi = gpu_style ? 16 : 1024, s2lo = gpu_style ? 1 : 2,
           s2hi = gpu_style ? 64 : 1024, s3lo = gpu_style ? 1 : 2, s3hi = gpu_style ? 64 : 1024,
           s4lo = gpu_style ? 1 : 2, s4hi = gpu_style ? 1 : 1024;
  int chained = !gpu_style;
  int n = 0;
  for (uint32_t a = bit_ceil32(s1lo); a <= s1hi; a <<= 1)
    for (uint32_t b = bit_ceil32(s2lo); b <= s2hi; b <<= 1) {
      uint32_t c3hi = chained ? (s3hi < b ? s3hi : b) : s3hi;
      for (uint32_t c = bit_ceil32(s3lo); c <= c3hi; c <<= 1) {
        uint32_t c4hi = chained ? (s4hi < c ? s4hi : c) : s4hi;
        for (uint32_t d = bit_ceil32(s4lo); d <= c4hi; d <<= 1) {
          if (out) {
            out[4 * n] = a;
            out[4 * n + 1] = b;
            out[4 * n + 2] = c;
            out[4 * n + 3] = d;
          }
          ++n;
        }
      }
    }
  return n;
}

static const uint32_t kBlurSides[6] = {1024, 2048, 4096, 8192, 16384, 32768}; /* datagen.hpp:28 */
static const uint32_t kMcFilter[3] = {3, 5, 7};                              /* datagen.hpp:24 */
static const uint32_t kMpAux[4] = {2, 3, 4, 5};                              /* datagen.hpp:25 */
static const uint32_t kMpPool[2] = {1, 2};                                   /* datagen.hpp:26 */

/* kernels.cpp:184-206 */
static uint64_t complexity(const params_t* p) {
  const uint64_t m = p->m, n = p->n, k = p->k;
  switch (p->kind) {
    case LANN_MM: return m * n * k;
    case LANN_MV: return m * n;
    case LANN_MC: return (m - p->r + 1) * (n - p->r + 1) * (uint64_t)p->r * p->r;
    case LANN_MP: {
      const uint64_t s = p->s;
      return ((n + s - 1) / s) * ((m + s - 1) / s) * s * s;
    }
    default: return n * n;
  }
}

/* features.cpp:23-54 (base features, no c); returns the count */
static int featurize_base(const params_t* p, int with_n_thd, double* f) {
  int n = 0;
  switch (p->kind) {
    case LANN_MM: f[n++] = p->m; f[n++] = p->n; f[n++] = p->k; f[n++] = p->d1; f[n++] = p->d2; break;
    case LANN_MV: f[n++] = p->m; f[n++] = p->n; f[n++] = p->d; break;
    case LANN_MC: f[n++] = p->m; f[n++] = p->n; f[n++] = p->r; f[n++] = p->d; break;
    case LANN_MP: f[n++] = p->m; f[n++] = p->n; f[n++] = p->r; f[n++] = p->s; f[n++] = p->d; break;
    default:
      f[n++] = p->n;
      for (int j = 0; j < 4; ++j) f[n++] = p->sched[j];
      with_n_thd = 0;
  }
  if (with_n_thd) f[n++] = p->n_thd;
  return n;
}

/* datagen.cpp:60-110 sample_params, generic over the draw source */
typedef uint64_t (*bounded_fn)(void* src, uint64_t n);

static int64_t uni_int(bounded_fn b, void* src, int64_t lo, int64_t hi) {
  return lo + (int64_t)b(src, (uint64_t)(hi - lo) + 1);
}

static void sample_params(int kind, int max_threads, int blur_gpu, bounded_fn b, void* src,
                          params_t* p) {
  double lad[72];
  const int inc_one = kind != LANN_MV; /* ParamSpace::defaults, datagen.cpp:18-24 */
  memset(p, 0, sizeof *p);
  p->kind = kind;
  p->d1 = p->d2 = p->d = 1.0;
  p->n_thd = 1;
  switch (kind) {
    case LANN_MM: {
      p->m = (uint32_t)uni_int(b, src, 1, 1024);
      p->n = (uint32_t)uni_int(b, src, 1, 1024);
      p->k = (uint32_t)uni_int(b, src, 1, 1024);
      int L = density_ladder((uint64_t)p->m * p->n, inc_one, lad);
      p->d1 = lad[b(src, L)];
      L = density_ladder((uint64_t)p->n * p->k, inc_one, lad);
      p->d2 = lad[b(src, L)];
      p->n_thd = (int)uni_int(b, src, 1, max_threads);
      break;
    }
    case LANN_MV: {
      p->m = (uint32_t)uni_int(b, src, 1, 1024);
      p->n = (uint32_t)uni_int(b, src, 1, 1024);
      int L = density_ladder((uint64_t)p->m * p->n, inc_one, lad);
      p->d = lad[b(src, L)];
      p->n_thd = (int)uni_int(b, src, 1, max_threads);
      break;
    }
    case LANN_MC: {
      p->r = kMcFilter[b(src, 3)];
      uint32_t lo = p->r > 1 ? p->r : 1, hi = 1024 > p->r ? 1024 : p->r;
      p->m = (uint32_t)uni_int(b, src, lo, hi);
      p->n = (uint32_t)uni_int(b, src, lo, hi);
      int L = density_ladder((uint64_t)p->m * p->n, inc_one, lad);
      p->d = lad[b(src, L)];
      p->n_thd = (int)uni_int(b, src, 1, max_threads);
      break;
    }
    case LANN_MP: {
      p->r = kMpAux[b(src, 4)];
      p->s = kMpPool[b(src, 2)];
      uint32_t lo = p->r > 1 ? p->r : 1, hi = 1024 > p->r ? 1024 : p->r;
      p->m = (uint32_t)uni_int(b, src, lo, hi);
      p->n = (uint32_t)uni_int(b, src, lo, hi);
      int L = density_ladder((uint64_t)p->m * p->n, inc_one, lad);
      p->d = lad[b(src, L)];
      p->n_thd = (int)uni_int(b, src, 1, max_threads);
      break;
    }
    default: {
      p->n = kBlurSides[b(src, 6)];
      static uint32_t lat[2][2200 * 4];
      static int lat_n[2] = {0, 0};
      int g = blur_gpu ? 1 : 0;
      if (!lat_n[g]) lat_n[g] = enumerate_lattice(g, lat[g]);
      uint64_t i = b(src, (uint64_t)lat_n[g]);
      memcpy(p->sched, &lat[g][4 * i], sizeof p->sched);
      break;
    }
  }
}

static uint64_t mt_bounded(void* src, uint64_t n) { return rng_bounded((rng_t*)src, n); }

/* ---- synthetic world probe (lann_engine.h lann_world; generalises
 * acceptance_main.cpp:271-279) ------------------------------------------------ */
static double world_runtime(const lann_world* w, const params_t* p, rng_t* noise_rng) {
  double g, fd = 1.0;
  if (p->kind == LANN_BLUR) {
    g = 1.0;
    for (int j = 0; j < 4; ++j) {
      const double d = (double)__builtin_ctz(p->sched[j]) - w->mu[j];
      g += w->kappa[j] * d * d;
    }
  } else {
    g = w->g0 + w->g1 / (double)p->n_thd;
    const double dens = p->kind == LANN_MM ? p->d1 : p->d;
    fd = (1.0 - w->delta) + w->delta * dens;
  }
  const double nz = 1.0 + rng_uniform_range(noise_rng, -w->noise, w->noise);
  return w->alpha * (double)complexity(p) * g * fd * nz + w->beta;
}

/* datagen.cpp:177-223 build_dataset with a probe */
int or_build_dataset(const lann_world* w, uint64_t seed, int count, double* feats, uint64_t* c,
                     double* rt, int* n_features) {
  if (count < 2) return LANN_PARAM_ERROR;
  if (w->max_threads < 1) return LANN_PARAM_ERROR;
  rng_t* rng = malloc(sizeof(rng_t));
  rng_t* noise = malloc(sizeof(rng_t));
  rng_seed(rng, or_derive_seed(seed, 0));
  rng_seed(noise, or_derive_seed(seed, 0x9015E));
  const int takes_thd = w->hw_class == LANN_HW_CPU && w->kind != LANN_BLUR; /* variants.hpp:30 */
  int status = 0;
  for (int i = 0; i < count; ++i) {
    params_t p;
    sample_params(w->kind, w->max_threads, w->blur_lattice == 1, mt_bounded, rng, &p);
    if (w->hw_class != LANN_HW_CPU) p.n_thd = 1;      /* FixedSingle, datagen.cpp:195 */
    if (w->kind == LANN_BLUR) p.n_thd = w->max_threads; /* datagen.cpp:196 */
    double* f = feats + (size_t)i * LANN_ROW;
    memset(f, 0, LANN_ROW * sizeof(double));
    *n_features = featurize_base(&p, takes_thd, f);
    c[i] = complexity(&p);
    rt[i] = world_runtime(w, &p, noise);
    if (!(rt[i] > 0.0)) { status = LANN_BUILD_ABORT; break; }
  }
  free(rng);
  free(noise);
  return status;
}

/* datagen.cpp:225-248: full Fisher-Yates from Rng(derive_seed(seed, 0x517)) */
int or_split_order(int n, double frac, uint64_t seed, int64_t* order, int* n_train) {
  if (!(frac > 0.0 && frac < 1.0)) return LANN_PARAM_ERROR;
  rng_t* rng = malloc(sizeof(rng_t));
  rng_seed(rng, or_derive_seed(seed, 0x517ULL));
  for (int i = 0; i < n; ++i) order[i] = i;
  for (int i = 0; i < n; ++i) {
    int64_t j = i + (int64_t)rng_bounded(rng, (uint64_t)(n - i));
    int64_t t = order[i];
    order[i] = order[j];
    order[j] = t;
  }
  free(rng);
  *n_train = (int)llround(frac * (double)n);
  return 0;
}

/* ---- mlp.cpp ------------------------------------------------------------------ */

/* mlp.cpp:9-25 Glorot-uniform, layer order, biases 0 */
int or_mlp_init(int n_dims, const int* dims, uint64_t seed, int raw_rng, double* params) {
  if (n_dims < 2) return -LANN_PARAM_ERROR;
  for (int l = 0; l < n_dims; ++l)
    if (dims[l] < 1) return -LANN_PARAM_ERROR;
  rng_t* rng = malloc(sizeof(rng_t));
  rng_seed(rng, raw_rng ? seed : or_derive_seed(seed, 0xA11CE));
  int off = 0;
  for (int l = 0; l + 1 < n_dims; ++l) {
    const int in = dims[l], out = dims[l + 1];
    const double bound = sqrt(6.0 / (in + out));
    for (int j = 0; j < in * out; ++j) params[off++] = rng_uniform_range(rng, -bound, bound);
    for (int o = 0; o < out; ++o) params[off++] = 0.0;
  }
  free(rng);
  return off;
}

#define MAXW 128 /* widest layer the oracle handles (unconstrained blur = 40, MM 64) */

/* mlp.cpp:36-52 forward_cached; acts[l] holds layer-l activations */
static void forward_cached(int n_dims, const int* dims, const double* params, const double* x,
                           double acts[][MAXW]) {
  for (int i = 0; i < dims[0]; ++i) acts[0][i] = x[i];
  int off = 0;
  for (int l = 0; l + 1 < n_dims; ++l) {
    const int in = dims[l], out = dims[l + 1];
    const double* w = params + off;
    const double* b = params + off + in * out;
    const int hidden = l + 2 < n_dims;
    for (int o = 0; o < out; ++o) {
      double z = b[o];
      for (int i = 0; i < in; ++i) z += w[o * in + i] * acts[l][i];
      acts[l + 1][o] = hidden ? (z > 0.0 ? z : 0.0) : z;
    }
    off += in * out + out;
  }
}

static int param_total(int n_dims, const int* dims) {
  int t = 0;
  for (int l = 0; l + 1 < n_dims; ++l) t += (dims[l] + 1) * dims[l + 1];
  return t;
}

/* mlp.cpp:75-122 mse_gradient, sequential over samples */
int or_mse_gradient(int n_dims, const int* dims, const double* params, int n, const double* X,
                    const double* y, double* loss, double* grad) {
  if (n < 1) return LANN_PARAM_ERROR;
  const int P = param_total(n_dims, dims);
  double acts[4][MAXW], delta[4][MAXW];
  for (int p = 0; p < P; ++p) grad[p] = 0.0;
  double L = 0.0;
  const double inv_n = 1.0 / (double)n;
  const int nl = n_dims - 1;
  for (int s = 0; s < n; ++s) {
    forward_cached(n_dims, dims, params, X + (size_t)s * LANN_ROW, acts);
    const double err = acts[nl][0] - y[s];
    L += err * err;
    delta[nl - 1][0] = 2.0 * err;
    /* walk layers backwards: next = layer l+1 */
    int off_next = 0;
    for (int l = 0; l + 1 < nl; ++l) off_next += (dims[l] + 1) * dims[l + 1];
    for (int l = nl - 1; l-- > 0;) {
      const int nin = dims[l + 1], nout = dims[l + 2];
      const double* nw = params + off_next;
      for (int i = 0; i < nin; ++i) {
        double acc = 0.0;
        for (int o = 0; o < nout; ++o) acc += nw[o * nin + i] * delta[l + 1][o];
        delta[l][i] = acts[l + 1][i] > 0.0 ? acc : 0.0;
      }
      off_next -= (dims[l] + 1) * dims[l + 1];
    }
    int off = 0;
    for (int l = 0; l < nl; ++l) {
      const int in = dims[l], out = dims[l + 1];
      double* gw = grad + off;
      for (int o = 0; o < out; ++o)
        for (int i = 0; i < in; ++i) gw[o * in + i] += inv_n * delta[l][o] * acts[l][i];
      off += in * out;
      double* gb = grad + off;
      for (int o = 0; o < out; ++o) gb[o] += inv_n * delta[l][o];
      off += out;
    }
  }
  *loss = L * inv_n;
  return 0;
}

/* mlp.cpp:142-175 Adam + train_full_batch */
int or_train_full_batch(int n_dims, const int* dims, double* params, int n, const double* X,
                        const double* y, double lr, int epochs, double* trace, int* bad_epoch) {
  *bad_epoch = -1;
  if (epochs < 1) return LANN_PARAM_ERROR;
  const int P = param_total(n_dims, dims);
  double* m = calloc((size_t)P, sizeof(double));
  double* v = calloc((size_t)P, sizeof(double));
  double* g = calloc((size_t)P, sizeof(double));
  const double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
  int status = 0;
  for (int e = 0; e < epochs; ++e) {
    double loss;
    or_mse_gradient(n_dims, dims, params, n, X, y, &loss, g);
    if (!isfinite(loss)) {
      *bad_epoch = e;
      status = LANN_TRAINING_ERROR;
      break;
    }
    if (trace) trace[e] = loss;
    const int step = e + 1;
    const double bc1 = 1.0 - pow(beta1, step);
    const double bc2 = 1.0 - pow(beta2, step);
    for (int i = 0; i < P; ++i) {
      m[i] = beta1 * m[i] + (1.0 - beta1) * g[i];
      v[i] = beta2 * v[i] + (1.0 - beta2) * g[i] * g[i];
      const double mhat = m[i] / bc1;
      const double vhat = v[i] / bc2;
      params[i] -= lr * mhat / (sqrt(vhat) + eps);
    }
  }
  free(m);
  free(v);
  free(g);
  return status;
}

/* ---- models.cpp --------------------------------------------------------------- */

/* models.cpp:89-116 NormStats::fit; norm = {f_min[8], f_max[8], t_min, t_max} */
void or_norm_fit(int n, int I, const double* X, const double* y, int log_target, double* norm) {
  for (int j = 0; j < 18; ++j) norm[j] = 0.0;
  for (int j = 0; j < I; ++j) {
    norm[j] = INFINITY;
    norm[8 + j] = -INFINITY;
  }
  for (int s = 0; s < n; ++s)
    for (int j = 0; j < I; ++j) {
      const double x = X[(size_t)s * LANN_ROW + j];
      norm[j] = x < norm[j] ? x : norm[j];             /* std::min(f_min, x) */
      norm[8 + j] = norm[8 + j] < x ? x : norm[8 + j]; /* std::max(f_max, x) */
    }
  double lo = y[0], hi = y[0];
  for (int s = 0; s < n; ++s) {
    lo = y[s] < lo ? y[s] : lo;
    hi = hi < y[s] ? y[s] : hi;
  }
  norm[16] = log_target ? log(lo) : lo;
  norm[17] = log_target ? log(hi) : hi;
}

/* models.cpp:118-127 */
static double norm_feature(const double* norm, int j, double x) {
  const double range = norm[8 + j] - norm[j];
  return range > 0.0 ? (x - norm[j]) / range : 0.0;
}
/* models.cpp:129-133 */
static double norm_target(const double* norm, int log_target, double t) {
  const double range = norm[17] - norm[16];
  const double v = log_target ? log(t) : t;
  return range > 0.0 ? (v - norm[16]) / range : 0.0;
}
/* models.cpp:135-139 */
static double denorm_target(const double* norm, int log_target, double ts) {
  const double range = norm[17] - norm[16];
  const double v = range > 0.0 ? norm[16] + ts * range : norm[16];
  return log_target ? exp(v) : v;
}

/* models.cpp:346-363 predict (MLP payload), x = model-input vector of length I */
double or_predict_row(int I, int n_hidden, const int* hidden, const double* params,
                      const double* norm, int log_target, const double* x) {
  int dims[4] = {I, hidden[0], n_hidden > 1 ? hidden[1] : 1, 1};
  const int nd = n_hidden + 2;
  double xn[LANN_ROW], acts[4][MAXW];
  for (int j = 0; j < I; ++j) xn[j] = norm_feature(norm, j, x[j]);
  forward_cached(nd, dims, params, xn, acts);
  const double v = denorm_target(norm, log_target, acts[nd - 1][0]);
  return v < 1e-9 ? 1e-9 : v; /* std::max(value, 1e-9) */
}

/* ---- eval.cpp ---------------------------------------------------------------- */

static int check_pair(int n, const double* t) {
  if (n < 1) return LANN_DOMAIN_ERROR;
  for (int i = 0; i < n; ++i)
    if (!(t[i] > 0.0)) return LANN_DOMAIN_ERROR;
  return 0;
}

/* eval.cpp:26-32 */
int or_mape(int n, const double* t, const double* p, double* out) {
  if (check_pair(n, t)) return LANN_DOMAIN_ERROR;
  double acc = 0.0;
  for (int i = 0; i < n; ++i) acc += fabs(t[i] - p[i]) / t[i];
  *out = 100.0 * acc / (double)n;
  return 0;
}

static const double* g_sort_key;
static int cmp_truth_index(const void* a, const void* b) {
  const int64_t i = *(const int64_t*)a, j = *(const int64_t*)b;
  if (g_sort_key[i] != g_sort_key[j]) return g_sort_key[i] < g_sort_key[j] ? -1 : 1;
  return i < j ? -1 : (i > j);
}

/* eval.cpp:34-57: drop floor(drop*n) smallest truths (ties by index), sum in sorted order */
int or_mape_thresholded(int n, const double* t, const double* p, double drop, double* out,
                        int* kept) {
  if (check_pair(n, t)) return LANN_DOMAIN_ERROR;
  if (drop < 0.0 || drop > 1.0) return LANN_DOMAIN_ERROR;
  const int n_drop = (int)floor(drop * (double)n + 1e-12);
  if (n_drop >= n) return LANN_DOMAIN_ERROR;
  int64_t* order = malloc(sizeof(int64_t) * (size_t)n);
  for (int i = 0; i < n; ++i) order[i] = i;
  g_sort_key = t;
  qsort(order, (size_t)n, sizeof(int64_t), cmp_truth_index);
  double acc = 0.0;
  for (int i = n_drop; i < n; ++i) {
    const int64_t j = order[i];
    acc += fabs(t[j] - p[j]) / t[j];
  }
  free(order);
  *kept = n - n_drop;
  *out = 100.0 * acc / (double)(*kept);
  return 0;
}

/* eval.cpp:59-75 average ranks (tie groups share the mean 1-based rank); computed
 * by counting, which equals the sort-based result exactly (ranks are halves) */
static void average_ranks(int n, const double* v, double* ranks) {
  for (int i = 0; i < n; ++i) {
    int64_t less = 0, eq = 0;
    for (int j = 0; j < n; ++j) {
      less += v[j] < v[i];
      eq += v[j] == v[i];
    }
    /* positions less .. less+eq-1 (0-based): (i + j) / 2 + 1 */
    ranks[i] = ((double)less + (double)(less + eq - 1)) / 2.0 + 1.0;
  }
}

/* eval.cpp:77-90 */
int or_spearman(int n, const double* t, const double* p, double* out) {
  if (n < 2) return LANN_DOMAIN_ERROR;
  double* rt = malloc(sizeof(double) * (size_t)n);
  double* rp = malloc(sizeof(double) * (size_t)n);
  average_ranks(n, t, rt);
  average_ranks(n, p, rp);
  const double nn = (double)n;
  double d2 = 0.0;
  for (int i = 0; i < n; ++i) {
    const double d = rt[i] - rp[i];
    d2 += d * d;
  }
  free(rt);
  free(rp);
  *out = 1.0 - 6.0 * d2 / (nn * (nn * nn - 1.0));
  return 0;
}

/* ---- selector.cpp ------------------------------------------------------------ */

static int lex_less(const uint32_t* a, const uint32_t* b) {
  for (int j = 0; j < 4; ++j)
    if (a[j] != b[j]) return a[j] < b[j];
  return 0;
}

/* selector.cpp:26-53: argmin of predict over blur candidates, ties -> lexicographic */
int64_t or_select_schedule(int family, int n_hidden, const int* hidden, const double* params,
                           const double* norm, int log_target, uint32_t n_img, int64_t n_cands,
                           const uint32_t* cands, double* score) {
  const int I = family == LANN_NNC ? 6 : 5;
  int64_t best = -1;
  double best_score = 0.0;
  for (int64_t i = 0; i < n_cands; ++i) {
    double x[LANN_ROW];
    x[0] = n_img;
    for (int j = 0; j < 4; ++j) x[1 + j] = cands[4 * i + j];
    x[5] = (double)((uint64_t)n_img * n_img);
    const double s = or_predict_row(I, n_hidden, hidden, params, norm, log_target, x);
    if (best < 0 || s < best_score ||
        (s == best_score && lex_less(cands + 4 * i, cands + 4 * best))) {
      best = i;
      best_score = s;
    }
  }
  *score = best_score;
  return best;
}

/* ---- counter-based candidates (engine definition, lann_engine.h) ---------------- */
static uint64_t sm_bounded(void* src, uint64_t n) {
  uint64_t* st = (uint64_t*)src;
  const uint64_t threshold = (0 - n) % n; /* rng.hpp:34-40 rejection rule */
  for (;;) {
    const uint64_t x = or_splitmix64(st);
    if (x >= threshold) return x % n;
  }
}

void or_candidate(int kind, int max_threads, uint64_t seed, int64_t idx, double* base,
                  uint64_t* c) {
  uint64_t st = or_derive_seed(seed, (uint64_t)idx);
  params_t p;
  sample_params(kind, max_threads, 0, sm_bounded, &st, &p);
  memset(base, 0, LANN_ROW * sizeof(double));
  featurize_base(&p, 1, base); /* n_thd last; models without it ignore the column */
  *c = complexity(&p);
}

static int base_count(int kind) {
  switch (kind) {
    case LANN_MM: return 5;
    case LANN_MV: return 3;
    case LANN_MC: return 4;
    case LANN_MP: return 5;
    default: return 5;
  }
}

void or_select_variants(const lann_model_set* ms, const int32_t* with_n_thd, int kind,
                        int max_threads, uint64_t seed, int64_t first, int64_t n_cands,
                        int32_t* out_idx, double* out_score) {
  for (int64_t i = 0; i < n_cands; ++i) {
    double base[LANN_ROW];
    uint64_t c;
    or_candidate(kind, max_threads, seed, first + i, base, &c);
    const int nb = base_count(kind);
    int32_t best = -1;
    double best_s = 0.0;
    for (int v = 0; v < ms->n_models; ++v) {
      double x[LANN_ROW];
      int I = 0;
      for (int j = 0; j < nb; ++j) x[I++] = base[j];
      if (with_n_thd[v]) x[I++] = base[nb];
      if (I < ms->n_inputs[v]) x[I++] = (double)c; /* augmented family appends c */
      int hidden[2] = {ms->h1[v], ms->h2[v]};
      const double s = or_predict_row(ms->n_inputs[v], ms->h2[v] > 0 ? 2 : 1, hidden,
                                      ms->params + ms->param_offset[v], ms->norm + 18 * v,
                                      ms->log_target[v], x);
      if (best < 0 || s < best_s) {
        best = v;
        best_s = s;
      }
    }
    out_idx[i] = best;
    out_score[i] = best_s;
  }
}

/* ---- models::train_nn + predict_dataset + make_report (models.cpp:279-303) ----- */
static int validate_config(const lann_job* j, int I) {
  if (j->n_hidden < 1 || j->n_hidden > 2) return LANN_PARAM_ERROR;
  for (int h = 0; h < j->n_hidden; ++h)
    if (j->hidden[h] < 1) return LANN_PARAM_ERROR;
  if (!(j->learning_rate == 1e-2 || j->learning_rate == 1e-3 || j->learning_rate == 1e-4))
    return LANN_PARAM_ERROR;
  if (j->epochs < 1) return LANN_PARAM_ERROR;
  int dims[4] = {I, j->hidden[0], j->n_hidden > 1 ? j->hidden[1] : 1, 1};
  if (!j->unconstrained && param_total(j->n_hidden + 2, dims) > 75) return LANN_PARAM_ERROR;
  return 0;
}

int or_run_job(const lann_job* j, lann_job_result* r, double* params_out, double* trace) {
  memset(r, 0, sizeof *r);
  r->nonfinite_epoch = -1;
  const int count = j->count;
  double* feats = malloc(sizeof(double) * LANN_ROW * (size_t)count);
  uint64_t* c = malloc(sizeof(uint64_t) * (size_t)count);
  double* rt = malloc(sizeof(double) * (size_t)count);
  int64_t* order = malloc(sizeof(int64_t) * (size_t)count);
  int nf = 0, n_train = 0;
  int st = or_build_dataset(&j->world, j->data_seed, count, feats, c, rt, &nf);
  if (!st) st = or_split_order(count, j->train_fraction, j->data_seed, order, &n_train);
  if (st) goto done;
  {
    /* index lists of the training and evaluation parts */
    int64_t* tr = malloc(sizeof(int64_t) * (size_t)count);
    int64_t* ev = malloc(sizeof(int64_t) * (size_t)count);
    int ntr = 0, nev = 0;
    if (j->n_folds >= 2) {
      const int b0 = n_train * j->fold / j->n_folds, b1 = n_train * (j->fold + 1) / j->n_folds;
      for (int i = 0; i < n_train; ++i) {
        if (i >= b0 && i < b1) ev[nev++] = order[i];
        else tr[ntr++] = order[i];
      }
    } else {
      for (int i = 0; i < n_train; ++i) tr[ntr++] = order[i];
      for (int i = n_train; i < count; ++i) ev[nev++] = order[i];
    }
    const int aug = j->family == LANN_NNC;
    const int I = nf + aug;
    if (ntr < 2) { st = LANN_PARAM_ERROR; goto done2; } /* models.cpp:173 */
    st = validate_config(j, I);
    if (st) goto done2;
    /* assemble (models.cpp:172-182) */
    double* X = calloc((size_t)ntr * LANN_ROW, sizeof(double));
    double* y = malloc(sizeof(double) * (size_t)ntr);
    for (int s = 0; s < ntr; ++s) {
      memcpy(X + (size_t)s * LANN_ROW, feats + tr[s] * LANN_ROW, sizeof(double) * (size_t)nf);
      if (aug) X[(size_t)s * LANN_ROW + nf] = (double)c[tr[s]];
      y[s] = rt[tr[s]];
    }
    double norm[18];
    or_norm_fit(ntr, I, X, y, j->log_target, norm);
    {
      double lo = y[0];
      for (int s = 0; s < ntr; ++s) lo = y[s] < lo ? y[s] : lo;
      if (j->log_target && !(lo > 0.0)) { st = LANN_PARAM_ERROR; free(X); free(y); goto done2; }
    }
    double* Xn = calloc((size_t)ntr * LANN_ROW, sizeof(double));
    double* yn = malloc(sizeof(double) * (size_t)ntr);
    for (int s = 0; s < ntr; ++s) {
      for (int k = 0; k < I; ++k)
        Xn[(size_t)s * LANN_ROW + k] = norm_feature(norm, k, X[(size_t)s * LANN_ROW + k]);
      yn[s] = norm_target(norm, j->log_target, y[s]);
    }
    int dims[4] = {I, j->hidden[0], j->n_hidden > 1 ? j->hidden[1] : 1, 1};
    const int nd = j->n_hidden + 2;
    const int P = param_total(nd, dims);
    double* params = malloc(sizeof(double) * (size_t)P);
    or_mlp_init(nd, dims, j->init_seed, 0, params);
    double* tr_buf = trace ? trace : malloc(sizeof(double) * (size_t)j->epochs);
    int bad = -1;
    st = or_train_full_batch(nd, dims, params, ntr, Xn, yn, j->learning_rate, j->epochs, tr_buf,
                             &bad);
    r->nonfinite_epoch = bad;
    r->n_inputs = I;
    r->n_params = P;
    r->n_train = ntr;
    r->n_eval = nev;
    if (!st) {
      r->final_loss = tr_buf[j->epochs - 1];
      double* truth = malloc(sizeof(double) * (size_t)(nev > 0 ? nev : 1));
      double* pred = malloc(sizeof(double) * (size_t)(nev > 0 ? nev : 1));
      for (int s = 0; s < nev; ++s) {
        double x[LANN_ROW] = {0};
        memcpy(x, feats + ev[s] * LANN_ROW, sizeof(double) * (size_t)nf);
        if (aug) x[nf] = (double)c[ev[s]];
        pred[s] = or_predict_row(I, j->n_hidden, j->hidden, params, norm, j->log_target, x);
        truth[s] = rt[ev[s]];
      }
      int kept = 0;
      st = or_mape(nev, truth, pred, &r->mape);
      if (!st) st = or_mape_thresholded(nev, truth, pred, 0.3, &r->mape_thr, &kept);
      if (!st) st = or_spearman(nev, truth, pred, &r->rho);
      r->n_kept = kept;
      free(truth);
      free(pred);
    }
    if (params_out) memcpy(params_out, params, sizeof(double) * (size_t)P);
    if (!trace) free(tr_buf);
    free(params);
    free(Xn);
    free(yn);
    free(X);
    free(y);
  done2:
    free(tr);
    free(ev);
  }
done:
  r->status = st;
  free(feats);
  free(c);
  free(rt);
  free(order);
  return st;
}

/* Cross-validation fold-mean model (engine definition, include/lann_engine.h "cross-validation
 * summary"; the reference has no k-fold driver). fold_jobs[f] is fold f of one seed (all other
 * fields equal), params[f] its trained weights. Each fold model predicts the split's test part
 * order[n_train..count) (datagen.cpp:225-248) with its own NormStats (fit on its training blocks,
 * models.cpp:89-116) as models::predict does (models.cpp:346-363); the predictions are summed in
 * fold order and divided by k. Writes n_test predictions and the truths beside them. */
int or_fold_mean(int k, const lann_job* fold_jobs, const double* const* params, double* pred, double* truth,
                 int* n_test) {
  const lann_job* j0 = &fold_jobs[0];
  const int count = j0->count;
  double* feats = malloc(sizeof(double) * LANN_ROW * (size_t)count);
  uint64_t* c = malloc(sizeof(uint64_t) * (size_t)count);
  double* rt = malloc(sizeof(double) * (size_t)count);
  int64_t* order = malloc(sizeof(int64_t) * (size_t)count);
  int nf = 0, n_train = 0;
  int st = or_build_dataset(&j0->world, j0->data_seed, count, feats, c, rt, &nf);
  if (!st) st = or_split_order(count, j0->train_fraction, j0->data_seed, order, &n_train);
  const int nt = count - n_train;
  *n_test = nt;
  const int aug = j0->family == LANN_NNC;
  const int I = nf + aug;
  double* X = calloc((size_t)(n_train > 0 ? n_train : 1) * LANN_ROW, sizeof(double));
  double* y = malloc(sizeof(double) * (size_t)(n_train > 0 ? n_train : 1));
  for (int f = 0; f < k && !st; ++f) {
    const lann_job* j = &fold_jobs[f];
    const int b0 = n_train * j->fold / j->n_folds, b1 = n_train * (j->fold + 1) / j->n_folds;
    int ntr = 0;
    for (int i = 0; i < n_train; ++i) {
      if (i >= b0 && i < b1) continue;
      memset(X + (size_t)ntr * LANN_ROW, 0, sizeof(double) * LANN_ROW);
      memcpy(X + (size_t)ntr * LANN_ROW, feats + order[i] * LANN_ROW, sizeof(double) * (size_t)nf);
      if (aug) X[(size_t)ntr * LANN_ROW + nf] = (double)c[order[i]];
      y[ntr++] = rt[order[i]];
    }
    double norm[18];
    or_norm_fit(ntr, I, X, y, j->log_target, norm);
    for (int s = 0; s < nt; ++s) {
      const int64_t idx = order[n_train + s];
      double x[LANN_ROW] = {0};
      memcpy(x, feats + idx * LANN_ROW, sizeof(double) * (size_t)nf);
      if (aug) x[nf] = (double)c[idx];
      const double p = or_predict_row(I, j->n_hidden, j->hidden, params[f], norm, j->log_target, x);
      pred[s] = f == 0 ? p : pred[s] + p;
      truth[s] = rt[idx];
    }
  }
  for (int s = 0; s < nt && !st; ++s) pred[s] = pred[s] / (double)k;
  free(X);
  free(y);
  free(feats);
  free(c);
  free(rt);
  free(order);
  return st;
}
