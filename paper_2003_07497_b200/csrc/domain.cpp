// domain.cpp — see domain.hpp. Reference behaviour is cited per function.
#include "domain.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>

namespace lann {

std::uint64_t complexity(const Instance& p) {
  const std::uint64_t m = p.m, n = p.n, k = p.k;
  switch (p.kind) {
    case LANN_MM: return m * n * k;
    case LANN_MV: return m * n;
    case LANN_MC: {
      const std::uint64_t r = p.r;
      return (m - r + 1) * (n - r + 1) * r * r;
    }
    case LANN_MP: {
      const std::uint64_t s = p.s;
      return ((n + s - 1) / s) * ((m + s - 1) / s) * s * s;
    }
    default: return n * n;
  }
}

int base_feature_count(int kind, bool with_n_thd) {
  static const int base[5] = {5, 3, 4, 5, 5};
  return base[kind] + ((with_n_thd && kind != LANN_BLUR) ? 1 : 0);
}

int base_features(const Instance& p, bool with_n_thd, double* f) {
  int n = 0;
  switch (p.kind) {
    case LANN_MM:
      for (double v : {double(p.m), double(p.n), double(p.k), p.d1, p.d2}) f[n++] = v;
      break;
    case LANN_MV:
      for (double v : {double(p.m), double(p.n), p.d}) f[n++] = v;
      break;
    case LANN_MC:
      for (double v : {double(p.m), double(p.n), double(p.r), p.d}) f[n++] = v;
      break;
    case LANN_MP:
      for (double v : {double(p.m), double(p.n), double(p.r), double(p.s), p.d}) f[n++] = v;
      break;
    default:
      f[n++] = double(p.n);
      for (int j = 0; j < 4; ++j) f[n++] = double(p.sched[j]);
      return n;  // blur never takes n_thd
  }
  if (with_n_thd) f[n++] = double(p.n_thd);
  return n;
}

const std::vector<std::uint32_t>& schedule_lattice(int gpu_style) {
  static std::vector<std::uint32_t> tables[2];
  static std::once_flag once;
  std::call_once(once, [] {
    for (int g = 0; g < 2; ++g) {
      const std::uint32_t lo[4] = {2, g ? 1u : 2u, g ? 1u : 2u, g ? 1u : 2u};
      const std::uint32_t hi[4] = {g ? 16u : 1024u, g ? 64u : 1024u, g ? 64u : 1024u, g ? 1u : 1024u};
      for (std::uint32_t a = std::bit_ceil(lo[0]); a <= hi[0]; a <<= 1)
        for (std::uint32_t b = std::bit_ceil(lo[1]); b <= hi[1]; b <<= 1)
          for (std::uint32_t c = std::bit_ceil(lo[2]); c <= (g ? hi[2] : std::min(hi[2], b)); c <<= 1)
            for (std::uint32_t d = std::bit_ceil(lo[3]); d <= (g ? hi[3] : std::min(hi[3], c)); d <<= 1)
              for (std::uint32_t v : {a, b, c, d}) tables[g].push_back(v);
    }
  });
  return tables[gpu_style ? 1 : 0];
}

namespace {

// datagen.cpp:38-45 — dyadic ladder {1, 1/2, ...} down to 2^-floor(log2 cells)
double pick_density(std::uint64_t cells, bool include_one, SeqRng& rng) {
  const int depth = int(std::bit_width(cells)) - 1;
  const int first = include_one ? 0 : 1;
  const int len = depth >= first ? depth - first + 1 : 0;
  if (len == 0) {
    (void)rng.bounded(1);
    return 1.0;
  }
  return std::ldexp(1.0, -(first + int(rng.bounded(std::uint64_t(len)))));
}

std::uint32_t uniform_dim(SeqRng& rng, std::uint32_t lo, std::uint32_t hi) {
  return std::uint32_t(std::int64_t(lo) + std::int64_t(rng.bounded(std::uint64_t(hi - lo) + 1)));
}

}  // namespace

Instance sample_instance(const SampleSpace& sp, SeqRng& rng) {
  const int kind = sp.kind, max_threads = sp.max_threads, gpu_lattice = sp.gpu_lattice;
  const std::uint32_t lo = sp.dim_min, hi = sp.dim_max;
  static const std::uint32_t mc_r[3] = {3, 5, 7}, mp_r[4] = {2, 3, 4, 5}, mp_s[2] = {1, 2};
  const bool inc_one = kind != LANN_MV;  // ParamSpace::defaults (datagen.cpp:18-24)
  Instance p;
  p.kind = kind;
  auto threads = [&] { return int(uniform_dim(rng, 1, std::uint32_t(max_threads))); };
  switch (kind) {
    case LANN_MM: {
      p.m = uniform_dim(rng, lo, hi);
      p.n = uniform_dim(rng, lo, hi);
      p.k = uniform_dim(rng, lo, hi);
      p.d1 = pick_density(std::uint64_t(p.m) * p.n, inc_one, rng);
      p.d2 = pick_density(std::uint64_t(p.n) * p.k, inc_one, rng);
      p.n_thd = threads();
      break;
    }
    case LANN_MV:
      p.m = uniform_dim(rng, lo, hi);
      p.n = uniform_dim(rng, lo, hi);
      p.d = pick_density(std::uint64_t(p.m) * p.n, inc_one, rng);
      p.n_thd = threads();
      break;
    case LANN_MC:
      p.r = mc_r[rng.bounded(3)];
      p.m = uniform_dim(rng, std::max(lo, p.r), std::max(hi, p.r));
      p.n = uniform_dim(rng, std::max(lo, p.r), std::max(hi, p.r));
      p.d = pick_density(std::uint64_t(p.m) * p.n, inc_one, rng);
      p.n_thd = threads();
      break;
    case LANN_MP:
      p.r = mp_r[rng.bounded(4)];
      p.s = mp_s[rng.bounded(2)];
      p.m = uniform_dim(rng, std::max(lo, p.r), std::max(hi, p.r));
      p.n = uniform_dim(rng, std::max(lo, p.r), std::max(hi, p.r));
      p.d = pick_density(std::uint64_t(p.m) * p.n, inc_one, rng);
      p.n_thd = threads();
      break;
    default: {
      p.n = sp.sides[rng.bounded(sp.sides.size())];
      const auto& lat = schedule_lattice(gpu_lattice);
      const std::uint64_t i = rng.bounded(lat.size() / 4);
      std::memcpy(p.sched, &lat[4 * i], sizeof p.sched);
      break;
    }
  }
  return p;
}

Instance sample_instance(int kind, int max_threads, int gpu_lattice, SeqRng& rng) {
  SampleSpace sp;
  sp.kind = kind;
  sp.max_threads = max_threads;
  sp.gpu_lattice = gpu_lattice;
  return sample_instance(sp, rng);
}

// perfsage.cpp:71-84 (mock_probe, the CLI's --mock-timer): hash the bits of the augmented
// feature vector (featurize(params, true): base features, n_thd except for blur, then c)
// through splitmix64 -> jitter in [0.5, 1.5) -> 1e-9 * c * jitter + 1e-6
double mock_runtime(const Instance& p) {
  double f[LANN_ROW + 1] = {0};
  int n = base_features(p, true, f);
  f[n++] = double(complexity(p));
  std::uint64_t h = 0x9e3779b97f4a7c15ULL;
  for (int i = 0; i < n; ++i) {
    std::uint64_t bits;
    std::memcpy(&bits, &f[i], sizeof bits);
    h ^= bits;
    splitmix64(h);
  }
  const double jitter = 0.5 + double(splitmix64(h) >> 11) * 0x1.0p-53;
  return 1e-9 * double(complexity(p)) * jitter + 1e-6;
}

Status build_mock_dataset(const SampleSpace& sp, bool single_threaded, std::uint64_t seed, int count, Dataset& ds) {
  if (count < 2) return {LANN_PARAM_ERROR, "build_dataset needs count >= 2"};
  if (sp.kind < 0 || sp.kind > LANN_BLUR) return {LANN_PARAM_ERROR, "unknown kernel kind"};
  if (sp.max_threads < 1) return {LANN_PARAM_ERROR, "param space needs max_threads >= 1"};
  if (sp.dim_min < 1 || sp.dim_max < sp.dim_min) return {LANN_PARAM_ERROR, "param space needs 1 <= dim_min <= dim_max"};
  if (sp.kind == LANN_BLUR && sp.sides.empty()) return {LANN_PARAM_ERROR, "blur space needs image sides"};
  const bool takes_thd = sp.kind != LANN_BLUR;  // native variants are CPU class (variants.hpp:29-31)
  ds.kind = sp.kind;
  ds.n_features = base_feature_count(sp.kind, takes_thd);
  ds.feats.assign(std::size_t(count) * LANN_ROW, 0.0);
  ds.c.assign(count, 0);
  ds.runtime.assign(count, 0.0);
  SeqRng rng(derive_seed(seed, 0));
  for (int i = 0; i < count; ++i) {
    Instance p = sample_instance(sp, rng);
    if (single_threaded) p.n_thd = 1;               // Threading::FixedSingle (datagen.cpp:195)
    if (sp.kind == LANN_BLUR) p.n_thd = sp.max_threads;  // datagen.cpp:196
    base_features(p, takes_thd, &ds.feats[std::size_t(i) * LANN_ROW]);
    ds.c[i] = complexity(p);
    ds.runtime[i] = mock_runtime(p);
  }
  return {};
}

namespace {

// lann_world probe (lann_engine.h); acceptance_main.cpp:271-279 is the special case
double world_runtime(const lann_world& w, const Instance& p, SeqRng& noise_rng) {
  double g, fd = 1.0;
  if (p.kind == LANN_BLUR) {
    g = 1.0;
    for (int j = 0; j < 4; ++j) {
      const double d = double(std::countr_zero(p.sched[j])) - w.mu[j];
      g += w.kappa[j] * d * d;
    }
  } else {
    g = w.g0 + w.g1 / double(p.n_thd);
    const double dens = p.kind == LANN_MM ? p.d1 : p.d;
    fd = (1.0 - w.delta) + w.delta * dens;
  }
  const double nz = 1.0 + noise_rng.uniform(-w.noise, w.noise);
  return w.alpha * double(complexity(p)) * g * fd * nz + w.beta;
}

}  // namespace

Status build_dataset(const lann_world& w, std::uint64_t seed, int count, Dataset& ds) {
  if (count < 2) return {LANN_PARAM_ERROR, "build_dataset needs count >= 2"};
  if (w.kind < 0 || w.kind > LANN_BLUR) return {LANN_PARAM_ERROR, "unknown kernel kind"};
  if (w.max_threads < 1) return {LANN_PARAM_ERROR, "param space needs max_threads >= 1"};
  const bool takes_thd = w.hw_class == LANN_HW_CPU && w.kind != LANN_BLUR;  // variants.hpp:29-31
  ds.kind = w.kind;
  ds.n_features = base_feature_count(w.kind, takes_thd);
  ds.feats.assign(std::size_t(count) * LANN_ROW, 0.0);
  ds.c.assign(count, 0);
  ds.runtime.assign(count, 0.0);
  SeqRng rng(derive_seed(seed, 0));
  SeqRng noise(derive_seed(seed, 0x9015E));
  SampleSpace sp;  // the default space, built once (its side list is a heap vector)
  sp.kind = w.kind;
  sp.max_threads = w.max_threads;
  sp.gpu_lattice = w.blur_lattice;
  for (int i = 0; i < count; ++i) {
    Instance p = sample_instance(sp, rng);
    if (w.hw_class != LANN_HW_CPU) p.n_thd = 1;      // Threading::FixedSingle (datagen.cpp:195)
    if (w.kind == LANN_BLUR) p.n_thd = w.max_threads; // datagen.cpp:196
    base_features(p, takes_thd, &ds.feats[std::size_t(i) * LANN_ROW]);
    ds.c[i] = complexity(p);
    ds.runtime[i] = world_runtime(w, p, noise);
    if (!(ds.runtime[i] > 0.0)) {
      ds.runtime.resize(i);
      return {LANN_BUILD_ABORT, "dataset build aborted after " + std::to_string(i) + "/" +
                                    std::to_string(count) + " samples: measured runtime must be > 0"};
    }
  }
  return {};
}

Status probe_schedules(const lann_world& w, std::uint64_t seed, std::uint32_t image_n, int n,
                       const std::uint32_t* sched, double* runtime) {
  if (w.kind != LANN_BLUR) return {LANN_PARAM_ERROR, "schedule probes need a blur world"};
  if (n < 0 || image_n == 0) return {LANN_PARAM_ERROR, "bad probe request"};
  SeqRng noise(derive_seed(seed, 0x9015E));
  for (int i = 0; i < n; ++i) {
    Instance p;
    p.kind = LANN_BLUR;
    p.n = image_n;
    p.n_thd = w.max_threads;
    for (int j = 0; j < 4; ++j) {
      p.sched[j] = sched[4 * i + j];
      if (p.sched[j] == 0 || (p.sched[j] & (p.sched[j] - 1)) != 0)
        return {LANN_PARAM_ERROR, "schedule factors must be positive powers of two"};
    }
    runtime[i] = world_runtime(w, p, noise);
  }
  return {};
}

Status split_order(int n, double frac, std::uint64_t seed, std::vector<std::int64_t>& order,
                   int& n_train) {
  if (!(frac > 0.0 && frac < 1.0)) return {LANN_PARAM_ERROR, "train fraction must lie in (0,1)"};
  order.resize(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  SeqRng rng(derive_seed(seed, 0x517ULL));
  for (int i = 0; i < n; ++i) std::swap(order[i], order[i + std::int64_t(rng.bounded(std::uint64_t(n - i)))]);
  n_train = int(std::llround(frac * double(n)));
  return {};
}

Status make_tile(const Dataset& ds, const std::vector<std::int64_t>& order, int n_train,
                 int n_folds, int fold, int family, bool log_target, Tile& t) {
  std::vector<std::int64_t> tr, ev;
  if (n_folds >= 2) {
    if (fold < 0 || fold >= n_folds) return {LANN_PARAM_ERROR, "fold index out of range"};
    const int b0 = n_train * fold / n_folds, b1 = n_train * (fold + 1) / n_folds;
    for (int i = 0; i < n_train; ++i) (i >= b0 && i < b1 ? ev : tr).push_back(order[i]);
  } else {
    tr.assign(order.begin(), order.begin() + n_train);
    ev.assign(order.begin() + n_train, order.end());
  }
  if (tr.size() < 2) return {LANN_PARAM_ERROR, "training needs at least 2 samples"};  // models.cpp:173
  const bool aug = family == LANN_NNC;
  const int nf = ds.n_features, I = nf + (aug ? 1 : 0);
  t.n_inputs = I;
  t.log_target = log_target;
  auto row_of = [&](std::int64_t s, double* dst) {
    std::fill(dst, dst + LANN_ROW, 0.0);
    std::memcpy(dst, &ds.feats[std::size_t(s) * LANN_ROW], sizeof(double) * nf);
    if (aug) dst[nf] = double(ds.c[s]);  // model_features (models.cpp:143-148)
  };
  // NormStats::fit (models.cpp:89-116)
  std::vector<double> raw(tr.size() * LANN_ROW);
  std::fill(t.norm, t.norm + 18, 0.0);
  for (int j = 0; j < I; ++j) {
    t.norm[j] = std::numeric_limits<double>::infinity();
    t.norm[8 + j] = -std::numeric_limits<double>::infinity();
  }
  for (std::size_t s = 0; s < tr.size(); ++s) {
    row_of(tr[s], &raw[s * LANN_ROW]);
    for (int j = 0; j < I; ++j) {
      t.norm[j] = std::min(t.norm[j], raw[s * LANN_ROW + j]);
      t.norm[8 + j] = std::max(t.norm[8 + j], raw[s * LANN_ROW + j]);
    }
  }
  double lo = ds.runtime[tr[0]], hi = lo;
  for (auto s : tr) {
    lo = std::min(lo, ds.runtime[s]);
    hi = std::max(hi, ds.runtime[s]);
  }
  if (log_target) {
    if (!(lo > 0.0)) return {LANN_PARAM_ERROR, "targets must be positive runtimes"};
    t.norm[16] = std::log(lo);
    t.norm[17] = std::log(hi);
  } else {
    t.norm[16] = lo;
    t.norm[17] = hi;
  }
  // normalize / normalize_target (models.cpp:118-133)
  t.Xn.assign(tr.size() * LANN_ROW, 0.0);
  t.yn.resize(tr.size());
  const double trange = t.norm[17] - t.norm[16];
  for (std::size_t s = 0; s < tr.size(); ++s) {
    for (int j = 0; j < I; ++j) {
      const double range = t.norm[8 + j] - t.norm[j];
      t.Xn[s * LANN_ROW + j] = range > 0.0 ? (raw[s * LANN_ROW + j] - t.norm[j]) / range : 0.0;
    }
    const double v = log_target ? std::log(ds.runtime[tr[s]]) : ds.runtime[tr[s]];
    t.yn[s] = trange > 0.0 ? (v - t.norm[16]) / trange : 0.0;
  }
  t.eval_rows.assign(ev.size() * LANN_ROW, 0.0);
  t.eval_truth.resize(ev.size());
  for (std::size_t s = 0; s < ev.size(); ++s) {
    row_of(ev[s], &t.eval_rows[s * LANN_ROW]);
    t.eval_truth[s] = ds.runtime[ev[s]];
  }
  // k-fold tiles also carry the split's test part (no fold trains or validates on it): the
  // rows the fold-mean model of a cross-validation ensemble is scored on
  t.test_rows.clear();
  t.test_truth.clear();
  if (n_folds >= 2) {
    const std::size_t n_test = order.size() - std::size_t(n_train);
    t.test_rows.assign(n_test * LANN_ROW, 0.0);
    t.test_truth.resize(n_test);
    for (std::size_t s = 0; s < n_test; ++s) {
      row_of(order[std::size_t(n_train) + s], &t.test_rows[s * LANN_ROW]);
      t.test_truth[s] = ds.runtime[order[std::size_t(n_train) + s]];
    }
  }
  return {};
}

int param_count(int n_inputs, int h1, int h2) {
  return h2 > 0 ? (n_inputs + 1) * h1 + (h1 + 1) * h2 + (h2 + 1) : (n_inputs + 1) * h1 + (h1 + 1);
}

Status validate_config(const lann_job& j, int n_inputs) {
  if (j.family != LANN_NNC && j.family != LANN_NN)
    return {LANN_PARAM_ERROR, "train_nn expects an NN family config"};
  if (j.n_hidden < 1 || j.n_hidden > 2)
    return {LANN_PARAM_ERROR, "networks use 1 hidden layer (prediction) or 2 (selection)"};
  for (int h = 0; h < j.n_hidden; ++h)
    if (j.hidden[h] < 1) return {LANN_PARAM_ERROR, "hidden widths must be >= 1"};
  const double lr = j.learning_rate;
  if (!(lr == 1e-2 || lr == 1e-3 || lr == 1e-4))
    return {LANN_PARAM_ERROR, "learning rate must be one of 1e-2, 1e-3, 1e-4"};
  if (j.epochs < 1) return {LANN_PARAM_ERROR, "epochs must be >= 1"};
  if (!j.unconstrained &&
      param_count(n_inputs, j.hidden[0], j.n_hidden > 1 ? j.hidden[1] : 0) > 75)
    return {LANN_PARAM_ERROR, "lightweight model exceeds the 75-parameter budget"};
  return {};
}

void glorot_init(int I, int h1, int h2, std::uint64_t seed, double* params) {
  SeqRng rng(derive_seed(seed, 0xA11CE));  // models.cpp:298
  const int dims[4] = {I, h1, h2 > 0 ? h2 : 1, 1};
  const int nl = h2 > 0 ? 3 : 2;
  int off = 0;
  for (int l = 0; l < nl; ++l) {
    const int in = dims[l], out = dims[l + 1];
    const double bound = std::sqrt(6.0 / (in + out));
    for (int j = 0; j < in * out; ++j) params[off++] = rng.uniform(-bound, bound);
    for (int o = 0; o < out; ++o) params[off++] = 0.0;
  }
}

const std::vector<double>& adam_bias_table(int epochs) {
  static std::mutex mu;
  static std::vector<double> table;
  std::lock_guard<std::mutex> lock(mu);
  const std::size_t have = table.size() / 2;
  if (have < std::size_t(epochs)) {
    const double beta1 = 0.9, beta2 = 0.999;  // AdamState defaults (mlp.hpp:52-55)
    table.resize(std::size_t(epochs) * 2);
    for (std::size_t t = have; t < std::size_t(epochs); ++t) {
      const int step = int(t) + 1;
      table[2 * t] = 1.0 - std::pow(beta1, step);
      table[2 * t + 1] = 1.0 - std::pow(beta2, step);
    }
  }
  return table;
}

std::vector<lann_world> default_combos() {
  // 4 kernels x 2 variants (dense / sparse) x 5 hardware classes (3 CPU hosts with
  // n_thd, 2 GPU-class black boxes without) = 40 prediction worlds, plus 8 blur
  // selection worlds. Combo 0 is the acceptance world (acceptance_main.cpp:271-279).
  std::vector<lann_world> out;
  const double kind_alpha[4] = {3e-9, 2e-9, 1.5e-9, 1e-9};
  struct Hw { int cls, threads; double mult, g0, g1, beta; };
  const Hw hws[5] = {{LANN_HW_CPU, 4, 1.0, 0.25, 0.75, 0.0},
                     {LANN_HW_CPU, 8, 0.7, 0.15, 0.85, 0.0},
                     {LANN_HW_CPU, 16, 1.3, 0.10, 0.90, 0.0},
                     {LANN_HW_GPU, 1, 0.02, 1.0, 0.0, 5e-6},
                     {LANN_HW_GPU, 1, 0.05, 1.0, 0.0, 2e-5}};
  for (int kind = 0; kind < 4; ++kind)
    for (int variant = 0; variant < 2; ++variant)
      for (const Hw& h : hws) {
        lann_world w{};
        w.kind = kind;
        w.hw_class = h.cls;
        w.max_threads = h.threads;
        w.alpha = kind_alpha[kind] * (variant ? 2.5 : 1.0) * h.mult;
        w.g0 = h.g0;
        w.g1 = h.g1;
        w.delta = variant ? 0.9 : 0.0;
        w.beta = h.beta;
        w.noise = 0.02;
        out.push_back(w);
      }
  struct Bl { int lattice; double alpha, beta; double mu[4], kappa[4]; };
  const Bl blurs[8] = {
      {0, 1.0e-9, 0.0, {3, 8, 7, 3}, {0.05, 0.02, 0.03, 0.04}},
      {0, 0.7e-9, 0.0, {4, 7, 6, 2}, {0.04, 0.03, 0.02, 0.05}},
      {0, 1.3e-9, 0.0, {2, 9, 8, 4}, {0.06, 0.01, 0.04, 0.03}},
      {1, 1e-11, 1e-5, {2, 4, 4, 0}, {0.20, 0.10, 0.10, 0.0}},
      {1, 2e-11, 2e-5, {3, 3, 5, 0}, {0.15, 0.12, 0.08, 0.0}},
      {0, 2.0e-9, 0.0, {5, 6, 5, 3}, {0.03, 0.05, 0.05, 0.02}},   // FFT stand-ins
      {0, 1.5e-9, 0.0, {6, 10, 9, 5}, {0.02, 0.04, 0.06, 0.01}},
      {0, 0.9e-9, 0.0, {1, 5, 3, 1}, {0.08, 0.02, 0.02, 0.06}},
  };
  for (const Bl& b : blurs) {
    lann_world w{};
    w.kind = LANN_BLUR;
    w.hw_class = LANN_HW_CPU;
    w.max_threads = 1;
    w.blur_lattice = b.lattice;
    w.alpha = b.alpha;
    w.g0 = 1.0;
    w.beta = b.beta;
    w.noise = 0.02;
    for (int j = 0; j < 4; ++j) {
      w.mu[j] = b.mu[j];
      w.kappa[j] = b.kappa[j];
    }
    out.push_back(w);
  }
  return out;
}

}  // namespace lann
