// perfsage_api.cpp — the drop-in perfsage:: C++ API (include/perfsage_b200/perfsage.hpp)
// implemented over the engine's C ABI. Host work is exactly the reference's per-model
// preparation (assemble, NormStats, Glorot init — models.cpp:172-303); all training,
// prediction, metric and selection arithmetic runs in the engine's CUDA kernels.
#include "../../include/perfsage_b200/perfsage.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <limits>
#include <map>
#include <memory>

#include "../../include/lann_engine.h"
#include "domain.hpp"

namespace perfsage {

// ---- engine handle per host thread ---------------------------------------------------------
namespace engine {
namespace {
struct State {
  Precision precision = Precision::Fp64Exact;
  int device = 0;
  lann_engine* handle = nullptr;
  ~State() {
    if (handle) lann_engine_destroy(handle);
  }
};
thread_local State g_state;
}  // namespace

void set_precision(Precision p) { g_state.precision = p; }
Precision precision() { return g_state.precision; }
void set_device(int device) {
  if (g_state.handle && device != g_state.device) {
    lann_engine_destroy(g_state.handle);
    g_state.handle = nullptr;
  }
  g_state.device = device;
}

lann_engine* get() {
  if (!g_state.handle) {
    const int st = lann_engine_create(g_state.device, &g_state.handle);
    if (st == LANN_NO_DEVICE) throw Error("no CUDA device: the LANN engine has no CPU fallback");
    if (st) throw Error("engine creation failed");
  }
  return g_state.handle;
}
int lann_precision() { return g_state.precision == Precision::Fp32 ? LANN_FP32 : LANN_FP64_EXACT; }
}  // namespace engine

namespace {

[[noreturn]] void raise(int st, const std::string& msg, int epoch = -1) {
  switch (st) {
    case LANN_SCHEMA_ERROR: throw SchemaError(msg);
    case LANN_DOMAIN_ERROR: throw DomainError(msg);
    case LANN_TRAINING_ERROR: throw TrainingError(msg, epoch);
    case LANN_BUILD_ABORT: throw BuildAbortError(msg, 0);
    case LANN_PARAM_ERROR: throw ParamError(msg);
    default: throw Error(msg);
  }
}

void check(int st, lann_engine* e) {
  if (st) raise(st, lann_last_error(e));
}

}  // namespace

// ---- kernels ------------------------------------------------------------------------------------
namespace kernels {

std::string to_string(KernelKind kind) {
  static const char* names[] = {"mm", "mv", "mc", "mp", "blur"};
  return names[static_cast<int>(kind)];
}

bool ScheduleCandidate::is_pow2() const {
  auto ok = [](std::uint32_t v) { return v > 0 && std::has_single_bit(v); };
  return ok(s1) && ok(s2) && ok(s3) && ok(s4);
}

std::string ScheduleCandidate::to_string() const {
  return "{" + std::to_string(s1) + "," + std::to_string(s2) + "," + std::to_string(s3) + "," +
         std::to_string(s4) + "}";
}

ScheduleSpace ScheduleSpace::cpu_default() { return {}; }

ScheduleSpace ScheduleSpace::gpu_style() {
  ScheduleSpace s;
  s.s1_min = 2; s.s1_max = 16;
  s.s2_min = 1; s.s2_max = 64;
  s.s3_min = 1; s.s3_max = 64;
  s.s4_min = 1; s.s4_max = 1;
  s.chained = false;
  return s;
}

bool ScheduleSpace::contains(const ScheduleCandidate& c) const {
  if (!c.is_pow2()) return false;
  if (c.s1 < s1_min || c.s1 > s1_max || c.s2 < s2_min || c.s2 > s2_max) return false;
  if (c.s3 < s3_min || c.s3 > (chained ? std::min(s3_max, c.s2) : s3_max)) return false;
  if (c.s4 < s4_min || c.s4 > (chained ? std::min(s4_max, c.s3) : s4_max)) return false;
  return true;
}

std::vector<ScheduleCandidate> ScheduleSpace::enumerate_all() const {
  std::vector<ScheduleCandidate> out;
  auto p2 = [](std::uint32_t lo, std::uint32_t hi) {
    std::vector<std::uint32_t> v;
    for (std::uint32_t x = std::bit_ceil(std::max<std::uint32_t>(lo, 1)); x <= hi; x <<= 1) v.push_back(x);
    return v;
  };
  for (auto a : p2(s1_min, s1_max))
    for (auto b : p2(s2_min, s2_max))
      for (auto c : p2(s3_min, chained ? std::min(s3_max, b) : s3_max))
        for (auto d : p2(s4_min, chained ? std::min(s4_max, c) : s4_max)) out.push_back({a, b, c, d});
  return out;
}

std::uint64_t ScheduleSpace::size() const { return enumerate_all().size(); }

}  // namespace kernels

// ---- datagen ---------------------------------------------------------------------------------------
namespace datagen {

std::vector<double> Dataset::runtimes() const {
  std::vector<double> out;
  out.reserve(samples.size());
  for (const auto& s : samples) out.push_back(s.runtime_s);
  return out;
}

std::pair<Dataset, Dataset> split(const Dataset& ds, double frac, std::uint64_t seed) {
  std::vector<std::int64_t> order;
  int ntr = 0;
  const lann::Status st = lann::split_order(int(ds.samples.size()), frac, seed, order, ntr);
  if (st) raise(st.code, st.msg);
  auto part = [&](std::size_t b, std::size_t e) {
    Dataset d;
    d.kind = ds.kind;
    d.feature_names = ds.feature_names;
    d.seed = ds.seed;
    d.host = ds.host;
    for (std::size_t i = b; i < e; ++i) d.samples.push_back(ds.samples[order[i]]);
    return d;
  };
  return {part(0, ntr), part(ntr, ds.samples.size())};
}

}  // namespace datagen

// ---- models ------------------------------------------------------------------------------------------
namespace models {

int Mlp::param_count() const {
  int n = 0;
  for (const auto& l : layers) n += (l.in + 1) * l.out;
  return n;
}

std::string to_string(ModelFamily f) {
  static const char* names[] = {"nnc", "nn", "const", "lrc", "nlrc"};
  return names[static_cast<int>(f)];
}

bool family_augmented(ModelFamily f) { return f != ModelFamily::Nn; }

int param_count_for(int input_dim, const std::vector<int>& hidden) {
  int count = 0, in = input_dim;
  for (int h : hidden) {
    count += (in + 1) * h;
    in = h;
  }
  return count + in + 1;
}

void ModelConfig::validate(int input_dim) const {
  if (family == ModelFamily::NnC || family == ModelFamily::Nn) {
    if (hidden_widths.empty() || hidden_widths.size() > 2)
      throw ParamError("networks use 1 hidden layer (prediction) or 2 (selection)");
    for (int h : hidden_widths)
      if (h < 1) throw ParamError("hidden widths must be >= 1");
    if (!(learning_rate == 1e-2 || learning_rate == 1e-3 || learning_rate == 1e-4))
      throw ParamError("learning rate must be one of 1e-2, 1e-3, 1e-4");
    if (epochs < 1) throw ParamError("epochs must be >= 1");
    if (!unconstrained && param_count_for(input_dim, hidden_widths) > kLightweightParamBudget)
      throw ParamError("lightweight model exceeds the 75-parameter budget");
  }
  if (family == ModelFamily::NlrC && (forest_trees < 1 || forest_depth < 1))
    throw ParamError("forest needs trees >= 1 and depth >= 1");
}

ModelConfig default_config(kernels::KernelKind kind, ModelFamily family, bool unconstrained) {
  ModelConfig cfg;
  cfg.family = family;
  cfg.unconstrained = unconstrained;
  if (kind == kernels::KernelKind::Blur) {
    cfg.hidden_widths = {5, 5};
    cfg.learning_rate = 1e-2;
    cfg.epochs = 20000;
    cfg.log_target = true;
  } else {
    cfg.hidden_widths = {8};
    cfg.learning_rate = 1e-2;
    cfg.epochs = 8000;
  }
  if (unconstrained)
    for (int& h : cfg.hidden_widths) h *= 8;
  return cfg;
}

NormStats NormStats::fit(const std::vector<std::vector<double>>& X, std::span<const double> y,
                         bool log_target) {
  if (X.empty()) throw ParamError("cannot fit normalization on an empty set");
  const std::size_t p = X[0].size();
  NormStats st;
  st.log_target = log_target;
  st.f_min.assign(p, std::numeric_limits<double>::infinity());
  st.f_max.assign(p, -std::numeric_limits<double>::infinity());
  for (const auto& row : X)
    for (std::size_t j = 0; j < p; ++j) {
      st.f_min[j] = std::min(st.f_min[j], row[j]);
      st.f_max[j] = std::max(st.f_max[j], row[j]);
    }
  double lo = y[0], hi = y[0];
  for (double t : y) {
    lo = std::min(lo, t);
    hi = std::max(hi, t);
  }
  if (log_target) {
    if (!(lo > 0.0)) throw ParamError("targets must be positive runtimes");
    st.t_min = std::log(lo);
    st.t_max = std::log(hi);
  } else {
    st.t_min = lo;
    st.t_max = hi;
  }
  return st;
}

std::vector<double> NormStats::normalize(std::span<const double> f) const {
  if (f.size() != f_min.size()) throw SchemaError("feature vector length does not match the model schema");
  std::vector<double> out(f.size());
  for (std::size_t j = 0; j < f.size(); ++j) {
    const double range = f_max[j] - f_min[j];
    out[j] = range > 0.0 ? (f[j] - f_min[j]) / range : 0.0;
  }
  return out;
}

double NormStats::normalize_target(double t) const {
  const double range = t_max - t_min;
  const double v = log_target ? std::log(t) : t;
  return range > 0.0 ? (v - t_min) / range : 0.0;
}

double NormStats::denormalize_target(double ts) const {
  const double range = t_max - t_min;
  const double v = range > 0.0 ? t_min + ts * range : t_min;
  return log_target ? std::exp(v) : v;
}

std::vector<double> model_features(const datagen::Sample& s, ModelFamily family) {
  if (family == ModelFamily::Const) return {double(s.c)};
  std::vector<double> f = s.features;
  if (family_augmented(family)) f.push_back(double(s.c));
  return f;
}

std::vector<double> flatten_params(const Mlp& net) {
  std::vector<double> flat;
  for (const auto& l : net.layers) {
    flat.insert(flat.end(), l.w.begin(), l.w.end());
    flat.insert(flat.end(), l.b.begin(), l.b.end());
  }
  return flat;
}

int param_count(const TrainedModel& m) {
  const auto* net = std::get_if<Mlp>(&m.payload);
  if (!net) throw ParamError("param_count is defined for NN-family models only");
  return net->param_count();
}

namespace {

std::vector<std::string> schema_of(const datagen::Dataset& ds, ModelFamily family) {
  if (family == ModelFamily::Const) return {"c"};
  auto names = ds.feature_names;
  if (family_augmented(family)) names.emplace_back("c");
  return names;
}

Mlp unflatten(const std::vector<int>& dims, const double* flat) {
  Mlp net;
  std::size_t off = 0;
  for (std::size_t l = 0; l + 1 < dims.size(); ++l) {
    DenseLayer L;
    L.in = dims[l];
    L.out = dims[l + 1];
    L.w.assign(flat + off, flat + off + std::size_t(L.in) * L.out);
    off += L.w.size();
    L.b.assign(flat + off, flat + off + L.out);
    off += L.out;
    net.layers.push_back(std::move(L));
  }
  return net;
}

struct Prepared {
  TrainedModel model;
  std::vector<int> dims;
  std::vector<double> Xn, yn;  // [n][8], [n]
  std::vector<double> init;
};

// models.cpp:279-299 — everything train_nn does before train_full_batch
Prepared prepare(const datagen::Dataset& train, const ModelConfig& config) {
  if (config.family != ModelFamily::NnC && config.family != ModelFamily::Nn)
    throw ParamError("train_nn expects an NN family config");
  if (train.samples.size() < 2) throw ParamError("training needs at least 2 samples");
  std::vector<std::vector<double>> X;
  std::vector<double> y;
  for (const auto& s : train.samples) {
    X.push_back(model_features(s, config.family));
    y.push_back(s.runtime_s);
  }
  const int I = int(X[0].size());
  if (I > 7) throw ParamError("model inputs must lie in 1..7");
  config.validate(I);
  Prepared p;
  p.model.config = config;
  p.model.kind = train.kind;
  p.model.schema = schema_of(train, config.family);
  p.model.norm = NormStats::fit(X, y, config.log_target);
  p.Xn.assign(X.size() * LANN_ROW, 0.0);
  p.yn.resize(y.size());
  for (std::size_t s = 0; s < X.size(); ++s) {
    const auto xn = p.model.norm.normalize(X[s]);
    std::copy(xn.begin(), xn.end(), p.Xn.begin() + s * LANN_ROW);
    p.yn[s] = p.model.norm.normalize_target(y[s]);
  }
  p.dims = {I};
  p.dims.insert(p.dims.end(), config.hidden_widths.begin(), config.hidden_widths.end());
  p.dims.push_back(1);
  p.init.resize(std::size_t(param_count_for(I, config.hidden_widths)));
  lann::glorot_init(I, config.hidden_widths[0],
                    config.hidden_widths.size() > 1 ? config.hidden_widths[1] : 0, config.seed,
                    p.init.data());
  return p;
}

}  // namespace

namespace {
std::vector<TrainedModel> train_nn_population(const std::vector<const datagen::Dataset*>& train,
                                              const std::vector<ModelConfig>& configs) {
  if (train.size() != configs.size()) throw ParamError("one dataset per model config");
  if (train.empty()) return {};
  std::vector<Prepared> prep;
  for (std::size_t i = 0; i < train.size(); ++i) prep.push_back(prepare(*train[i], configs[i]));
  const int M = int(prep.size());
  std::vector<int> rows, inputs, tile, h1, h2, epochs;
  std::vector<std::int64_t> toff, poff, troff;
  std::vector<double> X, Y, lr, params;
  std::int64_t r = 0, tr = 0;
  for (int m = 0; m < M; ++m) {
    const auto& p = prep[m];
    rows.push_back(int(p.yn.size()));
    inputs.push_back(p.dims[0]);
    toff.push_back(r);
    r += std::int64_t(p.yn.size());
    X.insert(X.end(), p.Xn.begin(), p.Xn.end());
    Y.insert(Y.end(), p.yn.begin(), p.yn.end());
    tile.push_back(m);
    h1.push_back(p.dims[1]);
    h2.push_back(p.dims.size() > 3 ? p.dims[2] : 0);
    lr.push_back(p.model.config.learning_rate);
    epochs.push_back(p.model.config.epochs);
    poff.push_back(std::int64_t(params.size()));
    params.insert(params.end(), p.init.begin(), p.init.end());
    troff.push_back(tr);
    tr += p.model.config.epochs;
  }
  std::vector<double> final_loss(M), trace(static_cast<std::size_t>(tr));
  std::vector<std::int32_t> bad(M, -1);
  lann_train_batch b{};
  b.n_models = M;
  b.precision = engine::lann_precision();
  b.n_tiles = M;
  b.tile_rows = rows.data();
  b.tile_inputs = inputs.data();
  b.tile_offset = toff.data();
  b.total_rows = r;
  b.X = X.data();
  b.y = Y.data();
  b.model_tile = tile.data();
  b.model_h1 = h1.data();
  b.model_h2 = h2.data();
  b.model_lr = lr.data();
  b.model_epochs = epochs.data();
  b.model_param_offset = poff.data();
  b.total_params = std::int64_t(params.size());
  b.params = params.data();
  b.final_loss = final_loss.data();
  b.nonfinite_epoch = bad.data();
  b.loss_trace = trace.data();
  b.trace_offset = troff.data();
  b.trace_stride = 1;
  lann_engine* e = engine::get();
  const int st = lann_train(e, &b);
  if (st == LANN_TRAINING_ERROR) {
    int epoch = -1;
    for (int m = 0; m < M && epoch < 0; ++m) epoch = bad[m];
    raise(st, lann_last_error(e), epoch);
  }
  check(st, e);
  std::vector<TrainedModel> out;
  for (int m = 0; m < M; ++m) {
    TrainedModel model = std::move(prep[m].model);
    model.payload = unflatten(prep[m].dims, params.data() + poff[m]);
    model.loss_trace.assign(trace.begin() + troff[m], trace.begin() + troff[m] + epochs[m]);
    out.push_back(std::move(model));
  }
  return out;
}

// models.cpp:176-182 — the raw design matrix of a baseline family
struct Design {
  std::vector<std::vector<double>> X;
  std::vector<double> y;
};
Design assemble(const datagen::Dataset& train, ModelFamily family) {
  if (train.samples.size() < 2) throw ParamError("training needs at least 2 samples");
  Design d;
  for (const auto& smp : train.samples) {
    d.X.push_back(model_features(smp, family));
    d.y.push_back(smp.runtime_s);
  }
  if (d.X[0].size() > LANN_ROW) throw ParamError("model inputs must lie in 1..8");
  return d;
}

TrainedModel base_model(const datagen::Dataset& train, const ModelConfig& config) {
  TrainedModel m;
  m.config = config;
  m.kind = train.kind;
  m.schema = schema_of(train, config.family);
  return m;
}

struct PackedDesign {
  std::vector<std::int32_t> rows, feats;
  std::vector<std::int64_t> off;
  std::vector<double> X, y;
  lann_design view() const {
    return {std::int32_t(rows.size()), rows.data(), feats.data(), off.data(), X.data(), y.data()};
  }
  void add(const Design& d) {
    off.push_back(std::int64_t(y.size()));
    rows.push_back(std::int32_t(d.y.size()));
    feats.push_back(std::int32_t(d.X[0].size()));
    for (const auto& r : d.X) {
      double row[LANN_ROW] = {0};
      std::copy(r.begin(), r.end(), row);
      X.insert(X.end(), row, row + LANN_ROW);
    }
    y.insert(y.end(), d.y.begin(), d.y.end());
  }
};

constexpr double kRidge = 1e-8;  // models.cpp:276

// const + lrc (models.cpp:305-320): one least-squares launch for all of them
void fit_linear_batch(const std::vector<const datagen::Dataset*>& train, const std::vector<ModelConfig>& cfgs,
                      const std::vector<int>& idx, std::vector<TrainedModel>& out) {
  PackedDesign pd;
  for (int i : idx) pd.add(assemble(*train[i], cfgs[i].family));
  const int M = int(idx.size());
  std::vector<double> w(std::size_t(M) * LANN_ROW), b(M);
  std::vector<std::int32_t> st(M);
  lann_engine* e = engine::get();
  const lann_design dv = pd.view();
  const int rc = lann_fit_linear(e, &dv, kRidge, w.data(), b.data(), st.data());
  if (rc == LANN_DOMAIN_ERROR) throw FitError("singular design matrix despite ridge");
  check(rc, e);
  for (int k = 0; k < M; ++k) {
    TrainedModel m = base_model(*train[idx[k]], cfgs[idx[k]]);
    LinearModel lin;
    lin.weights.assign(w.begin() + std::ptrdiff_t(k) * LANN_ROW, w.begin() + std::ptrdiff_t(k) * LANN_ROW + pd.feats[k]);
    lin.intercept = b[k];
    m.payload = std::move(lin);
    out[idx[k]] = std::move(m);
  }
}

// nlrc (models.cpp:322-333): one forest launch, models x trees CTAs; trees per launch must agree,
// so configs are grouped by (trees, depth)
void fit_forest_batch(const std::vector<const datagen::Dataset*>& train, const std::vector<ModelConfig>& cfgs,
                      const std::vector<int>& idx, std::vector<TrainedModel>& out) {
  std::map<std::pair<int, int>, std::vector<int>> groups;
  for (int i : idx) groups[{cfgs[i].forest_trees, cfgs[i].forest_depth}].push_back(i);
  for (const auto& [key, members] : groups) {
    PackedDesign pd;
    std::vector<std::uint64_t> seeds;
    int max_rows = 0;
    for (int i : members) {
      const Design d = assemble(*train[i], ModelFamily::NlrC);
      cfgs[i].validate(int(d.X[0].size()));
      if (d.y.size() < 10) throw ParamError("forest needs at least 10 samples");
      pd.add(d);
      seeds.push_back(cfgs[i].seed);
      max_rows = std::max(max_rows, int(d.y.size()));
    }
    const int M = int(members.size()), trees = key.first, npt = 2 * max_rows;
    const std::size_t total = std::size_t(M) * trees * npt;
    std::vector<std::int32_t> nf(total), nl(total), nr(total), nc(std::size_t(M) * trees);
    std::vector<double> nt(total), nv(total);
    lann_engine* e = engine::get();
    const lann_design dv = pd.view();
    check(lann_fit_forest(e, &dv, trees, key.second, 2, seeds.data(), nf.data(), nt.data(), nl.data(), nr.data(),
                          nv.data(), nc.data()),
          e);
    for (int k = 0; k < M; ++k) {
      TrainedModel m = base_model(*train[members[k]], cfgs[members[k]]);
      Forest forest;
      for (int t = 0; t < trees; ++t) {
        Tree tree;
        const std::size_t base = (std::size_t(k) * trees + t) * npt;
        for (int v = 0; v < nc[std::size_t(k) * trees + t]; ++v)
          tree.nodes.push_back({nf[base + v], nt[base + v], nl[base + v], nr[base + v], nv[base + v]});
        forest.trees.push_back(std::move(tree));
      }
      m.payload = std::move(forest);
      out[members[k]] = std::move(m);
    }
  }
}
}  // namespace

std::vector<TrainedModel> train_population(const std::vector<const datagen::Dataset*>& train,
                                           const std::vector<ModelConfig>& configs) {
  if (train.size() != configs.size()) throw ParamError("one dataset per model config");
  std::vector<int> nn, lin, forest;
  for (std::size_t i = 0; i < configs.size(); ++i) {
    switch (configs[i].family) {
      case ModelFamily::NnC:
      case ModelFamily::Nn: nn.push_back(int(i)); break;
      case ModelFamily::Const:
      case ModelFamily::LrC: lin.push_back(int(i)); break;
      case ModelFamily::NlrC: forest.push_back(int(i)); break;
    }
  }
  std::vector<TrainedModel> out(configs.size());
  if (!nn.empty()) {
    std::vector<const datagen::Dataset*> t;
    std::vector<ModelConfig> c;
    for (int i : nn) {
      t.push_back(train[i]);
      c.push_back(configs[i]);
    }
    auto res = train_nn_population(t, c);
    for (std::size_t k = 0; k < nn.size(); ++k) out[nn[k]] = std::move(res[k]);
  }
  if (!lin.empty()) fit_linear_batch(train, configs, lin, out);
  if (!forest.empty()) fit_forest_batch(train, configs, forest, out);
  return out;
}

TrainedModel train_nn(const datagen::Dataset& train, const ModelConfig& config) {
  if (config.family != ModelFamily::NnC && config.family != ModelFamily::Nn)
    throw ParamError("train_nn expects an NN family config");
  return std::move(train_population({&train}, {config}).front());
}

TrainedModel train_const(const datagen::Dataset& train, const ModelConfig& config) {
  if (config.family != ModelFamily::Const) throw ParamError("train_const expects family const");
  return std::move(train_population({&train}, {config}).front());
}

TrainedModel train_lrc(const datagen::Dataset& train, const ModelConfig& config) {
  if (config.family != ModelFamily::LrC) throw ParamError("train_lrc expects family lrc");
  return std::move(train_population({&train}, {config}).front());
}

TrainedModel train_nlrc(const datagen::Dataset& train, const ModelConfig& config) {
  if (config.family != ModelFamily::NlrC) throw ParamError("train_nlrc expects family nlrc");
  return std::move(train_population({&train}, {config}).front());
}

TrainedModel train_model(const datagen::Dataset& train, const ModelConfig& config) {
  return std::move(train_population({&train}, {config}).front());
}

namespace {
// rows of one model's dataset in its model_features layout (schema-checked, models.cpp:347-350)
void append_rows(const TrainedModel& t, const datagen::Dataset& data, int m, std::vector<double>& rows,
                 std::vector<std::int32_t>& row_model) {
  for (const auto& smp : data.samples) {
    const auto f = model_features(smp, t.config.family);
    if (f.size() != t.schema.size())
      throw SchemaError("feature vector length " + std::to_string(f.size()) + " does not match model schema of " +
                        std::to_string(t.schema.size()));
    double row[LANN_ROW] = {0};
    std::copy(f.begin(), f.end(), row);
    rows.insert(rows.end(), row, row + LANN_ROW);
    row_model.push_back(m);
  }
}

void predict_mlp(const std::vector<const TrainedModel*>& models, const std::vector<const datagen::Dataset*>& data,
                 const std::vector<int>& idx, std::vector<std::vector<double>>& res) {
  const int M = int(idx.size());
  std::vector<std::int32_t> n_in(M), h1(M), h2(M), logt(M), row_model;
  std::vector<std::int64_t> poff(M);
  std::vector<double> params, norm(std::size_t(M) * 18, 0.0), rows;
  for (int m = 0; m < M; ++m) {
    const TrainedModel& t = *models[idx[m]];
    const Mlp& net = std::get<Mlp>(t.payload);
    n_in[m] = net.input_dim();
    h1[m] = net.layers.size() > 1 ? net.layers[0].out : 1;
    h2[m] = net.layers.size() > 2 ? net.layers[1].out : 0;
    logt[m] = t.norm.log_target;
    poff[m] = std::int64_t(params.size());
    const auto flat = flatten_params(net);
    params.insert(params.end(), flat.begin(), flat.end());
    for (std::size_t j = 0; j < t.norm.f_min.size() && j < 8; ++j) {
      norm[18 * m + j] = t.norm.f_min[j];
      norm[18 * m + 8 + j] = t.norm.f_max[j];
    }
    norm[18 * m + 16] = t.norm.t_min;
    norm[18 * m + 17] = t.norm.t_max;
    append_rows(t, *data[idx[m]], m, rows, row_model);
  }
  std::vector<double> out(row_model.size());
  if (!row_model.empty()) {
    lann_model_set ms{M, engine::lann_precision(), n_in.data(), h1.data(), h2.data(), logt.data(),
                      poff.data(), params.data(), std::int64_t(params.size()), norm.data()};
    lann_engine* e = engine::get();
    check(lann_predict(e, &ms, std::int64_t(row_model.size()), rows.data(), row_model.data(), out.data()), e);
  }
  std::size_t k = 0;
  for (int m = 0; m < M; ++m)
    for (std::size_t i = 0; i < data[idx[m]]->samples.size(); ++i) res[idx[m]].push_back(out[k++]);
}

void predict_linear(const std::vector<const TrainedModel*>& models, const std::vector<const datagen::Dataset*>& data,
                    const std::vector<int>& idx, std::vector<std::vector<double>>& res) {
  const int M = int(idx.size());
  std::vector<std::int32_t> nf(M), row_model;
  std::vector<double> w(std::size_t(M) * LANN_ROW, 0.0), b(M), rows;
  for (int m = 0; m < M; ++m) {
    const TrainedModel& t = *models[idx[m]];
    const auto& lin = std::get<LinearModel>(t.payload);
    if (lin.weights.size() != t.schema.size() || lin.weights.size() > LANN_ROW)
      throw SchemaError("linear model weights do not match its schema");
    nf[m] = std::int32_t(lin.weights.size());
    std::copy(lin.weights.begin(), lin.weights.end(), w.begin() + std::ptrdiff_t(m) * LANN_ROW);
    b[m] = lin.intercept;
    append_rows(t, *data[idx[m]], m, rows, row_model);
  }
  std::vector<double> out(row_model.size());
  if (!row_model.empty()) {
    lann_engine* e = engine::get();
    check(lann_predict_linear(e, M, nf.data(), w.data(), b.data(), std::int64_t(row_model.size()), rows.data(),
                              row_model.data(), out.data()),
          e);
  }
  std::size_t k = 0;
  for (int m = 0; m < M; ++m)
    for (std::size_t i = 0; i < data[idx[m]]->samples.size(); ++i) res[idx[m]].push_back(out[k++]);
}

void predict_forest(const std::vector<const TrainedModel*>& models, const std::vector<const datagen::Dataset*>& data,
                    const std::vector<int>& idx, std::vector<std::vector<double>>& res) {
  std::map<std::size_t, std::vector<int>> by_trees;  // one launch per tree count
  for (int i : idx) {
    const auto& f = std::get<Forest>(models[i]->payload);
    if (f.trees.empty()) throw ParamError("empty forest");
    by_trees[f.trees.size()].push_back(i);
  }
  for (const auto& [trees, members] : by_trees) {
    const int M = int(members.size());
    int npt = 1;
    for (int i : members)
      for (const auto& t : std::get<Forest>(models[i]->payload).trees) npt = std::max(npt, int(t.nodes.size()));
    const std::size_t total = std::size_t(M) * trees * npt;
    std::vector<std::int32_t> nf(total, -1), nl(total, -1), nr(total, -1), row_model;
    std::vector<double> nt(total, 0.0), nv(total, 0.0), rows;
    for (int m = 0; m < M; ++m) {
      const TrainedModel& tm = *models[members[m]];
      const auto& f = std::get<Forest>(tm.payload);
      for (std::size_t t = 0; t < trees; ++t) {
        const auto& nodes = f.trees[t].nodes;
        if (nodes.empty()) throw ParamError("forest tree has no nodes");
        for (std::size_t v = 0; v < nodes.size(); ++v) {
          const std::size_t o = (std::size_t(m) * trees + t) * npt + v;
          nf[o] = nodes[v].feature;
          nt[o] = nodes[v].threshold;
          nl[o] = nodes[v].left;
          nr[o] = nodes[v].right;
          nv[o] = nodes[v].value;
        }
      }
      append_rows(tm, *data[members[m]], m, rows, row_model);
    }
    std::vector<double> out(row_model.size());
    if (!row_model.empty()) {
      lann_engine* e = engine::get();
      check(lann_predict_forest(e, M, int(trees), npt, nf.data(), nt.data(), nl.data(), nr.data(), nv.data(),
                                std::int64_t(row_model.size()), rows.data(), row_model.data(), out.data()),
            e);
    }
    std::size_t k = 0;
    for (int m = 0; m < M; ++m)
      for (std::size_t i = 0; i < data[members[m]]->samples.size(); ++i) res[members[m]].push_back(out[k++]);
  }
}
}  // namespace

std::vector<std::vector<double>> predict_population(const std::vector<const TrainedModel*>& models,
                                                    const std::vector<const datagen::Dataset*>& data) {
  if (models.size() != data.size()) throw ParamError("one dataset per model");
  std::vector<int> mlp, lin, forest;
  for (std::size_t i = 0; i < models.size(); ++i) {
    if (std::holds_alternative<Mlp>(models[i]->payload)) mlp.push_back(int(i));
    else if (std::holds_alternative<LinearModel>(models[i]->payload)) lin.push_back(int(i));
    else forest.push_back(int(i));
  }
  std::vector<std::vector<double>> res(models.size());
  if (!mlp.empty()) predict_mlp(models, data, mlp, res);
  if (!lin.empty()) predict_linear(models, data, lin, res);
  if (!forest.empty()) predict_forest(models, data, forest, res);
  return res;
}

std::vector<double> predict_dataset(const TrainedModel& model, const datagen::Dataset& data) {
  return predict_population({&model}, {&data}).front();
}

double predict(const TrainedModel& model, std::span<const double> features) {
  if (features.size() != model.schema.size())
    throw SchemaError("feature vector length " + std::to_string(features.size()) +
                      " does not match model schema of " + std::to_string(model.schema.size()));
  // predict() receives the model-input vector itself (c already appended for the
  // augmented family): route it through a family whose model_features is the identity
  TrainedModel alias = model;
  alias.config.family = ModelFamily::Nn;
  datagen::Dataset one;
  one.kind = model.kind;
  datagen::Sample s;
  s.features.assign(features.begin(), features.end());
  one.samples.push_back(std::move(s));
  return predict_population({&alias}, {&one}).front().front();
}

}  // namespace models

// ---- eval ------------------------------------------------------------------------------------------
namespace eval {
namespace {
struct Metrics {
  double mape, thr, rho;
  std::int32_t kept;
};
Metrics run(std::span<const double> t, std::span<const double> p, double drop) {
  if (t.size() != p.size()) throw DomainError("truth and prediction lengths differ");
  if (t.empty()) throw DomainError("metric needs at least one sample");
  for (double x : t)
    if (!(x > 0.0)) throw DomainError("all true runtimes must be > 0");
  const std::int64_t off = 0;
  const std::int32_t len = std::int32_t(t.size());
  Metrics m{};
  lann_engine* e = engine::get();
  if (t.size() == 1) {
    // the set kernel needs two samples (spearman); a duplicated single sample gives the
    // same MAPE bit for bit: 100*(2x)/2 == 100*x/1 (scaling by 2 commutes with rounding)
    const double t2[2] = {t[0], t[0]}, p2[2] = {p[0], p[0]};
    const std::int32_t two = 2;
    const int st = lann_eval(e, 1, &off, &two, t2, p2, 0.0, &m.mape, &m.thr, &m.kept, &m.rho);
    if (st) raise(st, lann_last_error(e));
    m.kept = 1;
    return m;
  }
  const int st = lann_eval(e, 1, &off, &len, t.data(), p.data(), drop, &m.mape, &m.thr, &m.kept, &m.rho);
  if (st) raise(st, lann_last_error(e));
  return m;
}
}  // namespace

double mape(std::span<const double> truth, std::span<const double> pred) {
  return run(truth, pred, 0.3).mape;
}

ThresholdedMape mape_thresholded(std::span<const double> truth, std::span<const double> pred, double drop) {
  if (drop < 0.0 || drop > 1.0) throw DomainError("drop fraction must lie in [0,1]");
  const auto n_drop = static_cast<std::size_t>(std::floor(drop * double(truth.size()) + 1e-12));
  if (n_drop >= truth.size() && !truth.empty()) throw DomainError("threshold would drop every sample");
  const Metrics m = run(truth, pred, drop);
  return {m.thr, std::size_t(m.kept)};
}

double spearman(std::span<const double> truth, std::span<const double> pred) {
  if (truth.size() != pred.size()) throw DomainError("truth and prediction lengths differ");
  if (truth.size() < 2) throw DomainError("spearman needs at least two samples");
  return run(truth, pred, 0.0).rho;
}

EvalReport make_report(std::span<const double> truth, std::span<const double> pred, double drop) {
  const auto thr = mape_thresholded(truth, pred, drop);
  if (truth.size() < 2) throw DomainError("spearman needs at least two samples");  // eval.cpp:80
  const Metrics m = run(truth, pred, drop);
  EvalReport r;
  r.mape_full = m.mape;
  r.mape_thresholded = thr.value;
  r.n_kept = thr.n_kept;
  r.rho = m.rho;
  r.n_total = truth.size();
  return r;
}

}  // namespace eval

// ---- selector ----------------------------------------------------------------------------------------
namespace selector {

std::vector<ScheduleCandidate> enumerate_candidates(const ScheduleSpace& space, std::size_t limit,
                                                    std::uint64_t seed) {
  if (limit < 1) throw ParamError("candidate limit must be >= 1");
  auto lattice = space.enumerate_all();
  if (lattice.empty()) throw DomainError("empty schedule space");
  if (limit >= lattice.size()) return lattice;
  lann::SeqRng rng(lann::derive_seed(seed, 0xCA4D));  // selector.cpp:20-21
  for (std::size_t i = 0; i < limit; ++i)
    std::swap(lattice[i], lattice[i + std::size_t(rng.bounded(lattice.size() - i))]);
  lattice.resize(limit);
  return lattice;
}

ScheduleCandidate select(const ScheduleScorer& scorer, const std::vector<ScheduleCandidate>& cands) {
  if (cands.empty()) throw ParamError("select needs at least one candidate");
  const ScheduleCandidate* best = &cands.front();
  double best_score = scorer(*best);
  for (std::size_t i = 1; i < cands.size(); ++i) {
    const double s = scorer(cands[i]);
    if (s < best_score || (s == best_score && cands[i] < *best)) {
      best = &cands[i];
      best_score = s;
    }
  }
  return *best;
}

ScheduleCandidate select(const models::TrainedModel& model, std::uint32_t image_n,
                         const std::vector<ScheduleCandidate>& cands) {
  if (model.kind != kernels::KernelKind::Blur)
    throw SchemaError("variant selection needs a model trained on the blur schema");
  if (cands.empty()) throw ParamError("select needs at least one candidate");
  const auto& net = std::get<models::Mlp>(model.payload);
  std::int32_t n_in = net.input_dim(), h1 = net.layers[0].out,
               h2 = net.layers.size() > 2 ? net.layers[1].out : 0, logt = model.norm.log_target;
  std::int64_t poff = 0;
  const auto params = models::flatten_params(net);
  double norm[18] = {0};
  for (std::size_t j = 0; j < model.norm.f_min.size() && j < 8; ++j) {
    norm[j] = model.norm.f_min[j];
    norm[8 + j] = model.norm.f_max[j];
  }
  norm[16] = model.norm.t_min;
  norm[17] = model.norm.t_max;
  std::vector<std::uint32_t> flat;
  for (const auto& c : cands) flat.insert(flat.end(), {c.s1, c.s2, c.s3, c.s4});
  lann_model_set ms{1, engine::lann_precision(), &n_in, &h1, &h2, &logt, &poff, params.data(),
                    std::int64_t(params.size()), norm};
  std::int64_t chosen = -1;
  double score = 0.0;
  lann_engine* e = engine::get();
  check(lann_select_schedule(e, &ms, image_n, std::int64_t(cands.size()), flat.data(), &chosen, &score), e);
  return cands[std::size_t(chosen)];
}

}  // namespace selector
}  // namespace perfsage
