// api_host.cpp — the host-side value types and helpers of the reference's perfsage:: API that a
// caller of the LANN path uses around the engine (kernels.hpp InstanceParams / complexity,
// datagen.hpp ParamSpace / sample_params / build_dataset with a probe, features.hpp featurize,
// mlp.hpp Mlp::init / unflatten_params), plus train_full_batch on the GPU. These are
// restatements of the reference's host logic (paths relative to proj/core/src); the arithmetic
// of training, prediction, metrics and selection stays in the engine's kernels.
#include <algorithm>
#include <cmath>

#include "../../include/lann_engine.h"
#include "../../include/perfsage_b200/perfsage.hpp"

namespace perfsage {

namespace engine {
lann_engine* get();
int lann_precision();
}  // namespace engine

// ---- kernels.cpp:89-206 --------------------------------------------------------------------------
namespace kernels {

InstanceParams InstanceParams::mm(std::uint32_t m, std::uint32_t n, std::uint32_t k, double d1, double d2,
                                  int n_thd) {
  InstanceParams p;
  p.kind = KernelKind::MM;
  p.m = m, p.n = n, p.k = k, p.d1 = d1, p.d2 = d2, p.n_thd = n_thd;
  return p;
}
InstanceParams InstanceParams::mv(std::uint32_t m, std::uint32_t n, double d, int n_thd) {
  InstanceParams p;
  p.kind = KernelKind::MV;
  p.m = m, p.n = n, p.d = d, p.n_thd = n_thd;
  return p;
}
InstanceParams InstanceParams::mc(std::uint32_t m, std::uint32_t n, std::uint32_t r, double d, int n_thd) {
  InstanceParams p;
  p.kind = KernelKind::MC;
  p.m = m, p.n = n, p.r = r, p.d = d, p.n_thd = n_thd;
  return p;
}
InstanceParams InstanceParams::mp(std::uint32_t m, std::uint32_t n, std::uint32_t r, std::uint32_t s, double d,
                                  int n_thd) {
  InstanceParams p;
  p.kind = KernelKind::MP;
  p.m = m, p.n = n, p.r = r, p.s = s, p.d = d, p.n_thd = n_thd;
  return p;
}
InstanceParams InstanceParams::blur(std::uint32_t n, const ScheduleCandidate& sched) {
  InstanceParams p;
  p.kind = KernelKind::Blur;
  p.n = n;
  p.schedule = sched;
  return p;
}

void InstanceParams::validate() const {
  auto need = [](bool ok, const char* what) {
    if (!ok) throw ParamError(what);
  };
  auto dens = [](double v) { return v > 0.0 && v <= 1.0; };
  need(n_thd >= 1, "n_thd must be >= 1");
  switch (kind) {
    case KernelKind::MM:
      need(m >= 1 && n >= 1 && k >= 1, "MM dims must be >= 1");
      need(dens(d1) && dens(d2), "MM densities must lie in (0,1]");
      need(r == 0 && s == 0 && !schedule, "MM carries no r/s/schedule");
      break;
    case KernelKind::MV:
      need(m >= 1 && n >= 1, "MV dims must be >= 1");
      need(dens(d), "MV density must lie in (0,1]");
      need(k == 0 && r == 0 && s == 0 && !schedule, "MV carries no k/r/s/schedule");
      break;
    case KernelKind::MC:
      need(r >= 1, "MC filter dim must be >= 1");
      need(m >= r && n >= r, "MC requires m >= r and n >= r");
      need(dens(d), "MC density must lie in (0,1]");
      need(k == 0 && s == 0 && !schedule, "MC carries no k/s/schedule");
      break;
    case KernelKind::MP:
      need(s >= 1, "MP pool dim must be >= 1");
      need(r >= 1, "MP aux dim must be >= 1");
      need(m >= s && n >= s, "MP requires m >= s and n >= s");
      need(dens(d), "MP density must lie in (0,1]");
      need(k == 0 && !schedule, "MP carries no k/schedule");
      break;
    case KernelKind::Blur:
      need(n >= 4, "blur image side must be >= 4");
      need(schedule.has_value(), "blur requires a schedule");
      need(schedule->is_pow2(), "blur schedule factors must be positive powers of two");
      need(m == 0 && k == 0 && r == 0 && s == 0, "blur carries only n and schedule");
      break;
  }
}

std::uint64_t complexity(const InstanceParams& p) {
  p.validate();
  const std::uint64_t m = p.m, n = p.n, k = p.k, r = p.r, s = p.s;
  switch (p.kind) {
    case KernelKind::MM: return m * n * k;
    case KernelKind::MV: return m * n;
    case KernelKind::MC: return (m - r + 1) * (n - r + 1) * r * r;
    case KernelKind::MP: return ((n + s - 1) / s) * ((m + s - 1) / s) * s * s;
    case KernelKind::Blur: return n * n;
  }
  return 0;
}

}  // namespace kernels

// ---- features.cpp:23-57, models.cpp:143-163 --------------------------------------------------------
namespace models {

std::vector<double> featurize(const kernels::InstanceParams& p, bool augmented, bool with_n_thd) {
  using K = kernels::KernelKind;
  p.validate();
  std::vector<double> f;
  switch (p.kind) {
    case K::MM: f = {double(p.m), double(p.n), double(p.k), p.d1, p.d2}; break;
    case K::MV: f = {double(p.m), double(p.n), p.d}; break;
    case K::MC: f = {double(p.m), double(p.n), double(p.r), p.d}; break;
    case K::MP: f = {double(p.m), double(p.n), double(p.r), double(p.s), p.d}; break;
    case K::Blur: {
      const auto& sc = *p.schedule;
      f = {double(p.n), double(sc.s1), double(sc.s2), double(sc.s3), double(sc.s4)};
      with_n_thd = false;
      break;
    }
  }
  if (with_n_thd) f.push_back(double(p.n_thd));
  if (augmented) f.push_back(double(kernels::complexity(p)));
  return f;
}

std::vector<double> featurize(const kernels::InstanceParams& p, bool augmented) { return featurize(p, augmented, true); }

std::vector<double> model_features(const kernels::InstanceParams& p, ModelFamily family, bool with_n_thd) {
  if (family == ModelFamily::Const) return {double(kernels::complexity(p))};
  return featurize(p, family_augmented(family), with_n_thd);
}

std::vector<std::string> model_schema(const std::vector<std::string>& base_names, ModelFamily family) {
  if (family == ModelFamily::Const) return {"c"};
  auto names = base_names;
  if (family_augmented(family)) names.emplace_back("c");
  return names;
}

Mlp Mlp::init(const std::vector<int>& dims, Rng& rng) {
  if (dims.size() < 2) throw ParamError("network needs at least input and output dims");
  for (int d : dims)
    if (d < 1) throw ParamError("network layer widths must be >= 1");
  Mlp net;
  for (std::size_t l = 0; l + 1 < dims.size(); ++l) {
    DenseLayer L;
    L.in = dims[l];
    L.out = dims[l + 1];
    const double bound = std::sqrt(6.0 / (L.in + L.out));
    L.w.resize(std::size_t(L.in) * std::size_t(L.out));
    for (auto& w : L.w) w = rng.uniform(-bound, bound);
    L.b.assign(std::size_t(L.out), 0.0);
    net.layers.push_back(std::move(L));
  }
  return net;
}

void unflatten_params(Mlp& net, std::span<const double> flat) {
  std::size_t off = 0;
  for (auto& L : net.layers) {
    if (off + L.w.size() + L.b.size() > flat.size()) throw ParamError("flat parameter size mismatch");
    for (auto& w : L.w) w = flat[off++];
    for (auto& b : L.b) b = flat[off++];
  }
  if (off != flat.size()) throw ParamError("flat parameter size mismatch");
}

namespace {
// one net as a lann_mlp_batch (the C ABI's generic-net entry points)
struct OneNet {
  std::vector<std::int32_t> dims;
  std::vector<double> params, X;
  std::int32_t n_dims = 0, n_rows = 0;
  lann_mlp_batch b{};
  OneNet(const Mlp& net, const std::vector<std::vector<double>>* rows, std::span<const double> single) {
    if (net.layers.empty()) throw ParamError("empty network");
    dims.push_back(net.layers.front().in);
    for (const auto& L : net.layers) dims.push_back(L.out);
    params = flatten_params(net);
    const std::size_t I = std::size_t(net.input_dim());
    if (rows) {
      for (const auto& r : *rows) {
        if (r.size() != I) throw SchemaError("feature vector length does not match the network input");
        X.insert(X.end(), r.begin(), r.end());
      }
      n_rows = std::int32_t(rows->size());
    } else {
      X.assign(single.begin(), single.end());
      n_rows = 1;
    }
    n_dims = std::int32_t(dims.size());
    b.n_nets = 1;
    b.n_dims = &n_dims;
    b.dims = dims.data();
    b.params = params.data();
    b.n_rows = &n_rows;
    b.X = X.data();
  }
};
void raise_mlp(int st) {
  lann_engine* e = engine::get();
  if (st == LANN_PARAM_ERROR) throw ParamError(lann_last_error(e));
  if (st == LANN_SCHEMA_ERROR) throw SchemaError(lann_last_error(e));
  if (st) throw Error(lann_last_error(e));
}
}  // namespace

double Mlp::forward(std::span<const double> x) const {
  if (static_cast<int>(x.size()) != input_dim())  // mlp.cpp:55-56
    throw SchemaError("feature vector length does not match the network input");
  OneNet one(*this, nullptr, x);
  double out = 0.0;
  raise_mlp(lann_mlp_forward(engine::get(), &one.b, &out));
  return out;
}

double mse_loss(const Mlp& net, const std::vector<std::vector<double>>& X, std::span<const double> y) {
  if (X.size() != y.size() || X.empty()) throw ParamError("bad training batch");  // mlp.cpp:66
  OneNet one(net, &X, {});
  one.b.y = y.data();
  double loss = 0.0;
  raise_mlp(lann_mse_loss(engine::get(), &one.b, &loss));
  return loss;
}

LossGrad mse_gradient(const Mlp& net, const std::vector<std::vector<double>>& X, std::span<const double> y) {
  if (X.size() != y.size() || X.empty()) throw ParamError("bad training batch");  // mlp.cpp:77
  OneNet one(net, &X, {});
  one.b.y = y.data();
  LossGrad r;
  r.grad.assign(one.params.size(), 0.0);
  raise_mlp(lann_mse_gradient(engine::get(), &one.b, &r.loss, r.grad.data()));
  return r;
}

void AdamState::update(std::span<double> params, std::span<const double> grad, double lr) {
  ++step;  // mlp.cpp:143
  if (grad.size() < params.size() || m.size() < params.size() || v.size() < params.size())
    throw ParamError("Adam state / gradient shorter than the parameter vector");
  raise_mlp(lann_adam_update(engine::get(), std::int64_t(params.size()), params.data(), grad.data(), m.data(),
                             v.data(), step, lr, beta1, beta2, epsilon));
}

std::vector<double> train_full_batch(Mlp& net, const std::vector<std::vector<double>>& X, std::span<const double> y,
                                     double lr, int epochs) {
  if (X.size() != y.size() || X.empty()) throw ParamError("feature/target size mismatch");
  if (net.layers.size() < 2 || net.layers.size() > 3 || net.layers.back().out != 1)
    throw ParamError("the engine trains nets with 1 or 2 hidden layers and one output");
  const int I = net.input_dim(), n = int(X.size());
  if (I < 1 || I > 7) throw ParamError("model inputs must lie in 1..7");
  std::vector<double> Xf(std::size_t(n) * LANN_ROW, 0.0);
  for (int s = 0; s < n; ++s) {
    if (int(X[std::size_t(s)].size()) != I)
      throw SchemaError("feature vector length " + std::to_string(X[std::size_t(s)].size()) +
                        " does not match network input " + std::to_string(I));
    std::copy(X[std::size_t(s)].begin(), X[std::size_t(s)].end(), Xf.begin() + std::ptrdiff_t(s) * LANN_ROW);
  }
  std::vector<double> params = flatten_params(net), yv(y.begin(), y.end()), trace(std::size_t(std::max(epochs, 0)));
  const int rows = n, tile = 0, h1 = net.layers[0].out, h2 = net.layers.size() == 3 ? net.layers[1].out : 0;
  const std::int64_t toff = 0, poff = 0, troff = 0;
  double final_loss = 0.0;
  std::int32_t bad = -1;
  lann_train_batch b{};
  b.n_models = 1;
  b.precision = engine::lann_precision();
  b.n_tiles = 1;
  b.tile_rows = &rows;
  b.tile_inputs = &I;
  b.tile_offset = &toff;
  b.total_rows = n;
  b.X = Xf.data();
  b.y = yv.data();
  b.model_tile = &tile;
  b.model_h1 = &h1;
  b.model_h2 = &h2;
  b.model_lr = &lr;
  b.model_epochs = &epochs;
  b.model_param_offset = &poff;
  b.total_params = std::int64_t(params.size());
  b.params = params.data();
  b.final_loss = &final_loss;
  b.nonfinite_epoch = &bad;
  b.loss_trace = trace.data();
  b.trace_offset = &troff;
  b.trace_stride = 1;
  lann_engine* e = engine::get();
  const int st = lann_train(e, &b);
  if (st == LANN_TRAINING_ERROR) throw TrainingError(lann_last_error(e), bad);
  if (st == LANN_PARAM_ERROR) throw ParamError(lann_last_error(e));
  if (st) throw Error(lann_last_error(e));
  unflatten_params(net, params);
  return trace;
}

}  // namespace models

// ---- datagen.cpp:18-124, 177-223 --------------------------------------------------------------------
namespace datagen {

ParamSpace ParamSpace::defaults(kernels::KernelKind kind, int max_threads) {
  ParamSpace s;
  s.kind = kind;
  s.max_threads = std::max(1, max_threads);
  if (kind == kernels::KernelKind::MV) s.density_ladder_includes_one = false;
  return s;
}

void ParamSpace::validate() const {
  using K = kernels::KernelKind;
  if (dim_min < 1 || dim_max < dim_min) throw ParamError("param space needs 1 <= dim_min <= dim_max");
  if (max_threads < 1) throw ParamError("param space needs max_threads >= 1");
  if (kind == K::MC && mc_filter_dims.empty()) throw ParamError("MC space needs filter dims");
  if (kind == K::MP && (mp_aux_dims.empty() || mp_pool_dims.empty())) throw ParamError("MP space needs aux and pool dims");
  if (kind == K::Blur && blur_sides.empty()) throw ParamError("blur space needs image sides");
}

std::vector<double> density_ladder(std::uint64_t cells, bool include_one) {
  const int depth = cells ? int(std::bit_width(cells)) - 1 : -1;  // floor(log2(cells))
  std::vector<double> ladder;
  for (int j = include_one ? 0 : 1; j <= depth; ++j) ladder.push_back(std::ldexp(1.0, -j));
  if (ladder.empty()) ladder.push_back(1.0);
  return ladder;
}

kernels::InstanceParams sample_params(const ParamSpace& space, Rng& rng) {
  using K = kernels::KernelKind;
  using P = kernels::InstanceParams;
  space.validate();
  auto dim = [&] { return std::uint32_t(rng.uniform_int(space.dim_min, space.dim_max)); };
  auto dim_at_least = [&](std::uint32_t lo) {
    return std::uint32_t(rng.uniform_int(std::max(space.dim_min, lo), std::max(space.dim_max, lo)));
  };
  auto threads = [&] { return int(rng.uniform_int(1, space.max_threads)); };
  auto density = [&](std::uint64_t cells) {
    const auto ladder = density_ladder(cells, space.density_ladder_includes_one);
    return ladder[std::size_t(rng.bounded(ladder.size()))];
  };
  auto pick = [&](const std::vector<std::uint32_t>& v) { return v[std::size_t(rng.bounded(v.size()))]; };
  switch (space.kind) {
    case K::MM: {
      const std::uint32_t m = dim(), n = dim(), k = dim();
      const double d1 = density(std::uint64_t(m) * n);
      const double d2 = density(std::uint64_t(n) * k);
      return P::mm(m, n, k, d1, d2, threads());
    }
    case K::MV: {
      const std::uint32_t m = dim(), n = dim();
      const double d = density(std::uint64_t(m) * n);
      return P::mv(m, n, d, threads());
    }
    case K::MC: {
      const std::uint32_t r = pick(space.mc_filter_dims);
      const std::uint32_t m = dim_at_least(r), n = dim_at_least(r);
      const double d = density(std::uint64_t(m) * n);
      return P::mc(m, n, r, d, threads());
    }
    case K::MP: {
      const std::uint32_t r = pick(space.mp_aux_dims), s = pick(space.mp_pool_dims);
      const std::uint32_t m = dim_at_least(r), n = dim_at_least(r);
      const double d = density(std::uint64_t(m) * n);
      return P::mp(m, n, r, s, d, threads());
    }
    case K::Blur: {
      const std::uint32_t n = pick(space.blur_sides);
      const auto lattice = space.schedules.enumerate_all();
      if (lattice.empty()) throw ParamError("empty schedule space");
      return P::blur(n, lattice[std::size_t(rng.bounded(lattice.size()))]);
    }
  }
  throw ParamError("unreachable kernel kind");
}

kernels::InstanceParams sample_params(const ParamSpace& space, std::uint64_t seed) {
  Rng rng(seed);
  return sample_params(space, rng);
}

double median_of(std::vector<double> values) {
  if (values.empty()) throw DomainError("median of empty sample");
  std::sort(values.begin(), values.end());
  const std::size_t n = values.size();
  return n % 2 ? values[n / 2] : 0.5 * (values[n / 2 - 1] + values[n / 2]);
}

Dataset build_dataset(const kernels::VariantDescriptor& variant, const ParamSpace& space, std::size_t count,
                      std::uint64_t seed, const BuildOptions& options) {
  if (count < 2) throw ParamError("build_dataset needs count >= 2");
  if (variant.kind != space.kind) throw ParamError("variant kernel does not match the parameter space");
  space.validate();
  if (!options.probe && !variant.is_external())
    throw ParamError("the B200 engine does not time the reference's CPU kernels: pass BuildOptions::probe, "
                     "use an external variant, or datagen::build_measured for B200 GPU variants");
  Dataset ds;
  ds.kind = space.kind;
  ds.feature_names = models::feature_names(space.kind, variant.takes_n_thd());
  ds.seed = seed;
  ds.host = variant.hardware_label;
  Rng rng(derive_seed(seed, 0));
  for (std::size_t i = 0; i < count; ++i) {
    try {
      auto params = sample_params(space, rng);
      if (variant.threading == kernels::Threading::FixedSingle) params.n_thd = 1;
      if (space.kind == kernels::KernelKind::Blur) params.n_thd = space.max_threads;
      Sample smp;
      smp.features = models::featurize(params, false, variant.takes_n_thd());
      smp.c = kernels::complexity(params);
      smp.variant_id = variant.variant_id;
      smp.runtime_s = options.probe ? options.probe(params) : run_external_variant(variant.launch_command, smp.features);
      if (!(smp.runtime_s > 0.0)) throw DomainError("measured runtime must be > 0");
      ds.samples.push_back(std::move(smp));
    } catch (const Error& e) {
      throw BuildAbortError("dataset build aborted after " + std::to_string(ds.samples.size()) + "/" +
                                std::to_string(count) + " samples: " + e.what(),
                            ds.samples.size());
    }
  }
  return ds;
}

}  // namespace datagen

namespace eval {
double speedup(double baseline_s, double chosen_s) {
  if (!(baseline_s > 0.0) || !(chosen_s > 0.0)) throw DomainError("speedup needs positive runtimes");
  return baseline_s / chosen_s;
}
}  // namespace eval

}  // namespace perfsage
