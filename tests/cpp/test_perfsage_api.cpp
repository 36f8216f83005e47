// C++ drop-in API test: the reference's own hot-path unit tests (proj/tests/test_models.cpp,
// test_eval.cpp, test_selector.cpp), restated against include/perfsage_b200/perfsage.hpp with
// unchanged call syntax, plus bit-exact pins from the reference's golden run. Built and run by
// tests/test_gpu_cpp_api.py on the GPU box. Exit code 0 = all checks passed.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <map>
#include <random>

#include "lann_engine.h"
#include "perfsage_b200/perfsage.hpp"

using namespace perfsage;
using namespace perfsage::models;
using datagen::Dataset;
using datagen::Sample;
using kernels::KernelKind;

static int g_fail = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
      ++g_fail;                                                            \
    }                                                                      \
  } while (0)
#define CHECK_THROWS(expr, type)                                           \
  do {                                                                     \
    bool thrown = false;                                                   \
    try {                                                                  \
      expr;                                                                \
    } catch (const type&) {                                                \
      thrown = true;                                                       \
    }                                                                      \
    if (!thrown) {                                                         \
      std::printf("FAIL %s:%d: %s did not throw\n", __FILE__, __LINE__, #expr); \
      ++g_fail;                                                            \
    }                                                                      \
  } while (0)

// test_models.cpp:28-48 synth_mm, with an mt19937_64-driven draw of (m, n, k, n_thd)
static Dataset synth_mm(std::size_t count, std::uint64_t seed,
                        const std::function<double(std::uint64_t c, int n_thd, std::mt19937_64&)>& fn) {
  Dataset ds;
  ds.kind = KernelKind::MM;
  ds.feature_names = {"m", "n", "k", "d1", "d2", "n_thd"};
  std::mt19937_64 rng(seed);
  for (std::size_t i = 0; i < count; ++i) {
    const std::uint32_t m = 1 + rng() % 1024, n = 1 + rng() % 1024, k = 1 + rng() % 1024;
    const int thd = int(1 + rng() % 4);
    Sample s;
    s.features = {double(m), double(n), double(k), 1.0, 1.0, double(thd)};
    s.c = std::uint64_t(m) * n * k;
    s.variant_id = "synthetic";
    s.runtime_s = fn(s.c, thd, rng);
    ds.samples.push_back(s);
  }
  return ds;
}

// test_models.cpp:176-196 near_relu_kink (= acceptance_main.cpp:172-190 has_relu_kink)
static bool near_relu_kink(const Mlp& net, const std::vector<std::vector<double>>& X, double margin) {
  for (const auto& x : X) {
    std::vector<double> act(x);
    for (std::size_t l = 0; l + 1 < net.layers.size(); ++l) {
      const auto& layer = net.layers[l];
      std::vector<double> next(layer.out);
      for (int o = 0; o < layer.out; ++o) {
        double z = layer.b[o];
        for (int i = 0; i < layer.in; ++i) z += layer.w[std::size_t(o) * layer.in + i] * act[i];
        if (std::abs(z) < margin) return true;
        next[o] = z > 0 ? z : 0.0;
      }
      act = std::move(next);
    }
  }
  return false;
}

// GradientCheck.AnalyticMatchesFiniteDifferences (test_models.cpp:200-235) with the seed, trial
// count, net sizes and sample count of the named source: mse_gradient and mse_loss on the GPU
static double gradient_check(std::uint64_t seed, int trials, int in_span, int h_span, int h2_span, int rows) {
  Rng rng(seed);
  double worst = 0.0;
  for (int trial = 0; trial < trials; ++trial) {
    const int inputs = 2 + int(rng.bounded(std::uint64_t(in_span)));
    std::vector<int> dims{inputs, 2 + int(rng.bounded(std::uint64_t(h_span)))};
    if (trial % 2 == 1) dims.push_back(2 + int(rng.bounded(std::uint64_t(h2_span))));
    dims.push_back(1);
    Mlp net = Mlp::init(dims, rng);
    std::vector<std::vector<double>> X(static_cast<std::size_t>(rows), std::vector<double>(static_cast<std::size_t>(inputs)));
    std::vector<double> y(X.size());
    do {
      for (auto& row : X)
        for (auto& v : row) v = rng.uniform(-1.0, 1.0);
    } while (near_relu_kink(net, X, 1e-3));
    for (auto& v : y) v = rng.uniform(0.0, 1.0);
    const auto lg = mse_gradient(net, X, y);
    auto params = flatten_params(net);
    const double h = 1e-5;
    for (std::size_t i = 0; i < params.size(); ++i) {
      const double saved = params[i];
      params[i] = saved + h;
      unflatten_params(net, params);
      const double up = mse_loss(net, X, y);
      params[i] = saved - h;
      unflatten_params(net, params);
      const double down = mse_loss(net, X, y);
      params[i] = saved;
      unflatten_params(net, params);
      const double numeric = (up - down) / (2 * h);
      const double denom = std::max({std::abs(numeric), std::abs(lg.grad[i]), 1e-6});
      const double rel = std::abs(numeric - lg.grad[i]) / denom;
      worst = std::max(worst, rel);
      CHECK(rel < 1e-4);
    }
  }
  return worst;
}

int main() {
  // GradientCheck (test_models.cpp:200-235: Rng(77), 6 nets, 5 rows) and acceptance criterion 3
  // (acceptance_main.cpp:194-239: Rng(0x6AD), 20 nets, 6 rows, worst relative error <= 1e-4)
  {
    const double w1 = gradient_check(77, 6, 4, 4, 3, 5);
    const double w3 = gradient_check(0x6AD, 20, 5, 5, 4, 6);
    std::printf("gradient check: test_models worst rel %.3g, criterion 3 (20 nets) worst rel %.3g\n", w1, w3);
    // Mlp::forward == the last sample's forward inside mse_loss; AdamState::update moves the
    // parameters against the gradient and counts steps
    Rng rng(5);
    Mlp net = Mlp::init({3, 4, 1}, rng);
    const std::vector<std::vector<double>> X{{0.1, 0.2, 0.3}};
    const std::vector<double> y{0.5};
    const double f = net.forward(X[0]);
    CHECK(mse_loss(net, X, y) == (f - 0.5) * (f - 0.5));
    CHECK_THROWS(net.forward(std::vector<double>{1.0}), SchemaError);
    CHECK_THROWS(mse_loss(net, {}, {}), ParamError);
    auto p = flatten_params(net);
    AdamState adam(p.size());
    const auto g = mse_gradient(net, X, y);
    const auto before = p;
    adam.update(p, g.grad, 1e-2);
    CHECK(adam.step == 1);
    for (std::size_t i = 0; i < p.size(); ++i)
      if (g.grad[i] != 0.0) CHECK((p[i] - before[i]) * g.grad[i] < 0.0);
  }
  // ParamCount (test_models.cpp:76-90)
  CHECK(param_count_for(7, {8}) == 73);
  CHECK(param_count_for(6, {5, 5}) == 71);
  {
    ModelConfig cfg;
    cfg.hidden_widths = {0};
    CHECK_THROWS(cfg.validate(7), ParamError);
    cfg.hidden_widths = {8, 8, 8};
    CHECK_THROWS(cfg.validate(7), ParamError);
    cfg.hidden_widths = {32};
    CHECK_THROWS(cfg.validate(7), ParamError);
    cfg.unconstrained = true;
    cfg.validate(7);
    cfg.learning_rate = 0.5;
    CHECK_THROWS(cfg.validate(7), ParamError);
  }
  // FitsConstantTarget (test_models.cpp:105-117)
  {
    const auto ds = synth_mm(40, 3, [](std::uint64_t, int, std::mt19937_64&) { return 0.125; });
    auto cfg = default_config(KernelKind::MM, ModelFamily::NnC);
    cfg.learning_rate = 1e-3;
    cfg.epochs = 4000;
    cfg.seed = 1;
    const auto model = train_nn(ds, cfg);
    // the reference's test bar is < 1e-6 on its own sampled dataset; on this dataset the
    // reference train_nn itself (linked from the reference core objects) ends at exactly:
    CHECK(model.loss_trace.back() == 5.2222559624722591e-06);
    for (const auto& s : ds.samples) {
      const double p = predict(model, model_features(s, ModelFamily::NnC));
      CHECK(std::fabs(p - 0.125) <= 0.125 * 1e-3);
    }
  }
  // DeterministicInSeed (test_models.cpp:119-133)
  {
    const auto ds = synth_mm(30, 5, [](std::uint64_t c, int, std::mt19937_64&) { return 1e-9 * double(c) + 1e-6; });
    auto cfg = default_config(KernelKind::MM, ModelFamily::NnC);
    cfg.epochs = 500;
    cfg.seed = 11;
    const auto a = train_nn(ds, cfg);
    const auto b = train_nn(ds, cfg);
    CHECK(std::get<Mlp>(a.payload).layers[0].w == std::get<Mlp>(b.payload).layers[0].w);
    CHECK(a.loss_trace == b.loss_trace);
    cfg.seed = 12;
    const auto c = train_nn(ds, cfg);
    CHECK(std::get<Mlp>(a.payload).layers[0].w != std::get<Mlp>(c.payload).layers[0].w);
  }
  // LearnsLinearComplexityWorld (test_models.cpp:135-155)
  {
    auto make = [](std::uint64_t seed) {
      return synth_mm(250, seed, [](std::uint64_t c, int, std::mt19937_64& r) {
        return 3e-9 * double(c) * (1.0 + (double(r() >> 11) * 0x1.0p-53 * 0.02 - 0.01));
      });
    };
    const auto tr = make(100), te = make(200);
    auto cfg = default_config(KernelKind::MM, ModelFamily::NnC);
    cfg.seed = 3;
    const auto model = train_nn(tr, cfg);
    const auto pred = predict_dataset(model, te);
    const auto thr = eval::mape_thresholded(te.runtimes(), pred, 0.3);
    CHECK(thr.value <= 10.0);
  }
  // RejectsSchemaMismatch (test_models.cpp:166-172)
  {
    const auto ds = synth_mm(20, 3, [](std::uint64_t, int, std::mt19937_64&) { return 0.5; });
    auto cfg = default_config(KernelKind::MM, ModelFamily::NnC);
    cfg.epochs = 10;
    const auto model = train_nn(ds, cfg);
    CHECK_THROWS(predict(model, std::vector<double>{1.0, 2.0}), SchemaError);
  }
  // Eval hand examples (test_eval.cpp:64-157)
  {
    CHECK(eval::mape(std::vector{1.0, 2.0, 3.0}, std::vector{1.0, 2.0, 3.0}) == 0.0);
    CHECK(eval::mape(std::vector{100.0}, std::vector{90.0}) == 10.0);
    CHECK(eval::mape(std::vector{1.0, 2.0}, std::vector{2.0, 1.0}) == 75.0);
    CHECK_THROWS(eval::mape(std::vector{0.0}, std::vector{1.0}), DomainError);
    std::vector<double> t(10), p(10);
    for (int i = 0; i < 10; ++i) {
      t[i] = i + 1;
      p[i] = (i + 1) * 1.1;
    }
    const auto r = eval::mape_thresholded(t, p, 0.3);
    CHECK(r.n_kept == 7u && std::fabs(r.value - 10.0) < 1e-9);
    CHECK(std::fabs(eval::spearman(std::vector{1.0, 2.0, 3.0, 4.0}, std::vector{1.0, 3.0, 2.0, 4.0}) - 0.8) < 1e-12);
    CHECK(eval::spearman(std::vector{0.1, 0.2, 0.5, 0.9}, std::vector{4.0, 3.0, 2.0, 1.0}) == -1.0);
    CHECK_THROWS(eval::spearman(std::vector{1.0}, std::vector{1.0}), DomainError);
    CHECK_THROWS(eval::mape_thresholded(std::vector{1.0, 2.0}, std::vector{1.0, 2.0}, 1.0), DomainError);
  }
  // Selector (test_selector.cpp:15-96)
  {
    CHECK(kernels::ScheduleSpace::cpu_default().size() == 2200u);
    CHECK(kernels::ScheduleSpace::gpu_style().size() == 196u);
    const kernels::ScheduleCandidate small{2, 4, 4, 2}, big{8, 8, 8, 8};
    CHECK(selector::select([](const kernels::ScheduleCandidate&) { return 0.5; }, {big, small}) == small);
    const auto a = selector::enumerate_candidates(kernels::ScheduleSpace::cpu_default(), 100, 4);
    const auto b = selector::enumerate_candidates(kernels::ScheduleSpace::cpu_default(), 100, 4);
    CHECK(a.size() == 100u && a == b);
    // memorizing predictor == brute-force argmin (100 random candidate sets)
    std::mt19937_64 rng(31);
    const auto lattice = kernels::ScheduleSpace::cpu_default().enumerate_all();
    for (int trial = 0; trial < 100; ++trial) {
      std::map<kernels::ScheduleCandidate, double> table;
      std::vector<kernels::ScheduleCandidate> cands;
      for (int i = 0; i < 40; ++i) {
        const auto& c = lattice[rng() % lattice.size()];
        if (!table.count(c)) {
          table[c] = double(rng() >> 11) * 0x1.0p-53;
          cands.push_back(c);
        }
      }
      const auto chosen = selector::select([&](const kernels::ScheduleCandidate& c) { return table.at(c); }, cands);
      auto best = cands[0];
      for (const auto& c : cands)
        if (table[c] < table[best] || (table[c] == table[best] && c < best)) best = c;
      CHECK(chosen == best);
    }
  }
  // Bit-exact pin: config 1 seed 1 through the drop-in API on the GPU (values from the
  // reference run, tests/golden/golden_r01.json): the acceptance-world dataset is rebuilt by
  // the caller exactly as acceptance_main.cpp:281-289 does, here from the engine's C ABI.
  {
    lann_world w{};
    w.kind = LANN_MM;
    w.hw_class = LANN_HW_CPU;
    w.max_threads = 4;
    w.alpha = 3e-9;
    w.g0 = 0.25;
    w.g1 = 0.75;
    w.noise = 0.02;
    std::vector<double> feats(500 * LANN_ROW), rt(500);
    std::vector<std::uint64_t> c(500);
    std::int32_t nf = 0;
    CHECK(lann_build_dataset(&w, 1, 500, feats.data(), c.data(), rt.data(), &nf) == 0);
    Dataset ds;
    ds.kind = KernelKind::MM;
    ds.feature_names = {"m", "n", "k", "d1", "d2", "n_thd"};
    for (int i = 0; i < 500; ++i) {
      Sample s;
      s.features.assign(feats.begin() + i * LANN_ROW, feats.begin() + i * LANN_ROW + nf);
      s.c = c[i];
      s.runtime_s = rt[i];
      s.variant_id = "dense_threaded";
      ds.samples.push_back(s);
    }
    const auto [train, test] = datagen::split(ds, 0.5, 1);
    auto cfg = default_config(KernelKind::MM, ModelFamily::NnC);
    cfg.seed = 1;
    engine::set_precision(engine::Precision::Fp64Exact);
    const auto model = train_model(train, cfg);
    const auto pred = predict_dataset(model, test);
    const auto rep = eval::make_report(test.runtimes(), pred, 0.3);
    CHECK(model.loss_trace.size() == 8000u);
    CHECK(model.loss_trace[0] == 0.324627613197639);
    CHECK(model.loss_trace.back() == 8.870984881723841e-05);
    CHECK(rep.mape_full == 21.40125600149908);
    CHECK(rep.mape_thresholded == 6.815106868884986);
    CHECK(rep.rho == 0.9934868717899487);
    std::printf("config1 seed1 via drop-in API: final loss %.17g thr-MAPE %.17g rho %.17g\n",
                model.loss_trace.back(), rep.mape_thresholded, rep.rho);
    // the batched overload trains 3 seeds in one call, each identical to its single call
    std::vector<ModelConfig> cfgs(3, cfg);
    cfgs[1].seed = 2;
    cfgs[2].seed = 3;
    const auto pop = train_population({&train, &train, &train}, cfgs);
    CHECK(pop[0].loss_trace == model.loss_trace);
    CHECK(std::get<Mlp>(pop[0].payload).layers[0].w == std::get<Mlp>(model.payload).layers[0].w);
    auto cfg3 = cfg;
    cfg3.seed = 3;
    CHECK(train_nn(train, cfg3).loss_trace == pop[2].loss_trace);
  }
  // TrainLinear.RecoversExactLine (test_models.cpp:269-285): t = 2c + 1 with small dims
  {
    // sample_params draws (densities vary: a full-rank design), dims <= 16, t = 2c + 1
    auto ds = datagen::build_mock(KernelKind::MM, "dense_threaded", 60, 13, 4, 16);
    for (auto& smp : ds.samples) smp.runtime_s = 2.0 * double(smp.c) + 1.0;
    ModelConfig cfg;
    cfg.family = ModelFamily::LrC;
    const auto model = train_lrc(ds, cfg);
    const auto& lin = std::get<LinearModel>(model.payload);
    CHECK(std::fabs(lin.weights.back() - 2.0) < 1e-6);
    CHECK(std::fabs(lin.intercept - 1.0) < 1e-6);
    for (std::size_t j = 0; j + 1 < lin.weights.size(); ++j) CHECK(std::fabs(lin.weights[j]) < 1e-5);
    CHECK_THROWS(param_count(model), ParamError);
  }
  // TrainConst.UsesOnlyComplexity (test_models.cpp:287-301)
  {
    const auto ds = synth_mm(60, 15, [](std::uint64_t c, int, std::mt19937_64&) { return 5e-9 * double(c) + 2e-6; });
    ModelConfig cfg;
    cfg.family = ModelFamily::Const;
    const auto model = train_const(ds, cfg);
    CHECK(model.schema == std::vector<std::string>{"c"});
    Sample smp = ds.samples[0];
    const double before = predict(model, model_features(smp, ModelFamily::Const));
    smp.features[0] += 100.0;
    smp.features[3] = 0.25;
    const double after = predict(model, model_features(smp, ModelFamily::Const));
    CHECK(before == after);
    CHECK(std::fabs(before - smp.runtime_s) <= smp.runtime_s * 1e-3);
  }
  // TrainForest.ConstantTargetAndDeterminism (test_models.cpp:303-326)
  {
    const auto ds = synth_mm(40, 3, [](std::uint64_t, int, std::mt19937_64&) { return 0.75; });
    ModelConfig cfg;
    cfg.family = ModelFamily::NlrC;
    cfg.seed = 5;
    const auto model = train_nlrc(ds, cfg);
    const auto preds = predict_dataset(model, ds);
    for (double v : preds) CHECK(v == 0.75);
    const auto noisy = synth_mm(50, 17, [](std::uint64_t c, int, std::mt19937_64& r) {
      return 1e-9 * double(c) + double(r() >> 11) * 0x1.0p-53 * 1e-6;
    });
    const auto a = train_nlrc(noisy, cfg), b = train_nlrc(noisy, cfg);
    CHECK(predict_dataset(a, noisy) == predict_dataset(b, noisy));
    Dataset tiny = ds;
    tiny.samples.resize(5);
    CHECK_THROWS(train_nlrc(tiny, cfg), ParamError);
  }
  // ModelIo.RoundTripPredictionsAreBitExact (test_models.cpp:328-350), all five families
  {
    const auto ds = synth_mm(40, 19, [](std::uint64_t c, int, std::mt19937_64& r) {
      return 2e-9 * double(c) * (1 + (double(r() >> 11) * 0x1.0p-53 - 0.5) * 0.2) + 1e-7;
    });
    for (ModelFamily family :
         {ModelFamily::NnC, ModelFamily::Nn, ModelFamily::Const, ModelFamily::LrC, ModelFamily::NlrC}) {
      ModelConfig cfg = default_config(KernelKind::MM, family);
      cfg.family = family;
      cfg.epochs = 200;
      cfg.seed = 23;
      const auto model = train_model(ds, cfg);
      const std::string path = "/tmp/lann_model_" + to_string(family) + ".json";
      save_model(model, path);
      const auto back = load_model(path);
      CHECK(back.schema == model.schema);
      CHECK(predict_dataset(model, ds) == predict_dataset(back, ds));
    }
    CHECK_THROWS(load_model("/tmp/lann_nonexistent_model.json"), LoadError);
  }
  std::printf("drop-in API: %d failures\n", g_fail);
  return g_fail == 0 ? 0 : 1;
}
