// Test helper for the on-disk formats of the perfsage:: API (no device needed): built and driven
// by tests/test_formats.py against the reference's own save/load (oracle/_ref shim).
//   formats_tool csv-roundtrip IN OUT      load_csv + save_csv
//   formats_tool csv-load IN               prints "ok <n>" or "<ErrorType>: <what>"
//   formats_tool model-roundtrip IN OUT    load_model + save_model
//   formats_tool model-load IN             prints "ok" or "<ErrorType>: <what>"
//   formats_tool model-synth OUT SEED      a model with awkward doubles (subnormals, -0, 0.1, ...)
//   formats_tool model-dump IN             %a of f_min, f_max, t_min, t_max, flat params, loss_trace
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>

#include "perfsage_b200/perfsage.hpp"

using namespace perfsage;

static int report(const std::exception& e) {
  const char* type = dynamic_cast<const LoadError*>(&e)    ? "LoadError"
                     : dynamic_cast<const ParamError*>(&e) ? "ParamError"
                                                           : "Error";
  std::printf("%s: %s\n", type, e.what());
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  const std::string mode = argv[1];
  try {
    if (mode == "csv-roundtrip") {
      datagen::save_csv(datagen::load_csv(argv[2]), argv[3]);
    } else if (mode == "csv-load") {
      try {
        std::printf("ok %zu\n", datagen::load_csv(argv[2]).size());
      } catch (const std::exception& e) {
        return report(e);
      }
    } else if (mode == "model-roundtrip") {
      models::save_model(models::load_model(argv[2]), argv[3]);
    } else if (mode == "model-load") {
      try {
        models::load_model(argv[2]);
        std::printf("ok\n");
      } catch (const std::exception& e) {
        return report(e);
      }
    } else if (mode == "model-synth") {
      std::mt19937_64 rng(std::strtoull(argv[3], nullptr, 10));
      std::uniform_real_distribution<double> u(-1.0, 1.0);
      const double awkward[] = {0.1, -0.0, 5e-324, DBL_MIN, DBL_MAX, 1.0 / 3.0, -2.2250738585072009e-308,
                                123456789.123456789, 1e-300, 6.02214076e23};
      models::TrainedModel m;
      m.kind = kernels::KernelKind::MM;
      m.config = models::default_config(m.kind, models::ModelFamily::NnC);
      m.config.seed = 0xFFFFFFFFFFFFFFFFULL;  // u64 seeds must survive the round trip
      m.schema = {"m", "n", "k", "d1", "d2", "n_thd", "c"};
      models::Mlp net;
      const int dims[] = {7, 8, 1};
      int k = 0;
      for (int l = 0; l < 2; ++l) {
        models::DenseLayer L;
        L.in = dims[l];
        L.out = dims[l + 1];
        for (int i = 0; i < L.in * L.out; ++i) L.w.push_back(k < 10 ? awkward[k++] : u(rng));
        for (int i = 0; i < L.out; ++i) L.b.push_back(u(rng) * 1e-7);
        net.layers.push_back(L);
      }
      m.payload = net;
      for (int j = 0; j < 7; ++j) {
        m.norm.f_min.push_back(u(rng));
        m.norm.f_max.push_back(u(rng) + 2.0);
      }
      m.norm.t_min = 1.2345e-7;
      m.norm.t_max = 3.0000000000000004;
      for (int e = 0; e < 50; ++e) m.loss_trace.push_back(std::ldexp(u(rng) + 1.5, -e));
      models::save_model(m, argv[2]);
    } else if (mode == "model-synth-linear" || mode == "model-synth-forest") {
      std::mt19937_64 rng(std::strtoull(argv[3], nullptr, 10));
      std::uniform_real_distribution<double> u(-1.0, 1.0);
      models::TrainedModel m;
      m.kind = kernels::KernelKind::MV;
      m.schema = {"m", "n", "d", "c"};
      if (mode == "model-synth-linear") {
        m.config = models::default_config(m.kind, models::ModelFamily::LrC);
        models::LinearModel lin;
        lin.weights = {1e-300, -0.0, u(rng), 0.1};
        lin.intercept = u(rng) * 1e-7;
        m.payload = lin;
      } else {
        m.config = models::default_config(m.kind, models::ModelFamily::NlrC);
        m.config.forest_trees = 3;
        models::Forest f;
        for (int t = 0; t < 3; ++t) {
          models::Tree tree;
          tree.nodes.push_back({int(t % 4), u(rng), 1, 2, u(rng)});
          tree.nodes.push_back({-1, 0.0, -1, -1, u(rng) * 1e-9});
          tree.nodes.push_back({-1, 0.0, -1, -1, 5e-324});
          f.trees.push_back(tree);
        }
        m.payload = f;
      }
      models::save_model(m, argv[2]);
    } else if (mode == "model-dump") {
      const auto m = models::load_model(argv[2]);
      for (double v : m.norm.f_min) std::printf("%a\n", v);
      for (double v : m.norm.f_max) std::printf("%a\n", v);
      std::printf("%a\n%a\n", m.norm.t_min, m.norm.t_max);
      for (double v : models::flatten_params(std::get<models::Mlp>(m.payload))) std::printf("%a\n", v);
      for (double v : m.loss_trace) std::printf("%a\n", v);
    } else {
      return 2;
    }
  } catch (const std::exception& e) {
    std::printf("unexpected %s\n", e.what());
    return 1;
  }
  return 0;
}
