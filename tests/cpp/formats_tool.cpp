// Test helper for the on-disk formats of the perfsage:: API (no device needed): built and driven
// by tests/test_formats.py against the reference's own save/load (oracle/_ref shim).
//   formats_tool csv-roundtrip IN OUT      load_csv + save_csv
//   formats_tool csv-load IN               prints "ok <n>" or "<ErrorType>: <what>"
//   formats_tool model-roundtrip IN OUT    load_model + save_model
//   formats_tool model-load IN             prints "ok" or "<ErrorType>: <what>"
//   formats_tool model-synth OUT SEED      a model with awkward doubles (subnormals, -0, 0.1, ...)
//   formats_tool model-dump IN             %a of f_min, f_max, t_min, t_max, flat params, loss_trace
//   formats_tool api-gen KIND VARIANT MAXTHR DIMMAX GPU COUNT SEED OUT [SIDES...]
//                                          datagen::build_dataset(descriptor, ParamSpace, ..., {probe})
//                                          with the reference CLI's mock probe (perfsage.cpp:71-84)
//   formats_tool api-init SEED D0 D1 ...   %a of Mlp::init(dims, Rng(SEED)) flattened
//   formats_tool api-params KIND SEED N    N sample_params draws: features (augmented, n_thd) as %a
//   formats_tool api-train SEED EPOCHS LR N D0 D1 ...
//                                          models::train_full_batch on the GPU (needs a device):
//                                          prints X, y, initial params, then trace + final params
//                                          or "TrainingError <epoch>"
//   formats_tool api-gen-errors            build_dataset's ParamError / BuildAbortError contract
//   formats_tool api-validate              InstanceParams::validate / complexity edge cases
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
  if (argc < 2) return 2;
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
    } else if (mode == "api-gen") {
      if (argc < 10) return 2;
      const auto kind = kernels::kind_from_string(argv[2]);
      const std::string vid = argv[3];
      auto space = datagen::ParamSpace::defaults(kind, std::atoi(argv[4]));
      space.dim_max = std::uint32_t(std::strtoul(argv[5], nullptr, 10));
      if (kind == kernels::KernelKind::Blur) {
        space.blur_sides.clear();
        for (int i = 10; i < argc; ++i) space.blur_sides.push_back(std::uint32_t(std::strtoul(argv[i], nullptr, 10)));
        space.schedules = std::atoi(argv[6]) ? kernels::ScheduleSpace::gpu_style() : kernels::ScheduleSpace::cpu_default();
      }
      kernels::VariantDescriptor v;
      v.variant_id = vid;
      v.kind = kind;
      v.threading = vid.ends_with("_single") ? kernels::Threading::FixedSingle : kernels::Threading::Threaded;
      datagen::BuildOptions opts;
      opts.probe = [](const kernels::InstanceParams& p) {  // perfsage.cpp:71-84
        std::uint64_t h = 0x9e3779b97f4a7c15ULL;
        for (double f : models::featurize(p, true)) {
          std::uint64_t bits;
          std::memcpy(&bits, &f, sizeof bits);
          h ^= bits;
          splitmix64(h);
        }
        const double jitter = 0.5 + double(splitmix64(h) >> 11) * 0x1.0p-53;
        return 1e-9 * double(kernels::complexity(p)) * jitter + 1e-6;
      };
      datagen::save_csv(datagen::build_dataset(v, space, std::size_t(std::atoi(argv[7])),
                                               std::strtoull(argv[8], nullptr, 10), opts),
                        argv[9]);
    } else if (mode == "api-init") {
      Rng rng(std::strtoull(argv[2], nullptr, 10));
      std::vector<int> dims;
      for (int i = 3; i < argc; ++i) dims.push_back(std::atoi(argv[i]));
      try {
        for (double v : models::flatten_params(models::Mlp::init(dims, rng))) std::printf("%a\n", v);
      } catch (const ParamError& e) {
        return report(e);
      }
    } else if (mode == "api-params") {
      if (argc < 5) return 2;
      const auto kind = kernels::kind_from_string(argv[2]);
      auto space = datagen::ParamSpace::defaults(kind, 8);
      Rng rng(std::strtoull(argv[3], nullptr, 10));
      for (int i = 0, n = std::atoi(argv[4]); i < n; ++i) {
        const auto p = datagen::sample_params(space, rng);
        for (double f : models::featurize(p, true)) std::printf("%a ", f);
        std::printf("\n");
      }
    } else if (mode == "api-train") {
      if (argc < 8) return 2;
      const std::uint64_t seed = std::strtoull(argv[2], nullptr, 10);
      const int epochs = std::atoi(argv[3]), n = std::atoi(argv[5]);
      const double lr = std::strtod(argv[4], nullptr);
      std::vector<int> dims;
      for (int i = 6; i < argc; ++i) dims.push_back(std::atoi(argv[i]));
      Rng rng(seed);
      auto net = models::Mlp::init(dims, rng);
      std::vector<std::vector<double>> X(static_cast<std::size_t>(n), std::vector<double>(static_cast<std::size_t>(dims[0])));
      std::vector<double> y(static_cast<std::size_t>(n));
      for (auto& row : X)
        for (auto& v : row) v = rng.uniform();
      for (auto& v : y) v = rng.uniform();
      std::printf("X");
      for (const auto& row : X)
        for (double v : row) std::printf(" %a", v);
      std::printf("\ny");
      for (double v : y) std::printf(" %a", v);
      std::printf("\np0");
      for (double v : models::flatten_params(net)) std::printf(" %a", v);
      std::printf("\n");
      try {
        const auto trace = models::train_full_batch(net, X, y, lr, epochs);
        std::printf("trace");
        for (double v : trace) std::printf(" %a", v);
        std::printf("\np1");
        for (double v : models::flatten_params(net)) std::printf(" %a", v);
        std::printf("\n");
      } catch (const TrainingError& e) {
        std::printf("TrainingError %d\n", e.epoch());
      }
    } else if (mode == "api-gen-errors") {
      auto space = datagen::ParamSpace::defaults(kernels::KernelKind::MM, 4);
      kernels::VariantDescriptor v;
      v.variant_id = "dense_threaded";
      datagen::BuildOptions opts;
      int calls = 0;
      opts.probe = [&](const kernels::InstanceParams&) { return ++calls == 3 ? 0.0 : 1e-3; };
      auto attempt = [&](const char* name, auto&& fn) {
        try {
          fn();
          std::printf("%s ok\n", name);
        } catch (const BuildAbortError& e) {
          std::printf("%s BuildAbortError %zu %s\n", name, e.completed(), e.what());
        } catch (const ParamError& e) {
          std::printf("%s ParamError %s\n", name, e.what());
        }
      };
      attempt("count1", [&] { datagen::build_dataset(v, space, 1, 1, opts); });
      attempt("kind", [&] {
        auto other = v;
        other.kind = kernels::KernelKind::MV;
        datagen::build_dataset(other, space, 5, 1, opts);
      });
      attempt("noprobe", [&] { datagen::build_dataset(v, space, 5, 1); });
      attempt("zero", [&] { datagen::build_dataset(v, space, 5, 1, opts); });
      datagen::BuildOptions bad;
      bad.probe = [](const kernels::InstanceParams&) -> double { throw ParamError("probe failed"); };
      attempt("throws", [&] { datagen::build_dataset(v, space, 5, 1, bad); });
    } else if (mode == "api-validate") {
      using P = kernels::InstanceParams;
      const std::pair<const char*, P> cases[] = {
          {"mm-ok", P::mm(3, 4, 5, 0.5, 1.0, 2)},
          {"mm-zero-dim", P::mm(0, 4, 5)},
          {"mm-density", P::mm(3, 4, 5, 0.0, 1.0)},
          {"mv-ok", P::mv(7, 9, 0.25, 1)},
          {"mc-ok", P::mc(9, 8, 3, 1.0, 1)},
          {"mc-small", P::mc(2, 8, 3)},
          {"mp-ok", P::mp(9, 8, 3, 2, 1.0, 1)},
          {"mp-small", P::mp(1, 8, 3, 2)},
          {"blur-ok", P::blur(1024, {8, 256, 128, 8})},
          {"blur-npow2", P::blur(1024, {8, 255, 128, 8})},
          {"blur-small", P::blur(2, {8, 256, 128, 8})},
      };
      for (const auto& [name, p] : cases) {
        try {
          std::printf("%s %llu\n", name, static_cast<unsigned long long>(kernels::complexity(p)));
        } catch (const ParamError&) {
          std::printf("%s ParamError\n", name);
        }
      }
      try {
        auto bad = P::mv(3, 3);
        bad.n_thd = 0;
        bad.validate();
        std::printf("n_thd0 ok\n");
      } catch (const ParamError&) {
        std::printf("n_thd0 ParamError\n");
      }
      std::printf("median %a %a\n", datagen::median_of({3.0, 1.0, 2.0}), datagen::median_of({4.0, 1.0, 2.0, 3.0}));
      std::printf("speedup %a\n", eval::speedup(2.0, 0.5));
      const auto lad = datagen::density_ladder(10, false);
      std::printf("ladder");
      for (double d : lad) std::printf(" %a", d);
      std::printf("\n");
    } else {
      return 2;
    }
  } catch (const std::exception& e) {
    std::printf("unexpected %s\n", e.what());
    return 1;
  }
  return 0;
}
