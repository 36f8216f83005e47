// cli.cpp — `perfsage`, the command-line caller of the engine.
//
// Mirrors the reference tool's subcommands, options, outputs and manifest
// (/root/reference/proj/tools/perfsage.cpp:32-422) on top of the drop-in perfsage:: API and the
// C ABI, with every training / prediction / metric / selection step on the GPU:
//   gen      dataset -> dataset_<kernel>_<variant>.csv, from one of three probes:
//            --measure --kernel K --variant V   real B200 kernel variants timed with CUDA events
//                                               (measure.cu; `gen --list-variants`)
//            --external-cmd CMD --kernel K      the reference's external black-box protocol
//            --world W                          the engine's closed-form synthetic worlds
//   measure-variant  serve the external protocol for a B200 variant (one feature line in ->
//            one runtime out), so the reference's own `gen --external-cmd` can measure B200s
//   bench    measure one instance of a B200 variant (the reference times one CPU kernel)
//   train    CSV -> split(seed 0x5b11) -> train_model -> model_<family>.json, train.csv, test.csv
//   eval     model JSON(s) x CSV -> eval.csv (+ --group-by aggregate)
//   compare  CSV -> the five families (nnc, nn, const, lrc, nlrc) batched per family group -> compare.csv
//   select   blur schedules: train on measured samples, GPU argmin over the candidates,
//            regret / speedups (selection.json, schedules.csv)
//   sweep    the 48-combination population x seeds x k folds (config 3 / config 5) through
//            the engine, sharded over --devices (one engine + host thread per GPU, contiguous
//            cost-balanced shards, no collective) -> sweep.csv + per-combination summary
//   select-variants  config 4: counter-generated candidate shapes scored by V variant models,
//            argmin per candidate -> variant histogram (variants.csv)
// Every run appends {command, argv, seed, timestamp, inputs, outputs} to <out>/manifest.json
// (perfsage.cpp:36-66). Errors print "error: <what>" and exit 1, like the reference.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <ctime>
#include <filesystem>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "../../include/lann_engine.h"
#include "../../include/perfsage_b200/perfsage.hpp"
#include "domain.hpp"
#include "json_lite.hpp"

namespace fs = std::filesystem;
using namespace perfsage;

namespace {

// ---- argument parsing (--key value, --flag, repeated keys) -------------------------------------
struct Args {
  std::string command;
  std::multimap<std::string, std::string> kv;
  std::vector<std::string> raw;

  bool has(const std::string& k) const { return kv.count(k) > 0; }
  std::string get(const std::string& k, const std::string& def) const {
    auto it = kv.find(k);
    return it == kv.end() ? def : it->second;
  }
  std::vector<std::string> all(const std::string& k) const {
    std::vector<std::string> out;
    auto [a, b] = kv.equal_range(k);
    for (auto it = a; it != b; ++it) out.push_back(it->second);
    return out;
  }
  long long integer(const std::string& k, long long def) const {
    if (!has(k)) return def;
    const std::string v = get(k, "");
    char* end = nullptr;
    const long long x = std::strtoll(v.c_str(), &end, 10);
    if (v.empty() || *end) throw ParamError("--" + k + " expects an integer, got '" + v + "'");
    return x;
  }
  std::uint64_t u64(const std::string& k, std::uint64_t def) const {
    if (!has(k)) return def;
    const std::string v = get(k, "");
    char* end = nullptr;
    const unsigned long long x = std::strtoull(v.c_str(), &end, 10);
    if (v.empty() || *end) throw ParamError("--" + k + " expects an unsigned integer, got '" + v + "'");
    return x;
  }
  double real(const std::string& k, double def) const {
    if (!has(k)) return def;
    const std::string v = get(k, "");
    char* end = nullptr;
    const double x = std::strtod(v.c_str(), &end);
    if (v.empty() || *end) throw ParamError("--" + k + " expects a number, got '" + v + "'");
    return x;
  }
};

const std::vector<std::string> kFlags = {"unconstrained", "list", "help", "both-families", "measure",
                                         "gpu-class", "list-variants", "mock-timer"};

Args parse(int argc, char** argv) {
  Args a;
  if (argc < 2) throw ParamError("missing subcommand (gen, train, eval, compare, select, sweep, select-variants)");
  a.command = argv[1];
  for (int i = 1; i < argc; ++i) a.raw.emplace_back(argv[i]);
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) throw ParamError("unexpected argument '" + k + "'");
    k = k.substr(2);
    const auto eq = k.find('=');
    if (eq != std::string::npos) {
      a.kv.emplace(k.substr(0, eq), k.substr(eq + 1));
    } else if (std::find(kFlags.begin(), kFlags.end(), k) != kFlags.end()) {
      a.kv.emplace(k, "1");
    } else {
      if (i + 1 >= argc) throw ParamError("--" + k + " needs a value");
      a.kv.emplace(k, argv[++i]);
    }
  }
  return a;
}

// ---- manifest (perfsage.cpp:36-66) ------------------------------------------------------------
std::int64_t manifest_timestamp() {
  if (const char* env = std::getenv("PERFSAGE_TIMESTAMP")) return std::atoll(env);
  return static_cast<std::int64_t>(std::time(nullptr));
}

std::string host_label() {
  std::string model = "unknown-cpu";
  std::ifstream is("/proc/cpuinfo");
  std::string line;
  while (std::getline(is, line))
    if (line.rfind("model name", 0) == 0) {
      model = line.substr(line.find(':') + 2);
      break;
    }
  return model + " x" + std::to_string(std::thread::hardware_concurrency()) + " + B200 engine";
}

void record_run(const fs::path& out, const Args& a, std::uint64_t seed, const std::vector<std::string>& inputs,
                const std::vector<std::string>& outputs) {
  using namespace lann::jsonl;
  fs::create_directories(out);
  const fs::path path = out / "manifest.json";
  std::string host = host_label();
  std::vector<std::string> runs;  // previous runs, re-serialised
  if (fs::exists(path)) {
    std::ifstream is(path, std::ios::binary);
    std::stringstream buf;
    buf << is.rdbuf();
    Json m;
    try {
      m = Parser(buf.str()).document();
    } catch (const LoadError&) {
      throw LoadError("existing manifest '" + path.string() + "' is not valid JSON");
    }
    if (const Json* h = m.find("host")) host = h->str();
    if (const Json* r = m.find("runs"))
      for (const auto& run : r->items) {
        std::ostringstream o;
        o << "{\"command\": " << quote(run.at("command").str()) << ", \"argv\": [";
        for (std::size_t i = 0; i < run.at("argv").items.size(); ++i)
          o << (i ? ", " : "") << quote(run.at("argv").items[i].str());
        o << "], \"seed\": " << run.at("seed").text << ", \"timestamp\": " << run.at("timestamp").text
          << ", \"inputs\": [";
        for (std::size_t i = 0; i < run.at("inputs").items.size(); ++i)
          o << (i ? ", " : "") << quote(run.at("inputs").items[i].str());
        o << "], \"outputs\": [";
        for (std::size_t i = 0; i < run.at("outputs").items.size(); ++i)
          o << (i ? ", " : "") << quote(run.at("outputs").items[i].str());
        o << "]}";
        runs.push_back(o.str());
      }
  }
  std::ostringstream o;
  o << "{\"command\": " << quote(a.command) << ", \"argv\": " << jarr(a.raw) << ", \"seed\": " << seed
    << ", \"timestamp\": " << manifest_timestamp() << ", \"inputs\": " << jarr(inputs)
    << ", \"outputs\": " << jarr(outputs) << "}";
  runs.push_back(o.str());
  std::ofstream os(path, std::ios::binary);
  os << "{\n  \"host\": " << quote(host) << ",\n  \"runs\": [\n";
  for (std::size_t i = 0; i < runs.size(); ++i) os << "    " << runs[i] << (i + 1 < runs.size() ? ",\n" : "\n");
  os << "  ]\n}\n";
}

// ---- shared helpers ------------------------------------------------------------------------------
void setup_engine(const Args& a) {
  const std::string p = a.get("precision", "fp64");
  if (p == "fp64") engine::set_precision(engine::Precision::Fp64Exact);
  else if (p == "fp32") engine::set_precision(engine::Precision::Fp32);
  else throw ParamError("--precision must be fp64 or fp32");
  engine::set_device(int(a.integer("device", 0)));
}

std::vector<int> parse_ints(const std::string& s) {
  std::vector<int> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ',')) {
    char* end = nullptr;
    const long v = std::strtol(tok.c_str(), &end, 10);
    if (tok.empty() || *end) throw ParamError("expected a comma-separated integer list, got '" + s + "'");
    out.push_back(int(v));
  }
  return out;
}

kernels::ScheduleCandidate parse_schedule(const std::string& text) {  // perfsage.cpp:86-96
  const auto v = parse_ints(text);
  if (v.size() != 4) throw ParamError("schedule must be four comma-separated factors, e.g. 8,256,128,8");
  kernels::ScheduleCandidate c;
  c.s1 = std::uint32_t(v[0]);
  c.s2 = std::uint32_t(v[1]);
  c.s3 = std::uint32_t(v[2]);
  c.s4 = std::uint32_t(v[3]);
  if (!c.is_pow2()) throw ParamError("schedule factors must be positive powers of two");
  return c;
}

models::ModelConfig make_config(kernels::KernelKind kind, models::ModelFamily family, const Args& a,
                                std::uint64_t seed) {  // perfsage.cpp:111-123
  auto cfg = models::default_config(kind, family, a.has("unconstrained"));
  cfg.family = family;
  cfg.seed = seed;
  if (a.has("epochs")) cfg.epochs = int(a.integer("epochs", cfg.epochs));
  if (a.has("lr")) cfg.learning_rate = a.real("lr", cfg.learning_rate);
  if (a.has("hidden")) cfg.hidden_widths = parse_ints(a.get("hidden", ""));
  return cfg;
}

eval::EvalReport evaluate_model_on(const models::TrainedModel& m, const datagen::Dataset& data, double drop,
                                   const std::vector<double>& pred) {  // perfsage.cpp:98-108
  const auto truth = data.runtimes();
  auto rep = eval::make_report(truth, pred, drop);
  rep.kernel = kernels::to_string(data.kind);
  rep.variant = data.samples.empty() ? "" : data.samples.front().variant_id;
  rep.model_family = models::to_string(m.config.family);
  return rep;
}

std::string sanitize(std::string s) {
  for (char& ch : s)
    if (ch == '@' || ch == '/' || ch == ' ') ch = '_';
  return s;
}

// hostinfo.cpp:26-34: hardware threads, capped by PERFSAGE_THREADS
int host_max_threads() {
  int hw = int(std::thread::hardware_concurrency());
  if (hw < 1) hw = 1;
  if (const char* env = std::getenv("PERFSAGE_THREADS")) {
    const int cap = std::atoi(env);
    if (cap >= 1) hw = std::min(hw, cap);
  }
  return hw;
}

// ---- subcommands ---------------------------------------------------------------------------------
int cmd_gen(const Args& a) {
  if (a.has("list-variants")) {
    std::cout << "kernel  B200 variant\n";
    for (auto k : {kernels::KernelKind::MM, kernels::KernelKind::MV, kernels::KernelKind::MC, kernels::KernelKind::MP,
                   kernels::KernelKind::Blur})
      for (const auto& v : datagen::measured_variants(k))
        std::cout << std::left << std::setw(8) << kernels::to_string(k) << v << "\n";
    return 0;
  }
  if (a.has("mock-timer")) {  // perfsage.cpp:197-248 with --mock-timer: byte-identical dataset
    const auto kind = kernels::kind_from_string(a.get("kernel", "mm"));
    std::string variant = a.get("variant", "dense_threaded");
    if (kind == kernels::KernelKind::Blur && variant == "dense_threaded") variant = "tiled";  // the only blur variant
    const int mt = int(a.integer("max-threads", 0));
    const int threads = mt > 0 ? mt : host_max_threads();
    std::vector<std::uint32_t> sides;
    for (const auto& v : a.all("blur-n")) sides.push_back(std::uint32_t(std::strtoul(v.c_str(), nullptr, 10)));
    if (sides.empty()) sides = {1024};
    const std::uint64_t seed = a.u64("seed", 1);
    const auto ds = datagen::build_mock(kind, variant, std::size_t(a.integer("count", 500)), seed, threads,
                                        std::uint32_t(a.integer("dim-max", 1024)), sides,
                                        a.get("blur-space", "cpu") == "gpu");
    const fs::path out = a.get("out", "perfsage_out");
    fs::create_directories(out);
    const fs::path csv = out / ("dataset_" + a.get("kernel", "mm") + "_" + variant + ".csv");
    datagen::save_csv(ds, csv.string());
    record_run(out, a, seed, {}, {csv.string()});
    std::cout << "wrote " << ds.size() << " samples to " << csv.string() << "\n";
    return 0;
  }
  if (a.has("measure") || a.has("external-cmd")) {
    const auto kind = kernels::kind_from_string(a.get("kernel", "mm"));
    const std::size_t count = std::size_t(a.integer("count", 500));
    const std::uint64_t seed = a.u64("seed", 1);
    const fs::path out = a.get("out", "perfsage_out");
    datagen::Dataset ds;
    std::string vid;
    if (a.has("measure")) {
      const std::string variant = a.get("variant", "");
      if (variant.empty()) throw ParamError("--measure needs --variant (see gen --list-variants)");
      const datagen::TimingPolicy pol{int(a.integer("warmups", 1)), int(a.integer("reps", 5))};
      ds = datagen::build_measured(kind, variant, count, seed, pol, a.get("blur-space", "gpu") == "gpu",
                                   std::uint32_t(a.integer("blur-side", 1024)));
      vid = variant + "@b200";
    } else {
      vid = a.get("variant-id", a.get("external-id", "external"));
      ds = datagen::build_external(kind, a.get("external-cmd", ""), vid, a.has("gpu-class"),
                                   int(a.integer("max-threads", 4)), count, seed);
    }
    fs::create_directories(out);
    const fs::path csv = out / ("dataset_" + kernels::to_string(kind) + "_" + sanitize(vid) + ".csv");
    datagen::save_csv(ds, csv.string());
    record_run(out, a, seed, {}, {csv.string()});
    std::cout << "wrote " << ds.size() << " samples to " << csv.string() << "\n";
    return 0;
  }
  if (a.has("kernel") && !a.has("world"))
    throw ParamError("measuring the reference's CPU kernels is not part of this engine: use --mock-timer, "
                     "--measure (B200 variants, gen --list-variants), --external-cmd or --world (gen --list)");
  if (a.has("list")) {
    std::cout << "world  kernel  variant\n";
    for (int i = 0; i < datagen::synthetic_world_count(); ++i) {
      const auto ds = datagen::build_synthetic(i, 2, 1);
      std::cout << std::left << std::setw(7) << i << std::setw(8) << kernels::to_string(ds.kind)
                << datagen::combo_variant_id(i) << "\n";
    }
    return 0;
  }
  const int world = int(a.integer("world", 0));
  const std::size_t count = std::size_t(a.integer("count", 500));
  const std::uint64_t seed = a.u64("seed", 1);
  const fs::path out = a.get("out", "perfsage_out");
  const auto ds = datagen::build_synthetic(world, count, seed);
  fs::create_directories(out);
  const fs::path csv =
      out / ("dataset_" + kernels::to_string(ds.kind) + "_" + sanitize(datagen::combo_variant_id(world)) + ".csv");
  datagen::save_csv(ds, csv.string());
  record_run(out, a, seed, {}, {csv.string()});
  std::cout << "wrote " << ds.size() << " samples to " << csv.string() << "\n";
  return 0;
}

int cmd_train(const Args& a) {  // perfsage.cpp:250-278
  setup_engine(a);
  const std::string data = a.get("data", "");
  if (data.empty()) throw ParamError("--data is required");
  const std::string fam = a.get("family", "nnc");
  const auto family = models::family_from_string(fam);
  const std::uint64_t seed = a.u64("seed", 0);
  const auto dataset = datagen::load_csv(data);
  const auto [train_set, test_set] = datagen::split(dataset, a.real("train-frac", 0.5), lann::derive_seed(seed, 0x5b11));
  const auto cfg = make_config(dataset.kind, family, a, seed);
  const auto model = models::train_model(train_set, cfg);
  const fs::path out = a.get("out", "perfsage_out");
  fs::create_directories(out);
  const fs::path mp = out / ("model_" + fam + ".json"), tr = out / "train.csv", te = out / "test.csv";
  models::save_model(model, mp.string());
  datagen::save_csv(train_set, tr.string());
  datagen::save_csv(test_set, te.string());
  record_run(out, a, seed, {data}, {mp.string(), tr.string(), te.string()});
  std::cout << "trained " << fam << " on " << train_set.size() << " samples";
  if (std::holds_alternative<models::Mlp>(model.payload))
    std::cout << " (" << models::param_count(model) << " parameters, final loss " << model.loss_trace.back() << ")";
  std::cout << "\nmodel: " << mp.string() << "\n";
  return 0;
}

int cmd_eval(const Args& a) {  // perfsage.cpp:280-305
  setup_engine(a);
  const std::string data_path = a.get("data", "");
  const auto paths = a.all("model");
  if (data_path.empty() || paths.empty()) throw ParamError("--data and at least one --model are required");
  const auto data = datagen::load_csv(data_path);
  if (data.samples.empty()) throw DomainError("evaluation dataset is empty");
  std::vector<models::TrainedModel> ms;
  for (const auto& p : paths) ms.push_back(models::load_model(p));
  std::vector<const models::TrainedModel*> mp;
  std::vector<const datagen::Dataset*> dp;
  for (const auto& m : ms) {
    mp.push_back(&m);
    dp.push_back(&data);
  }
  const auto preds = models::predict_population(mp, dp);  // every model in one engine call
  const double drop = a.real("drop", 0.3);
  std::vector<eval::EvalReport> reports;
  for (std::size_t i = 0; i < ms.size(); ++i) reports.push_back(evaluate_model_on(ms[i], data, drop, preds[i]));
  const fs::path out = a.get("out", "perfsage_out");
  fs::create_directories(out);
  const fs::path csv = out / "eval.csv";
  {
    std::ofstream os(csv, std::ios::binary);
    eval::write_reports_csv(os, reports);
  }
  eval::print_reports(std::cout, reports);
  if (a.has("group-by")) {
    const std::string g = a.get("group-by", "kernel");
    eval::GroupBy gb = eval::GroupBy::Kernel;
    if (g == "variant") gb = eval::GroupBy::Variant;
    else if (g == "family") gb = eval::GroupBy::ModelFamily;
    else if (g != "kernel") throw ParamError("--group-by must be kernel, variant, or family");
    eval::print_aggregate(std::cout, eval::aggregate(reports, gb));
  }
  record_run(out, a, 0, paths, {csv.string()});
  return 0;
}

int cmd_compare(const Args& a) {  // perfsage.cpp:384-414, NN families batched
  setup_engine(a);
  const std::string data = a.get("data", "");
  if (data.empty()) throw ParamError("--data is required");
  const std::uint64_t seed = a.u64("seed", 0);
  const auto dataset = datagen::load_csv(data);
  const auto [train_set, test_set] = datagen::split(dataset, a.real("train-frac", 0.5), lann::derive_seed(seed, 0x5b11));
  const std::vector<models::ModelFamily> fams = {models::ModelFamily::NnC, models::ModelFamily::Nn,
                                                 models::ModelFamily::Const, models::ModelFamily::LrC,
                                                 models::ModelFamily::NlrC};
  std::vector<models::ModelConfig> cfgs;
  std::vector<const datagen::Dataset*> trains, tests;
  for (auto f : fams) {
    cfgs.push_back(make_config(dataset.kind, f, a, seed));
    trains.push_back(&train_set);
    tests.push_back(&test_set);
  }
  const auto ms = models::train_population(trains, cfgs);  // NN pair in one launch set, LS, forest
  std::vector<const models::TrainedModel*> mp;
  for (const auto& m : ms) mp.push_back(&m);
  const auto preds = models::predict_population(mp, tests);
  const double drop = a.real("drop", 0.3);
  std::vector<eval::EvalReport> reports;
  for (std::size_t i = 0; i < ms.size(); ++i) reports.push_back(evaluate_model_on(ms[i], test_set, drop, preds[i]));
  std::size_t best = 0;
  for (std::size_t i = 1; i < reports.size(); ++i)
    if (reports[i].mape_thresholded < reports[best].mape_thresholded) best = i;
  const fs::path out = a.get("out", "perfsage_out");
  fs::create_directories(out);
  const fs::path csv = out / "compare.csv";
  {
    std::ofstream os(csv, std::ios::binary);
    eval::write_reports_csv(os, reports);
  }
  eval::print_reports(std::cout, reports);
  std::cout << "best thresholded MAPE: " << reports[best].model_family << " (" << reports[best].mape_thresholded
            << "%)\n";
  record_run(out, a, seed, {data}, {csv.string()});
  return 0;
}

int cmd_select(const Args& a) {  // perfsage.cpp:307-382
  setup_engine(a);
  const auto default_sched = parse_schedule(a.get("default", a.get("default-schedule", "8,256,128,8")));
  const std::uint32_t n = std::uint32_t(a.integer("n", 1024));
  const std::uint64_t seed = a.u64("seed", 0);
  datagen::Dataset measured;
  measured.kind = kernels::KernelKind::Blur;
  measured.feature_names = models::feature_names(kernels::KernelKind::Blur, false);
  measured.seed = seed;
  std::vector<kernels::ScheduleCandidate> candidates;
  selector::MeasuredCandidates table;
  std::vector<std::string> inputs;
  if (a.has("data")) {
    const std::string path = a.get("data", "");
    inputs.push_back(path);
    measured = datagen::load_csv(path);
    if (measured.kind != kernels::KernelKind::Blur) throw ParamError("--data must hold blur schedule samples");
    for (const auto& s : measured.samples) {
      if (std::uint32_t(s.features[0]) != n) continue;
      kernels::ScheduleCandidate c{std::uint32_t(s.features[1]), std::uint32_t(s.features[2]),
                                   std::uint32_t(s.features[3]), std::uint32_t(s.features[4])};
      candidates.push_back(c);
      table.emplace_back(c, s.runtime_s);
    }
    if (candidates.empty()) throw ParamError("no samples with n=" + std::to_string(n) + " in " + path);
  } else if (a.has("measure")) {
    // real B200 timings of the blur_sched variant at every candidate schedule (measure.cu)
    const bool gpu = a.get("lattice", "gpu") == "gpu";
    candidates = selector::enumerate_candidates(gpu ? kernels::ScheduleSpace::gpu_style()
                                                    : kernels::ScheduleSpace::cpu_default(),
                                                std::size_t(a.integer("candidates", 200)), seed);
    if (std::find(candidates.begin(), candidates.end(), default_sched) == candidates.end())
      candidates.push_back(default_sched);
    std::vector<double> feats(candidates.size() * LANN_ROW, 0.0), rt(candidates.size());
    for (std::size_t i = 0; i < candidates.size(); ++i) {
      const auto& c = candidates[i];
      double* f = &feats[i * LANN_ROW];
      f[0] = n, f[1] = c.s1, f[2] = c.s2, f[3] = c.s3, f[4] = c.s4;
    }
    lann_engine* e = nullptr;
    if (lann_engine_create(int(a.integer("device", 0)), &e) != LANN_OK)
      throw Error("no CUDA device: the LANN engine has no CPU fallback");
    const int st = lann_measure(e, LANN_BLUR, "blur_sched", int(candidates.size()), feats.data(),
                                int(a.integer("warmups", 2)), int(a.integer("reps", 7)), lann::derive_seed(seed, 0x1417),
                                rt.data(), nullptr);
    const std::string err = st ? lann_last_error(e) : "";
    lann_engine_destroy(e);
    if (st) throw ParamError("measurement failed: " + err);
    for (std::size_t i = 0; i < candidates.size(); ++i) {
      table.emplace_back(candidates[i], rt[i]);
      datagen::Sample smp;
      const auto& c = candidates[i];
      smp.features = {double(n), double(c.s1), double(c.s2), double(c.s3), double(c.s4)};
      smp.c = std::uint64_t(n) * n;
      smp.runtime_s = rt[i];
      smp.variant_id = "blur_sched@b200";
      measured.samples.push_back(std::move(smp));
    }
  } else if (a.has("mock-timer")) {
    // perfsage.cpp:340-362 with --mock-timer: every candidate (plus the default) probed by the
    // deterministic mock timer on blur(n, schedule) with n_thd = the worker threads
    const int mt = int(a.integer("max-threads", 0));
    const int threads = mt > 0 ? mt : host_max_threads();
    candidates = selector::enumerate_candidates(kernels::ScheduleSpace::cpu_default(),
                                                std::size_t(a.integer("candidates", 200)), seed);
    if (std::find(candidates.begin(), candidates.end(), default_sched) == candidates.end())
      candidates.push_back(default_sched);
    std::vector<std::uint32_t> flat;
    for (const auto& c : candidates) flat.insert(flat.end(), {c.s1, c.s2, c.s3, c.s4});
    std::vector<double> rt(candidates.size());
    if (lann_mock_schedules(n, threads, int(candidates.size()), flat.data(), rt.data()))
      throw ParamError("schedule probe failed");
    for (std::size_t i = 0; i < candidates.size(); ++i) {
      table.emplace_back(candidates[i], rt[i]);
      datagen::Sample smp;
      const auto& c = candidates[i];
      smp.features = {double(n), double(c.s1), double(c.s2), double(c.s3), double(c.s4)};
      smp.c = std::uint64_t(n) * n;
      smp.runtime_s = rt[i];
      smp.variant_id = "tiled";
      measured.samples.push_back(std::move(smp));
    }
  } else {
    // the synthetic blur world stands in for measuring the tiled kernel (out of scope)
    const int world = int(a.integer("world", 40));
    const auto worlds = lann::default_combos();
    if (world < 0 || world >= int(worlds.size()) || worlds[std::size_t(world)].kind != LANN_BLUR)
      throw ParamError("--world must name a blur world (40..47)");
    candidates = selector::enumerate_candidates(kernels::ScheduleSpace::cpu_default(),
                                                std::size_t(a.integer("candidates", 200)), seed);
    if (std::find(candidates.begin(), candidates.end(), default_sched) == candidates.end())
      candidates.push_back(default_sched);
    std::vector<std::uint32_t> flat;
    for (const auto& c : candidates) flat.insert(flat.end(), {c.s1, c.s2, c.s3, c.s4});
    std::vector<double> rt(candidates.size());
    const int st = lann_probe_schedules(&worlds[std::size_t(world)], lann::derive_seed(seed, 0x1417), n,
                                        int(candidates.size()), flat.data(), rt.data());
    if (st) throw ParamError("schedule probe failed");
    const std::string vid = datagen::combo_variant_id(world);
    for (std::size_t i = 0; i < candidates.size(); ++i) {
      table.emplace_back(candidates[i], rt[i]);
      datagen::Sample s;
      const auto& c = candidates[i];
      s.features = {double(n), double(c.s1), double(c.s2), double(c.s3), double(c.s4)};
      s.c = std::uint64_t(n) * n;
      s.runtime_s = rt[i];
      s.variant_id = vid;
      measured.samples.push_back(std::move(s));
    }
  }
  const auto family = models::family_from_string(a.get("family", "nnc"));
  // --seeds K: train K init seeds (seed .. seed+K-1) as ONE population and keep the model with the
  // lowest final training loss (the protocol of acceptance criterion 8, acceptance_main.cpp:438-450)
  const int n_seeds = std::max(1, int(a.integer("seeds", 1)));
  std::vector<models::ModelConfig> cfgs;
  std::vector<const datagen::Dataset*> sets;
  for (int k = 0; k < n_seeds; ++k) {
    cfgs.push_back(make_config(kernels::KernelKind::Blur, family, a, seed + std::uint64_t(k)));
    sets.push_back(&measured);
  }
  auto trained = models::train_population(sets, cfgs);
  std::size_t pick = 0;
  for (std::size_t k = 1; k < trained.size(); ++k)
    if (!trained[k].loss_trace.empty() && trained[k].loss_trace.back() < trained[pick].loss_trace.back()) pick = k;
  const models::TrainedModel model = std::move(trained[pick]);
  const auto chosen = selector::select(model, n, candidates);
  std::vector<double> feats = {double(n), double(chosen.s1), double(chosen.s2), double(chosen.s3), double(chosen.s4)};
  if (models::family_augmented(family)) feats.push_back(double(std::uint64_t(n) * n));
  const double predicted = models::predict(model, feats);
  const auto report = selector::evaluate_selection(chosen, table, default_sched, std::nullopt, predicted);
  const fs::path out = a.get("out", "perfsage_out");
  fs::create_directories(out);
  const fs::path jp = out / "selection.json", cp = out / "schedules.csv";
  {
    std::ofstream os(jp, std::ios::binary);
    os << report.to_json() << '\n';
  }
  datagen::save_csv(measured, cp.string());
  record_run(out, a, seed, inputs, {jp.string(), cp.string()});
  std::cout << report.summary() << "\n";
  return 0;
}

// models::default_config (models.cpp:66-85) in job form
void default_model(const lann_world& w, lann_job& j, bool unconstrained) {
  if (w.kind == LANN_BLUR) {
    j.n_hidden = 2;
    j.hidden[0] = j.hidden[1] = unconstrained ? 40 : 5;
    j.learning_rate = 1e-2;
    j.epochs = 20000;
    j.log_target = 1;
  } else {
    j.n_hidden = 1;
    j.hidden[0] = unconstrained ? 64 : 8;
    j.hidden[1] = 0;
    j.learning_rate = 1e-2;
    j.epochs = 8000;
    j.log_target = 0;
  }
  j.unconstrained = unconstrained ? 1 : 0;
}

int cmd_sweep(const Args& a) {
  const std::uint64_t root = a.u64("root-seed", 1);
  const int n_seeds = int(a.integer("seeds", 256));
  const int n_folds = int(a.integer("folds", 5));
  const int count = int(a.integer("count", 500));
  const std::string fam = a.get("family", "nnc");
  const std::string prec = a.get("precision", "fp32");
  const int precision = prec == "fp64" ? LANN_FP64_EXACT : LANN_FP32;
  if (prec != "fp64" && prec != "fp32") throw ParamError("--precision must be fp64 or fp32");
  std::vector<int> families;
  if (fam == "nnc" || fam == "both") families.push_back(LANN_NNC);
  if (fam == "nn" || fam == "both") families.push_back(LANN_NN);
  if (families.empty()) throw ParamError("--family must be nnc, nn or both");
  if (n_seeds < 1 || (n_folds != 0 && n_folds < 2)) throw ParamError("--seeds >= 1 and --folds 0 or >= 2");
  const auto worlds = lann::default_combos();
  std::vector<int> combos;
  if (a.has("combos")) combos = parse_ints(a.get("combos", ""));
  else
    for (int i = 0; i < int(worlds.size()); ++i) combos.push_back(i);
  // config3_jobs (paper_2003_07497_b200/population.py): combo seed derive_seed(root, i),
  // init seed derive_seed(combo seed, 1 + s), fold f = block f of the split's train part
  std::vector<lann_job> jobs;
  struct Meta { int combo, family, seed, fold; };
  std::vector<Meta> meta;
  const double scale = a.real("epochs-scale", 1.0);
  for (int f : families)
    for (int i : combos) {
      if (i < 0 || i >= int(worlds.size())) throw ParamError("combination index out of range");
      const std::uint64_t ds = lann::derive_seed(root, std::uint64_t(i));
      for (int s = 0; s < n_seeds; ++s)
        for (int k = 0; k < std::max(1, n_folds); ++k) {
          lann_job j{};
          j.world = worlds[std::size_t(i)];
          j.data_seed = ds;
          j.count = count;
          j.train_fraction = 0.5;
          j.n_folds = n_folds;
          j.fold = k;
          j.family = f;
          default_model(j.world, j, a.has("unconstrained"));
          j.epochs = std::max(1, int(j.epochs * scale));
          j.init_seed = lann::derive_seed(ds, std::uint64_t(1 + s));
          jobs.push_back(j);
          meta.push_back({i, f, s, k});
        }
    }
  // one engine per device (--devices 0,1,... or a range 0-7; default --device, 0): contiguous
  // cost-balanced shards, one host thread per device, results gathered in job order, no NCCL
  std::vector<std::int32_t> devices;
  if (a.has("devices")) {
    const std::string d = a.get("devices", "0");
    if (const auto dash = d.find('-'); dash != std::string::npos && d.find(',') == std::string::npos) {
      const int lo = std::stoi(d.substr(0, dash)), hi = std::stoi(d.substr(dash + 1));
      if (lo < 0 || hi < lo) throw ParamError("--devices range must be lo-hi with 0 <= lo <= hi");
      for (int i = lo; i <= hi; ++i) devices.push_back(i);
    } else {
      for (int v : parse_ints(d)) devices.push_back(v);
    }
  } else {
    devices.push_back(std::int32_t(a.integer("device", 0)));
  }
  lann_group* group = nullptr;
  if (lann_group_create(std::int32_t(devices.size()), devices.data(), &group) != LANN_OK)
    throw Error("no CUDA device: the LANN engine has no CPU fallback");
  std::vector<std::int32_t> bounds(devices.size() + 1);
  lann_group_shard_bounds(group, std::int32_t(jobs.size()), jobs.data(), bounds.data());
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<lann_job_result> res(jobs.size());
  // k-fold sweeps also return the cross-validation summary (fold-mean test scores per seed,
  // per-combination fold and test statistics), computed on the devices
  std::int32_t n_groups = 0, n_ens = 0;
  lann_cv_layout(std::int32_t(jobs.size()), jobs.data(), &n_groups, &n_ens);
  std::vector<lann_cv_group> cvg(std::size_t(std::max(1, n_groups)));
  std::vector<lann_cv_ensemble> cve(std::size_t(std::max(1, n_ens)));
  const int st = n_groups > 0
                     ? lann_group_run_cv(group, std::int32_t(jobs.size()), jobs.data(), precision, res.data(),
                                         cvg.data(), cve.data())
                     : lann_group_run_population(group, std::int32_t(jobs.size()), jobs.data(), precision,
                                                 res.data(), nullptr, nullptr, nullptr, nullptr);
  const auto t2 = std::chrono::steady_clock::now();
  const double dev_ms = lann_group_last_device_ms(group);
  double flop = 0.0;  // algorithmic FLOP of the trainers
  for (std::size_t m = 0; m < jobs.size(); ++m)
    if (res[m].status == LANN_OK) {
      const auto& j = jobs[m];
      const int I = res[m].n_inputs, h1 = j.hidden[0], h2 = j.n_hidden > 1 ? j.hidden[1] : 0;
      const double fs = h2 > 0 ? 4.0 * I * h1 + 6.0 * h1 * h2 + 6.0 * h2 + h1 + 5 : 4.0 * I * h1 + 6.0 * h1 + 5;
      flop += double(j.epochs) * (res[m].n_train * fs + 14.0 * res[m].n_params);
    }
  const std::string err = st ? lann_group_last_error(group) : "";
  lann_group_destroy(group);
  if (st) throw Error("population run failed: " + err);
  const fs::path out = a.get("out", "perfsage_out");
  fs::create_directories(out);
  const fs::path csv = out / "sweep.csv";
  std::ofstream os(csv, std::ios::binary);
  os << "combo,kernel,variant,family,seed_index,fold,status,nonfinite_epoch,n_train,n_eval,final_loss,mape,"
        "mape_thresholded,rho,n_kept\n";
  os << std::setprecision(17);
  std::map<std::pair<int, int>, std::vector<double>> thr;
  long long model_epochs = 0;
  for (std::size_t m = 0; m < jobs.size(); ++m) {
    const auto& r = res[m];
    const auto& mt = meta[m];
    model_epochs += jobs[m].epochs;
    os << mt.combo << ',' << kernels::to_string(kernels::KernelKind(worlds[std::size_t(mt.combo)].kind)) << ','
       << datagen::combo_variant_id(mt.combo) << ',' << (mt.family == LANN_NNC ? "nnc" : "nn") << ',' << mt.seed
       << ',' << mt.fold << ',' << r.status << ',' << r.nonfinite_epoch << ',' << r.n_train << ',' << r.n_eval
       << ',' << r.final_loss << ',' << r.mape << ',' << r.mape_thr << ',' << r.rho << ',' << r.n_kept << '\n';
    if (r.status == LANN_OK) thr[{mt.family, mt.combo}].push_back(r.mape_thr);
  }
  os.close();
  if (n_groups == 0)
    std::cout << std::left << std::setw(7) << "combo" << std::setw(8) << "kernel" << std::setw(22) << "variant"
              << std::setw(7) << "model" << std::right << std::setw(10) << "models" << std::setw(14)
              << "median MAPE30%" << "\n";
  for (const auto& [key, v] : thr) {
    if (n_groups > 0) break;
    auto s = v;
    std::sort(s.begin(), s.end());
    const double med = s.size() % 2 ? s[s.size() / 2] : 0.5 * (s[s.size() / 2 - 1] + s[s.size() / 2]);
    std::cout << std::left << std::setw(7) << key.second << std::setw(8)
              << kernels::to_string(kernels::KernelKind(worlds[std::size_t(key.second)].kind)) << std::setw(22)
              << datagen::combo_variant_id(key.second) << std::setw(7) << (key.first == LANN_NNC ? "nnc" : "nn")
              << std::right << std::setw(10) << v.size() << std::fixed << std::setprecision(2) << std::setw(14)
              << med << "\n";
    std::cout.unsetf(std::ios::fixed);
  }
  const double all_s = std::chrono::duration<double>(t2 - t0).count();
  std::cout << jobs.size() << " models, " << model_epochs << " model-epochs on " << devices.size()
            << " device(s): device " << dev_ms << " ms (max over devices; " << double(model_epochs) / (dev_ms / 1e3)
            << " model-epochs/s, " << flop / (dev_ms / 1e3) / 1e12 << " TFLOP/s algorithmic), end to end " << all_s
            << " s\n";
  if (devices.size() > 1) {
    std::cout << "shards (jobs per device):";
    for (std::size_t d = 0; d < devices.size(); ++d)
      std::cout << ' ' << devices[d] << ':' << bounds[d + 1] - bounds[d];
    std::cout << "\n";
  }
  std::vector<std::string> outputs{csv.string()};
  if (n_groups > 0) {
    // cv.csv: one row per combination x family: held-out fold statistics over its seeds x folds
    // and the fold-mean model's test-part statistics over its seeds (mean, median)
    const fs::path cvp = out / "cv.csv";
    std::ofstream cs(cvp, std::ios::binary);
    cs << "combo,kernel,variant,family,n_folds,n_models,n_models_ok,n_ensembles,n_ensembles_ok,n_test,"
          "fold_mape_mean,fold_mape_median,fold_mape_thr_mean,fold_mape_thr_median,fold_rho_mean,fold_rho_median,"
          "test_mape_mean,test_mape_median,test_mape_thr_mean,test_mape_thr_median,test_rho_mean,test_rho_median\n";
    cs << std::setprecision(17);
    std::cout << std::left << std::setw(7) << "combo" << std::setw(8) << "kernel" << std::setw(22) << "variant"
              << std::setw(7) << "model" << std::right << std::setw(16) << "fold MAPE30% md" << std::setw(18)
              << "fold-mean MAPE%" << std::setw(18) << "fold-mean MAPE30%" << "\n";
    for (int gi = 0; gi < n_groups; ++gi) {
      const lann_cv_group& g = cvg[std::size_t(gi)];
      const auto& mt = meta[std::size_t(g.first_job)];
      const std::string kname = kernels::to_string(kernels::KernelKind(worlds[std::size_t(mt.combo)].kind));
      const std::string vname = datagen::combo_variant_id(mt.combo), fname = mt.family == LANN_NNC ? "nnc" : "nn";
      cs << mt.combo << ',' << kname << ',' << vname << ',' << fname << ',' << g.n_folds << ',' << g.n_models << ','
         << g.n_models_ok << ',' << g.n_ensembles << ',' << g.n_ensembles_ok << ',' << g.n_test;
      for (const lann_cv_stat& v : {g.fold_mape, g.fold_mape_thr, g.fold_rho, g.test_mape, g.test_mape_thr, g.test_rho})
        cs << ',' << v.mean << ',' << v.median;
      cs << '\n';
      std::cout << std::left << std::setw(7) << mt.combo << std::setw(8) << kname << std::setw(22) << vname
                << std::setw(7) << fname << std::right << std::fixed << std::setprecision(2) << std::setw(16)
                << g.fold_mape_thr.median << std::setw(18) << g.test_mape.mean << std::setw(18)
                << g.test_mape_thr.mean << "\n";
      std::cout.unsetf(std::ios::fixed);
    }
    outputs.push_back(cvp.string());
  }
  record_run(out, a, root, {}, outputs);
  return 0;
}

int cmd_select_variants(const Args& a) {
  setup_engine(a);
  const auto paths = a.all("model");
  if (paths.empty()) throw ParamError("at least one --model is required");
  std::vector<models::TrainedModel> ms;
  for (const auto& p : paths) ms.push_back(models::load_model(p));
  const auto kind = ms.front().kind;
  if (kind == kernels::KernelKind::Blur) throw ParamError("select-variants scores the prediction kernels (mm, mv, mc, mp)");
  std::vector<std::int32_t> n_in, h1, h2, logt, thd;
  std::vector<std::int64_t> poff;
  std::vector<double> params, norm;
  for (const auto& m : ms) {
    if (m.kind != kind) throw ParamError("all --model files must predict the same kernel kind");
    const auto& net = std::get<models::Mlp>(m.payload);
    if (net.layers.size() != 2) throw ParamError("select-variants expects one-hidden-layer prediction nets");
    n_in.push_back(net.layers[0].in);
    h1.push_back(net.layers[0].out);
    h2.push_back(0);
    logt.push_back(m.norm.log_target ? 1 : 0);
    const bool with_thd = std::find(m.schema.begin(), m.schema.end(), "n_thd") != m.schema.end();
    thd.push_back(with_thd ? 1 : 0);
    poff.push_back(std::int64_t(params.size()));
    const auto flat = models::flatten_params(net);
    params.insert(params.end(), flat.begin(), flat.end());
    double nrm[18] = {0};
    for (std::size_t i = 0; i < m.norm.f_min.size() && i < 8; ++i) {
      nrm[i] = m.norm.f_min[i];
      nrm[8 + i] = m.norm.f_max[i];
    }
    nrm[16] = m.norm.t_min;
    nrm[17] = m.norm.t_max;
    norm.insert(norm.end(), nrm, nrm + 18);
  }
  lann_model_set set{};
  set.n_models = int(ms.size());
  set.precision = engine::precision() == engine::Precision::Fp32 ? LANN_FP32 : LANN_FP64_EXACT;
  set.n_inputs = n_in.data();
  set.h1 = h1.data();
  set.h2 = h2.data();
  set.log_target = logt.data();
  set.param_offset = poff.data();
  set.params = params.data();
  set.total_params = std::int64_t(params.size());
  set.norm = norm.data();
  const std::int64_t n = a.integer("candidates", 1000000);
  const std::int64_t first = a.integer("first", 0);
  const std::uint64_t seed = a.u64("seed", 7);
  std::vector<std::int32_t> idx(std::size_t(std::max<std::int64_t>(n, 0)));
  std::vector<double> score(idx.size());
  lann_engine* e = nullptr;
  if (lann_engine_create(int(a.integer("device", 0)), &e) != LANN_OK)
    throw Error("no CUDA device: the LANN engine has no CPU fallback");
  const int st = lann_select_variants(e, &set, thd.data(), int(kind), int(a.integer("max-threads", 16)), seed, first,
                                      n, idx.data(), score.data());
  const double ms_dev = lann_last_train_ms(e);
  const std::string err = st ? lann_last_error(e) : "";
  lann_engine_destroy(e);
  if (st) throw ParamError("variant selection failed: " + err);
  std::vector<long long> hist(ms.size(), 0);
  for (auto v : idx) hist[std::size_t(v)] += 1;
  const fs::path out = a.get("out", "perfsage_out");
  fs::create_directories(out);
  const fs::path csv = out / "variants.csv";
  {
    std::ofstream os(csv, std::ios::binary);
    os << "model,variant,chosen\n";
    for (std::size_t v = 0; v < ms.size(); ++v) os << paths[v] << ',' << v << ',' << hist[v] << '\n';
  }
  std::cout << n << " candidate " << kernels::to_string(kind) << " shapes x " << ms.size() << " variant models: "
            << double(n) * double(ms.size()) / (ms_dev / 1e3) << " predictions/s (scoring kernel " << ms_dev
            << " ms)\n";
  for (std::size_t v = 0; v < ms.size(); ++v)
    std::cout << "  variant " << v << " (" << paths[v] << "): fastest for " << hist[v] << " candidates\n";
  record_run(out, a, seed, paths, {csv.string()});
  return 0;
}

// perfsage.cpp:424-472 `bench`: measure ONE kernel instance — here a B200 GPU-class variant
// (median of reps CUDA-event timings); --list names the variants.
int cmd_bench(const Args& a) {
  if (a.has("list")) {
    std::cout << "kernel  B200 variant\n";
    for (auto k : {kernels::KernelKind::MM, kernels::KernelKind::MV, kernels::KernelKind::MC, kernels::KernelKind::MP,
                   kernels::KernelKind::Blur})
      for (const auto& v : datagen::measured_variants(k))
        std::cout << std::left << std::setw(8) << kernels::to_string(k) << v << "\n";
    return 0;
  }
  const auto kind = kernels::kind_from_string(a.get("kernel", "mm"));
  const auto names = datagen::measured_variants(kind);
  const std::string variant = a.get("variant", names.front());
  const double m = a.real("m", 256), n = a.real("n", 256), k = a.real("k", 256), r = a.real("r", 3), st = a.real("s", 2);
  const double d = a.real("d", 1.0), d2 = a.real("d2", 1.0);
  double f[LANN_ROW] = {0};
  std::uint64_t c = 0;
  switch (kind) {  // GPU-class base features (features.cpp:10-21 without n_thd) and kernels.cpp:184-206
    case kernels::KernelKind::MM:
      f[0] = m, f[1] = n, f[2] = k, f[3] = d, f[4] = d2;
      c = std::uint64_t(m) * std::uint64_t(n) * std::uint64_t(k);
      break;
    case kernels::KernelKind::MV:
      f[0] = m, f[1] = n, f[2] = d;
      c = std::uint64_t(m) * std::uint64_t(n);
      break;
    case kernels::KernelKind::MC:
      f[0] = m, f[1] = n, f[2] = r, f[3] = d;
      c = std::uint64_t(m - r + 1) * std::uint64_t(n - r + 1) * std::uint64_t(r * r);
      break;
    case kernels::KernelKind::MP:
      f[0] = m, f[1] = n, f[2] = r, f[3] = st, f[4] = d;
      c = std::uint64_t((n + st - 1) / st) * std::uint64_t((m + st - 1) / st) * std::uint64_t(st * st);
      break;
    case kernels::KernelKind::Blur: {
      const auto sc = parse_schedule(a.get("schedule", "8,256,128,8"));
      f[0] = n, f[1] = sc.s1, f[2] = sc.s2, f[3] = sc.s3, f[4] = sc.s4;
      c = std::uint64_t(n) * std::uint64_t(n);
      break;
    }
  }
  lann_engine* e = nullptr;
  if (lann_engine_create(int(a.integer("device", 0)), &e) != LANN_OK)
    throw Error("no CUDA device: the LANN engine has no CPU fallback");
  double rt = 0.0;
  const int status = lann_measure(e, int(kind), variant.c_str(), 1, f, int(a.integer("warmups", 1)),
                                  int(a.integer("reps", 5)), a.u64("seed", 1), &rt, nullptr);
  const std::string err = status ? lann_last_error(e) : "";
  lann_engine_destroy(e);
  if (status) throw ParamError(err);
  std::cout << kernels::to_string(kind) << "/" << variant << " c=" << c << " median_s=" << rt << "\n";
  return 0;
}

// The reference's external-variant protocol (external.cpp:46-118) served by a B200 variant:
// every stdin line of GPU-class features -> one line with the median runtime in seconds.
int cmd_measure_variant(const Args& a) {
  const auto kind = kernels::kind_from_string(a.get("kernel", "mm"));
  const std::string variant = a.get("variant", "");
  const int warmups = int(a.integer("warmups", 1)), reps = int(a.integer("reps", 5));
  const std::uint64_t seed = a.u64("seed", 1);
  lann_engine* e = nullptr;
  if (lann_engine_create(int(a.integer("device", 0)), &e) != LANN_OK)
    throw Error("no CUDA device: the LANN engine has no CPU fallback");
  std::string line;
  int st = 0;
  while (std::getline(std::cin, line)) {
    std::stringstream ss(line);
    double f[LANN_ROW] = {0};
    int n = 0;
    for (double v; n < LANN_ROW && ss >> v;) f[n++] = v;
    if (n == 0) continue;
    double rt = 0.0;
    st = lann_measure(e, int(kind), variant.c_str(), 1, f, warmups, reps, seed, &rt, nullptr);
    if (st) break;
    std::printf("%.17g\n", rt);
    std::fflush(stdout);
  }
  const std::string err = st ? lann_last_error(e) : "";
  lann_engine_destroy(e);
  if (st) throw ParamError("measurement failed: " + err);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.command == "gen") return cmd_gen(a);
    if (a.command == "train") return cmd_train(a);
    if (a.command == "eval") return cmd_eval(a);
    if (a.command == "compare") return cmd_compare(a);
    if (a.command == "select") return cmd_select(a);
    if (a.command == "sweep") return cmd_sweep(a);
    if (a.command == "select-variants") return cmd_select_variants(a);
    if (a.command == "measure-variant") return cmd_measure_variant(a);
    if (a.command == "bench") return cmd_bench(a);
    throw ParamError("unknown subcommand '" + a.command + "'");
  } catch (const std::exception& ex) {
    std::cerr << "error: " << ex.what() << "\n";
    return 1;
  }
}
