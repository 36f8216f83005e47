// io.cpp — the on-disk formats and report writers of the perfsage:: API at population scale
// (SURVEY.md 8(f) rows 1-2), host-only C++:
//   * datagen::save_csv / load_csv        — the reference's dataset CSV (csv.cpp:43-102)
//   * models::save_model / load_model     — the "perfsage-model" v1 JSON (model_io.cpp:114-173)
//   * eval::aggregate / write_reports_csv / print_reports / print_aggregate (eval.cpp:110-197)
//   * models::feature_names / kind_from_feature_names (features.cpp:10-21, 59-72)
//   * datagen::build_synthetic            — the engine's synthetic generator as a Dataset
// The JSON reader/writer is a small self-contained one (the reference uses nlohmann json,
// which is not a dependency of this engine). Doubles are written with 17 significant digits
// ("%.17g"), which round-trips every finite double exactly, so save -> load is bit-exact and
// the files load unchanged in the reference (and the reference's files load here).
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <map>
#include <memory>
#include <ostream>
#include <sstream>
#include <csignal>
#include <mutex>

#include <sys/wait.h>
#include <unistd.h>

#include "../../include/lann_engine.h"
#include "../../include/perfsage_b200/perfsage.hpp"
#include "domain.hpp"
#include "json_lite.hpp"

namespace perfsage {

namespace kernels {
KernelKind kind_from_string(const std::string& name) {
  if (name == "mm") return KernelKind::MM;
  if (name == "mv") return KernelKind::MV;
  if (name == "mc") return KernelKind::MC;
  if (name == "mp") return KernelKind::MP;
  if (name == "blur") return KernelKind::Blur;
  throw ParamError("unknown kernel kind: '" + name + "'");
}
}  // namespace kernels

namespace models {
ModelFamily family_from_string(const std::string& name) {
  if (name == "nnc") return ModelFamily::NnC;
  if (name == "nn") return ModelFamily::Nn;
  if (name == "const") return ModelFamily::Const;
  if (name == "lrc") return ModelFamily::LrC;
  if (name == "nlrc") return ModelFamily::NlrC;
  throw ParamError("unknown model family: '" + name + "'");
}

std::vector<std::string> feature_names(kernels::KernelKind kind, bool with_n_thd) {
  using K = kernels::KernelKind;
  std::vector<std::string> names;
  switch (kind) {
    case K::MM: names = {"m", "n", "k", "d1", "d2"}; break;
    case K::MV: names = {"m", "n", "d"}; break;
    case K::MC: names = {"m", "n", "r", "d"}; break;
    case K::MP: names = {"m", "n", "r", "s", "d"}; break;
    case K::Blur: return {"n", "s1", "s2", "s3", "s4"};
  }
  if (with_n_thd) names.emplace_back("n_thd");
  return names;
}

std::pair<kernels::KernelKind, bool> kind_from_feature_names(const std::vector<std::string>& names) {
  using K = kernels::KernelKind;
  for (K kind : {K::MM, K::MV, K::MC, K::MP, K::Blur})
    for (bool thd : {true, false})
      if (names == feature_names(kind, thd)) return {kind, thd};
  std::string joined;
  for (const auto& n : names) joined += (joined.empty() ? "" : ",") + n;
  throw LoadError("unrecognized feature schema: [" + joined + "]");
}
}  // namespace models

using namespace lann::jsonl;

// ---- datagen: CSV + synthetic generator --------------------------------------------------------
namespace datagen {

void save_csv(const Dataset& ds, const std::string& path) {
  std::ofstream os(path, std::ios::binary);
  if (!os) throw LoadError("cannot open '" + path + "' for writing");
  os << "kernel,variant";
  for (const auto& n : ds.feature_names) os << ',' << n;
  os << ",c,runtime_s\n";
  const std::string kind = kernels::to_string(ds.kind);
  for (const auto& s : ds.samples) {
    os << kind << ',' << s.variant_id;
    for (double f : s.features) os << ',' << fmt17(f);
    os << ',' << s.c << ',' << fmt17(s.runtime_s) << '\n';
  }
  if (!os) throw LoadError("write to '" + path + "' failed");
}

Dataset load_csv(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw LoadError("cannot open '" + path + "'");
  std::string line;
  if (!std::getline(is, line)) throw LoadError(path + ": missing header row");
  if (!line.empty() && line.back() == '\r') line.pop_back();
  const auto header = split_fields(line);
  if (header.size() < 4 || header[0] != "kernel" || header[1] != "variant" ||
      header[header.size() - 2] != "c" || header.back() != "runtime_s")
    throw LoadError(path + ":1: header must be kernel,variant,<features...>,c,runtime_s");
  Dataset ds;
  ds.feature_names.assign(header.begin() + 2, header.end() - 2);
  ds.kind = models::kind_from_feature_names(ds.feature_names).first;
  const std::string kind = kernels::to_string(ds.kind);
  const std::size_t expected = header.size();
  std::size_t lineno = 1;
  while (std::getline(is, line)) {
    ++lineno;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    const std::string where = path + ":" + std::to_string(lineno);
    const auto f = split_fields(line);
    if (f.size() != expected)
      throw LoadError(where + ": expected " + std::to_string(expected) + " fields, got " +
                      std::to_string(f.size()));
    if (f[0] != kind) throw LoadError(where + ": kernel column does not match the schema kernel");
    Sample s;
    s.variant_id = f[1];
    for (std::size_t i = 2; i + 2 < expected; ++i) s.features.push_back(parse_number(f[i], where));
    const double c = parse_number(f[expected - 2], where);
    if (c < 0.0) throw LoadError(where + ": negative c");
    s.c = static_cast<std::uint64_t>(c);
    s.runtime_s = parse_number(f[expected - 1], where);
    if (!(s.runtime_s > 0.0)) throw LoadError(where + ": runtime_s must be > 0");
    ds.samples.push_back(std::move(s));
  }
  return ds;
}

int synthetic_world_count() { return int(lann::default_combos().size()); }

std::string combo_variant_id(int index) {
  const auto worlds = lann::default_combos();
  if (index < 0 || index >= int(worlds.size())) throw ParamError("synthetic world index out of range");
  const lann_world& w = worlds[std::size_t(index)];
  if (w.kind == LANN_BLUR) {
    const int b = index - 40;
    if (b >= 5) return "fft_standin" + std::to_string(b - 5);
    return w.blur_lattice ? "tiled_gpu" + std::to_string(b - 3) : "tiled@cpu" + std::to_string(b);
  }
  const int local = index % 10;  // (variant, hw) within the kernel kind
  const std::string storage = local < 5 ? "dense" : "sparse";
  if (w.hw_class == LANN_HW_CPU) return storage + "_threaded@cpu" + std::to_string(w.max_threads);
  return storage + "@gpu" + std::string(1, char('a' + (local % 5) - 3));
}

Dataset build_synthetic(int index, std::size_t count, std::uint64_t seed) {
  const auto worlds = lann::default_combos();
  if (index < 0 || index >= int(worlds.size())) throw ParamError("synthetic world index out of range");
  if (count == 0) throw ParamError("count must be >= 1");
  const lann_world& w = worlds[std::size_t(index)];
  std::vector<double> feats(count * LANN_ROW), rt(count);
  std::vector<std::uint64_t> c(count);
  int nf = 0;
  const int st = lann_build_dataset(&w, seed, int(count), feats.data(), c.data(), rt.data(), &nf);
  if (st == LANN_PARAM_ERROR) throw ParamError("invalid synthetic dataset request");
  if (st) throw Error("synthetic dataset generation failed");
  Dataset ds;
  ds.kind = static_cast<kernels::KernelKind>(w.kind);
  ds.feature_names = models::feature_names(ds.kind, w.hw_class == LANN_HW_CPU && w.kind != LANN_BLUR);
  ds.seed = seed;
  ds.host = "synthetic-world-" + std::to_string(index);
  const std::string vid = combo_variant_id(index);
  for (std::size_t i = 0; i < count; ++i) {
    Sample s;
    s.features.assign(feats.begin() + std::ptrdiff_t(i * LANN_ROW), feats.begin() + std::ptrdiff_t(i * LANN_ROW + nf));
    s.c = c[i];
    s.runtime_s = rt[i];
    s.variant_id = vid;
    ds.samples.push_back(std::move(s));
  }
  return ds;
}

std::vector<std::string> measured_variants(kernels::KernelKind kind) {
  std::vector<std::string> out;
  for (int i = 0; i < lann_measure_variant_count(int(kind)); ++i) out.emplace_back(lann_measure_variant_name(int(kind), i));
  return out;
}

std::vector<std::string> native_variants(kernels::KernelKind kind) {  // variants.cpp:225-247
  if (kind == kernels::KernelKind::Blur) return {"tiled"};
  std::vector<std::string> v = {"dense_single", "dense_threaded", "sparse_single"};
  if (kind == kernels::KernelKind::MM) v.emplace_back("tiled_threaded");
  return v;
}

Dataset build_mock(kernels::KernelKind kind, const std::string& variant_id, std::size_t count, std::uint64_t seed,
                   int max_threads, std::uint32_t dim_max, std::vector<std::uint32_t> blur_sides, bool gpu_lattice) {
  const auto names = native_variants(kind);
  if (std::find(names.begin(), names.end(), variant_id) == names.end())
    throw ParamError("no variant '" + variant_id + "' registered for kernel " + kernels::to_string(kind));
  const bool single = variant_id.size() > 7 && variant_id.compare(variant_id.size() - 7, 7, "_single") == 0;
  std::vector<double> feats(count * LANN_ROW), rt(count);
  std::vector<std::uint64_t> c(count);
  int nf = 0;
  const int st = lann_build_mock_dataset(int(kind), single ? 1 : 0, max_threads, dim_max, int(blur_sides.size()),
                                         blur_sides.data(), gpu_lattice ? 1 : 0, int(count), seed, feats.data(),
                                         c.data(), rt.data(), &nf);
  if (st) throw ParamError("invalid parameter space for the mock dataset");
  Dataset ds;
  ds.kind = kind;
  ds.feature_names = models::feature_names(kind, kind != kernels::KernelKind::Blur);
  ds.seed = seed;
  ds.host = "mock-timer";
  for (std::size_t i = 0; i < count; ++i) {
    Sample smp;
    smp.features.assign(feats.begin() + std::ptrdiff_t(i * LANN_ROW), feats.begin() + std::ptrdiff_t(i * LANN_ROW + nf));
    smp.c = c[i];
    smp.runtime_s = rt[i];
    smp.variant_id = variant_id;
    ds.samples.push_back(std::move(smp));
  }
  return ds;
}

Dataset build_measured(kernels::KernelKind kind, const std::string& variant, std::size_t count, std::uint64_t seed,
                       TimingPolicy policy, bool gpu_lattice, std::uint32_t blur_side) {
  if (count < 2) throw ParamError("build_dataset needs count >= 2");
  if (policy.reps < 1) throw ParamError("timing policy needs reps >= 1");
  if (policy.warmups < 0) throw ParamError("timing policy needs warmups >= 0");
  lann_engine* e = nullptr;
  if (lann_engine_create(0, &e) != LANN_OK) throw Error("no CUDA device: the LANN engine has no CPU fallback");
  std::vector<double> feats(count * LANN_ROW), rt(count);
  std::vector<std::uint64_t> c(count);
  int nf = 0;
  const int st = lann_build_measured_dataset(e, int(kind), variant.c_str(), gpu_lattice ? 1 : 0, int(blur_side),
                                             int(count), seed, policy.warmups, policy.reps, feats.data(), c.data(),
                                             rt.data(), &nf);
  const std::string msg = st ? lann_last_error(e) : "";
  lann_engine_destroy(e);
  if (st == LANN_PARAM_ERROR) throw ParamError(msg);
  if (st) throw Error("measurement failed: " + msg);
  Dataset ds;
  ds.kind = kind;
  ds.feature_names = models::feature_names(kind, false);
  ds.seed = seed;
  ds.host = "NVIDIA B200";
  for (std::size_t i = 0; i < count; ++i) {
    Sample smp;
    smp.features.assign(feats.begin() + std::ptrdiff_t(i * LANN_ROW), feats.begin() + std::ptrdiff_t(i * LANN_ROW + nf));
    smp.c = c[i];
    smp.runtime_s = rt[i];
    smp.variant_id = variant + "@b200";
    ds.samples.push_back(std::move(smp));
  }
  return ds;
}

double run_external_variant(const std::string& command, std::span<const double> features) {
  if (command.empty()) throw ExternalVariantError("empty launch command");
  static std::once_flag once;  // the child may exit without reading its stdin
  std::call_once(once, [] { std::signal(SIGPIPE, SIG_IGN); });
  int to_child[2], from_child[2];
  if (pipe(to_child) != 0) throw ExternalVariantError("pipe() failed");
  if (pipe(from_child) != 0) {
    close(to_child[0]);
    close(to_child[1]);
    throw ExternalVariantError("pipe() failed");
  }
  const pid_t pid = fork();
  if (pid < 0) {
    for (int fd : {to_child[0], to_child[1], from_child[0], from_child[1]}) close(fd);
    throw ExternalVariantError("fork() failed for '" + command + "'");
  }
  if (pid == 0) {
    if (dup2(to_child[0], STDIN_FILENO) < 0 || dup2(from_child[1], STDOUT_FILENO) < 0) _exit(127);
    for (int fd : {to_child[0], to_child[1], from_child[0], from_child[1]}) close(fd);
    execl("/bin/sh", "sh", "-c", command.c_str(), static_cast<char*>(nullptr));
    _exit(127);
  }
  close(to_child[0]);
  close(from_child[1]);
  std::string line;
  for (std::size_t i = 0; i < features.size(); ++i) line += (i ? " " : "") + fmt17(features[i]);
  line += '\n';
  for (std::size_t off = 0; off < line.size();) {
    const ssize_t w = write(to_child[1], line.data() + off, line.size() - off);
    if (w <= 0) break;
    off += std::size_t(w);
  }
  close(to_child[1]);
  std::string reply;
  char buf[256];
  for (ssize_t r; (r = read(from_child[0], buf, sizeof buf)) > 0;) reply.append(buf, std::size_t(r));
  close(from_child[0]);
  int status = 0;
  if (waitpid(pid, &status, 0) < 0) throw ExternalVariantError("waitpid() failed for '" + command + "'");
  if (!WIFEXITED(status) || WEXITSTATUS(status) != 0)
    throw ExternalVariantError("variant command '" + command + "' exited with status " +
                               std::to_string(WIFEXITED(status) ? WEXITSTATUS(status) : -1));
  std::string tok = reply.substr(0, reply.find('\n'));
  while (!tok.empty() && (tok.back() == '\r' || tok.back() == ' ')) tok.pop_back();
  const std::size_t b = tok.find_first_not_of(' ');
  if (b == std::string::npos) throw ExternalVariantError("variant command '" + command + "' replied with no runtime");
  tok = tok.substr(b);
  char* end = nullptr;
  const double v = std::strtod(tok.c_str(), &end);
  if (end == tok.c_str() || *end != '\0')
    throw ExternalVariantError("variant command '" + command + "' replied with non-numeric runtime '" + tok + "'");
  if (!(v > 0.0)) throw ExternalVariantError("variant command '" + command + "' replied with non-positive runtime");
  return v;
}

Dataset build_external(kernels::KernelKind kind, const std::string& command, const std::string& variant_id,
                       bool gpu_class, int max_threads, std::size_t count, std::uint64_t seed) {
  if (count < 2) throw ParamError("build_dataset needs count >= 2");
  if (max_threads < 1) throw ParamError("param space needs max_threads >= 1");
  const bool takes_thd = !gpu_class && kind != kernels::KernelKind::Blur;  // variants.hpp:29-31
  lann::SeqRng rng(lann::derive_seed(seed, 0));
  Dataset ds;
  ds.kind = kind;
  ds.feature_names = models::feature_names(kind, takes_thd);
  ds.seed = seed;
  ds.host = "external";
  for (std::size_t i = 0; i < count; ++i) {
    lann::Instance p = lann::sample_instance(int(kind), max_threads, gpu_class ? 1 : 0, rng);
    if (gpu_class) p.n_thd = 1;  // Threading::FixedSingle (datagen.cpp:195)
    double f[LANN_ROW] = {0};
    const int nf = lann::base_features(p, takes_thd, f);
    Sample smp;
    smp.features.assign(f, f + nf);
    smp.c = lann::complexity(p);
    smp.runtime_s = run_external_variant(command, smp.features);
    smp.variant_id = variant_id;
    ds.samples.push_back(std::move(smp));
  }
  return ds;
}

}  // namespace datagen

// ---- models: JSON ------------------------------------------------------------------------------
namespace models {

void save_model(const TrainedModel& m, const std::string& path) {
  const auto& c = m.config;
  std::ostringstream o;
  o << "{\n";
  o << "  \"format\": \"perfsage-model\",\n";
  o << "  \"version\": 1,\n";
  o << "  \"family\": " << quote(to_string(c.family)) << ",\n";
  o << "  \"kernel\": " << quote(kernels::to_string(m.kind)) << ",\n";
  o << "  \"schema\": " << jarr(m.schema) << ",\n";
  o << "  \"config\": {\n";
  o << "    \"family\": " << quote(to_string(c.family)) << ",\n";
  o << "    \"hidden_widths\": " << jarr(c.hidden_widths) << ",\n";
  o << "    \"learning_rate\": " << jnum(c.learning_rate) << ",\n";
  o << "    \"epochs\": " << c.epochs << ",\n";
  o << "    \"seed\": " << c.seed << ",\n";
  o << "    \"unconstrained\": " << (c.unconstrained ? "true" : "false") << ",\n";
  o << "    \"log_target\": " << (c.log_target ? "true" : "false") << ",\n";
  o << "    \"forest_trees\": " << c.forest_trees << ",\n";
  o << "    \"forest_depth\": " << c.forest_depth << "\n";
  o << "  },\n";
  o << "  \"norm_stats\": {\n";
  o << "    \"f_min\": " << jarr(m.norm.f_min) << ",\n";
  o << "    \"f_max\": " << jarr(m.norm.f_max) << ",\n";
  o << "    \"t_min\": " << jnum(m.norm.t_min) << ",\n";
  o << "    \"t_max\": " << jnum(m.norm.t_max) << ",\n";
  o << "    \"log_target\": " << (m.norm.log_target ? "true" : "false") << "\n";
  o << "  },\n";
  o << "  \"payload\": {\n";
  if (const auto* net = std::get_if<Mlp>(&m.payload)) {
    o << "    \"layers\": [\n";
    for (std::size_t l = 0; l < net->layers.size(); ++l) {
      const auto& L = net->layers[l];
      o << "      {\"rows\": " << L.out << ", \"cols\": " << L.in << ", \"weights\": " << jarr(L.w)
        << ", \"biases\": " << jarr(L.b) << "}" << (l + 1 < net->layers.size() ? "," : "") << "\n";
    }
    o << "    ]\n  },\n";
    o << "  \"metrics\": {\n";
    o << "    \"param_count\": " << net->param_count() << ",\n";
    if (!m.loss_trace.empty()) o << "    \"final_loss\": " << jnum(m.loss_trace.back()) << ",\n";
    o << "    \"loss_trace\": " << jarr(m.loss_trace) << "\n";
    o << "  }\n}\n";
  } else {
    if (const auto* lin = std::get_if<LinearModel>(&m.payload)) {
      o << "    \"linear\": {\"weights\": " << jarr(lin->weights) << ", \"intercept\": " << jnum(lin->intercept)
        << "}\n";
    } else {
      const auto& forest = std::get<Forest>(m.payload);
      o << "    \"forest\": [\n";
      for (std::size_t t = 0; t < forest.trees.size(); ++t) {
        o << "      [";
        const auto& nodes = forest.trees[t].nodes;
        for (std::size_t v = 0; v < nodes.size(); ++v)
          o << (v ? ", " : "") << "{\"feature\": " << nodes[v].feature << ", \"threshold\": "
            << jnum(nodes[v].threshold) << ", \"left\": " << nodes[v].left << ", \"right\": " << nodes[v].right
            << ", \"value\": " << jnum(nodes[v].value) << "}";
        o << "]" << (t + 1 < forest.trees.size() ? "," : "") << "\n";
      }
      o << "    ]\n";
    }
    o << "  },\n  \"metrics\": null\n}\n";  // model_io.cpp:140-146: metrics only for NN payloads
  }
  std::ofstream os(path, std::ios::binary);
  if (!os) throw LoadError("cannot open '" + path + "' for writing");
  os << o.str();
  if (!os) throw LoadError("write to '" + path + "' failed");
}

TrainedModel load_model(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw LoadError("cannot open '" + path + "'");
  std::stringstream buf;
  buf << is.rdbuf();
  const std::string text = buf.str();
  Json j;
  try {
    j = Parser(text).document();
  } catch (const LoadError& e) {
    throw LoadError("'" + path + "' is not a valid model file: " + e.what());
  }
  try {
    if (j.at("format").str() != "perfsage-model") throw LoadError("'" + path + "' is not a perfsage model file");
    if (j.at("version").i32() != 1)
      throw LoadError("'" + path + "' has unsupported model version " + j.at("version").text);
    TrainedModel m;
    const Json& c = j.at("config");
    m.config.family = family_from_string(c.at("family").str());
    m.config.hidden_widths.clear();
    for (const auto& h : c.at("hidden_widths").items) m.config.hidden_widths.push_back(h.i32());
    m.config.learning_rate = c.at("learning_rate").num();
    m.config.epochs = c.at("epochs").i32();
    m.config.seed = c.at("seed").u64();
    m.config.unconstrained = c.at("unconstrained").boolean();
    m.config.log_target = c.at("log_target").boolean();
    m.config.forest_trees = c.at("forest_trees").i32();
    m.config.forest_depth = c.at("forest_depth").i32();
    m.kind = kernels::kind_from_string(j.at("kernel").str());
    for (const auto& s : j.at("schema").items) m.schema.push_back(s.str());
    const Json& n = j.at("norm_stats");
    m.norm.f_min = n.at("f_min").doubles();
    m.norm.f_max = n.at("f_max").doubles();
    m.norm.t_min = n.at("t_min").num();
    m.norm.t_max = n.at("t_max").num();
    m.norm.log_target = n.at("log_target").boolean();
    const Json& p = j.at("payload");
    if (p.find("layers")) {
      Mlp net;
      for (const auto& lj : p.at("layers").items) {
        DenseLayer L;
        L.out = lj.at("rows").i32();
        L.in = lj.at("cols").i32();
        L.w = lj.at("weights").doubles();
        L.b = lj.at("biases").doubles();
        if (L.w.size() != std::size_t(L.in) * std::size_t(L.out) || L.b.size() != std::size_t(L.out))
          throw LoadError("layer shape does not match its weight payload");
        net.layers.push_back(std::move(L));
      }
      if (net.layers.empty()) throw LoadError("model has no layers");
      m.payload = std::move(net);
    } else if (p.find("linear")) {
      LinearModel lin;
      lin.weights = p.at("linear").at("weights").doubles();
      lin.intercept = p.at("linear").at("intercept").num();
      m.payload = std::move(lin);
    } else if (p.find("forest")) {
      Forest forest;
      for (const auto& tj : p.at("forest").items) {
        Tree t;
        for (const auto& nj : tj.items)
          t.nodes.push_back({nj.at("feature").i32(), nj.at("threshold").num(), nj.at("left").i32(),
                             nj.at("right").i32(), nj.at("value").num()});
        if (t.nodes.empty()) throw LoadError("forest tree has no nodes");
        forest.trees.push_back(std::move(t));
      }
      if (forest.trees.empty()) throw LoadError("forest has no trees");
      m.payload = std::move(forest);
    } else {
      throw LoadError("model payload missing (expected layers, linear, or forest)");
    }
    if (const Json* mt = j.find("metrics"))
      if (const Json* lt = mt->find("loss_trace")) m.loss_trace = lt->doubles();
    return m;
  } catch (const ParamError& e) {
    throw LoadError("'" + path + "' has invalid model fields: " + e.what());
  }
}

}  // namespace models

// ---- eval: reports -------------------------------------------------------------------------------
namespace eval {

std::vector<AggregateRow> aggregate(const std::vector<EvalReport>& reports, GroupBy group_by) {
  if (reports.empty()) throw DomainError("nothing to aggregate");
  auto key_of = [&](const EvalReport& r) -> const std::string& {
    switch (group_by) {
      case GroupBy::Variant: return r.variant;
      case GroupBy::ModelFamily: return r.model_family;
      default: return r.kernel;
    }
  };
  std::map<std::string, AggregateRow> groups;
  AggregateRow overall;
  overall.group = "overall";
  for (const auto& r : reports) {
    for (AggregateRow* row : {&groups[key_of(r)], &overall}) {
      row->mape_full += r.mape_full;
      row->mape_thresholded += r.mape_thresholded;
      row->rho += r.rho;
      row->reports += 1;
    }
    groups[key_of(r)].group = key_of(r);
  }
  auto finish = [](AggregateRow row) {
    const double n = double(row.reports);
    row.mape_full /= n;
    row.mape_thresholded /= n;
    row.rho /= n;
    return row;
  };
  std::vector<AggregateRow> out;
  for (auto& [key, row] : groups) out.push_back(finish(row));
  out.push_back(finish(overall));
  return out;
}

void write_reports_csv(std::ostream& os, const std::vector<EvalReport>& reports) {
  os << "kernel,variant,model_family,mape_full,mape_thresholded,rho,n_total,n_kept\n";
  const auto old = os.precision(17);
  for (const auto& r : reports)
    os << r.kernel << ',' << r.variant << ',' << r.model_family << ',' << r.mape_full << ','
       << r.mape_thresholded << ',' << r.rho << ',' << r.n_total << ',' << r.n_kept << '\n';
  os.precision(old);
}

void print_reports(std::ostream& os, const std::vector<EvalReport>& reports) {
  os << std::left << std::setw(8) << "kernel" << std::setw(16) << "variant" << std::setw(8) << "model"
     << std::right << std::setw(12) << "MAPE%" << std::setw(12) << "MAPE30%" << std::setw(9) << "rho"
     << std::setw(8) << "kept" << '\n';
  for (const auto& r : reports) {
    os << std::left << std::setw(8) << r.kernel << std::setw(16) << r.variant << std::setw(8)
       << r.model_family << std::right << std::fixed << std::setprecision(2) << std::setw(12) << r.mape_full
       << std::setw(12) << r.mape_thresholded << std::setprecision(3) << std::setw(9) << r.rho
       << std::setw(7) << r.n_kept << '/' << r.n_total << '\n';
    os.unsetf(std::ios::fixed);
  }
}

void print_aggregate(std::ostream& os, const std::vector<AggregateRow>& rows) {
  os << std::left << std::setw(20) << "group" << std::right << std::setw(12) << "MAPE%" << std::setw(12)
     << "MAPE30%" << std::setw(9) << "rho" << std::setw(9) << "reports" << '\n';
  for (const auto& row : rows) {
    os << std::left << std::setw(20) << row.group << std::right << std::fixed << std::setprecision(2)
       << std::setw(12) << row.mape_full << std::setw(12) << row.mape_thresholded << std::setprecision(3)
       << std::setw(9) << row.rho << std::setw(9) << row.reports << '\n';
    os.unsetf(std::ios::fixed);
  }
}

}  // namespace eval

// ---- selector: selection report ----------------------------------------------------------------
namespace selector {

SelectionReport evaluate_selection(const ScheduleCandidate& chosen, const MeasuredCandidates& measured,
                                   const ScheduleCandidate& default_schedule,
                                   std::optional<double> default_runtime_s, double predicted_s) {
  if (measured.empty()) throw ParamError("no measured candidates");
  SelectionReport rep;
  rep.chosen = chosen;
  rep.predicted_s = predicted_s;
  rep.default_schedule = default_schedule;
  double sum = 0.0;
  const std::pair<ScheduleCandidate, double>* at_chosen = nullptr;
  const std::pair<ScheduleCandidate, double>* best = nullptr;
  const std::pair<ScheduleCandidate, double>* at_default = nullptr;
  for (const auto& row : measured) {
    if (!(row.second > 0.0)) throw DomainError("measured runtimes must be > 0");
    sum += row.second;
    if (row.first == chosen) at_chosen = &row;
    if (row.first == default_schedule) at_default = &row;
    if (!best || row.second < best->second || (row.second == best->second && row.first < best->first))
      best = &row;
  }
  if (!at_chosen) throw ParamError("chosen schedule " + chosen.to_string() + " has no measured runtime");
  if (!default_runtime_s && !at_default)
    throw ParamError("default schedule " + default_schedule.to_string() + " has no measured runtime");
  rep.measured_s = at_chosen->second;
  rep.true_best = best->first;
  rep.true_best_s = best->second;
  rep.default_s = default_runtime_s ? *default_runtime_s : at_default->second;
  if (!(rep.default_s > 0.0)) throw DomainError("default runtime must be > 0");
  rep.regret = rep.measured_s / rep.true_best_s;
  rep.speedup_vs_default = rep.default_s / rep.measured_s;
  rep.speedup_vs_random_mean = (sum / double(measured.size())) / rep.measured_s;
  return rep;
}

namespace {
std::string sched_json(const ScheduleCandidate& c, const char* indent) {
  return std::string("{\n") + indent + "  \"s1\": " + std::to_string(c.s1) + ",\n" + indent + "  \"s2\": " +
         std::to_string(c.s2) + ",\n" + indent + "  \"s3\": " + std::to_string(c.s3) + ",\n" + indent +
         "  \"s4\": " + std::to_string(c.s4) + "\n" + indent + "}";
}
}  // namespace

std::string SelectionReport::to_json() const {
  std::ostringstream o;
  o << "{\n  \"chosen\": " << sched_json(chosen, "  ") << ",\n  \"predicted_s\": " << jnum(predicted_s)
    << ",\n  \"measured_s\": " << jnum(measured_s) << ",\n  \"true_best\": " << sched_json(true_best, "  ")
    << ",\n  \"true_best_s\": " << jnum(true_best_s) << ",\n  \"default_schedule\": "
    << sched_json(default_schedule, "  ") << ",\n  \"default_s\": " << jnum(default_s)
    << ",\n  \"regret\": " << jnum(regret) << ",\n  \"speedup_vs_default\": " << jnum(speedup_vs_default)
    << ",\n  \"speedup_vs_random_mean\": " << jnum(speedup_vs_random_mean) << "\n}";
  return o.str();
}

std::string SelectionReport::summary() const {
  std::ostringstream os;
  os << "chosen schedule   " << chosen.to_string() << "  measured " << measured_s << " s (predicted "
     << predicted_s << " s)\n"
     << "true best         " << true_best.to_string() << "  " << true_best_s << " s  (regret " << regret
     << "x)\n"
     << "default schedule  " << default_schedule.to_string() << "  " << default_s
     << " s  (speedup vs default " << speedup_vs_default << "x)\n"
     << "speedup vs mean candidate: " << speedup_vs_random_mean << "x";
  return os.str();
}

}  // namespace selector
}  // namespace perfsage
