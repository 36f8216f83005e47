// perfsage_b200/perfsage.hpp — drop-in C++ API for the reference's LANN hot path.
//
// Same namespaces, type names, fields and function signatures as the reference
// perfsage core (paths relative to /root/reference/proj/core/include/perfsage/) for
// the data-parallel path the engine replaces:
//   errors.hpp      Error, ParamError, SchemaError, DomainError, TrainingError, BuildAbortError
//   kernels.hpp     KernelKind, ScheduleCandidate, ScheduleSpace (cpu_default / gpu_style / enumerate_all)
//   datagen.hpp     Sample, Dataset, split
//   models.hpp      ModelFamily, ModelConfig, default_config, param_count_for, NormStats,
//                   TrainedModel, train_nn, train_model (NN families), predict, predict_dataset
//   mlp.hpp         DenseLayer, Mlp
//   eval.hpp        mape, mape_thresholded, spearman, make_report, speedup
//   selector.hpp    enumerate_candidates, select(ScheduleScorer...), select(TrainedModel, n, cands)
//   features.hpp    feature_names, kind_from_feature_names
//   csv.cpp         datagen::save_csv / load_csv (same columns, %.17g doubles)
//   model_io.hpp    models::save_model / load_model (same "perfsage-model" v1 JSON document)
//   eval.hpp        aggregate, write_reports_csv, print_reports, print_aggregate
// plus the batched overloads the engine exists for: models::train_population and
// models::predict_population, and datagen::build_synthetic (a dataset from one of the
// engine's synthetic runtime worlds, the generator the population runs use). Every compute call runs on the GPU through the C ABI
// (include/lann_engine.h); there is no CPU fallback. Link: -lperfsage_b200.
#pragma once

#include <cstdint>
#include <functional>
#include <iosfwd>
#include <optional>
#include <random>
#include <algorithm>
#include <utility>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <variant>
#include <vector>

namespace perfsage {

// ---- errors.hpp:9-69 ------------------------------------------------------------------------
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};
class ParamError : public Error { public: using Error::Error; };
class DomainError : public Error { public: using Error::Error; };
class SchemaError : public Error { public: using Error::Error; };
class TrainingError : public Error {
 public:
  TrainingError(const std::string& msg, int epoch) : Error(msg), epoch_(epoch) {}
  int epoch() const { return epoch_; }

 private:
  int epoch_;
};
class LoadError : public Error { public: using Error::Error; };  // errors.hpp:49-52
class FitError : public Error { public: using Error::Error; };   // errors.hpp:42-46
class ExternalVariantError : public Error { public: using Error::Error; };  // errors.hpp
class BuildAbortError : public Error {
 public:
  BuildAbortError(const std::string& msg, std::size_t completed) : Error(msg), completed_(completed) {}
  std::size_t completed() const { return completed_; }

 private:
  std::size_t completed_;
};

namespace engine {
enum class Precision { Fp64Exact, Fp32 };
// Arithmetic mode of the perfsage:: calls on this thread (default: Fp64Exact, bit-identical
// to the reference). Each host thread owns one engine (CUDA stream) on `device`.
void set_precision(Precision p);
Precision precision();
void set_device(int device);
}  // namespace engine

// ---- kernels.hpp -------------------------------------------------------------------------------
// ---- rng.hpp: the reference's seeded streams (mt19937_64 with hand-rolled draws) ---------------
inline std::uint64_t splitmix64(std::uint64_t& state) {
  std::uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline std::uint64_t derive_seed(std::uint64_t root, std::uint64_t stream) {
  std::uint64_t s = root ^ (0x9e3779b97f4a7c15ULL * (stream + 1));
  splitmix64(s);
  return splitmix64(s);
}
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : engine_(seed) {}
  std::uint64_t next() { return engine_(); }
  std::uint64_t bounded(std::uint64_t n) {  // unbiased: reject below 2^64 mod n
    const std::uint64_t threshold = (0 - n) % n;
    for (;;)
      if (const std::uint64_t r = engine_(); r >= threshold) return r % n;
  }
  std::int64_t uniform_int(std::int64_t lo, std::int64_t hi) {
    return lo + static_cast<std::int64_t>(bounded(static_cast<std::uint64_t>(hi - lo) + 1));
  }
  double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  template <typename T>
  void partial_shuffle(std::vector<T>& v, std::size_t k) {
    k = std::min(k, v.size());
    for (std::size_t i = 0; i < k; ++i) std::swap(v[i], v[i + static_cast<std::size_t>(bounded(v.size() - i))]);
  }

 private:
  std::mt19937_64 engine_;
};

namespace kernels {
enum class KernelKind { MM, MV, MC, MP, Blur };
std::string to_string(KernelKind kind);
KernelKind kind_from_string(const std::string& s);  // kernels.cpp (ParamError on unknown)

struct ScheduleCandidate {
  std::uint32_t s1 = 8, s2 = 256, s3 = 128, s4 = 8;
  auto tie() const { return std::tie(s1, s2, s3, s4); }
  bool operator==(const ScheduleCandidate& o) const { return tie() == o.tie(); }
  bool operator<(const ScheduleCandidate& o) const { return tie() < o.tie(); }
  bool is_pow2() const;
  std::string to_string() const;
};

struct ScheduleSpace {
  std::uint32_t s1_min = 2, s1_max = 1024, s2_min = 2, s2_max = 1024;
  std::uint32_t s3_min = 2, s3_max = 1024, s4_min = 2, s4_max = 1024;
  bool chained = true;
  static ScheduleSpace cpu_default();
  static ScheduleSpace gpu_style();
  bool contains(const ScheduleCandidate& c) const;
  std::uint64_t size() const;
  std::vector<ScheduleCandidate> enumerate_all() const;
};

/// kernels.hpp:58-98 — one kernel instance's parameters (host-side value type).
struct InstanceParams {
  KernelKind kind = KernelKind::MM;
  std::uint32_t m = 0, n = 0, k = 0, r = 0, s = 0;
  double d1 = 1.0, d2 = 1.0, d = 1.0;
  int n_thd = 1;
  std::optional<ScheduleCandidate> schedule;
  static InstanceParams mm(std::uint32_t m, std::uint32_t n, std::uint32_t k, double d1 = 1.0, double d2 = 1.0,
                           int n_thd = 1);
  static InstanceParams mv(std::uint32_t m, std::uint32_t n, double d = 1.0, int n_thd = 1);
  static InstanceParams mc(std::uint32_t m, std::uint32_t n, std::uint32_t r, double d = 1.0, int n_thd = 1);
  static InstanceParams mp(std::uint32_t m, std::uint32_t n, std::uint32_t r, std::uint32_t s, double d = 1.0,
                           int n_thd = 1);
  static InstanceParams blur(std::uint32_t n, const ScheduleCandidate& sched);
  void validate() const;  // ParamError on an out-of-domain field (kernels.cpp:149-182)
};
/// kernels.cpp:184-206: mm m*n*k, mv m*n, mc (m-r+1)(n-r+1)r^2, mp ceil(n/s)ceil(m/s)s^2, blur n^2
std::uint64_t complexity(const InstanceParams& params);

/// variants.hpp:12-32 — the descriptor of a benchmarked variant (the engine measures none of the
/// reference's CPU kernels; datagen::build_dataset needs a probe or an external variant).
enum class Storage { Dense, Sparse };
enum class Threading { Threaded, FixedSingle };
enum class ImplKind { Naive, Tiled, External };
enum class HardwareClass { Cpu, Gpu };
struct VariantDescriptor {
  std::string variant_id;
  KernelKind kind = KernelKind::MM;
  Storage storage = Storage::Dense;
  Threading threading = Threading::Threaded;
  ImplKind impl = ImplKind::Naive;
  HardwareClass hw_class = HardwareClass::Cpu;
  std::string hardware_label;
  std::string launch_command;  // external variants only
  bool is_external() const { return impl == ImplKind::External; }
  bool takes_n_thd() const { return hw_class == HardwareClass::Cpu && kind != KernelKind::Blur; }
};
}  // namespace kernels

// ---- datagen.hpp:72-116 -------------------------------------------------------------------------
namespace datagen {
struct Sample {
  std::vector<double> features;
  std::uint64_t c = 0;
  double runtime_s = 0.0;
  std::string variant_id;
  bool operator==(const Sample&) const = default;
};

struct Dataset {
  kernels::KernelKind kind = kernels::KernelKind::MM;
  std::vector<std::string> feature_names;
  std::vector<Sample> samples;
  std::uint64_t seed = 0;
  std::string host;
  std::size_t size() const { return samples.size(); }
  std::vector<double> runtimes() const;
};

/// datagen.hpp:44-51 / datagen.cpp:118-160: untimed warm-ups, then the median of `reps` runs.
struct TimingPolicy {
  int warmups = 1;
  int reps = 5;
};

/// datagen.hpp:15-40 / datagen.cpp:18-110: the sampling space and its draws (host-side).
struct ParamSpace {
  kernels::KernelKind kind = kernels::KernelKind::MM;
  std::uint32_t dim_min = 1, dim_max = 1024;
  int max_threads = 1;
  std::vector<std::uint32_t> mc_filter_dims = {3, 5, 7};
  std::vector<std::uint32_t> mp_aux_dims = {2, 3, 4, 5};
  std::vector<std::uint32_t> mp_pool_dims = {1, 2};
  bool density_ladder_includes_one = true;
  std::vector<std::uint32_t> blur_sides = {1024, 2048, 4096, 8192, 16384, 32768};
  kernels::ScheduleSpace schedules = kernels::ScheduleSpace::cpu_default();
  static ParamSpace defaults(kernels::KernelKind kind, int max_threads);
  void validate() const;
};
std::vector<double> density_ladder(std::uint64_t cells, bool include_one);
kernels::InstanceParams sample_params(const ParamSpace& space, Rng& rng);
kernels::InstanceParams sample_params(const ParamSpace& space, std::uint64_t seed);
double median_of(std::vector<double> values);  // datagen.cpp:118-124 (DomainError when empty)

/// datagen.hpp:94-116: build_dataset with a runtime probe. Without a probe the reference times
/// its CPU kernels, which this engine does not: external variants run the black-box protocol,
/// anything else throws ParamError (use build_measured for B200 variants). Probe or external
/// failures abort with BuildAbortError carrying the completed sample count.
using RuntimeProbe = std::function<double(const kernels::InstanceParams&)>;
struct BuildOptions {
  TimingPolicy policy;
  RuntimeProbe probe;
};
Dataset build_dataset(const kernels::VariantDescriptor& variant, const ParamSpace& space, std::size_t count,
                      std::uint64_t seed, const BuildOptions& options = {});

/// Disjoint, exhaustive, seeded-shuffle partition (datagen.cpp:225-248).
std::pair<Dataset, Dataset> split(const Dataset& dataset, double train_fraction, std::uint64_t seed);

/// csv.cpp:43-102: header kernel,variant,<features...>,c,runtime_s; doubles as %.17g, LF
/// line endings; LoadError on a bad header, field count, number, negative c or runtime <= 0.
void save_csv(const Dataset& dataset, const std::string& path);
Dataset load_csv(const std::string& path);

/// The engine's synthetic dataset generator (lann_build_dataset): `count` samples of
/// datagen::sample_params draws from Rng(derive_seed(seed, 0)) probed by the closed-form
/// runtime world `world_index` of the 48 default combinations (0 = the acceptance world,
/// acceptance_main.cpp:271-279). variant_id names the combination (combo_variant_id).
Dataset build_synthetic(int world_index, std::size_t count, std::uint64_t seed);

/// Real measurement on the B200 (lann_build_measured_dataset): `count` sample_params draws of
/// the GPU-class space (no n_thd), each timed as B200 kernel variant `variant` (CUDA events,
/// TimingPolicy median). Variants per kind: measured_variants(kind). variant_id = variant@b200.
Dataset build_measured(kernels::KernelKind kind, const std::string& variant, std::size_t count,
                       std::uint64_t seed, TimingPolicy policy = {}, bool gpu_lattice = true,
                       std::uint32_t blur_side = 1024);
std::vector<std::string> measured_variants(kernels::KernelKind kind);
/// The reference CLI's `gen --mock-timer` dataset for a builtin native variant
/// (variants.cpp:225-247: dense_single, dense_threaded, sparse_single per kind, tiled_threaded
/// for mm, tiled for blur): ParamSpace::defaults(kind, max_threads) with dims U{1..dim_max},
/// blur sides / lattice, the mock probe (perfsage.cpp:71-84). ParamError on an unknown variant.
Dataset build_mock(kernels::KernelKind kind, const std::string& variant_id, std::size_t count, std::uint64_t seed,
                   int max_threads, std::uint32_t dim_max = 1024, std::vector<std::uint32_t> blur_sides = {1024},
                   bool gpu_lattice = false);
std::vector<std::string> native_variants(kernels::KernelKind kind);
/// external.cpp:46-118: run `command` via /bin/sh, write the features as one line of %.17g
/// values to its stdin, read one positive decimal runtime (seconds) from the first stdout line.
/// Throws ExternalVariantError on spawn failure, non-zero exit or a malformed reply.
double run_external_variant(const std::string& command, std::span<const double> features);
/// datagen::build_dataset with an external variant as the probe (perfsage.cpp cmd_gen
/// --external-cmd): sample_params draws (CPU class: n_thd in 1..max_threads, pinned to 1 for a
/// GPU-class variant), features without c sent to the command.
Dataset build_external(kernels::KernelKind kind, const std::string& command, const std::string& variant_id,
                       bool gpu_class, int max_threads, std::size_t count, std::uint64_t seed);
int synthetic_world_count();
std::string combo_variant_id(int world_index);
}  // namespace datagen

// ---- mlp.hpp / models.hpp ----------------------------------------------------------------------
namespace models {
struct DenseLayer {
  int in = 0;
  int out = 0;
  std::vector<double> w;
  std::vector<double> b;
};

struct Mlp {
  std::vector<DenseLayer> layers;
  /// mlp.cpp:9-25: Glorot-uniform weights U(-sqrt(6/(in+out)), +sqrt(6/(in+out))) drawn in layer /
  /// row order from `rng`, biases 0 (host-side, bit-identical to the reference)
  static Mlp init(const std::vector<int>& dims, Rng& rng);
  /// mlp.hpp:27 / mlp.cpp:54-62 on the GPU (lann_mlp_forward): the network output for one
  /// feature vector, bit-identical to the reference's; SchemaError on a length mismatch
  double forward(std::span<const double> x) const;
  int input_dim() const { return layers.empty() ? 0 : layers.front().in; }
  int param_count() const;
};

/// mlp.hpp:34-35 / mlp.cpp:64-73 on the GPU (lann_mse_loss): mean squared error over rows of X
double mse_loss(const Mlp& net, const std::vector<std::vector<double>>& X, std::span<const double> y);

/// mlp.hpp:37-44 / mlp.cpp:75-122 on the GPU (lann_mse_gradient): the analytic gradient of
/// mse_loss, flattened in layer order (weights then biases per layer), and the loss
struct LossGrad {
  double loss = 0.0;
  std::vector<double> grad;
};
LossGrad mse_gradient(const Mlp& net, const std::vector<std::vector<double>>& X, std::span<const double> y);

/// mlp.hpp:50-60 / mlp.cpp:142-154: Adam over a flat parameter vector; update() runs on the
/// GPU (lann_adam_update) with the bias corrections from the host libm, as the reference
struct AdamState {
  std::vector<double> m;
  std::vector<double> v;
  int step = 0;
  double beta1 = 0.9;
  double beta2 = 0.999;
  double epsilon = 1e-8;

  explicit AdamState(std::size_t n) : m(n, 0.0), v(n, 0.0) {}
  void update(std::span<double> params, std::span<const double> grad, double lr);
};

void unflatten_params(Mlp& net, std::span<const double> flat);  // mlp.cpp:132-140
/// mlp.hpp:64-66 / mlp.cpp:156-175 on the GPU (one-model lann_train): `epochs` full-batch Adam
/// epochs over normalised rows X (one vector per sample) and targets y; net's weights updated in
/// place; returns the pre-update loss trace. TrainingError(epoch) on a non-finite loss.
std::vector<double> train_full_batch(Mlp& net, const std::vector<std::vector<double>>& X,
                                     std::span<const double> y, double lr, int epochs);

enum class ModelFamily { NnC, Nn, Const, LrC, NlrC };
std::string to_string(ModelFamily family);
ModelFamily family_from_string(const std::string& s);  // models.cpp (ParamError on unknown)

/// features.cpp:10-72
std::vector<std::string> feature_names(kernels::KernelKind kind, bool with_n_thd);
std::vector<double> featurize(const kernels::InstanceParams& params, bool augmented, bool with_n_thd);
std::vector<double> featurize(const kernels::InstanceParams& params, bool augmented);  // with n_thd
std::vector<std::string> model_schema(const std::vector<std::string>& base_names, ModelFamily family);
std::pair<kernels::KernelKind, bool> kind_from_feature_names(const std::vector<std::string>& names);
bool family_augmented(ModelFamily family);

struct ModelConfig {
  ModelFamily family = ModelFamily::NnC;
  std::vector<int> hidden_widths = {8};
  double learning_rate = 1e-3;
  int epochs = 5000;
  std::uint64_t seed = 0;
  bool unconstrained = false;
  bool log_target = false;
  int forest_trees = 100;
  int forest_depth = 12;
  void validate(int input_dim) const;
};

constexpr int kLightweightParamBudget = 75;
ModelConfig default_config(kernels::KernelKind kind, ModelFamily family, bool unconstrained = false);
int param_count_for(int input_dim, const std::vector<int>& hidden_widths);

struct NormStats {
  std::vector<double> f_min, f_max;
  double t_min = 0.0, t_max = 1.0;
  bool log_target = false;
  std::vector<double> normalize(std::span<const double> features) const;
  double normalize_target(double t) const;
  double denormalize_target(double t_scaled) const;
  static NormStats fit(const std::vector<std::vector<double>>& X, std::span<const double> y,
                       bool log_target = false);
};

/// models.hpp:56-60 — the const / lrc payload: runtime = intercept + sum_j weights[j] * x[j]
struct LinearModel {
  std::vector<double> weights;
  double intercept = 0.0;
};
/// forest.hpp:10-30 — the nlrc payload (nodes in depth-first preorder, leaves have feature -1).
/// Prediction runs on the GPU through models::predict / predict_dataset.
struct TreeNode {
  int feature = -1;
  double threshold = 0.0;
  int left = -1;
  int right = -1;
  double value = 0.0;
  bool is_leaf() const { return feature < 0; }
};
struct Tree {
  std::vector<TreeNode> nodes;
};
struct Forest {
  std::vector<Tree> trees;
};

struct TrainedModel {
  ModelConfig config;
  kernels::KernelKind kind = kernels::KernelKind::MM;
  std::vector<std::string> schema;
  NormStats norm;  // NN families only (the baselines fit raw features)
  std::variant<Mlp, LinearModel, Forest> payload;
  std::vector<double> loss_trace;
};

std::vector<double> model_features(const datagen::Sample& sample, ModelFamily family);
std::vector<double> model_features(const kernels::InstanceParams& params, ModelFamily family, bool with_n_thd = true);

/// models.cpp:279-303 — trained on the GPU (one-model population).
TrainedModel train_nn(const datagen::Dataset& train, const ModelConfig& config);
/// models.cpp:335-344 — every family on the GPU: nnc / nn (train_nn), const / lrc (least squares,
/// bit-identical), nlrc (random forest).
TrainedModel train_model(const datagen::Dataset& train, const ModelConfig& config);
TrainedModel train_const(const datagen::Dataset& train, const ModelConfig& config);  // models.cpp:305-312
TrainedModel train_lrc(const datagen::Dataset& train, const ModelConfig& config);    // models.cpp:314-320
TrainedModel train_nlrc(const datagen::Dataset& train, const ModelConfig& config);   // models.cpp:322-333
/// Batched overload: every (dataset, config) pair trained in one engine call per family group
/// (NN families: one trainer launch set; const + lrc: one least-squares launch; nlrc: one forest
/// launch of models x trees CTAs).
std::vector<TrainedModel> train_population(const std::vector<const datagen::Dataset*>& train,
                                           const std::vector<ModelConfig>& configs);

/// models.cpp:346-363 / 372-378 — evaluated on the GPU.
double predict(const TrainedModel& model, std::span<const double> features);
std::vector<double> predict_dataset(const TrainedModel& model, const datagen::Dataset& data);
/// Batched overload: predictions of many (model, dataset) pairs in one call.
std::vector<std::vector<double>> predict_population(const std::vector<const TrainedModel*>& models,
                                                    const std::vector<const datagen::Dataset*>& data);
int param_count(const TrainedModel& model);
std::vector<double> flatten_params(const Mlp& net);

/// model_io.cpp:114-173: the "perfsage-model" version-1 JSON document (config, schema,
/// norm_stats, payload.layers[rows, cols, weights, biases], metrics.loss_trace); doubles are
/// written with 17 significant digits, so save -> load is bit-exact. LoadError on bad files.
void save_model(const TrainedModel& model, const std::string& path);
TrainedModel load_model(const std::string& path);
}  // namespace models

// ---- eval.hpp:13-49 ------------------------------------------------------------------------------
namespace eval {
double mape(std::span<const double> truth, std::span<const double> pred);
struct ThresholdedMape {
  double value = 0.0;
  std::size_t n_kept = 0;
};
ThresholdedMape mape_thresholded(std::span<const double> truth, std::span<const double> pred,
                                 double drop_fraction = 0.3);
double spearman(std::span<const double> truth, std::span<const double> pred);
struct EvalReport {
  std::string kernel, variant, model_family;
  double mape_full = 0.0, mape_thresholded = 0.0, rho = 0.0;
  std::size_t n_total = 0, n_kept = 0;
};
EvalReport make_report(std::span<const double> truth, std::span<const double> pred,
                       double drop_fraction = 0.3);
double speedup(double baseline_s, double chosen_s);  // eval.cpp: baseline / chosen (DomainError if <= 0)

/// eval.cpp:110-197: per-group means (std::map key order) + an "overall" row.
enum class GroupBy { Kernel, Variant, ModelFamily };
struct AggregateRow {
  std::string group;
  double mape_full = 0.0, mape_thresholded = 0.0, rho = 0.0;
  std::size_t reports = 0;
};
std::vector<AggregateRow> aggregate(const std::vector<EvalReport>& reports, GroupBy group_by);
void write_reports_csv(std::ostream& os, const std::vector<EvalReport>& reports);
void print_reports(std::ostream& os, const std::vector<EvalReport>& reports);
void print_aggregate(std::ostream& os, const std::vector<AggregateRow>& rows);
}  // namespace eval

// ---- selector.hpp:21-36 --------------------------------------------------------------------------
namespace selector {
using kernels::ScheduleCandidate;
using kernels::ScheduleSpace;
std::vector<ScheduleCandidate> enumerate_candidates(const ScheduleSpace& space, std::size_t limit,
                                                    std::uint64_t seed);
using ScheduleScorer = std::function<double(const ScheduleCandidate&)>;
ScheduleCandidate select(const ScheduleScorer& scorer, const std::vector<ScheduleCandidate>& candidates);
/// selector.cpp:42-53 — all candidates scored and reduced on the GPU.
ScheduleCandidate select(const models::TrainedModel& model, std::uint32_t image_n,
                         const std::vector<ScheduleCandidate>& candidates);

/// selector.hpp:37-62 / selector.cpp:55-140: regret and speedups of a chosen schedule
/// against measured runtimes (true best: lowest runtime, ties to the smaller schedule).
struct SelectionReport {
  ScheduleCandidate chosen;
  double predicted_s = 0.0, measured_s = 0.0;
  ScheduleCandidate true_best;
  double true_best_s = 0.0;
  ScheduleCandidate default_schedule;
  double default_s = 0.0;
  double regret = 0.0;                  // measured_s / true_best_s
  double speedup_vs_default = 0.0;      // default_s / measured_s
  double speedup_vs_random_mean = 0.0;  // mean candidate runtime / measured_s
  std::string to_json() const;
  std::string summary() const;
};
using MeasuredCandidates = std::vector<std::pair<ScheduleCandidate, double>>;
SelectionReport evaluate_selection(const ScheduleCandidate& chosen, const MeasuredCandidates& measured,
                                   const ScheduleCandidate& default_schedule,
                                   std::optional<double> default_runtime_s, double predicted_s);
}  // namespace selector

}  // namespace perfsage
