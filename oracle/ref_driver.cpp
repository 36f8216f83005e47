// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library (perfsage core,
// compiled from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libperfsage_ref.so). It lets the tests, the golden-vector
// generator and bench.py's reference arm call the reference's own code through
// ctypes. Nothing in the product links or loads this file.
//
// Every function only marshals arguments and calls the reference API:
//   datagen::build_dataset / split  (datagen.cpp:177-248)
//   models::train_nn / predict / predict_dataset (models.cpp:279-378)
//   models::mse_gradient / Mlp::init (mlp.cpp:9-122)
//   eval::mape / mape_thresholded / spearman (eval.cpp:26-90)
//   selector::select / enumerate_candidates (selector.cpp:13-53)
//   datagen::save_csv / load_csv (csv.cpp), models::save_model / load_model (model_io.cpp),
//   and the body of the CLI's train command (tools/perfsage.cpp:250-278)
#include <algorithm>
#include <atomic>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "perfsage/datagen.hpp"
#include "perfsage/errors.hpp"
#include "perfsage/eval.hpp"
#include "perfsage/features.hpp"
#include "perfsage/kernels.hpp"
#include "perfsage/models.hpp"
#include "perfsage/rng.hpp"
#include "perfsage/selector.hpp"
#include "perfsage/variants.hpp"

#include "../include/lann_engine.h"

using namespace perfsage;

namespace {

thread_local std::string g_err;

int status_of(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const TrainingError*>(&e)) return LANN_TRAINING_ERROR;
    if (dynamic_cast<const SchemaError*>(&e)) return LANN_SCHEMA_ERROR;
    if (dynamic_cast<const DomainError*>(&e)) return LANN_DOMAIN_ERROR;
    if (dynamic_cast<const BuildAbortError*>(&e)) return LANN_BUILD_ABORT;
    return LANN_PARAM_ERROR;
}

kernels::KernelKind kind_of(int k) { return static_cast<kernels::KernelKind>(k); }

datagen::ParamSpace space_of(const lann_world& w) {
    auto space = datagen::ParamSpace::defaults(kind_of(w.kind), w.max_threads);
    if (w.kind == LANN_BLUR && w.blur_lattice == 1)
        space.schedules = kernels::ScheduleSpace::gpu_style();
    return space;
}

kernels::VariantDescriptor variant_of(const lann_world& w) {
    kernels::VariantDescriptor v;
    v.variant_id = w.hw_class == LANN_HW_CPU ? "cpu_variant" : "gpu_variant";
    v.kind = kind_of(w.kind);
    v.hw_class = w.hw_class == LANN_HW_CPU ? kernels::HardwareClass::Cpu
                                           : kernels::HardwareClass::Gpu;
    v.threading = w.hw_class == LANN_HW_CPU ? kernels::Threading::Threaded
                                            : kernels::Threading::FixedSingle;
    v.hardware_label = "synthetic";
    return v;
}

// The probe of lann_engine.h's lann_world, written in the style of the
// acceptance world (acceptance_main.cpp:271-279) with the same stream.
datagen::RuntimeProbe world_probe(const lann_world& w, std::uint64_t noise_seed) {
    auto rng = std::make_shared<Rng>(noise_seed);
    return [rng, w](const kernels::InstanceParams& p) {
        double g, fd = 1.0;
        if (p.kind == kernels::KernelKind::Blur) {
            const auto& s = *p.schedule;
            const std::uint32_t f[4] = {s.s1, s.s2, s.s3, s.s4};
            g = 1.0;
            for (int j = 0; j < 4; ++j) {
                const double d = double(std::countr_zero(f[j])) - w.mu[j];
                g += w.kappa[j] * d * d;
            }
        } else {
            g = w.g0 + w.g1 / double(p.n_thd);
            const double dens = p.kind == kernels::KernelKind::MM ? p.d1 : p.d;
            fd = (1.0 - w.delta) + w.delta * dens;
        }
        const double noise = 1.0 + rng->uniform(-w.noise, w.noise);
        return w.alpha * double(kernels::complexity(p)) * g * fd * noise + w.beta;
    };
}

datagen::Dataset make_dataset(const lann_world& w, std::uint64_t seed, int count) {
    datagen::BuildOptions opts;
    opts.probe = world_probe(w, derive_seed(seed, 0x9015E));
    return datagen::build_dataset(variant_of(w), space_of(w), count, seed, opts);
}

datagen::Dataset from_flat(int kind, int with_n_thd, int n, const double* feats,
                           const std::uint64_t* c, const double* rt) {
    datagen::Dataset ds;
    ds.kind = kind_of(kind);
    ds.feature_names = models::feature_names(ds.kind, with_n_thd != 0);
    const std::size_t nf = ds.feature_names.size();
    for (int i = 0; i < n; ++i) {
        datagen::Sample s;
        s.features.assign(feats + std::size_t(i) * LANN_ROW, feats + std::size_t(i) * LANN_ROW + nf);
        s.c = c[i];
        s.runtime_s = rt ? rt[i] : 1.0;
        s.variant_id = "v";
        ds.samples.push_back(std::move(s));
    }
    return ds;
}

models::ModelConfig config_of(int family, int n_hidden, const int* hidden, double lr,
                              int epochs, std::uint64_t seed, int log_target,
                              int unconstrained) {
    models::ModelConfig cfg;
    cfg.family = family == LANN_NN ? models::ModelFamily::Nn : models::ModelFamily::NnC;
    cfg.hidden_widths.assign(hidden, hidden + n_hidden);
    cfg.learning_rate = lr;
    cfg.epochs = epochs;
    cfg.seed = seed;
    cfg.log_target = log_target != 0;
    cfg.unconstrained = unconstrained != 0;
    return cfg;
}

models::TrainedModel model_of(int kind, int with_n_thd, int family, int n_hidden,
                              const int* hidden, const double* params, const double* norm,
                              int log_target) {
    models::TrainedModel m;
    m.config = config_of(family, n_hidden, hidden, 1e-2, 1, 0, log_target, 1);
    m.kind = kind_of(kind);
    m.schema = models::model_schema(models::feature_names(m.kind, with_n_thd != 0),
                                    m.config.family);
    const int in = int(m.schema.size());
    std::vector<int> dims{in};
    dims.insert(dims.end(), hidden, hidden + n_hidden);
    dims.push_back(1);
    Rng rng(0);
    auto net = models::Mlp::init(dims, rng);
    std::size_t total = 0;
    for (auto& l : net.layers) total += l.w.size() + l.b.size();
    models::unflatten_params(net, std::span<const double>(params, total));
    m.payload = std::move(net);
    m.norm.f_min.assign(norm, norm + in);
    m.norm.f_max.assign(norm + 8, norm + 8 + in);
    m.norm.t_min = norm[16];
    m.norm.t_max = norm[17];
    m.norm.log_target = log_target != 0;
    return m;
}

void export_norm(const models::NormStats& st, double* norm) {
    std::fill(norm, norm + 18, 0.0);
    for (std::size_t j = 0; j < st.f_min.size(); ++j) {
        norm[j] = st.f_min[j];
        norm[8 + j] = st.f_max[j];
    }
    norm[16] = st.t_min;
    norm[17] = st.t_max;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_build_dataset(const lann_world* w, std::uint64_t seed, int count, double* feats,
                      std::uint64_t* c, double* rt, int* n_features) {
    try {
        const auto ds = make_dataset(*w, seed, count);
        *n_features = int(ds.feature_names.size());
        for (int i = 0; i < count; ++i) {
            const auto& s = ds.samples[i];
            for (int j = 0; j < LANN_ROW; ++j)
                feats[std::size_t(i) * LANN_ROW + j] = j < int(s.features.size()) ? s.features[j] : 0.0;
            c[i] = s.c;
            rt[i] = s.runtime_s;
        }
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// Permutation applied by datagen::split (datagen.cpp:225-248), recovered by
// splitting a dataset whose runtimes are the sample indices.
int ref_split_order(int n, double frac, std::uint64_t seed, std::int64_t* order,
                    int* n_train) {
    try {
        datagen::Dataset ds;
        ds.kind = kernels::KernelKind::MM;
        for (int i = 0; i < n; ++i) {
            datagen::Sample s;
            s.runtime_s = double(i);
            ds.samples.push_back(s);
        }
        const auto [tr, te] = datagen::split(ds, frac, seed);
        int k = 0;
        for (const auto& s : tr.samples) order[k++] = std::int64_t(s.runtime_s);
        for (const auto& s : te.samples) order[k++] = std::int64_t(s.runtime_s);
        *n_train = int(tr.samples.size());
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_mlp_init(int n_dims, const int* dims, std::uint64_t seed, int raw_rng, double* params) {
    try {
        std::vector<int> d(dims, dims + n_dims);
        Rng rng(raw_rng ? seed : derive_seed(seed, 0xA11CE));
        const auto net = models::Mlp::init(d, rng);
        const auto flat = models::flatten_params(net);
        std::copy(flat.begin(), flat.end(), params);
        return int(flat.size());
    } catch (const std::exception& e) {
        return -status_of(e);
    }
}

int ref_mse_gradient(int n_dims, const int* dims, const double* params, int n,
                     const double* X, const double* y, double* loss, double* grad) {
    try {
        std::vector<int> d(dims, dims + n_dims);
        Rng rng(0);
        auto net = models::Mlp::init(d, rng);
        std::size_t total = 0;
        for (auto& l : net.layers) total += l.w.size() + l.b.size();
        models::unflatten_params(net, std::span<const double>(params, total));
        std::vector<std::vector<double>> rows;
        for (int i = 0; i < n; ++i)
            rows.emplace_back(X + std::size_t(i) * LANN_ROW, X + std::size_t(i) * LANN_ROW + dims[0]);
        const auto lg = models::mse_gradient(net, rows, std::span<const double>(y, n));
        *loss = lg.loss;
        std::copy(lg.grad.begin(), lg.grad.end(), grad);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

namespace {
models::Mlp net_from(int n_dims, const int* dims, const double* params) {
    std::vector<int> d(dims, dims + n_dims);
    Rng rng(0);
    auto net = models::Mlp::init(d, rng);
    std::size_t total = 0;
    for (auto& l : net.layers) total += l.w.size() + l.b.size();
    models::unflatten_params(net, std::span<const double>(params, total));
    return net;
}
}  // namespace

// Mlp::forward (mlp.cpp:54-62) per row, rows at stride LANN_ROW
int ref_mlp_forward(int n_dims, const int* dims, const double* params, int n, const double* X, double* out) {
    try {
        const auto net = net_from(n_dims, dims, params);
        for (int i = 0; i < n; ++i)
            out[i] = net.forward(std::span<const double>(X + std::size_t(i) * LANN_ROW, std::size_t(dims[0])));
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// mse_loss (mlp.cpp:64-73)
int ref_mse_loss(int n_dims, const int* dims, const double* params, int n, const double* X, const double* y,
                 double* loss) {
    try {
        const auto net = net_from(n_dims, dims, params);
        std::vector<std::vector<double>> rows;
        for (int i = 0; i < n; ++i)
            rows.emplace_back(X + std::size_t(i) * LANN_ROW, X + std::size_t(i) * LANN_ROW + dims[0]);
        *loss = models::mse_loss(net, rows, std::span<const double>(y, std::size_t(n)));
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// `steps` AdamState::update calls (mlp.cpp:142-154) with gradients grads[step][n]; m, v out
int ref_adam_steps(int n, double* params, const double* grads, int steps, double lr, double* m, double* v) {
    models::AdamState st(static_cast<std::size_t>(n));
    for (int k = 0; k < steps; ++k)
        st.update(std::span<double>(params, std::size_t(n)),
                  std::span<const double>(grads + std::size_t(k) * n, std::size_t(n)), lr);
    std::copy(st.m.begin(), st.m.end(), m);
    std::copy(st.v.begin(), st.v.end(), v);
    return 0;
}

// train_full_batch on caller-normalized rows (mlp.cpp:156-175).
int ref_train_full_batch(int n_dims, const int* dims, double* params, int n,
                         const double* X, const double* y, double lr, int epochs,
                         double* trace, int* bad_epoch) {
    try {
        std::vector<int> d(dims, dims + n_dims);
        Rng rng(0);
        auto net = models::Mlp::init(d, rng);
        std::size_t total = 0;
        for (auto& l : net.layers) total += l.w.size() + l.b.size();
        models::unflatten_params(net, std::span<const double>(params, total));
        std::vector<std::vector<double>> rows;
        for (int i = 0; i < n; ++i)
            rows.emplace_back(X + std::size_t(i) * LANN_ROW, X + std::size_t(i) * LANN_ROW + dims[0]);
        *bad_epoch = -1;
        const auto tr = models::train_full_batch(net, rows, std::span<const double>(y, n), lr, epochs);
        std::copy(tr.begin(), tr.end(), trace);
        const auto flat = models::flatten_params(net);
        std::copy(flat.begin(), flat.end(), params);
        return 0;
    } catch (const TrainingError& e) {
        *bad_epoch = e.epoch();
        return status_of(e);
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// models::train_nn on a flat dataset (models.cpp:279-303).
int ref_train_nn(int kind, int with_n_thd, int family, int n, const double* feats,
                 const std::uint64_t* c, const double* rt, int n_hidden, const int* hidden,
                 double lr, int epochs, std::uint64_t seed, int log_target, int unconstrained,
                 double* params, int* n_params, double* trace, double* norm, int* bad_epoch) {
    try {
        *bad_epoch = -1;
        const auto ds = from_flat(kind, with_n_thd, n, feats, c, rt);
        const auto cfg = config_of(family, n_hidden, hidden, lr, epochs, seed, log_target,
                                   unconstrained);
        const auto model = models::train_nn(ds, cfg);
        const auto flat = models::flatten_params(std::get<models::Mlp>(model.payload));
        std::copy(flat.begin(), flat.end(), params);
        *n_params = int(flat.size());
        if (trace) std::copy(model.loss_trace.begin(), model.loss_trace.end(), trace);
        export_norm(model.norm, norm);
        return 0;
    } catch (const TrainingError& e) {
        *bad_epoch = e.epoch();
        return status_of(e);
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// models::predict per row (models.cpp:346-363); feats are base features, c appended
// for the augmented family by model_features (models.cpp:143-148).
int ref_predict(int kind, int with_n_thd, int family, int n_hidden, const int* hidden,
                const double* params, const double* norm, int log_target, int n,
                const double* feats, const std::uint64_t* c, double* out) {
    try {
        const auto m = model_of(kind, with_n_thd, family, n_hidden, hidden, params, norm,
                                log_target);
        const auto ds = from_flat(kind, with_n_thd, n, feats, c, nullptr);
        const auto p = models::predict_dataset(m, ds);
        std::copy(p.begin(), p.end(), out);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// predict on explicit model-input vectors (schema length checked, SchemaError).
int ref_predict_raw(int kind, int with_n_thd, int family, int n_hidden, const int* hidden,
                    const double* params, const double* norm, int log_target, int len,
                    const double* x, double* out) {
    try {
        const auto m = model_of(kind, with_n_thd, family, n_hidden, hidden, params, norm,
                                log_target);
        *out = models::predict(m, std::span<const double>(x, len));
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_mape(int n, const double* t, const double* p, double* out) {
    try {
        *out = eval::mape(std::span<const double>(t, n), std::span<const double>(p, n));
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_mape_thresholded(int n, const double* t, const double* p, double drop, double* out,
                         int* kept) {
    try {
        const auto r = eval::mape_thresholded(std::span<const double>(t, n),
                                              std::span<const double>(p, n), drop);
        *out = r.value;
        *kept = int(r.n_kept);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_spearman(int n, const double* t, const double* p, double* out) {
    try {
        *out = eval::spearman(std::span<const double>(t, n), std::span<const double>(p, n));
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_enumerate_candidates(int lattice, std::uint64_t limit, std::uint64_t seed,
                             std::uint32_t* out, std::uint64_t cap) {
    try {
        const auto space = lattice == 1 ? kernels::ScheduleSpace::gpu_style()
                                        : kernels::ScheduleSpace::cpu_default();
        const auto c = selector::enumerate_candidates(space, limit, seed);
        for (std::size_t i = 0; i < c.size() && i < cap; ++i) {
            out[4 * i] = c[i].s1;
            out[4 * i + 1] = c[i].s2;
            out[4 * i + 2] = c[i].s3;
            out[4 * i + 3] = c[i].s4;
        }
        return int(c.size());
    } catch (const std::exception& e) {
        return -status_of(e);
    }
}

// selector::select(TrainedModel, n, candidates) (selector.cpp:42-53).
int ref_select_schedule(int family, int n_hidden, const int* hidden, const double* params,
                        const double* norm, int log_target, std::uint32_t n_img, int n_cands,
                        const std::uint32_t* cands, std::int64_t* chosen, double* score) {
    try {
        const auto m = model_of(LANN_BLUR, 0, family, n_hidden, hidden, params, norm, log_target);
        std::vector<kernels::ScheduleCandidate> cs;
        for (int i = 0; i < n_cands; ++i)
            cs.push_back({cands[4 * i], cands[4 * i + 1], cands[4 * i + 2], cands[4 * i + 3]});
        const auto best = selector::select(m, n_img, cs);
        for (int i = 0; i < n_cands; ++i)
            if (cs[i] == best) { *chosen = i; break; }
        const auto params_b = kernels::InstanceParams::blur(n_img, best);
        *score = models::predict(m, models::model_features(params_b, m.config.family));
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// ---- whole-pipeline runner (reference arm of bench.py, golden population) ----------
// One job = build_dataset -> split -> [fold] -> train_nn -> predict_dataset -> make_report,
// exactly the acceptance-criterion-5 protocol (acceptance_main.cpp:283-328).
static int run_job(const lann_job& j, lann_job_result* r, double* params, double* trace) {
    r->nonfinite_epoch = -1;
    try {
        const auto ds = make_dataset(j.world, j.data_seed, j.count);
        auto [train, test] = datagen::split(ds, j.train_fraction, j.data_seed);
        if (j.n_folds >= 2) {
            const std::size_t n = train.samples.size();
            const std::size_t b0 = n * j.fold / j.n_folds, b1 = n * (j.fold + 1) / j.n_folds;
            datagen::Dataset tr = train, ev = train;
            tr.samples.clear();
            ev.samples.clear();
            for (std::size_t i = 0; i < n; ++i)
                (i >= b0 && i < b1 ? ev : tr).samples.push_back(train.samples[i]);
            train = std::move(tr);
            test = std::move(ev);
        }
        const auto cfg = config_of(j.family, j.n_hidden, j.hidden, j.learning_rate, j.epochs,
                                   j.init_seed, j.log_target, j.unconstrained);
        const auto model = models::train_nn(train, cfg);
        const auto pred = models::predict_dataset(model, test);
        const auto rep = eval::make_report(test.runtimes(), pred, 0.3);
        const auto flat = models::flatten_params(std::get<models::Mlp>(model.payload));
        r->status = 0;
        r->n_inputs = int(model.schema.size());
        r->n_params = int(flat.size());
        r->n_train = int(train.samples.size());
        r->n_eval = int(test.samples.size());
        r->final_loss = model.loss_trace.back();
        r->mape = rep.mape_full;
        r->mape_thr = rep.mape_thresholded;
        r->rho = rep.rho;
        r->n_kept = int(rep.n_kept);
        if (params) std::copy(flat.begin(), flat.end(), params);
        if (trace) std::copy(model.loss_trace.begin(), model.loss_trace.end(), trace);
        return 0;
    } catch (const TrainingError& e) {
        r->nonfinite_epoch = e.epoch();
        r->status = status_of(e);
        return r->status;
    } catch (const std::exception& e) {
        r->status = status_of(e);
        return r->status;
    }
}

// Runs jobs on a pool of `threads` std::threads (one whole model per task, the
// reference trainer being single-threaded per model).
// Returns wall seconds.
double ref_run_population(int n_jobs, const lann_job* jobs, lann_job_result* results,
                          double* params, const std::int64_t* params_offset, double* trace,
                          const std::int64_t* trace_offset, int threads) {
    std::atomic<int> next{0};
    const auto t0 = std::chrono::steady_clock::now();
    auto worker = [&] {
        for (;;) {
            const int i = next.fetch_add(1);
            if (i >= n_jobs) return;
            run_job(jobs[i], &results[i], params ? params + params_offset[i] : nullptr,
                    trace ? trace + trace_offset[i] : nullptr);
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads) - 1; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---- on-disk formats and the CLI train pipeline (csv.cpp, model_io.cpp, perfsage.cpp) ----

// build_dataset with the world probe, every sample's variant_id set, then datagen::save_csv
int ref_save_dataset_csv(const lann_world* w, std::uint64_t seed, int count, const char* variant_id,
                         const char* path) {
    try {
        auto ds = make_dataset(*w, seed, count);
        for (auto& smp : ds.samples) smp.variant_id = variant_id;
        datagen::save_csv(ds, path);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_csv_roundtrip(const char* in, const char* out) {
    try {
        datagen::save_csv(datagen::load_csv(in), out);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_model_roundtrip(const char* in, const char* out) {
    try {
        models::save_model(models::load_model(in), out);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// load_model -> [f_min.., f_max.., t_min, t_max, flat params.., loss_trace..]; returns count
int ref_model_dump(const char* path, double* out, int cap) {
    try {
        const auto m = models::load_model(path);
        std::vector<double> v(m.norm.f_min.begin(), m.norm.f_min.end());
        v.insert(v.end(), m.norm.f_max.begin(), m.norm.f_max.end());
        v.push_back(m.norm.t_min);
        v.push_back(m.norm.t_max);
        const auto flat = models::flatten_params(std::get<models::Mlp>(m.payload));
        v.insert(v.end(), flat.begin(), flat.end());
        v.insert(v.end(), m.loss_trace.begin(), m.loss_trace.end());
        if (int(v.size()) > cap) return -1;
        std::copy(v.begin(), v.end(), out);
        return int(v.size());
    } catch (const std::exception& e) {
        status_of(e);
        return -1;
    }
}

// perfsage.cpp cmd_train (:250-278) minus the manifest: load_csv -> split(derive_seed(seed,
// 0x5b11)) -> default_config(kind, family) with seed (+ epochs override) -> train_model ->
// save_model / save_csv x2
int ref_cli_train(const char* csv, std::uint64_t seed, const char* family, int epochs,
                  const char* model_out, const char* train_out, const char* test_out) {
    try {
        const auto fam = models::family_from_string(family);
        const auto ds = datagen::load_csv(csv);
        const auto [tr, te] = datagen::split(ds, 0.5, derive_seed(seed, 0x5b11));
        auto cfg = models::default_config(ds.kind, fam, false);
        cfg.family = fam;
        cfg.seed = seed;
        if (epochs > 0) cfg.epochs = epochs;
        const auto model = models::train_model(tr, cfg);
        models::save_model(model, model_out);
        datagen::save_csv(tr, train_out);
        datagen::save_csv(te, test_out);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// perfsage.cpp cmd_gen with --external-cmd (:197-248): an external variant as the probe,
// datagen::build_dataset, every sample's variant_id set, save_csv
int ref_save_external_csv(int kind, int gpu_class, int max_threads, const char* command, const char* variant_id,
                          int count, std::uint64_t seed, const char* path) {
    try {
        kernels::VariantDescriptor ext;
        ext.variant_id = variant_id;
        ext.kind = kind_of(kind);
        ext.impl = kernels::ImplKind::External;
        ext.hw_class = gpu_class ? kernels::HardwareClass::Gpu : kernels::HardwareClass::Cpu;
        ext.hardware_label = "external";
        ext.launch_command = command;
        auto space = datagen::ParamSpace::defaults(kind_of(kind), max_threads);
        const auto ds = datagen::build_dataset(ext, space, std::size_t(count), seed, {});
        datagen::save_csv(ds, path);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// The reference CLI's mock_probe (tools/perfsage.cpp:71-84), restated here because the CLI itself
// needs CLI11 (absent); it only calls reference library functions.
datagen::RuntimeProbe ref_mock_probe() {
    return [](const kernels::InstanceParams& params) {
        const auto feats = models::featurize(params, true);
        std::uint64_t h = 0x9e3779b97f4a7c15ULL;
        for (double f : feats) {
            std::uint64_t bits;
            std::memcpy(&bits, &f, sizeof bits);
            h ^= bits;
            splitmix64(h);
        }
        const double jitter = 0.5 + double(splitmix64(h) >> 11) * 0x1.0p-53;
        return 1e-9 * double(kernels::complexity(params)) * jitter + 1e-6;
    };
}

// cmd_gen (perfsage.cpp:197-248) with --mock-timer, minus the manifest
int ref_cli_gen_mock(int kind, const char* variant_id, int max_threads, unsigned dim_max, int n_sides,
                     const unsigned* sides, int gpu_lattice, int count, std::uint64_t seed, const char* path) {
    try {
        auto space = datagen::ParamSpace::defaults(kind_of(kind), max_threads);
        space.dim_max = dim_max;
        if (kind_of(kind) == kernels::KernelKind::Blur) {
            space.blur_sides.assign(sides, sides + n_sides);
            space.schedules = gpu_lattice ? kernels::ScheduleSpace::gpu_style() : kernels::ScheduleSpace::cpu_default();
        }
        const auto registry = kernels::VariantRegistry::builtin();
        const auto& variant = registry.get(kind_of(kind), variant_id);
        datagen::BuildOptions opts;
        opts.probe = ref_mock_probe();
        datagen::save_csv(datagen::build_dataset(variant, space, std::size_t(count), seed, opts), path);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// cmd_select (perfsage.cpp:307-382) with --mock-timer and no --data: out = {chosen s1..s4,
// predicted_s, measured_s, true_best s1..s4, true_best_s, default_s, regret, speedup_vs_default,
// speedup_vs_random_mean}
int ref_cli_select_mock(unsigned n, int n_cands, std::uint64_t seed, int epochs, int threads, double* out) {
    try {
        const kernels::ScheduleCandidate default_sched{8, 256, 128, 8};
        auto candidates = selector::enumerate_candidates(kernels::ScheduleSpace::cpu_default(), std::size_t(n_cands), seed);
        const auto probe = ref_mock_probe();
        datagen::Dataset measured;
        measured.kind = kernels::KernelKind::Blur;
        measured.feature_names = models::feature_names(kernels::KernelKind::Blur, false);
        measured.seed = seed;
        selector::MeasuredCandidates table;
        auto instance = kernels::make_instance(kernels::InstanceParams::blur(n, default_sched), derive_seed(seed, 0x1417));
        instance.params.n_thd = threads;
        bool default_present = false;
        for (const auto& c : candidates) default_present |= (c == default_sched);
        if (!default_present) candidates.push_back(default_sched);
        for (const auto& c : candidates) {
            instance.params.schedule = c;
            const double runtime = probe(instance.params);
            table.emplace_back(c, runtime);
            datagen::Sample smp;
            smp.features = models::featurize(instance.params, false, false);
            smp.c = kernels::complexity(instance.params);
            smp.runtime_s = runtime;
            smp.variant_id = "tiled";
            measured.samples.push_back(std::move(smp));
        }
        auto cfg = models::default_config(kernels::KernelKind::Blur, models::ModelFamily::NnC, false);
        cfg.family = models::ModelFamily::NnC;
        cfg.seed = seed;
        if (epochs > 0) cfg.epochs = epochs;
        const auto model = models::train_model(measured, cfg);
        const auto chosen = selector::select(model, n, candidates);
        const auto chosen_params = kernels::InstanceParams::blur(n, chosen);
        const double predicted = models::predict(model, models::model_features(chosen_params, cfg.family));
        const auto rep = selector::evaluate_selection(chosen, table, default_sched, std::nullopt, predicted);
        const double v[] = {double(rep.chosen.s1), double(rep.chosen.s2), double(rep.chosen.s3), double(rep.chosen.s4),
                            rep.predicted_s, rep.measured_s, double(rep.true_best.s1), double(rep.true_best.s2),
                            double(rep.true_best.s3), double(rep.true_best.s4), rep.true_best_s, rep.default_s,
                            rep.regret, rep.speedup_vs_default, rep.speedup_vs_random_mean};
        std::copy(std::begin(v), std::end(v), out);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// perfsage.cpp evaluate_model_on (:98-108): out = {mape_full, mape_thr, rho, n_kept}
int ref_eval_model(const char* model_path, const char* csv, double drop, double* out) {
    try {
        const auto m = models::load_model(model_path);
        const auto data = datagen::load_csv(csv);
        const auto pred = models::predict_dataset(m, data);
        const auto rep = eval::make_report(data.runtimes(), pred, drop);
        out[0] = rep.mape_full;
        out[1] = rep.mape_thresholded;
        out[2] = rep.rho;
        out[3] = double(rep.n_kept);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// n sample_params draws (datagen.cpp:60-110) of ParamSpace::defaults(kind, 8) from Rng(seed):
// featurize(p, true) rows padded to LANN_ROW; returns the feature count.
int ref_sample_features(int kind, std::uint64_t seed, int n, double* out) {
    try {
        const auto space = datagen::ParamSpace::defaults(kind_of(kind), 8);
        Rng rng(seed);
        int nf = 0;
        for (int i = 0; i < n; ++i) {
            const auto f = models::featurize(datagen::sample_params(space, rng), true);
            nf = int(f.size());
            std::copy(f.begin(), f.end(), out + std::size_t(i) * LANN_ROW);
        }
        return nf;
    } catch (const std::exception& e) {
        return -status_of(e);
    }
}

}  // extern "C"
