/*
 * lann_engine.h — C ABI of the B200 LANN engine (drop-in for the perfsage
 * models / eval / selector / datagen hot path).
 *
 * Every entry point is plain C: caller-owned HOST buffers, sizes as integers,
 * integer status codes, no exceptions, no torch types. The engine owns its
 * device memory. Calls are synchronous (they return after the D2H copy).
 *
 * Reference interfaces each entry point replaces (paths into the reference
 * tree proj/core/):
 *   lann_train            models::train_full_batch       include/perfsage/mlp.hpp:64-66
 *   lann_mlp_forward      Mlp::forward                   include/perfsage/mlp.hpp:27
 *   lann_mse_loss         mse_loss                       include/perfsage/mlp.hpp:34-35
 *   lann_mse_gradient     mse_gradient + LossGrad        include/perfsage/mlp.hpp:37-44
 *   lann_adam_update      AdamState::update              include/perfsage/mlp.hpp:50-60
 *   lann_predict          models::predict / predict_dataset include/perfsage/models.hpp:109,119-120
 *   lann_eval             eval::mape / mape_thresholded / spearman / make_report
 *                                                         include/perfsage/eval.hpp:13-49
 *   lann_select_schedule  selector::select(TrainedModel, n, candidates)
 *                                                         include/perfsage/selector.hpp:35-36
 *   lann_select_variants  (no reference equivalent: multi-variant argmin built
 *                          from selector::select's tie rule, selector.cpp:26-40)
 *   lann_build_dataset    datagen::build_dataset + split  include/perfsage/datagen.hpp:109-116
 *   lann_run_population   models::train_nn + predict_dataset + eval::make_report
 *                          over a whole population (batched overload of
 *                          models.hpp:95,119 and eval.hpp:49)
 *
 * Status codes map 1:1 onto the reference's exception types
 * (include/perfsage/errors.hpp): ParamError, SchemaError, TrainingError,
 * DomainError, BuildAbortError.
 */
#ifndef LANN_ENGINE_H
#define LANN_ENGINE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status ------------------------------------------------------------ */
enum lann_status {
  LANN_OK = 0,
  LANN_PARAM_ERROR = 1,    /* perfsage::ParamError   (errors.hpp:15-18)  */
  LANN_SCHEMA_ERROR = 2,   /* perfsage::SchemaError  (errors.hpp:55-58)  */
  LANN_TRAINING_ERROR = 3, /* perfsage::TrainingError(errors.hpp:33-40)  */
  LANN_DOMAIN_ERROR = 4,   /* perfsage::DomainError  (errors.hpp:21-24)  */
  LANN_BUILD_ABORT = 5,    /* perfsage::BuildAbortError (errors.hpp:61-69) */
  LANN_CUDA_ERROR = 6,     /* device failure (no reference equivalent)    */
  LANN_NO_DEVICE = 7       /* no CUDA device: the engine never falls back */
};

/* ---- arithmetic modes ---------------------------------------------------- */
enum lann_precision {
  /* FP64 with the reference's exact operation order and no FMA contraction:
   * loss traces and weights are bit-identical to models::train_nn. */
  LANN_FP64_EXACT = 0,
  /* FP32 FMA throughput mode (tree reductions over samples). */
  LANN_FP32 = 1
};

/* ---- domain enums (kernels.hpp:13, models.hpp:19) -------------------------- */
enum lann_kind { LANN_MM = 0, LANN_MV = 1, LANN_MC = 2, LANN_MP = 3, LANN_BLUR = 4 };
enum lann_family { LANN_NNC = 0, LANN_NN = 1 };
enum lann_hw_class { LANN_HW_CPU = 0, LANN_HW_GPU = 1 }; /* variants.hpp:16 */

#define LANN_ROW 8 /* padded feature-row width: up to 7 inputs (+ 1 spare) */

/* ---- synthetic runtime world (a generalisation of the reference's
 * acceptance-test probe, proj/tests/acceptance/acceptance_main.cpp:271-279):
 *   non-blur: t = ((((alpha * c) * g) * fd) * nz) + beta,
 *             g  = g0 + g1 / n_thd,  fd = (1 - delta) + delta * d,
 *             nz = 1 + U(-noise, noise)
 *   blur:     same with g = 1 + sum_j kappa[j] * (log2 s_j - mu[j])^2, fd = 1
 * with nz drawn from Rng(derive_seed(data_seed, 0x9015E)) one draw per sample.
 * (alpha=3e-9, g0=0.25, g1=0.75, delta=0, beta=0, noise=0.02) is the
 * acceptance world bit for bit. */
typedef struct lann_world {
  int32_t kind;         /* lann_kind */
  int32_t hw_class;     /* lann_hw_class: CPU variants take n_thd (variants.hpp:29-31) */
  int32_t max_threads;  /* ParamSpace::max_threads (datagen.hpp:23) */
  int32_t blur_lattice; /* 0 = ScheduleSpace::cpu_default, 1 = gpu_style */
  double alpha, g0, g1, delta, beta, noise;
  double mu[4], kappa[4];
} lann_world;

/* One model of a population: dataset recipe + ModelConfig (models.hpp:27-40). */
typedef struct lann_job {
  lann_world world;
  uint64_t data_seed;    /* build_dataset seed; split uses the same seed */
  int32_t count;         /* dataset size (>= 2) */
  double train_fraction; /* datagen::split fraction */
  int32_t n_folds;       /* 0: train on the split's train part, evaluate on its test part;
                            k>=2: k-fold CV over the train part, see fold */
  int32_t fold;          /* held-out block index when n_folds >= 2 */
  int32_t family;        /* lann_family */
  int32_t n_hidden;      /* 1 or 2 */
  int32_t hidden[2];
  double learning_rate;  /* 1e-2, 1e-3 or 1e-4 (ModelConfig::validate) */
  int32_t epochs;
  uint64_t init_seed;    /* ModelConfig::seed */
  int32_t log_target;
  int32_t unconstrained;
} lann_job;

typedef struct lann_job_result {
  int32_t status;          /* lann_status of this job */
  int32_t nonfinite_epoch; /* TrainingError epoch, else -1 */
  int32_t n_inputs;        /* model inputs I */
  int32_t n_params;        /* trainable parameters P */
  int32_t n_train, n_eval; /* sample counts */
  double final_loss;       /* loss_trace.back() */
  double mape, mape_thr, rho; /* on the evaluation part */
  int32_t n_kept;
  int32_t precision_run;   /* lann_precision the trainer actually ran (-1: not trained): LANN_FP32 requests
                              run in FP32 for every shape with hidden layers of <= 64 units and <= 5120
                              parameters (packed kernels for the LANN shapes, a generic CTA kernel for
                              the rest); wider nets, and LANN shapes whose tile exceeds 96 KB, run in
                              LANN_FP64_EXACT and say so here */
} lann_job_result;

/* ---- engine ---------------------------------------------------------------- */
typedef struct lann_engine lann_engine;

int lann_engine_create(int device, lann_engine** out);
void lann_engine_destroy(lann_engine* engine);
const char* lann_last_error(const lann_engine* engine);
/* Device time (ms) of the most recent call's kernels, measured with CUDA
 * events on the engine stream; 0 if nothing ran. */
double lann_last_device_ms(const lann_engine* engine);
/* Number of engine kernels launched by the most recent call. */
int64_t lann_last_launches(const lann_engine* engine);
/* Device time (ms) of the dominant kernel of the most recent call: the
 * trainer launches of lann_train / lann_population_run (summed over steps), or
 * the scoring kernel of lann_select_variants(_compact), or the predictor of
 * lann_predict (inputs already on the device); CUDA events on the launch stream. */
double lann_last_train_ms(const lann_engine* engine);

/* ---- training (train_full_batch, batched) ----------------------------------
 * Tiles hold min-max-normalised training rows (NormStats, models.cpp:118-133):
 * X is [total_rows][LANN_ROW] doubles (columns >= I ignored), y [total_rows].
 * Models reference a tile; params is the flat reference layout
 * (L0.w row-major out x in, L0.b, L1.w, L1.b, ...; mlp.cpp:124-131), holding
 * the initial weights on entry and the trained weights on return. */
typedef struct lann_train_batch {
  int32_t n_models;
  int32_t precision;          /* lann_precision */
  int32_t n_tiles;
  const int32_t* tile_rows;   /* N per tile (>= 1) */
  const int32_t* tile_inputs; /* I per tile (1..7) */
  const int64_t* tile_offset; /* first row of the tile */
  int64_t total_rows;
  const double* X;
  const double* y;
  const int32_t* model_tile;
  const int32_t* model_h1;
  const int32_t* model_h2;    /* 0 = one hidden layer */
  const double* model_lr;
  const int32_t* model_epochs;
  const int64_t* model_param_offset;
  int64_t total_params;
  double* params;             /* in/out */
  double* final_loss;         /* out [n_models] */
  int32_t* nonfinite_epoch;   /* out [n_models]: -1 or TrainingError epoch */
  double* loss_trace;         /* optional out; NULL = not recorded */
  const int64_t* trace_offset;/* per model offset into loss_trace */
  int32_t trace_stride;       /* keep epochs e with e % stride == 0 */
} lann_train_batch;

int lann_train(lann_engine* engine, const lann_train_batch* batch);

/* ---- prediction (models::predict, models.cpp:346-363) ----------------------
 * Raw (un-normalised) feature rows [n_rows][LANN_ROW]; each row is scored by
 * row_model[row]. norm = per model {f_min[8], f_max[8], t_min, t_max} = 18 doubles;
 * output max(denormalize(forward(normalize(x))), 1e-9). */
typedef struct lann_model_set {
  int32_t n_models;
  int32_t precision;
  const int32_t* n_inputs;
  const int32_t* h1;
  const int32_t* h2;
  const int32_t* log_target;
  const int64_t* param_offset;
  const double* params;
  int64_t total_params;
  const double* norm;          /* [n_models][18] */
} lann_model_set;

int lann_predict(lann_engine* engine, const lann_model_set* models, int64_t n_rows,
                 const double* rows, const int32_t* row_model, double* out);

/* ---- metrics (eval.cpp:26-108) ----------------------------------------------
 * n_sets independent (truth, pred) sets packed back to back; set i spans
 * [offset[i], offset[i]+len[i]). Outputs per set. */
int lann_eval(lann_engine* engine, int32_t n_sets, const int64_t* offset, const int32_t* len,
              const double* truth, const double* pred, double drop_fraction,
              double* mape, double* mape_thr, int32_t* n_kept, double* rho);

/* ---- mlp.hpp building blocks on the GPU, batched over nets -------------------------
 * Mlp::forward (mlp.cpp:54-62), mse_loss (mlp.cpp:64-73), mse_gradient + LossGrad
 * (mlp.hpp:34-44, mlp.cpp:75-122) and AdamState::update (mlp.hpp:50-60, mlp.cpp:142-154)
 * for generic nets: any depth up to 8 layers, every width up to 64 (the reference's Mlp;
 * the population trainers compile the LANN shapes instead). Nets are concatenated: net k has
 * n_dims[k] dims (inputs, hidden..., outputs), its flat parameters (mlp.cpp:124-131 layout)
 * follow the previous net's, and its n_rows[k] rows of dims[0] doubles (and targets) follow
 * the previous net's rows. Exact reference operation order: results are bit-identical. */
typedef struct lann_mlp_batch {
  int32_t n_nets;
  const int32_t* n_dims;  /* per net, 2..9 */
  const int32_t* dims;    /* concatenated */
  const double* params;   /* concatenated flat parameters */
  const int32_t* n_rows;  /* per net, >= 1 */
  const double* X;        /* concatenated rows */
  const double* y;        /* concatenated targets (unused by lann_mlp_forward) */
} lann_mlp_batch;

/* out[row]: the network output (output unit 0) of every row of every net */
int lann_mlp_forward(lann_engine* engine, const lann_mlp_batch* batch, double* out);
/* loss[net] = (sum over rows in order of (f(x) - y)^2) / n_rows */
int lann_mse_loss(lann_engine* engine, const lann_mlp_batch* batch, double* loss);
/* loss[net] and grad (concatenated like params); the last layer must have one output */
int lann_mse_gradient(lann_engine* engine, const lann_mlp_batch* batch, double* loss, double* grad);
/* One Adam step over n parameters in place (params, m, v); `step` is the step count AFTER
 * the increment AdamState::update performs first; bias corrections 1 - pow(beta, step) are
 * taken from the host libm exactly as the reference computes them. */
int lann_adam_update(lann_engine* engine, int64_t n, double* params, const double* grad, double* m, double* v,
                     int32_t step, double lr, double beta1, double beta2, double epsilon);

/* ---- selection ------------------------------------------------------------------
 * Blur schedule selection (selector.cpp:42-53): candidates [n][4] u32 schedules,
 * model index 0 of the set, image side n_img. Returns the chosen index and its
 * predicted runtime; ties go to the lexicographically smaller schedule. */
int lann_select_schedule(lann_engine* engine, const lann_model_set* models, uint32_t n_img,
                         int64_t n_cands, const uint32_t* cands, int64_t* chosen,
                         double* chosen_score);

/* Multi-variant argmin: n_cands candidate shapes of `kind` generated
 * counter-based from seed (candidate i uses splitmix64 draws from
 * derive_seed(seed, first + i), same ranges as sample_params), each scored by
 * every model of the set (a model with with_n_thd[v] = 0 ignores n_thd);
 * out_idx[i] = argmin variant (ties -> lower index), out_score[i] = its score. */
int lann_select_variants(lann_engine* engine, const lann_model_set* models,
                         const int32_t* with_n_thd, int32_t kind, int32_t max_threads,
                         uint64_t seed, int64_t first, int64_t n_cands,
                         int32_t* out_idx, double* out_score);

/* lann_select_variants with compact, streamed outputs: out_idx[i] (uint8) and out_score[i]
 * (float: the FP32 scorer's own precision; FP64-exact models round their score once) for
 * candidate first + i, and hist[v] = number of candidates whose argmin is model v. Any of the
 * three outputs may be NULL (hist alone moves M counters, not per-candidate data). The range is
 * scored in chunks whose device-to-host copies overlap the next chunk's scoring; outputs in
 * pinned host memory (lann_host_alloc) are written by DMA directly, pageable ones through the
 * engine's pinned staging buffer. At most 255 models. */
int lann_select_variants_compact(lann_engine* engine, const lann_model_set* models, const int32_t* with_n_thd,
                                 int32_t kind, int32_t max_threads, uint64_t seed, int64_t first, int64_t n_cands,
                                 uint8_t* out_idx, float* out_score, int64_t* hist);

/* Pinned (page-locked) host memory for engine outputs: device-to-host copies into it run at
 * full link bandwidth and overlap compute. */
int lann_host_alloc(size_t bytes, void** out);
void lann_host_free(void* ptr);

/* ---- synthetic data (datagen::build_dataset + split, datagen.cpp:177-248) ----
 * feats [count][LANN_ROW] base features (no c), c [count], runtime [count];
 * order [count] = the split permutation of split(ds, train_fraction, seed). */
int lann_build_dataset(const lann_world* world, uint64_t seed, int32_t count,
                       double* feats, uint64_t* c, double* runtime, int32_t* n_features);
int lann_split_order(int32_t n, uint64_t seed, int64_t* order);

/* datagen::build_dataset of a native CPU-class variant with the reference CLI's --mock-timer
 * probe (perfsage.cpp:71-84: 1e-9 * c * jitter(hash of the augmented features) + 1e-6), over
 * ParamSpace{kind, max_threads, dims U{1..dim_max}, blur sides[n_sides], blur_lattice};
 * single_threaded pins n_thd = 1 (Threading::FixedSingle). Byte-identical to the reference CLI's
 * `gen --mock-timer` dataset. feats [count][LANN_ROW] (base features with n_thd). */
int lann_build_mock_dataset(int32_t kind, int32_t single_threaded, int32_t max_threads, uint32_t dim_max,
                            int32_t n_sides, const uint32_t* sides, int32_t blur_lattice, int32_t count,
                            uint64_t seed, double* feats, uint64_t* c, double* runtime, int32_t* n_features);
/* the mock probe at GIVEN blur schedules (cmd_select --mock-timer, perfsage.cpp:340-360) */
int lann_mock_schedules(uint32_t image_n, int32_t n_thd, int32_t n, const uint32_t* sched, double* runtime);

/* The synthetic world's runtime probe at GIVEN blur schedules (the stand-in for
 * datagen::measure of the tiled blur kernel in perfsage.cpp cmd_select:297-316):
 * instance blur(image_n, sched[i]) with n_thd = world.max_threads, noise drawn from
 * Rng(derive_seed(seed, 0x9015E)) one draw per schedule in order. sched [n][4]. */
int lann_probe_schedules(const lann_world* world, uint64_t seed, uint32_t image_n, int32_t n,
                         const uint32_t* sched, double* runtime);

/* ---- real measurement on the B200 (datagen::measure, datagen.cpp:118-160; the paper's
 * GPU-class variants, section IV-A) ----------------------------------------------------
 * Times GPU kernel variant `variant` of kernel kind `kind` on every instance: feats
 * [n][LANN_ROW] are the GPU-class base features (mm: m,n,k,d1,d2; mv: m,n,d; mc: m,n,r,d;
 * mp: m,n,r,s,d; blur: n,s1,s2,s3,s4), operands are generated on the device from `seed`,
 * `warmups` untimed runs then the median of `reps` CUDA-event-timed runs, in seconds.
 * checksum (optional) = sum of the output elements (FP64) for verification. */
int lann_measure(lann_engine* engine, int32_t kind, const char* variant, int32_t n, const double* feats,
                 int32_t warmups, int32_t reps, uint64_t seed, double* runtime_s, double* checksum);
int lann_measure_variant_count(int32_t kind);
const char* lann_measure_variant_name(int32_t kind, int32_t idx);
/* datagen::build_dataset with the measured probe: `count` instances drawn as sample_params
 * (Rng(derive_seed(seed, 0)), GPU class: no n_thd; blur from the `blur_lattice` schedule
 * space at side `blur_side`, 0 = the default sides), each measured by lann_measure. */
int lann_build_measured_dataset(lann_engine* engine, int32_t kind, const char* variant,
                                int32_t blur_lattice, int32_t blur_side, int32_t count, uint64_t seed,
                                int32_t warmups, int32_t reps, double* feats, uint64_t* c,
                                double* runtime, int32_t* n_features);

/* ---- the baseline families of the five-family comparison (models.cpp:184-333,
 * forest.cpp): const (C: t ~ c), lrc (LR+C) least squares and the nlrc random forest,
 * fitted on RAW features (no normalisation), batched over models. -------------------- */
typedef struct lann_design {
  int32_t n_models;
  const int32_t* n_rows;      /* samples per model */
  const int32_t* n_feats;     /* design columns per model (<= LANN_ROW; const: 1 = c) */
  const int64_t* row_offset;  /* first row of each model in X / y */
  const double* X;            /* [rows][LANN_ROW] model features (model_features order) */
  const double* y;            /* runtimes in seconds */
} lann_design;
/* fit_least_squares (models.cpp:220-265), bit-identical: weights [n_models][LANN_ROW],
 * intercept [n_models]; status[m] = 0, or LANN_DOMAIN_ERROR for FitError (singular despite
 * the ridge). */
int lann_fit_linear(lann_engine* engine, const lann_design* design, double ridge, double* weights,
                    double* intercept, int32_t* status);
/* fit_forest (forest.cpp:124-143): Rng(derive_seed(seeds[m], t)) bootstraps, trees of up to
 * nodes_per_tree = 2 * max(n_rows) nodes each, written in the reference's depth-first preorder
 * to node_* [n_models][trees][nodes_per_tree]; node_count [n_models][trees]. */
int lann_fit_forest(lann_engine* engine, const lann_design* design, int32_t trees, int32_t max_depth,
                    int32_t min_samples_split, const uint64_t* seeds, int32_t* node_feature,
                    double* node_threshold, int32_t* node_left, int32_t* node_right, double* node_value,
                    int32_t* node_count);
/* LinearModel / Forest prediction (models.cpp:357-362, forest.cpp:13-27), max(v, 1e-9). */
int lann_predict_linear(lann_engine* engine, int32_t n_models, const int32_t* n_feats, const double* weights,
                        const double* intercept, int64_t n_rows, const double* rows, const int32_t* row_model,
                        double* out);
int lann_predict_forest(lann_engine* engine, int32_t n_models, int32_t trees, int32_t nodes_per_tree,
                        const int32_t* node_feature, const double* node_threshold, const int32_t* node_left,
                        const int32_t* node_right, const double* node_value, int64_t n_rows, const double* rows,
                        const int32_t* row_model, double* out);

/* Glorot-uniform init (Mlp::init, mlp.cpp:9-25) with Rng(derive_seed(seed, 0xA11CE)). */
int lann_init_params(int32_t n_dims, const int32_t* dims, uint64_t seed, double* params);

/* ---- whole-population pipeline ----------------------------------------------------
 * For every job: build dataset -> split -> (fold) -> NormStats -> init ->
 * train (one batched launch set) -> predict on the evaluation part -> metrics.
 * params_out (optional) receives trained weights at results-indexed offsets
 * params_offset[j]; trace (optional) full loss traces at trace_offset[j]. */
int lann_run_population(lann_engine* engine, int32_t n_jobs, const lann_job* jobs,
                        int32_t precision, lann_job_result* results,
                        double* params_out, const int64_t* params_offset,
                        double* trace_out, const int64_t* trace_offset);

/* Prepared population: the same pipeline split so that the host preparation and
 * the uploads happen once (create), device-only passes can be repeated with all
 * inputs resident in HBM (run: weights reset from the resident initial copy,
 * train, predict, metrics; n_steps passes back to back), and results are copied
 * out on demand (fetch). lann_run_population == create + run(1) + fetch. */
typedef struct lann_population lann_population;
int lann_population_create(lann_engine* engine, int32_t n_jobs, const lann_job* jobs,
                           int32_t precision, int32_t record_trace, lann_population** out);
int lann_population_run(lann_population* pop, int32_t n_steps);
int lann_population_fetch(lann_population* pop, lann_job_result* results, double* params_out,
                          const int64_t* params_offset, double* trace_out,
                          const int64_t* trace_offset);
/* algorithmic training FLOP of one pass (sum E * (N*F_s + 14P)) */
double lann_population_flop(const lann_population* pop);
/* per job: the model's NormStats {f_min[8], f_max[8], t_min, t_max} (zeros for failed jobs) */
int lann_population_norm(const lann_population* pop, double* norm_out);
/* host->device / device->host bytes moved by this thread's engine calls since the last reset */
void lann_transfer_bytes(int64_t* h2d, int64_t* d2h, int32_t reset);
int64_t lann_population_models(const lann_population* pop);
/* frees the population; destroying its engine frees every population still alive (their handles
 * are then invalid, and destroying one of them again is a no-op) */
void lann_population_destroy(lann_population* pop);

/* ---- cross-validation summary of a k-fold sweep (BASELINE config 3) -------------
 * The reference has no k-fold driver; its primitives are split (datagen.cpp:225-248),
 * predict_dataset (models.cpp:365-378), make_report (eval.cpp:98-108) and aggregate's per-group
 * means (eval.cpp:110-146). Definitions (restated in oracle/lann_oracle.c, or_fold_mean):
 *  - CV GROUP: the k-fold jobs (n_folds >= 2) equal in every field except fold and init_seed
 *    (one combination x family x hyper-parameters); groups in order of first appearance.
 *  - ENSEMBLE: one init_seed of a group (order of first appearance). When all k folds are present
 *    and every one trained and evaluated OK, its FOLD-MEAN model predicts the split's test part
 *    (the samples no fold trains or validates on) as (p_0 + p_1 + ... + p_{k-1}) / k, summed in
 *    fold order, each p_f = models::predict of fold f's model with its own NormStats, and is
 *    scored with make_report (drop fraction 0.3).
 *  - Group statistics over the group's OK models (held-out fold metrics, job order) and its OK
 *    ensembles (fold-mean test metrics, ensemble order): mean = the values summed sequentially in
 *    that order / count (aggregate's rule); median = the middle of the sorted values, (a + b) / 2
 *    of the two middles for an even count.
 * A prepared population with k-fold jobs computes all of it on the device in every pass
 * (lann_population_run), after training and the held-out metrics. */
typedef struct lann_cv_stat {
  double mean, median;
} lann_cv_stat;
typedef struct lann_cv_group {
  int32_t first_job;       /* the group's first job (its world / family / hyper-parameters) */
  int32_t n_folds;
  int32_t n_models;        /* the group's jobs */
  int32_t n_models_ok;     /* ... that trained and evaluated OK (fold statistics are over these) */
  int32_t n_ensembles;     /* distinct init seeds */
  int32_t n_ensembles_ok;  /* ... complete, every member OK, test metrics OK */
  int32_t n_test;          /* test-part samples */
  int32_t reserved;
  lann_cv_stat fold_mape, fold_mape_thr, fold_rho; /* held-out fold metrics */
  lann_cv_stat test_mape, test_mape_thr, test_rho; /* fold-mean model on the test part */
} lann_cv_group;
typedef struct lann_cv_ensemble {
  int32_t group;           /* index into the groups */
  int32_t status;          /* LANN_OK; else why no fold-mean score: a missing fold (LANN_PARAM_ERROR),
                              a member's own status, or make_report's (LANN_DOMAIN_ERROR) */
  uint64_t init_seed;
  double mape, mape_thr, rho;
  int32_t n_kept, n_test;
} lann_cv_ensemble;
/* host only (no device): how many groups / ensembles a job list forms */
int lann_cv_layout(int32_t n_jobs, const lann_job* jobs, int32_t* n_groups, int32_t* n_ensembles);
/* the last pass's summary; arrays sized by lann_cv_layout (or lann_population_cv_count) */
int lann_population_cv_count(const lann_population* pop, int32_t* n_groups, int32_t* n_ensembles);
int lann_population_cv(lann_population* pop, lann_cv_group* groups, lann_cv_ensemble* ensembles);
/* the group statistics from per-job results and per-ensemble scores already on the host (merging
 * shards that ran on several devices or processes), computed on the engine's device; ensembles in
 * lann_cv_layout order, groups written (sized by lann_cv_layout) */
int lann_cv_summarize(lann_engine* engine, int32_t n_jobs, const lann_job* jobs, const lann_job_result* results,
                      const lann_cv_ensemble* ensembles, lann_cv_group* groups);

/* The 48 kernel-variant-hardware combinations of BASELINE config 2 (worlds
 * only). Writes up to cap entries, returns the count. */
int lann_default_combos(lann_world* out, int32_t cap);

/* ---- multi-GPU populations ("multiple models may be trained concurrently",
 * SPEC.md:327) ---------------------------------------------------------------------------
 * A group owns one engine per listed device. lann_group_run_population cuts the job list into
 * contiguous, cost-balanced shards (cost = epochs x train rows x parameters, so a combination's
 * seeds and folds stay together and share their tile), runs every shard through
 * lann_run_population on its own device from its own host thread, and writes the results (and
 * optional weights / loss traces, offsets as in lann_run_population) into the caller's arrays in
 * job order. Shards exchange nothing: no device-to-device traffic, no collective, no NCCL. A
 * device may be listed more than once (its shards then share it). FP64-exact results do not
 * depend on the sharding. */
typedef struct lann_group lann_group;
int lann_group_create(int32_t n_devices, const int32_t* devices, lann_group** out);
void lann_group_destroy(lann_group* group);
const char* lann_group_last_error(const lann_group* group);
int32_t lann_group_size(const lann_group* group);
/* the shard cut for n_jobs jobs over n_shards devices (host only, no device needed):
 * bounds[0] = 0 <= bounds[1] <= ... <= bounds[n_shards] = n_jobs; cost-balanced, each cut then
 * moved forward past adjacent jobs of the same cross-validation ensemble */
int lann_shard_bounds(int32_t n_shards, int32_t n_jobs, const lann_job* jobs, int32_t* bounds);
int lann_group_shard_bounds(const lann_group* group, int32_t n_jobs, const lann_job* jobs, int32_t* bounds);
int lann_group_run_population(lann_group* group, int32_t n_jobs, const lann_job* jobs, int32_t precision,
                              lann_job_result* results, double* params_out, const int64_t* params_offset,
                              double* trace_out, const int64_t* trace_offset);
/* lann_group_run_population with the cross-validation summary of the whole job list: the jobs
 * of every ensemble are placed next to each other (ensembles in order of first appearance) and
 * shard cuts never split an ensemble, each device scores its ensembles' fold-mean models, and the
 * group statistics over all shards are computed on the first device (lann_cv_summarize). Results
 * come back in job order; groups / ensembles sized by lann_cv_layout. FP64-exact summaries do not
 * depend on the number of devices. */
int lann_group_run_cv(lann_group* group, int32_t n_jobs, const lann_job* jobs, int32_t precision,
                      lann_job_result* results, lann_cv_group* groups, lann_cv_ensemble* ensembles);
/* device time of the last run: the maximum over the group's devices (their shards run
 * concurrently), and the wall time of the whole call */
double lann_group_last_device_ms(const lann_group* group);
double lann_group_last_wall_ms(const lann_group* group);

#ifdef __cplusplus
}
#endif
#endif /* LANN_ENGINE_H */
