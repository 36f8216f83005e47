// kernels.cuh — device-side argument blocks shared by the engine's CUDA kernels
// and the host launcher (engine.cpp). Plain structs of device pointers.
#pragma once

#include <cstdint>
#include <string>

#include <cuda_runtime.h>

namespace lann {

// One launch of the trainer over a population (see lann_train_batch).
struct TrainArgs {
  int n_models;
  const int* order;          // model processing order (longest first)
  const int* tile_rows;
  const int* tile_inputs;
  const int64_t* tile_offset;
  const double* X;           // [rows][8] normalised inputs
  const double* y;           // [rows]
  const int* model_tile;
  const int* h1;
  const int* h2;
  const double* lr;
  const int* epochs;
  const int64_t* param_offset;
  double* params;            // in/out
  double* final_loss;
  int* nonfinite_epoch;
  double* loss_trace;        // may be null
  const int64_t* trace_offset;
  int trace_stride;
  const double2* bias_corr;  // [max_epochs] {1-0.9^t, 1-0.999^t} from the host libm
  double* scratch;           // global per-sample records for models too big for smem
  const int64_t* scratch_offset;
  int smem_records;          // 1: per-sample records live in shared memory
  int rec_products;          // 1: phase A also stores every weight's per-sample product row
  int rec_chunk = 0;         // > 0: shared-memory records hold this many samples at a time (chunks
                             // of the sample range processed in order; the chains carry over)
  long long* phase_cycles;   // optional (LANN_PHASE_PROFILE): CTA 0's clock64 per phase
  int prof_flags = 0;        // profiling experiments (LANN_PROF_FLAGS), only read under phase_cycles
};

// FP32 throughput trainer: models grouped into warps that share one tile.
struct TrainF32Args {
  int n_groups;
  const int* group_first;    // first model (index into the sorted model list) of each group
  const int* group_count;    // models in the group (<= 32 / lanes-per-model)
  const int* sorted_model;   // engine model index for each sorted slot
  const float* rows;         // [rows][8]: x0..x6 (padded), y at column 7
  const int* tile_rows;
  const int64_t* tile_offset;
  const int* model_tile;
  const double* lr;
  const int* epochs;
  const int64_t* param_offset;
  double* params;            // in/out (fp64 in the ABI, fp32 inside)
  double* final_loss;
  int* nonfinite_epoch;
  double* loss_trace;
  const int64_t* trace_offset;
  int trace_stride;
  long long* phase_cycles;   // optional (LANN_PHASE_PROFILE): CTA 0's clock64 per phase
  const float2* bias_rcp;    // [max_epochs] {1/(1-0.9^t), 1/(1-0.999^t)} from the host (CTA kernel)
};

// FP32 trainer for the shapes without a compiled FP32 kernel (unconstrained widths, any 1-2 hidden
// layers up to 64 units, I <= 7): one model per CTA, records in shared memory a chunk of samples
// at a time (train_fp32.cu, train_fp32_wide_kernel).
struct TrainWideArgs {
  int n_models;
  const int* order;          // engine model indices of the launch
  const float* rows;         // packed FP32 rows [rows][8]: x0..x6, y at column 7
  const int* tile_rows;
  const int* tile_inputs;
  const int64_t* tile_offset;
  const int* model_tile;
  const int* h1;
  const int* h2;
  const double* lr;
  const int* epochs;
  const int64_t* param_offset;
  double* params;            // in/out (fp64 in the ABI, fp32 inside)
  double* final_loss;
  int* nonfinite_epoch;
  double* loss_trace;
  const int64_t* trace_offset;
  int trace_stride;
  const float2* bias_rcp;    // [max_epochs] {1/(1-0.9^t), 1/(1-0.999^t)}
  int chunk;                 // samples per shared-memory record chunk
  int max_p;                 // largest parameter count of the launch
};
bool fp32_wide_supported(int in, int h1, int h2);
int fp32_wide_rows(int h1, int h2);
size_t fp32_wide_smem_bytes(int max_p, int rows, int chunk);
void launch_train_fp32_wide(const TrainWideArgs& a, int dyn_bytes, cudaStream_t s);

// Prediction over rows (models.cpp:346-363).
struct PredictArgs {
  int64_t n_rows;
  const double* rows;        // raw model inputs [n][8]
  const int* row_model;
  const int* n_inputs;
  const int* h1;
  const int* h2;
  const int* log_target;
  const int64_t* param_offset;
  const double* params;
  const double* norm;        // [models][18]
  double* out;
};

// Metrics over packed (truth, pred) sets (eval.cpp:26-90).
struct EvalArgs {
  int n_sets;
  const int64_t* offset;
  const int* len;
  const double* truth;
  const double* pred;
  double drop_fraction;
  double* mape;
  double* mape_thr;
  int* n_kept;
  double* rho;
  int* status;
};

// Cross-validation fold-mean models (lann_engine.h, "cross-validation summary"): every ensemble's
// k fold models predict its test part, the predictions are averaged in fold order.
struct FoldMeanArgs {
  int n_ens;
  int kmax;
  const int* ens_k;          // folds of the ensemble
  const int* ens_models;     // [n_ens][kmax] engine model index of fold f
  const int64_t* ens_rows;   // first test row of the ensemble's test set (into rows / truth)
  const int* ens_len;        // test rows
  const int64_t* ens_out;    // first output slot
  const double* rows;        // raw model inputs [n][8]
  const double* truth;       // [n]
  const int* model_bad;      // per model: non-finite epoch (>= 0: TrainingError)
  const int* model_status;   // per model: held-out metrics status (0 ok)
  double* pred;              // [total] fold-mean predictions
  double* truth_out;         // [total] the ensemble's truth beside them (an eval set)
  int* ens_bad;              // per ensemble: -1, or 2 f + (0: fold f diverged, 1: fold f had no metrics)
};

// Group statistics (mean in item order, median of the sorted values) of three metrics over the
// OK items of each group: item i is OK when status[i] == 0 and bad[i] < 0.
struct CvStatsArgs {
  int n_groups;
  const int64_t* item_off;
  const int* item_len;
  const int* items;          // item ids, per group in order
  const double* m0;          // metric arrays indexed by item id
  const double* m1;
  const double* m2;
  const int* status;
  const int* bad;
  double* out;               // [group][6]: mean, median of m0, m1, m2
  int* n_ok;                 // [group]
  double* scratch;           // [total items]: the compacted values of one metric
};

// shape = {I, H1, H2} when every model of the launch has that compiled shape, else null
void launch_train_fp64(const TrainArgs& a, int max_p, int dyn_bytes, const int* shape, cudaStream_t s);
bool fp64_shape_compiled(int in, int h1, int h2);
// pipelined exact trainer (train_fp64_pipe.cu): compiled shapes with N <= 256
bool fp64_pipe_shape(int in, int h1, int h2);
bool launch_train_fp64_pipe(const TrainArgs& a, int I, int H1, int H2, int producer_warps, cudaStream_t s);
// FP64 trainer footprint (see train_fp64.cu): record matrix of a model, model state
size_t fp64_record_bytes(int in, int h1, int h2, int n);
size_t fp64_product_record_bytes(int in, int h1, int h2, int n);
size_t fp64_state_bytes(int p);
int fp64_record_rows(int h1, int h2);
int fp64_chunk_ld(int ch);  // row stride (doubles) of chunked shared-memory records
bool launch_train_fp32(const TrainF32Args& a, int in, int h1, int h2, int lanes, int tile_bytes,
                       cudaStream_t s);
bool fp32_shape_supported(int in, int h1, int h2);
int fp32_warp_slots_per_sm(int in, int h1, int h2, int lanes, int tile_bytes);
void launch_predict_fp64(const PredictArgs& a, cudaStream_t s);
void launch_predict_fp32(const PredictArgs& a, int n_models, int64_t n_params, cudaStream_t s);
void launch_eval(const EvalArgs& a, int max_len, int max_smem, int64_t total, cudaStream_t s);
int eval_launch_count(int max_len, int max_smem);
// fold-mean predictions of every ensemble (the population's PredictArgs give the models);
// FP32 populations predict with the FP32 forward like launch_predict_fp32
void launch_fold_mean(const PredictArgs& pa, const FoldMeanArgs& f, int max_len, bool exact, int n_models,
                      int64_t n_params, cudaStream_t s);
void launch_cv_stats(const CvStatsArgs& a, cudaStream_t s);

}  // namespace lann

namespace lann {
// select.cu
int select_schedule_launch(int64_t n, const uint32_t* d_cands, uint32_t n_img, int I, int H1,
                           int H2, int logt, const double* d_w, const double* d_nrm,
                           double* d_blk_score, int64_t* d_blk_idx, cudaStream_t s);
bool select_variants_supported(int n_models, int max_params);
// FP32 fast path (one hidden layer of 8, <= 16 models): weights folded with the
// normalisation on the host, passed as a __grid_constant__ parameter. Host pointers.
bool select_variants_fast_launch(int n_models, int kind, int max_threads, uint64_t seed, int64_t first,
                                 int64_t n, const int* n_inputs, const int* h1, const int* h2,
                                 const int* logt, const int* with_thd, const int64_t* param_offset,
                                 const double* params, const double* norm, void* d_idx, void* d_score,
                                 bool compact, unsigned long long* d_hist, int sms, cudaStream_t s);
int select_variants_launch(int n_models, int precision, int kind, int max_threads, uint64_t seed,
                           int64_t first, int64_t n, const int* d_in, const int* d_h1,
                           const int* d_h2, const int* d_logt, const int* d_thd,
                           const int64_t* d_poff, const double* d_params, const double* d_norm,
                           void* d_idx, void* d_score, bool compact, unsigned long long* d_hist, int sms,
                           cudaStream_t s);
}  // namespace lann

namespace lann {
void launch_pack_rows(const double* X, const double* y, int64_t n, float* out, cudaStream_t s);
}  // namespace lann

namespace lann {
// measure.cu — B200 GPU-class kernel variants timed with CUDA events
int measure_variant_count(int kind);
const char* measure_variant_name(int kind, int idx);
int measure_instances(int kind, const char* variant, int n, const double* feats, int warmups, int reps,
                      uint64_t seed, double* runtime_s, double* checksum, cudaStream_t s, std::string& err);
}  // namespace lann

namespace lann {
// baselines.cu — const / lrc least squares and the nlrc forest
struct LinearArgs {
  int n_models;
  const int* n_rows;
  const int* n_feats;         // columns of the design (1 for const)
  const int64_t* row_offset;
  const double* X;            // raw features [rows][LANN_ROW]
  const double* y;            // raw runtimes
  double ridge;
  double* weights;            // [n_models][LANN_ROW]
  double* intercept;
  int* status;                // 0 ok, 1 singular despite ridge (FitError)
};
struct PredictLinearArgs {
  int64_t n_rows;
  const double* rows;         // [n][LANN_ROW] raw features
  const int* row_model;
  const int* n_feats;
  const double* weights;
  const double* intercept;
  double* out;
};
struct ForestArgs {
  int n_models, trees, max_depth, min_samples_split, max_rows;
  const int* n_rows;
  const int* n_feats;
  const int64_t* row_offset;
  const double* X;
  const double* y;
  const uint16_t* bootstrap;  // [model][tree][max_rows] sorted sample indices
  int* node_feature;          // [model][tree][2 max_rows], breadth-first
  double* node_threshold;
  int* node_left;
  int* node_right;
  double* node_value;
  int* node_count;            // [model][tree]
  double* scratch_sse;        // [model][tree][max_rows][LANN_ROW]
  double* scratch_thr;
  unsigned char* scratch_ws = nullptr;  // non-null: the working set in global memory, ws_stride B per CTA
  size_t ws_stride = 0;
};
struct PredictForestArgs {
  int64_t n_rows;
  const double* rows;
  const int* row_model;
  int trees, nodes_per_tree;
  const int* node_feature;    // [model][tree][nodes_per_tree]
  const double* node_threshold;
  const int* node_left;
  const int* node_right;
  const double* node_value;
  double* out;
};
void launch_fit_linear(const LinearArgs& a, cudaStream_t s);
void launch_predict_linear(const PredictLinearArgs& a, cudaStream_t s);
size_t forest_smem_bytes(int max_rows);
void launch_fit_forest(const ForestArgs& a, cudaStream_t s);
void launch_predict_forest(const PredictForestArgs& a, cudaStream_t s);
}  // namespace lann

namespace lann {
// mlp_ops.cu: mlp.hpp's per-net operations (Mlp::forward, mse_loss, mse_gradient,
// AdamState::update) on the GPU, batched over nets of any depth <= kMaxLayers
constexpr int kMaxLayers = 8;
constexpr int kMaxMlpWidth = 64;
struct MlpArgs {
  int n_nets;
  const int* n_dims;          // per net: L + 1 (inputs, hidden..., outputs)
  const int64_t* dims_offset; // into dims
  const int* dims;
  const int64_t* param_offset;
  const int* n_params;
  const double* params;
  const int64_t* row_offset;  // first row of the net (into y and the global row index)
  const int* n_rows;
  const int64_t* x_offset;    // first double of the net's rows (row stride = dims[0])
  const double* X;
  const double* y;
  const int* row_net;         // per global row: its net
  int64_t total_rows;
};
struct AdamArgs {
  int64_t n;
  double* params;
  const double* grad;
  double* m;
  double* v;
  double beta1, beta2, eps, lr, bc1, bc2;
};
void launch_mlp_forward(const MlpArgs& a, double* out, cudaStream_t s);
void launch_mlp_loss(const MlpArgs& a, const double* fwd, double* loss, cudaStream_t s);
void launch_mlp_grad(const MlpArgs& a, double* scratch, const int64_t* scratch_offset, double* loss, double* grad,
                     cudaStream_t s);
void launch_adam(const AdamArgs& a, cudaStream_t s);
}  // namespace lann
