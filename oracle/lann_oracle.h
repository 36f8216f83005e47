/*
 * oracle/lann_oracle.h — TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * Plain-C restatement of the reference's LANN hot path (perfsage core,
 * proj/core/src/{rng,kernels,features,datagen,mlp,models,eval,selector}) in
 * FP64 with the reference's exact operation order. Only tests/, the smoke()
 * check and bench.py's cpu_baseline leg may load it; the product never does.
 * Pinned against the reference itself (oracle/_ref/libperfsage_ref.so, built
 * from the reference sources) and the golden vectors in tests/golden/.
 */
#ifndef LANN_ORACLE_H
#define LANN_ORACLE_H

#include <stdint.h>

#include "../include/lann_engine.h"

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp */
uint64_t or_splitmix64(uint64_t* state);
uint64_t or_derive_seed(uint64_t root, uint64_t stream);

/* dataset build + split (datagen.cpp:177-248); feats rows are LANN_ROW wide */
int or_build_dataset(const lann_world* w, uint64_t seed, int count, double* feats, uint64_t* c,
                     double* rt, int* n_features);
int or_split_order(int n, double frac, uint64_t seed, int64_t* order, int* n_train);

/* mlp.cpp */
int or_mlp_init(int n_dims, const int* dims, uint64_t seed, int raw_rng, double* params);
int or_mse_gradient(int n_dims, const int* dims, const double* params, int n, const double* X,
                    const double* y, double* loss, double* grad);
int or_train_full_batch(int n_dims, const int* dims, double* params, int n, const double* X,
                        const double* y, double lr, int epochs, double* trace, int* bad_epoch);

/* models.cpp: NormStats fit on model-input rows (I wide inside LANN_ROW rows) */
void or_norm_fit(int n, int I, const double* X, const double* y, int log_target, double* norm);
double or_predict_row(int I, int n_hidden, const int* hidden, const double* params,
                      const double* norm, int log_target, const double* x);

/* eval.cpp */
int or_mape(int n, const double* t, const double* p, double* out);
int or_mape_thresholded(int n, const double* t, const double* p, double drop, double* out,
                        int* kept);
int or_spearman(int n, const double* t, const double* p, double* out);

/* selector.cpp:26-53 */
int64_t or_select_schedule(int family, int n_hidden, const int* hidden, const double* params,
                           const double* norm, int log_target, uint32_t n_img, int64_t n_cands,
                           const uint32_t* cands, double* score);

/* counter-based candidate shapes + multi-variant argmin (engine definition) */
void or_candidate(int kind, int max_threads, uint64_t seed, int64_t idx, double* base,
                  uint64_t* c);
void or_select_variants(const lann_model_set* models, const int32_t* with_n_thd, int kind,
                        int max_threads, uint64_t seed, int64_t first, int64_t n_cands,
                        int32_t* out_idx, double* out_score);

/* whole job (acceptance criterion-5 protocol, acceptance_main.cpp:283-328) */
int or_run_job(const lann_job* job, lann_job_result* r, double* params, double* trace);
/* cross-validation fold-mean model of one seed's k fold models on the split's test part */
int or_fold_mean(int k, const lann_job* fold_jobs, const double* const* params, double* pred, double* truth,
                 int* n_test);

#ifdef __cplusplus
}
#endif
#endif
