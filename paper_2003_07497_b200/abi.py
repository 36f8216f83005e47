"""ctypes mirrors of the plain structs in include/lann_engine.h (layout only, no logic)."""
from __future__ import annotations

import ctypes as C

ROW = 8  # LANN_ROW

# lann_status
OK, PARAM_ERROR, SCHEMA_ERROR, TRAINING_ERROR, DOMAIN_ERROR, BUILD_ABORT, CUDA_ERROR, NO_DEVICE = range(8)
# lann_precision
FP64_EXACT, FP32 = 0, 1
# lann_kind (kernels.hpp:13)
MM, MV, MC, MP, BLUR = range(5)
# lann_family
NNC, NN = 0, 1
HW_CPU, HW_GPU = 0, 1


class World(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("hw_class", C.c_int32), ("max_threads", C.c_int32), ("blur_lattice", C.c_int32),
        ("alpha", C.c_double), ("g0", C.c_double), ("g1", C.c_double), ("delta", C.c_double),
        ("beta", C.c_double), ("noise", C.c_double),
        ("mu", C.c_double * 4), ("kappa", C.c_double * 4),
    ]


class Job(C.Structure):
    _fields_ = [
        ("world", World), ("data_seed", C.c_uint64), ("count", C.c_int32), ("train_fraction", C.c_double),
        ("n_folds", C.c_int32), ("fold", C.c_int32), ("family", C.c_int32), ("n_hidden", C.c_int32),
        ("hidden", C.c_int32 * 2), ("learning_rate", C.c_double), ("epochs", C.c_int32),
        ("init_seed", C.c_uint64), ("log_target", C.c_int32), ("unconstrained", C.c_int32),
    ]


class JobResult(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("nonfinite_epoch", C.c_int32), ("n_inputs", C.c_int32), ("n_params", C.c_int32),
        ("n_train", C.c_int32), ("n_eval", C.c_int32), ("final_loss", C.c_double), ("mape", C.c_double),
        ("mape_thr", C.c_double), ("rho", C.c_double), ("n_kept", C.c_int32), ("precision_run", C.c_int32),
    ]


class CvStat(C.Structure):
    _fields_ = [("mean", C.c_double), ("median", C.c_double)]


class CvGroup(C.Structure):
    """lann_cv_group: one combination x family x hyper-parameters of a k-fold sweep."""
    _fields_ = [
        ("first_job", C.c_int32), ("n_folds", C.c_int32), ("n_models", C.c_int32), ("n_models_ok", C.c_int32),
        ("n_ensembles", C.c_int32), ("n_ensembles_ok", C.c_int32), ("n_test", C.c_int32), ("reserved", C.c_int32),
        ("fold_mape", CvStat), ("fold_mape_thr", CvStat), ("fold_rho", CvStat),
        ("test_mape", CvStat), ("test_mape_thr", CvStat), ("test_rho", CvStat),
    ]


class CvEnsemble(C.Structure):
    """lann_cv_ensemble: one init seed's fold-mean model scored on the split's test part."""
    _fields_ = [
        ("group", C.c_int32), ("status", C.c_int32), ("init_seed", C.c_uint64), ("mape", C.c_double),
        ("mape_thr", C.c_double), ("rho", C.c_double), ("n_kept", C.c_int32), ("n_test", C.c_int32),
    ]


class TrainBatch(C.Structure):
    _fields_ = [
        ("n_models", C.c_int32), ("precision", C.c_int32), ("n_tiles", C.c_int32),
        ("tile_rows", C.c_void_p), ("tile_inputs", C.c_void_p), ("tile_offset", C.c_void_p),
        ("total_rows", C.c_int64), ("X", C.c_void_p), ("y", C.c_void_p),
        ("model_tile", C.c_void_p), ("model_h1", C.c_void_p), ("model_h2", C.c_void_p),
        ("model_lr", C.c_void_p), ("model_epochs", C.c_void_p), ("model_param_offset", C.c_void_p),
        ("total_params", C.c_int64), ("params", C.c_void_p), ("final_loss", C.c_void_p),
        ("nonfinite_epoch", C.c_void_p), ("loss_trace", C.c_void_p), ("trace_offset", C.c_void_p),
        ("trace_stride", C.c_int32),
    ]


class ModelSet(C.Structure):
    _fields_ = [
        ("n_models", C.c_int32), ("precision", C.c_int32),
        ("n_inputs", C.c_void_p), ("h1", C.c_void_p), ("h2", C.c_void_p), ("log_target", C.c_void_p),
        ("param_offset", C.c_void_p), ("params", C.c_void_p), ("total_params", C.c_int64), ("norm", C.c_void_p),
    ]


class MlpBatch(C.Structure):
    """lann_mlp_batch: generic nets for lann_mlp_forward / lann_mse_loss / lann_mse_gradient."""
    _fields_ = [
        ("n_nets", C.c_int32), ("n_dims", C.c_void_p), ("dims", C.c_void_p), ("params", C.c_void_p),
        ("n_rows", C.c_void_p), ("X", C.c_void_p), ("y", C.c_void_p),
    ]


def acceptance_world() -> World:
    """acceptance_main.cpp:271-289: MM dense_threaded, max_threads 4, t = 3e-9 c (0.25+0.75/n_thd)(1+U(-2%,2%))."""
    return World(kind=MM, hw_class=HW_CPU, max_threads=4, blur_lattice=0, alpha=3e-9, g0=0.25, g1=0.75,
                 delta=0.0, beta=0.0, noise=0.02)


def make_job(world: World, data_seed: int, *, count=500, train_fraction=0.5, n_folds=0, fold=0, family=NNC,
             hidden=(8,), lr=1e-2, epochs=8000, init_seed=None, log_target=False, unconstrained=False) -> Job:
    j = Job()
    j.world = world
    j.data_seed = data_seed
    j.count = count
    j.train_fraction = train_fraction
    j.n_folds = n_folds
    j.fold = fold
    j.family = family
    j.n_hidden = len(hidden)
    j.hidden[0] = hidden[0]
    j.hidden[1] = hidden[1] if len(hidden) > 1 else 0
    j.learning_rate = lr
    j.epochs = epochs
    j.init_seed = data_seed if init_seed is None else init_seed
    j.log_target = int(log_target)
    j.unconstrained = int(unconstrained)
    return j
