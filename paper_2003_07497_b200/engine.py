"""Python host binding of the engine's C ABI (include/lann_engine.h) via ctypes.

The compute path is the in-tree CUDA library ``lib/libperfsage_b200.so``. There is no
Python or CPU fallback: if the library is missing, loading fails loudly; if no CUDA
device is present, ``Engine()`` raises ``NoDeviceError``.

Error behaviour mirrors the reference's exceptions (include/perfsage/errors.hpp):
status codes are re-raised as ``ParamError``, ``SchemaError``, ``TrainingError``
(with ``.epoch``), ``DomainError`` and ``BuildAbortError``.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref

import numpy as np

from . import abi
from .abi import ROW, CvEnsemble, CvGroup, Job, JobResult, MlpBatch, ModelSet, TrainBatch, World

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libperfsage_b200.so")


class Error(RuntimeError):
    """perfsage::Error"""


class ParamError(Error):
    pass


class SchemaError(Error):
    pass


class DomainError(Error):
    pass


class BuildAbortError(Error):
    pass


class CudaError(Error):
    pass


class NoDeviceError(Error):
    pass


class TrainingError(Error):
    def __init__(self, msg, epoch):
        super().__init__(msg)
        self.epoch = epoch


_ERR = {abi.PARAM_ERROR: ParamError, abi.SCHEMA_ERROR: SchemaError, abi.DOMAIN_ERROR: DomainError,
        abi.BUILD_ABORT: BuildAbortError, abi.CUDA_ERROR: CudaError, abi.NO_DEVICE: NoDeviceError}

_lib = None

# every symbol include/lann_engine.h declares
EXPORTS = ["lann_engine_create", "lann_engine_destroy", "lann_last_error", "lann_last_device_ms",
           "lann_last_launches", "lann_last_train_ms", "lann_train", "lann_predict", "lann_eval",
           "lann_select_schedule", "lann_select_variants", "lann_build_dataset", "lann_split_order", "lann_probe_schedules", "lann_measure",
           "lann_measure_variant_count", "lann_measure_variant_name", "lann_build_measured_dataset",
           "lann_fit_linear", "lann_fit_forest", "lann_predict_linear", "lann_predict_forest",
           "lann_build_mock_dataset", "lann_mock_schedules",
           "lann_init_params", "lann_population_create", "lann_population_run", "lann_population_fetch",
           "lann_population_flop", "lann_population_models", "lann_population_destroy",
           "lann_population_norm", "lann_transfer_bytes", "lann_run_population", "lann_default_combos",
           "lann_mlp_forward", "lann_mse_loss", "lann_mse_gradient", "lann_adam_update",
           "lann_group_create", "lann_group_destroy", "lann_group_last_error", "lann_group_size",
           "lann_shard_bounds", "lann_group_shard_bounds", "lann_group_run_population",
           "lann_group_last_device_ms", "lann_group_last_wall_ms",
           "lann_select_variants_compact", "lann_host_alloc", "lann_host_free",
           "lann_cv_layout", "lann_population_cv_count", "lann_population_cv", "lann_cv_summarize",
           "lann_group_run_cv"]


def transfer_bytes(reset=False):
    """(h2d, d2h) bytes moved by this thread's engine calls since the last reset."""
    L = load_library()
    h, d = C.c_int64(0), C.c_int64(0)
    L.lann_transfer_bytes(C.addressof(h), C.addressof(d), int(reset))
    return h.value, d.value


def load_library(path: str = LIB_PATH):
    """Load the engine's shared library (raises OSError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OSError(f"engine library {path} is missing: run __graft_entry__.build() / make -C "
                      f"paper_2003_07497_b200/csrc")
    L = C.CDLL(path)
    vp = C.c_void_p
    L.lann_engine_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.lann_engine_destroy.argtypes = [vp]
    L.lann_last_error.argtypes = [vp]
    L.lann_last_error.restype = C.c_char_p
    L.lann_last_device_ms.argtypes = [vp]
    L.lann_last_device_ms.restype = C.c_double
    L.lann_last_launches.argtypes = [vp]
    L.lann_last_launches.restype = C.c_int64
    L.lann_last_train_ms.argtypes = [vp]
    L.lann_last_train_ms.restype = C.c_double
    L.lann_population_create.argtypes = [vp, C.c_int32, C.POINTER(Job), C.c_int32, C.c_int32, C.POINTER(vp)]
    L.lann_population_run.argtypes = [vp, C.c_int32]
    L.lann_population_fetch.argtypes = [vp, C.POINTER(JobResult), vp, vp, vp, vp]
    L.lann_population_flop.argtypes = [vp]
    L.lann_population_flop.restype = C.c_double
    L.lann_population_models.argtypes = [vp]
    L.lann_population_models.restype = C.c_int64
    L.lann_population_destroy.argtypes = [vp]
    L.lann_population_norm.argtypes = [vp, vp]
    L.lann_transfer_bytes.argtypes = [vp, vp, C.c_int32]
    L.lann_cv_layout.argtypes = [C.c_int32, C.POINTER(Job), vp, vp]
    L.lann_population_cv_count.argtypes = [vp, vp, vp]
    L.lann_population_cv.argtypes = [vp, C.POINTER(CvGroup), C.POINTER(CvEnsemble)]
    L.lann_cv_summarize.argtypes = [vp, C.c_int32, C.POINTER(Job), C.POINTER(JobResult), C.POINTER(CvEnsemble),
                                    C.POINTER(CvGroup)]
    L.lann_group_run_cv.argtypes = [vp, C.c_int32, C.POINTER(Job), C.c_int32, C.POINTER(JobResult),
                                    C.POINTER(CvGroup), C.POINTER(CvEnsemble)]
    L.lann_train.argtypes = [vp, C.POINTER(TrainBatch)]
    L.lann_predict.argtypes = [vp, C.POINTER(ModelSet), C.c_int64, vp, vp, vp]
    L.lann_eval.argtypes = [vp, C.c_int32, vp, vp, vp, vp, C.c_double, vp, vp, vp, vp]
    L.lann_select_schedule.argtypes = [vp, C.POINTER(ModelSet), C.c_uint32, C.c_int64, vp, vp, vp]
    L.lann_select_variants.argtypes = [vp, C.POINTER(ModelSet), vp, C.c_int32, C.c_int32, C.c_uint64,
                                       C.c_int64, C.c_int64, vp, vp]
    L.lann_build_dataset.argtypes = [C.POINTER(World), C.c_uint64, C.c_int32, vp, vp, vp, vp]
    L.lann_split_order.argtypes = [C.c_int32, C.c_uint64, vp]
    L.lann_init_params.argtypes = [C.c_int32, vp, C.c_uint64, vp]
    L.lann_run_population.argtypes = [vp, C.c_int32, C.POINTER(Job), C.c_int32, C.POINTER(JobResult),
                                      vp, vp, vp, vp]
    L.lann_default_combos.argtypes = [C.POINTER(World), C.c_int32]
    L.lann_mlp_forward.argtypes = [vp, C.POINTER(MlpBatch), vp]
    L.lann_mse_loss.argtypes = [vp, C.POINTER(MlpBatch), vp]
    L.lann_mse_gradient.argtypes = [vp, C.POINTER(MlpBatch), vp, vp]
    L.lann_adam_update.argtypes = [vp, C.c_int64, vp, vp, vp, vp, C.c_int32, C.c_double, C.c_double, C.c_double,
                                   C.c_double]
    L.lann_select_variants_compact.argtypes = [vp, C.POINTER(ModelSet), vp, C.c_int32, C.c_int32, C.c_uint64,
                                               C.c_int64, C.c_int64, vp, vp, vp]
    L.lann_host_alloc.argtypes = [C.c_size_t, C.POINTER(vp)]
    L.lann_host_free.argtypes = [vp]
    L.lann_group_create.argtypes = [C.c_int32, vp, C.POINTER(vp)]
    L.lann_group_destroy.argtypes = [vp]
    L.lann_group_last_error.argtypes = [vp]
    L.lann_group_last_error.restype = C.c_char_p
    L.lann_group_size.argtypes = [vp]
    L.lann_shard_bounds.argtypes = [C.c_int32, C.c_int32, C.POINTER(Job), vp]
    L.lann_group_shard_bounds.argtypes = [vp, C.c_int32, C.POINTER(Job), vp]
    L.lann_group_run_population.argtypes = [vp, C.c_int32, C.POINTER(Job), C.c_int32, C.POINTER(JobResult),
                                            vp, vp, vp, vp]
    L.lann_group_last_device_ms.argtypes = [vp]
    L.lann_group_last_device_ms.restype = C.c_double
    L.lann_group_last_wall_ms.argtypes = [vp]
    L.lann_group_last_wall_ms.restype = C.c_double
    _lib = L
    return L


def cv_layout(jobs):
    """(groups, ensembles) a job list forms (lann_cv_layout; host only)."""
    L = load_library()
    n = len(jobs)
    arr = (Job * max(1, n))(*jobs)
    ng, ne = C.c_int32(), C.c_int32()
    st = L.lann_cv_layout(n, arr, C.byref(ng), C.byref(ne))
    if st:
        raise ParamError("lann_cv_layout failed")
    return ng.value, ne.value


def _ptr(a):
    return a.ctypes.data if a is not None else None


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def param_count(n_inputs, h1, h2=0):
    """models.cpp:37-46"""
    if h2:
        return (n_inputs + 1) * h1 + (h1 + 1) * h2 + h2 + 1
    return (n_inputs + 1) * h1 + h1 + 1


def default_combos():
    L = load_library()
    arr = (World * 64)()
    n = L.lann_default_combos(arr, 64)
    return [arr[i] for i in range(n)]


def build_dataset(world: World, seed: int, count: int):
    """datagen::build_dataset with the world's probe -> (feats[count][8], c, runtime, n_features)."""
    L = load_library()
    feats = np.zeros((count, ROW))
    c = np.zeros(count, dtype=np.uint64)
    rt = np.zeros(count)
    nf = C.c_int32(0)
    st = L.lann_build_dataset(C.byref(world), seed, count, _ptr(feats), _ptr(c), _ptr(rt), C.addressof(nf))
    if st:
        raise _ERR.get(st, Error)(f"build_dataset failed ({st})")
    return feats, c, rt, nf.value


def init_params(dims, seed):
    """Mlp::init with Rng(derive_seed(seed, 0xA11CE)) (models.cpp:298, mlp.cpp:9-25)."""
    L = load_library()
    d = _c(dims, np.int32)
    P = int(sum((d[i] + 1) * d[i + 1] for i in range(len(d) - 1)))
    out = np.zeros(P)
    st = L.lann_init_params(len(d), _ptr(d), seed, _ptr(out))
    if st:
        raise _ERR.get(st, Error)("bad network dims")
    return out


class Engine:
    """One engine per device (and per host thread): owns a CUDA stream and device memory."""

    def __init__(self, device: int = 0):
        self.L = load_library()
        h = C.c_void_p()
        st = self.L.lann_engine_create(device, C.byref(h))
        if st == abi.NO_DEVICE:
            raise NoDeviceError("no CUDA device: the LANN engine has no CPU fallback")
        if st:
            raise _ERR.get(st, Error)(f"engine creation failed ({st})")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            for p in list(getattr(self, "_pops", ())):  # prepared populations go first
                p.close()
            self.L.lann_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- diagnostics ----
    @property
    def last_error(self) -> str:
        return self.L.lann_last_error(self.h).decode()

    @property
    def last_device_ms(self) -> float:
        return self.L.lann_last_device_ms(self.h)

    @property
    def last_launches(self) -> int:
        return self.L.lann_last_launches(self.h)

    @property
    def last_train_ms(self) -> float:
        return self.L.lann_last_train_ms(self.h)

    def prepare(self, jobs, precision=abi.FP32, record_trace=False):
        """lann_population_create: host preparation + one upload; returns a Population."""
        return Population(self, jobs, precision, record_trace)

    def _raise(self, st, epoch=-1):
        if st == abi.TRAINING_ERROR:
            raise TrainingError(self.last_error, epoch)
        raise _ERR.get(st, Error)(self.last_error or f"status {st}")

    # ---- train_full_batch, batched (mlp.cpp:156-175) ----
    def train(self, tiles_X, tiles_y, models, precision=abi.FP64_EXACT, trace=False, trace_stride=1,
              raise_on_error=True):
        """tiles_X: list of [N][8] arrays (normalised rows), tiles_y: list of [N];
        models: list of dicts {tile, h1, h2, lr, epochs, params}. Returns
        (params list, final_loss, nonfinite_epoch, traces or None)."""
        n_tiles = len(tiles_X)
        rows = np.array([len(y) for y in tiles_y], dtype=np.int32)
        offs = np.concatenate([[0], np.cumsum(rows)[:-1]]).astype(np.int64)
        X = np.zeros((int(rows.sum()), ROW))
        y = np.zeros(int(rows.sum()))
        for k in range(n_tiles):
            xk = np.asarray(tiles_X[k], dtype=np.float64)
            X[offs[k]:offs[k] + rows[k], : xk.shape[1]] = xk
            y[offs[k]:offs[k] + rows[k]] = tiles_y[k]
        inputs = np.array([np.asarray(tiles_X[k]).shape[1] for k in range(n_tiles)], dtype=np.int32)
        M = len(models)
        mt = np.array([m["tile"] for m in models], dtype=np.int32)
        h1 = np.array([m["h1"] for m in models], dtype=np.int32)
        h2 = np.array([m.get("h2", 0) for m in models], dtype=np.int32)
        lr = np.array([m["lr"] for m in models], dtype=np.float64)
        ep = np.array([m["epochs"] for m in models], dtype=np.int32)
        sizes = np.array([len(m["params"]) for m in models], dtype=np.int64)
        poff = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
        params = np.concatenate([np.asarray(m["params"], dtype=np.float64) for m in models])
        final = np.zeros(M)
        bad = np.zeros(M, dtype=np.int32)
        stride = max(1, int(trace_stride))
        tl = (ep + stride - 1) // stride
        toff = np.concatenate([[0], np.cumsum(tl)[:-1]]).astype(np.int64)
        tr = np.zeros(int(tl.sum())) if trace else None
        b = TrainBatch(n_models=M, precision=precision, n_tiles=n_tiles, tile_rows=_ptr(rows),
                       tile_inputs=_ptr(inputs), tile_offset=_ptr(offs), total_rows=len(y), X=_ptr(X), y=_ptr(y),
                       model_tile=_ptr(mt), model_h1=_ptr(h1), model_h2=_ptr(h2), model_lr=_ptr(lr),
                       model_epochs=_ptr(ep), model_param_offset=_ptr(poff), total_params=len(params),
                       params=_ptr(params), final_loss=_ptr(final), nonfinite_epoch=_ptr(bad),
                       loss_trace=_ptr(tr), trace_offset=_ptr(toff), trace_stride=stride)
        st = self.L.lann_train(self.h, C.byref(b))
        if st and raise_on_error:
            self._raise(st, int(bad[bad >= 0][0]) if (bad >= 0).any() else -1)
        out_p = [params[poff[i]:poff[i] + sizes[i]].copy() for i in range(M)]
        traces = [tr[toff[i]:toff[i] + tl[i]].copy() for i in range(M)] if trace else None
        return out_p, final, bad, traces

    # ---- models::predict over rows (models.cpp:346-363) ----
    def predict(self, models, rows, row_model, precision=abi.FP64_EXACT, out=None):
        """lann_predict. Rows already [n][8] float64 C-contiguous (e.g. in pinned memory, Pinned)
        are passed as they are; out (float64[n]) may be a caller buffer."""
        ms, keep = _model_set(models, precision)
        rows = np.asarray(rows)
        n = rows.shape[0]
        if rows.dtype == np.float64 and rows.ndim == 2 and rows.shape[1] == ROW and rows.flags.c_contiguous:
            full = rows
        else:
            full = np.zeros((n, ROW))
            full[:, : rows.shape[1]] = rows
        rm = row_model if (isinstance(row_model, np.ndarray) and row_model.dtype == np.int32
                           and row_model.flags.c_contiguous) else _c(row_model, np.int32)
        if out is None:
            out = np.zeros(n)
        st = self.L.lann_predict(self.h, C.byref(ms), n, _ptr(full), _ptr(rm), _ptr(out))
        if st:
            self._raise(st)
        return out

    # ---- mlp.hpp building blocks over generic nets (Mlp::forward, mse_loss, mse_gradient) ----
    def _mlp_batch(self, nets, need_y):
        """nets: list of (dims, params, X [n][dims[0]], y or None)."""
        nd = np.array([len(d) for d, _, _, _ in nets], dtype=np.int32)
        dims = np.concatenate([np.asarray(d, dtype=np.int32) for d, _, _, _ in nets])
        params = np.concatenate([np.asarray(p, dtype=np.float64) for _, p, _, _ in nets])
        rows = np.array([len(x) for _, _, x, _ in nets], dtype=np.int32)
        X = np.concatenate([np.asarray(x, dtype=np.float64).ravel() for _, _, x, _ in nets])
        keep = [nd, dims, params, rows, X]
        b = MlpBatch(len(nets), _ptr(nd), _ptr(dims), _ptr(params), _ptr(rows), _ptr(X), None)
        if need_y:
            y = np.concatenate([np.asarray(t, dtype=np.float64) for _, _, _, t in nets])
            keep.append(y)
            b.y = _ptr(y)
        return b, keep, int(rows.sum()), len(params)

    def mlp_forward(self, nets):
        b, keep, n_rows, _ = self._mlp_batch([(d, p, x, None) for d, p, x in nets], False)
        out = np.zeros(n_rows)
        st = self.L.lann_mlp_forward(self.h, C.byref(b), _ptr(out))
        if st:
            self._raise(st)
        return out

    def mse_loss(self, nets):
        b, keep, _, _ = self._mlp_batch(nets, True)
        loss = np.zeros(len(nets))
        st = self.L.lann_mse_loss(self.h, C.byref(b), _ptr(loss))
        if st:
            self._raise(st)
        return loss

    def mse_gradient(self, nets):
        """Returns (loss per net, list of gradient vectors)."""
        b, keep, _, n_params = self._mlp_batch(nets, True)
        loss, grad = np.zeros(len(nets)), np.zeros(n_params)
        st = self.L.lann_mse_gradient(self.h, C.byref(b), _ptr(loss), _ptr(grad))
        if st:
            self._raise(st)
        sizes = np.cumsum([len(p) for _, p, _, _ in nets])[:-1]
        return loss, np.split(grad, sizes)

    def adam_update(self, params, grad, m, v, step, lr, beta1=0.9, beta2=0.999, eps=1e-8):
        """AdamState::update in place on float64 arrays (step = the count after increment)."""
        st = self.L.lann_adam_update(self.h, len(params), _ptr(params), _ptr(np.ascontiguousarray(grad)), _ptr(m),
                                     _ptr(v), step, lr, beta1, beta2, eps)
        if st:
            self._raise(st)

    # ---- eval::mape / mape_thresholded / spearman over many sets ----
    def eval(self, truths, preds, drop=0.3):
        lens = np.array([len(t) for t in truths], dtype=np.int32)
        off = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
        t = np.concatenate([np.asarray(x, dtype=np.float64) for x in truths])
        p = np.concatenate([np.asarray(x, dtype=np.float64) for x in preds])
        n = len(truths)
        mape, thr, rho = np.zeros(n), np.zeros(n), np.zeros(n)
        kept = np.zeros(n, dtype=np.int32)
        st = self.L.lann_eval(self.h, n, _ptr(off), _ptr(lens), _ptr(t), _ptr(p), drop, _ptr(mape), _ptr(thr),
                              _ptr(kept), _ptr(rho))
        if st:
            self._raise(st)
        return mape, thr, kept, rho

    def select_schedule(self, model, n_img, cands, precision=abi.FP64_EXACT):
        ms, keep = _model_set([model], precision)
        c = _c(cands, np.uint32)
        chosen = C.c_int64(-1)
        score = C.c_double(0)
        st = self.L.lann_select_schedule(self.h, C.byref(ms), n_img, len(c), _ptr(c), C.addressof(chosen),
                                         C.addressof(score))
        if st:
            self._raise(st)
        return chosen.value, score.value

    def select_variants(self, models, with_n_thd, kind, max_threads, seed, first, n, precision=abi.FP32):
        ms, keep = _model_set(models, precision)
        thd = _c(with_n_thd, np.int32)
        idx = np.zeros(n, dtype=np.int32)
        score = np.zeros(n)
        st = self.L.lann_select_variants(self.h, C.byref(ms), _ptr(thd), kind, max_threads, seed, first, n,
                                         _ptr(idx), _ptr(score))
        if st:
            self._raise(st)
        return idx, score

    def select_variants_compact(self, models, with_n_thd, kind, max_threads, seed, first, n, precision=abi.FP32,
                                idx=None, score=None, want_hist=True):
        """lann_select_variants_compact: idx / score are caller arrays (uint8 / float32, pinned or
        not) or None; returns (idx, score, hist)."""
        ms, keep = _model_set(models, precision)
        thd = _c(with_n_thd, np.int32)
        hist = np.zeros(len(models), dtype=np.int64) if want_hist else None
        st = self.L.lann_select_variants_compact(self.h, C.byref(ms), _ptr(thd), kind, max_threads, seed, first, n,
                                                 _ptr(idx), _ptr(score), _ptr(hist))
        if st:
            self._raise(st)
        return idx, score, hist

    # ---- models::train_nn + predict_dataset + make_report over a population ----
    def cv_summarize(self, jobs, results, ensembles):
        """lann_cv_summarize: group statistics from host results and ensemble scores (merging
        shards from several devices or processes) computed on this engine's device."""
        n = len(jobs)
        ng, ne = cv_layout(jobs)
        arr = (Job * max(1, n))(*jobs)
        res = (JobResult * max(1, n))(*results)
        ens = (CvEnsemble * max(1, ne))(*ensembles)
        groups = (CvGroup * max(1, ng))()
        st = self.L.lann_cv_summarize(self.h, n, arr, res, ens, groups)
        if st:
            self._raise(st)
        return list(groups)[:ng]

    def run_population(self, jobs, precision=abi.FP64_EXACT, want_params=False, want_trace=False):
        n = len(jobs)
        arr = (Job * n)(*jobs)
        res = (JobResult * n)()
        params = off = trace = toff = None
        if want_params:
            params = np.zeros(n * 2048)
            off = (np.arange(n, dtype=np.int64) * 2048)
        if want_trace:
            ep = np.array([j.epochs for j in jobs], dtype=np.int64)
            toff = np.concatenate([[0], np.cumsum(ep)[:-1]]).astype(np.int64)
            trace = np.zeros(int(ep.sum()))
        st = self.L.lann_run_population(self.h, n, arr, precision, res, _ptr(params), _ptr(off), _ptr(trace),
                                        _ptr(toff))
        results = list(res)
        out_params = [params[off[i]:off[i] + results[i].n_params].copy() for i in range(n)] if want_params else None
        out_trace = [trace[toff[i]:toff[i] + jobs[i].epochs].copy() for i in range(n)] if want_trace else None
        return st, results, out_params, out_trace


class Population:
    """A prepared population (lann_population_*): inputs resident in HBM, device-only passes."""

    def __init__(self, eng: Engine, jobs, precision, record_trace=False):
        self.eng = eng
        self.jobs = list(jobs)
        n = len(self.jobs)
        self._arr = (Job * n)(*self.jobs)
        h = C.c_void_p()
        if not eng.h:
            raise Error("engine is closed")
        st = eng.L.lann_population_create(eng.h, n, self._arr, precision, int(record_trace), C.byref(h))
        if st and not h.value:
            eng._raise(st)
        self.h = h
        self.record_trace = record_trace
        if not hasattr(eng, "_pops"):
            eng._pops = weakref.WeakSet()
        eng._pops.add(self)

    @property
    def flop(self) -> float:
        return self.eng.L.lann_population_flop(self.h)

    @property
    def n_models(self) -> int:
        return self.eng.L.lann_population_models(self.h)

    def run(self, n_steps=1):
        if not self.h:
            raise Error("population is closed (or its engine was)")
        st = self.eng.L.lann_population_run(self.h, n_steps)
        if st:
            self.eng._raise(st)

    def norms(self):
        if not self.h:
            raise Error("population is closed (or its engine was)")
        out = np.zeros((len(self.jobs), 18))
        self.eng.L.lann_population_norm(self.h, _ptr(out))
        return out

    def fetch(self, want_params=False, want_trace=False):
        if not self.h:
            raise Error("population is closed (or its engine was)")
        n = len(self.jobs)
        res = (JobResult * n)()
        params = off = trace = toff = None
        if want_params:
            params = np.zeros(n * 2048)
            off = (np.arange(n, dtype=np.int64) * 2048)
        if want_trace and self.record_trace:
            ep = np.array([j.epochs for j in self.jobs], dtype=np.int64)
            toff = np.concatenate([[0], np.cumsum(ep)[:-1]]).astype(np.int64)
            trace = np.zeros(int(ep.sum()))
        st = self.eng.L.lann_population_fetch(self.h, res, _ptr(params), _ptr(off), _ptr(trace), _ptr(toff))
        results = list(res)
        out_p = [params[off[i]:off[i] + results[i].n_params].copy() for i in range(n)] if want_params else None
        out_t = [trace[toff[i]:toff[i] + self.jobs[i].epochs].copy() for i in range(n)] if trace is not None else None
        return st, results, out_p, out_t

    def cv(self):
        """The last pass's cross-validation summary (lann_population_cv): (groups, ensembles)."""
        if not self.h:
            raise Error("population is closed (or its engine was)")
        ng, ne = C.c_int32(), C.c_int32()
        self.eng.L.lann_population_cv_count(self.h, C.byref(ng), C.byref(ne))
        groups = (CvGroup * max(1, ng.value))()
        ens = (CvEnsemble * max(1, ne.value))()
        st = self.eng.L.lann_population_cv(self.h, groups, ens)
        if st:
            self.eng._raise(st)
        return list(groups)[:ng.value], list(ens)[:ne.value]

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            self.eng.L.lann_population_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        self.close()


def _model_set(models, precision):
    """models: list of dicts {inputs, h1, h2, log_target, params, norm(18)}"""
    M = len(models)
    I = np.array([m["inputs"] for m in models], dtype=np.int32)
    h1 = np.array([m["h1"] for m in models], dtype=np.int32)
    h2 = np.array([m.get("h2", 0) for m in models], dtype=np.int32)
    lt = np.array([int(m.get("log_target", 0)) for m in models], dtype=np.int32)
    sizes = np.array([len(m["params"]) for m in models], dtype=np.int64)
    poff = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    params = np.concatenate([np.asarray(m["params"], dtype=np.float64) for m in models])
    norm = np.concatenate([np.asarray(m["norm"], dtype=np.float64) for m in models])
    ms = ModelSet(n_models=M, precision=precision, n_inputs=_ptr(I), h1=_ptr(h1), h2=_ptr(h2), log_target=_ptr(lt),
                  param_offset=_ptr(poff), params=_ptr(params), total_params=len(params), norm=_ptr(norm))
    return ms, (I, h1, h2, lt, poff, params, norm)


def shard_bounds(jobs, n_shards: int):
    """lann_shard_bounds: the engine's contiguous cost-balanced cut of a job list (host only)."""
    L = load_library()
    n = len(jobs)
    arr = (Job * max(n, 1))(*jobs)
    b = np.zeros(n_shards + 1, dtype=np.int32)
    st = L.lann_shard_bounds(n_shards, n, arr, _ptr(b))
    if st:
        raise ParamError(f"lann_shard_bounds status {st}")
    return [int(x) for x in b]


class Group:
    """lann_group_*: one engine and one host thread per listed device; a population is cut into
    contiguous cost-balanced shards that run concurrently and are gathered in job order on the
    host (no device-to-device traffic, no NCCL)."""

    def __init__(self, devices):
        self.L = load_library()
        devs = np.asarray(list(devices), dtype=np.int32)
        self.h = C.c_void_p()
        st = self.L.lann_group_create(len(devs), _ptr(devs), C.byref(self.h))
        if st:
            raise _ERR.get(st, Error)(f"lann_group_create status {st}")
        self.devices = [int(d) for d in devs]

    def close(self):
        if self.h:
            self.L.lann_group_destroy(self.h)
            self.h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def last_error(self) -> str:
        return self.L.lann_group_last_error(self.h).decode()

    @property
    def last_device_ms(self) -> float:
        return self.L.lann_group_last_device_ms(self.h)

    @property
    def last_wall_ms(self) -> float:
        return self.L.lann_group_last_wall_ms(self.h)

    def shard_bounds(self, jobs):
        n = len(jobs)
        arr = (Job * n)(*jobs)
        b = np.zeros(len(self.devices) + 1, dtype=np.int32)
        self.L.lann_group_shard_bounds(self.h, n, arr, _ptr(b))
        return [int(x) for x in b]

    def run_population(self, jobs, precision=abi.FP64_EXACT, want_params=False):
        """Returns (status, results, params list or None)."""
        n = len(jobs)
        arr = (Job * n)(*jobs)
        res = (JobResult * n)()
        params = off = None
        if want_params:  # 2048 slots per model, as Engine.run_population
            params = np.zeros(n * 2048)
            off = np.arange(n, dtype=np.int64) * 2048
        st = self.L.lann_group_run_population(self.h, n, arr, precision, res, _ptr(params), _ptr(off), None, None)
        plist = None
        if want_params:
            plist = [params[off[k]: off[k] + res[k].n_params].copy() for k in range(n)]
        return st, list(res), plist

    def run_cv(self, jobs, precision=abi.FP64_EXACT):
        """lann_group_run_cv -> (status, results, cv groups, cv ensembles)."""
        n = len(jobs)
        arr = (Job * n)(*jobs)
        res = (JobResult * n)()
        ng, ne = cv_layout(jobs)
        groups = (CvGroup * max(1, ng))()
        ens = (CvEnsemble * max(1, ne))()
        st = self.L.lann_group_run_cv(self.h, n, arr, precision, res, groups, ens)
        return st, list(res), list(groups)[:ng], list(ens)[:ne]


class Pinned:
    """A numpy array in pinned host memory (lann_host_alloc): engine outputs written into it by
    DMA at full link bandwidth."""

    def __init__(self, n, dtype):
        self.L = load_library()
        dt = np.dtype(dtype)
        self.ptr = C.c_void_p()
        st = self.L.lann_host_alloc(max(1, n) * dt.itemsize, C.byref(self.ptr))
        if st or not self.ptr.value:
            raise NoDeviceError("lann_host_alloc failed (no CUDA device?)")
        buf = (C.c_byte * (max(1, n) * dt.itemsize)).from_address(self.ptr.value)
        self.array = np.frombuffer(buf, dtype=dt, count=n)

    def free(self):
        if self.ptr and self.ptr.value:
            self.array = None
            self.L.lann_host_free(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
