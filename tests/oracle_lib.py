"""ctypes bindings for the TEST-ONLY checkers under oracle/.

* ``Oracle``: oracle/_ref/liblann_oracle.so, the plain-C restatement (lann_oracle.c).
* ``Reference``: oracle/_ref/libperfsage_ref.so, the unmodified reference core compiled
  from /root/reference sources + the ref_driver.cpp shim (present only where it was built).

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs use this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
REF_DIR = os.path.join(ORACLE_DIR, "_ref")
ROW = 8

from paper_2003_07497_b200.abi import World, Job, JobResult, ModelSet  # noqa: E402  (plain structs)

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")


def build_oracle():
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


class _Lib:
    prefix = ""

    def __init__(self, path):
        self.lib = C.CDLL(path)
        p = self.prefix
        L = self.lib
        getattr(L, p + "build_dataset").argtypes = [C.POINTER(World), C.c_uint64, C.c_int, _dp, _u64p, _dp, C.POINTER(C.c_int)]
        getattr(L, p + "split_order").argtypes = [C.c_int, C.c_double, C.c_uint64, _i64p, C.POINTER(C.c_int)]
        getattr(L, p + "mlp_init").argtypes = [C.c_int, _i32p, C.c_uint64, C.c_int, _dp]
        getattr(L, p + "mse_gradient").argtypes = [C.c_int, _i32p, _dp, C.c_int, _dp, _dp, C.POINTER(C.c_double), _dp]
        getattr(L, p + "train_full_batch").argtypes = [C.c_int, _i32p, _dp, C.c_int, _dp, _dp, C.c_double, C.c_int, _dp, C.POINTER(C.c_int)]
        getattr(L, p + "mape").argtypes = [C.c_int, _dp, _dp, C.POINTER(C.c_double)]
        getattr(L, p + "mape_thresholded").argtypes = [C.c_int, _dp, _dp, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_int)]
        getattr(L, p + "spearman").argtypes = [C.c_int, _dp, _dp, C.POINTER(C.c_double)]

    def _f(self, name):
        return getattr(self.lib, self.prefix + name)

    def build_dataset(self, world: World, seed: int, count: int):
        feats = np.zeros((count, ROW))
        c = np.zeros(count, dtype=np.uint64)
        rt = np.zeros(count)
        nf = C.c_int(0)
        st = self._f("build_dataset")(C.byref(world), seed, count, feats, c, rt, C.byref(nf))
        return st, feats, c, rt, nf.value

    def split_order(self, n, frac, seed):
        order = np.zeros(n, dtype=np.int64)
        ntr = C.c_int(0)
        st = self._f("split_order")(n, frac, seed, order, C.byref(ntr))
        return st, order, ntr.value

    def mlp_init(self, dims, seed, raw=False):
        dims = np.asarray(dims, dtype=np.int32)
        P = int(sum((dims[i] + 1) * dims[i + 1] for i in range(len(dims) - 1)))
        out = np.zeros(max(P, 1))
        n = self._f("mlp_init")(len(dims), dims, seed, int(raw), out)
        return n, out[:P]

    def mse_gradient(self, dims, params, X, y):
        dims = np.asarray(dims, dtype=np.int32)
        loss = C.c_double(0)
        grad = np.zeros_like(params)
        st = self._f("mse_gradient")(len(dims), dims, np.ascontiguousarray(params), len(y),
                                     np.ascontiguousarray(X), np.ascontiguousarray(y), C.byref(loss), grad)
        return st, loss.value, grad

    def train_full_batch(self, dims, params, X, y, lr, epochs):
        dims = np.asarray(dims, dtype=np.int32)
        p = np.array(params, dtype=np.float64)
        trace = np.zeros(epochs)
        bad = C.c_int(-1)
        st = self._f("train_full_batch")(len(dims), dims, p, len(y), np.ascontiguousarray(X),
                                         np.ascontiguousarray(y), lr, epochs, trace, C.byref(bad))
        return st, p, trace, bad.value

    def mlp_forward(self, dims, params, X):
        dims = np.asarray(dims, dtype=np.int32)
        out = np.zeros(len(X))
        st = self._f("mlp_forward")(len(dims), dims, np.ascontiguousarray(params), len(X), np.ascontiguousarray(X), out)
        return st, out

    def mse_loss(self, dims, params, X, y):
        dims = np.asarray(dims, dtype=np.int32)
        loss = C.c_double(0)
        st = self._f("mse_loss")(len(dims), dims, np.ascontiguousarray(params), len(y), np.ascontiguousarray(X),
                                 np.ascontiguousarray(y), C.byref(loss))
        return st, loss.value

    def adam_steps(self, params, grads, lr):
        p = np.array(params, dtype=np.float64)
        g = np.ascontiguousarray(grads, dtype=np.float64)
        m, v = np.zeros_like(p), np.zeros_like(p)
        st = self._f("adam_steps")(len(p), p, g, len(g), lr, m, v)
        return st, p, m, v

    def mape(self, t, p):
        o = C.c_double(0)
        st = self._f("mape")(len(t), np.ascontiguousarray(t, dtype=np.float64), np.ascontiguousarray(p, dtype=np.float64), C.byref(o))
        return st, o.value

    def mape_thresholded(self, t, p, drop=0.3):
        o = C.c_double(0)
        k = C.c_int(0)
        st = self._f("mape_thresholded")(len(t), np.ascontiguousarray(t, dtype=np.float64), np.ascontiguousarray(p, dtype=np.float64), drop, C.byref(o), C.byref(k))
        return st, o.value, k.value

    def spearman(self, t, p):
        o = C.c_double(0)
        st = self._f("spearman")(len(t), np.ascontiguousarray(t, dtype=np.float64), np.ascontiguousarray(p, dtype=np.float64), C.byref(o))
        return st, o.value


class Oracle(_Lib):
    prefix = "or_"

    def __init__(self):
        path = os.path.join(REF_DIR, "liblann_oracle.so")
        if not os.path.exists(path):
            build_oracle()
        super().__init__(path)
        L = self.lib
        L.or_run_job.argtypes = [C.POINTER(Job), C.POINTER(JobResult), C.c_void_p, C.c_void_p]
        L.or_predict_row.argtypes = [C.c_int, C.c_int, _i32p, _dp, _dp, C.c_int, _dp]
        L.or_predict_row.restype = C.c_double
        L.or_norm_fit.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_int, _dp]
        L.or_select_schedule.argtypes = [C.c_int, C.c_int, _i32p, _dp, _dp, C.c_int, C.c_uint32, C.c_int64, _u32p, C.POINTER(C.c_double)]
        L.or_select_schedule.restype = C.c_int64
        L.or_candidate.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int64, _dp, C.POINTER(C.c_uint64)]
        L.or_select_variants.argtypes = [C.POINTER(ModelSet), _i32p, C.c_int, C.c_int, C.c_uint64, C.c_int64, C.c_int64, _i32p, _dp]
        L.or_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.or_derive_seed.restype = C.c_uint64
        L.or_fold_mean.argtypes = [C.c_int, C.POINTER(Job), C.POINTER(_dp), _dp, _dp, C.POINTER(C.c_int)]

    def run_job(self, job: Job, want_params=False, want_trace=False):
        r = JobResult()
        params = np.zeros(4096) if want_params else None
        trace = np.zeros(job.epochs) if want_trace else None
        self.lib.or_run_job(C.byref(job), C.byref(r),
                            params.ctypes.data if params is not None else None,
                            trace.ctypes.data if trace is not None else None)
        if params is not None:
            params = params[: r.n_params]
        return r, params, trace

    def predict_row(self, I, hidden, params, norm, log_target, x):
        h = np.asarray(list(hidden) + [0] * (2 - len(hidden)), dtype=np.int32)
        xx = np.zeros(ROW)
        xx[: len(x)] = x
        return self.lib.or_predict_row(I, len(hidden), h, np.ascontiguousarray(params), np.ascontiguousarray(norm), int(log_target), xx)

    def norm_fit(self, X, y, I, log_target=False):
        norm = np.zeros(18)
        self.lib.or_norm_fit(len(y), I, np.ascontiguousarray(X), np.ascontiguousarray(y), int(log_target), norm)
        return norm

    def select_schedule(self, family, hidden, params, norm, log_target, n_img, cands):
        h = np.asarray(list(hidden) + [0] * (2 - len(hidden)), dtype=np.int32)
        s = C.c_double(0)
        i = self.lib.or_select_schedule(family, len(hidden), h, np.ascontiguousarray(params), np.ascontiguousarray(norm),
                                        int(log_target), n_img, len(cands), np.ascontiguousarray(cands, dtype=np.uint32), C.byref(s))
        return i, s.value

    def candidate(self, kind, max_threads, seed, idx):
        base = np.zeros(ROW)
        c = C.c_uint64(0)
        self.lib.or_candidate(kind, max_threads, seed, idx, base, C.byref(c))
        return base, c.value


    def fold_mean(self, fold_jobs, params):
        """or_fold_mean: the fold-mean model of one seed's k fold models on the split's test part
        -> (pred, truth)."""
        k = len(fold_jobs)
        arr = (Job * k)(*fold_jobs)
        keep = [np.ascontiguousarray(p, dtype=np.float64) for p in params]
        pp = (_dp * k)(*[q.ctypes.data_as(_dp) for q in keep])
        n = fold_jobs[0].count
        pred, truth, nt = np.zeros(n), np.zeros(n), C.c_int(0)
        st = self.lib.or_fold_mean(k, arr, pp, pred, truth, C.byref(nt))
        assert st == 0, st
        return pred[: nt.value], truth[: nt.value]

    def cv_summary(self, jobs, results, params):
        """The cross-validation summary (include/lann_engine.h) restated in Python over the
        oracle's per-job results and weights: groups keyed by every job field except fold and
        init_seed, ensembles by (group, init_seed); fold-mean test metrics through or_fold_mean and
        the oracle's make_report; mean = sequential sum / n, median = sorted middle(s)."""
        def gkey(j):
            return (bytes(j.world), j.data_seed, j.count, j.train_fraction, j.n_folds, j.family, j.n_hidden,
                    tuple(j.hidden), j.learning_rate, j.epochs, j.log_target, j.unconstrained)
        groups, ens = {}, {}
        for i, j in enumerate(jobs):
            if j.n_folds < 2:
                continue
            g = groups.setdefault(gkey(j), {"first": i, "k": j.n_folds, "models": [], "ens": []})
            g["models"].append(i)
            key = (gkey(j), j.init_seed)
            if key not in ens:
                ens[key] = {"group": list(groups).index(gkey(j)), "seed": j.init_seed, "member": [-1] * j.n_folds}
                g["ens"].append(key)
            if 0 <= j.fold < j.n_folds and ens[key]["member"][j.fold] < 0:
                ens[key]["member"][j.fold] = i
        ok = lambda r: r.status == 0  # noqa: E731
        out_ens = []
        for key, e in ens.items():
            rec = {"group": e["group"], "seed": e["seed"], "status": 0}
            if any(m < 0 for m in e["member"]):
                rec["status"] = 1  # LANN_PARAM_ERROR: a fold is missing
            elif not all(ok(results[m]) for m in e["member"]):
                rec["status"] = next(results[m].status for m in e["member"] if not ok(results[m]))
            else:
                pred, truth = self.fold_mean([jobs[m] for m in e["member"]], [params[m] for m in e["member"]])
                st1, rec["mape"] = self.mape(truth, pred)
                st2, rec["mape_thr"], rec["n_kept"] = self.mape_thresholded(truth, pred)
                st3, rec["rho"] = self.spearman(truth, pred)
                rec["status"] = st1 or st2 or st3
                rec["n_test"] = len(truth)
            out_ens.append(rec)

        def stats(vals):
            if not vals:
                return (0.0, 0.0)
            acc = 0.0
            for v in vals:
                acc += v
            s_ = sorted(vals)
            n = len(s_)
            return (acc / n, s_[n // 2] if n % 2 else (s_[n // 2 - 1] + s_[n // 2]) / 2)
        out_groups = []
        ens_list = list(ens)
        for gk, g in groups.items():
            rows = [results[m] for m in g["models"] if ok(results[m])]
            eo = [out_ens[ens_list.index(k)] for k in g["ens"]]
            eo = [e for e in eo if e["status"] == 0]
            out_groups.append({
                "first_job": g["first"], "n_folds": g["k"], "n_models": len(g["models"]), "n_models_ok": len(rows),
                "n_ensembles": len(g["ens"]), "n_ensembles_ok": len(eo),
                "fold_mape": stats([r.mape for r in rows]), "fold_mape_thr": stats([r.mape_thr for r in rows]),
                "fold_rho": stats([r.rho for r in rows]),
                "test_mape": stats([e["mape"] for e in eo]), "test_mape_thr": stats([e["mape_thr"] for e in eo]),
                "test_rho": stats([e["rho"] for e in eo]),
            })
        return out_groups, out_ens


class Reference(_Lib):
    prefix = "ref_"

    @staticmethod
    def available():
        return os.path.exists(os.path.join(REF_DIR, "libperfsage_ref.so"))

    def __init__(self):
        super().__init__(os.path.join(REF_DIR, "libperfsage_ref.so"))
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_mlp_forward.argtypes = [C.c_int, _i32p, _dp, C.c_int, _dp, _dp]
        L.ref_mse_loss.argtypes = [C.c_int, _i32p, _dp, C.c_int, _dp, _dp, C.POINTER(C.c_double)]
        L.ref_adam_steps.argtypes = [C.c_int, _dp, _dp, C.c_int, C.c_double, _dp, _dp]
        L.ref_train_nn.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _u64p, _dp, C.c_int, _i32p, C.c_double, C.c_int,
                                   C.c_uint64, C.c_int, C.c_int, _dp, C.POINTER(C.c_int), C.c_void_p, _dp, C.POINTER(C.c_int)]
        L.ref_predict.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _i32p, _dp, _dp, C.c_int, C.c_int, _dp, _u64p, _dp]
        L.ref_predict_raw.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _i32p, _dp, _dp, C.c_int, C.c_int, _dp, C.POINTER(C.c_double)]
        L.ref_enumerate_candidates.argtypes = [C.c_int, C.c_uint64, C.c_uint64, _u32p, C.c_uint64]
        L.ref_select_schedule.argtypes = [C.c_int, C.c_int, _i32p, _dp, _dp, C.c_int, C.c_uint32, C.c_int, _u32p, C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        L.ref_run_population.argtypes = [C.c_int, C.POINTER(Job), C.POINTER(JobResult), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        L.ref_run_population.restype = C.c_double
        L.ref_save_dataset_csv.argtypes = [C.POINTER(World), C.c_uint64, C.c_int, C.c_char_p, C.c_char_p]
        L.ref_csv_roundtrip.argtypes = [C.c_char_p, C.c_char_p]
        L.ref_model_roundtrip.argtypes = [C.c_char_p, C.c_char_p]
        L.ref_model_dump.argtypes = [C.c_char_p, _dp, C.c_int]
        L.ref_cli_train.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_int, C.c_char_p, C.c_char_p, C.c_char_p]
        L.ref_eval_model.argtypes = [C.c_char_p, C.c_char_p, C.c_double, _dp]
        L.ref_cli_gen_mock.argtypes = [C.c_int, C.c_char_p, C.c_int, C.c_uint, C.c_int, _u32p, C.c_int, C.c_int,
                                       C.c_uint64, C.c_char_p]
        L.ref_sample_features.argtypes = [C.c_int, C.c_uint64, C.c_int, _dp]
        L.ref_cli_select_mock.argtypes = [C.c_uint, C.c_int, C.c_uint64, C.c_int, C.c_int, _dp]
        L.ref_save_external_csv.argtypes = [C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_char_p, C.c_int, C.c_uint64,
                                            C.c_char_p]

    # ---- on-disk formats (csv.cpp, model_io.cpp) and the CLI train body (perfsage.cpp) ----
    def save_dataset_csv(self, world, seed, count, variant_id, path):
        return self.lib.ref_save_dataset_csv(C.byref(world), seed, count, variant_id.encode(), str(path).encode())

    def csv_roundtrip(self, src, dst):
        return self.lib.ref_csv_roundtrip(str(src).encode(), str(dst).encode())

    def model_roundtrip(self, src, dst):
        return self.lib.ref_model_roundtrip(str(src).encode(), str(dst).encode())

    def model_dump(self, path):
        out = np.zeros(1 << 20)
        n = self.lib.ref_model_dump(str(path).encode(), out, len(out))
        assert n >= 0, self.last_error()
        return out[:n]

    def cli_train(self, csv, seed, family, epochs, model_out, train_out, test_out):
        return self.lib.ref_cli_train(str(csv).encode(), seed, family.encode(), epochs, str(model_out).encode(),
                                      str(train_out).encode(), str(test_out).encode())

    def cli_gen_mock(self, kind, variant_id, max_threads, dim_max, sides, gpu_lattice, count, seed, path):
        sides = np.ascontiguousarray(sides, dtype=np.uint32)
        return self.lib.ref_cli_gen_mock(kind, variant_id.encode(), max_threads, dim_max, len(sides), sides,
                                         int(gpu_lattice), count, seed, str(path).encode())

    def sample_features(self, kind, seed, n):
        out = np.zeros(n * 8)
        nf = self.lib.ref_sample_features(kind, seed, n, out)
        return nf, out.reshape(n, 8)[:, :max(nf, 0)]

    def cli_select_mock(self, n, n_cands, seed, epochs, threads):
        out = np.zeros(15)
        st = self.lib.ref_cli_select_mock(n, n_cands, seed, epochs, threads, out)
        return st, out

    def save_external_csv(self, kind, gpu_class, max_threads, command, variant_id, count, seed, path):
        return self.lib.ref_save_external_csv(kind, int(gpu_class), max_threads, command.encode(), variant_id.encode(),
                                              count, seed, str(path).encode())

    def eval_model(self, model, csv, drop=0.3):
        out = np.zeros(4)
        st = self.lib.ref_eval_model(str(model).encode(), str(csv).encode(), drop, out)
        return st, out

    def last_error(self):
        return self.lib.ref_last_error().decode()

    def train_nn(self, kind, with_n_thd, family, feats, c, rt, hidden, lr, epochs, seed, log_target=False, unconstrained=False):
        h = np.asarray(list(hidden) + [0] * (2 - len(hidden)), dtype=np.int32)
        params = np.zeros(4096)
        npar = C.c_int(0)
        trace = np.zeros(epochs)
        norm = np.zeros(18)
        bad = C.c_int(-1)
        st = self.lib.ref_train_nn(kind, int(with_n_thd), family, len(rt), np.ascontiguousarray(feats), np.ascontiguousarray(c, dtype=np.uint64),
                                   np.ascontiguousarray(rt), len(hidden), h, lr, epochs, seed, int(log_target), int(unconstrained),
                                   params, C.byref(npar), trace.ctypes.data, norm, C.byref(bad))
        return st, params[: npar.value], trace, norm, bad.value

    def predict(self, kind, with_n_thd, family, hidden, params, norm, log_target, feats, c):
        h = np.asarray(list(hidden) + [0] * (2 - len(hidden)), dtype=np.int32)
        out = np.zeros(len(c))
        st = self.lib.ref_predict(kind, int(with_n_thd), family, len(hidden), h, np.ascontiguousarray(params), np.ascontiguousarray(norm),
                                  int(log_target), len(c), np.ascontiguousarray(feats), np.ascontiguousarray(c, dtype=np.uint64), out)
        return st, out

    def enumerate_candidates(self, lattice, limit, seed):
        out = np.zeros((2200, 4), dtype=np.uint32)
        n = self.lib.ref_enumerate_candidates(lattice, limit, seed, out, 2200)
        return out[: max(n, 0)]

    def select_schedule(self, family, hidden, params, norm, log_target, n_img, cands):
        h = np.asarray(list(hidden) + [0] * (2 - len(hidden)), dtype=np.int32)
        chosen = C.c_int64(-1)
        s = C.c_double(0)
        st = self.lib.ref_select_schedule(family, len(hidden), h, np.ascontiguousarray(params), np.ascontiguousarray(norm), int(log_target),
                                          n_img, len(cands), np.ascontiguousarray(cands, dtype=np.uint32), C.byref(chosen), C.byref(s))
        return st, chosen.value, s.value

    def run_population(self, jobs, threads=1, want_params=False):
        n = len(jobs)
        arr = (Job * n)(*jobs)
        res = (JobResult * n)()
        params = off = None
        if want_params:
            params = np.zeros(n * 4096)
            off = (np.arange(n, dtype=np.int64) * 4096)
        secs = self.lib.ref_run_population(n, arr, res, params.ctypes.data if params is not None else None,
                                           off.ctypes.data if off is not None else None, None, None, threads)
        return secs, list(res), params
