"""Generate tests/golden/golden_r01.json from the REFERENCE ITSELF.

Runs the unmodified reference core compiled from /root/reference (oracle/_ref/libperfsage_ref.so,
built by oracle/Makefile) through the ref_driver.cpp shim and records its outputs. The JSON pins
the C oracle (CPU tests) and the CUDA engine (GPU tests); /root/reference is not needed at test
time. Regenerate with:  make -C oracle && python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_lib import Reference  # noqa: E402
from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import population as P  # noqa: E402


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def world_dict(w):
    return {f: (list(getattr(w, f)) if f in ("mu", "kappa") else getattr(w, f)) for f, _ in abi.World._fields_}


def world_from(d):
    w = abi.World()
    for k, v in d.items():
        if k in ("mu", "kappa"):
            for i, x in enumerate(v):
                getattr(w, k)[i] = x
        else:
            setattr(w, k, v)
    return w


def job_dict(j):
    return {"world": world_dict(j.world), "data_seed": j.data_seed, "count": j.count,
            "train_fraction": j.train_fraction, "n_folds": j.n_folds, "fold": j.fold, "family": j.family,
            "hidden": list(j.hidden)[: j.n_hidden], "lr": j.learning_rate, "epochs": j.epochs,
            "init_seed": j.init_seed, "log_target": j.log_target, "unconstrained": j.unconstrained}


def job_from(d):
    return abi.make_job(world_from(d["world"]), d["data_seed"], count=d["count"], train_fraction=d["train_fraction"],
                        n_folds=d["n_folds"], fold=d["fold"], family=d["family"], hidden=tuple(d["hidden"]),
                        lr=d["lr"], epochs=d["epochs"], init_seed=d["init_seed"], log_target=bool(d["log_target"]),
                        unconstrained=bool(d["unconstrained"]))


def result_dict(r, params=None, trace=None):
    d = {"status": r.status, "final_loss": r.final_loss, "mape": r.mape, "mape_thr": r.mape_thr, "rho": r.rho,
         "n_kept": r.n_kept, "n_inputs": r.n_inputs, "n_params": r.n_params, "n_train": r.n_train,
         "n_eval": r.n_eval, "nonfinite_epoch": r.nonfinite_epoch}
    if params is not None:
        d["params"] = [float(x) for x in params]
    if trace is not None:
        d["trace_head"] = [float(x) for x in trace[:5]]
        d["trace_sha256"] = sha(np.asarray(trace, dtype=np.float64))
    return d


def run_jobs_with_traces(ref, jobs):
    """Each job through the reference pipeline, keeping params and full trace."""
    out = []
    for j in jobs:
        arr = (abi.Job * 1)(j)
        res = (abi.JobResult * 1)()
        params = np.zeros(4096)
        po = np.zeros(1, dtype=np.int64)
        trace = np.zeros(j.epochs)
        to = np.zeros(1, dtype=np.int64)
        ref.lib.ref_run_population(1, arr, res, params.ctypes.data, po.ctypes.data, trace.ctypes.data,
                                   to.ctypes.data, 1)
        r = res[0]
        out.append(result_dict(r, params[: r.n_params], trace))
    return out


def main():
    ref = Reference()
    g = {"generator": "tests/golden/make_golden.py", "source": "reference core compiled from /root/reference "
         "(oracle/_ref/libperfsage_ref.so) via oracle/ref_driver.cpp"}
    # 1. config 1 = acceptance criterion 5 protocol, seeds 1..5, full 8000 epochs
    c1 = P.config1_jobs()
    g["config1"] = {"jobs": [job_dict(j) for j in c1], "results": run_jobs_with_traces(ref, c1)}
    # NN (no complexity input) for the same seeds (criterion 5's comparison arm)
    c1nn = P.config1_jobs(family=abi.NN)
    g["config1_nn"] = {"jobs": [job_dict(j) for j in c1nn], "results": run_jobs_with_traces(ref, c1nn)}
    # 2. the 48 combo worlds: datasets (sha256 of features / c / runtimes) + split orders
    from paper_2003_07497_b200 import engine as E
    combos = E.default_combos()
    ds = []
    for i, w in enumerate(combos):
        seed = P.combo_seed(1, i)
        st, feats, c, rt, nf = ref.build_dataset(w, seed, 500)
        assert st == 0, ref.last_error()
        _, order, ntr = ref.split_order(500, 0.5, seed)
        ds.append({"world": world_dict(w), "seed": seed, "n_features": nf, "sha256": sha(feats, c, rt),
                   "runtime_head": [float(x) for x in rt[:3]], "c_head": [int(x) for x in c[:3]],
                   "split_sha256": sha(order), "n_train": ntr})
    g["combos"] = ds
    # 3. the config-2 population with short training (200 epochs), full pipeline per job
    c2 = P.config2_jobs(root_seed=1, epochs_scale=0.01)
    secs, res, params = ref.run_population(c2, threads=8, want_params=True)
    g["config2_short"] = {"jobs": [job_dict(j) for j in c2],
                          "results": [result_dict(r, params[i * 4096:i * 4096 + r.n_params]) for i, r in enumerate(res)]}
    # 4. k-fold sweep slice: 3 combos (MM cpu, MV gpu, blur) x 2 seeds x 5 folds, 150 epochs
    pick = [combos[0], combos[13], combos[40]]
    kf = []
    for w in pick:
        for j in P.config3_jobs(root_seed=1, n_seeds=2, combos=[w]):
            j.epochs = 150
            kf.append(j)
    secs, res, params = ref.run_population(kf, threads=8, want_params=True)
    g["config3_kfold_short"] = {"jobs": [job_dict(j) for j in kf],
                                "results": [result_dict(r, params[i * 4096:i * 4096 + r.n_params]) for i, r in enumerate(res)]}
    # 5. metric KATs (test_eval.cpp:64-157) + random vectors with ties
    rng = np.random.default_rng(7)
    kat = []
    for t, p in [([1.0, 2.0, 3.0], [1.0, 2.0, 3.0]), ([100.0], [90.0]), ([1.0, 2.0], [2.0, 1.0]),
                 ([1.0, 2.0, 3.0, 4.0], [1.0, 3.0, 2.0, 4.0]), ([0.1, 0.2, 0.5, 0.9], [4.0, 3.0, 2.0, 1.0]),
                 ([1e-6, 1.0, 1.1, 1.2, 1.3, 1.4, 1.5, 1.6, 1.7, 1.8], [51e-6, 1.0, 1.1, 1.2, 1.3, 1.4, 1.5, 1.6, 1.7, 1.8])]:
        kat.append((t, p))
    for n in (2, 7, 50, 250, 1000):
        t = np.round(rng.uniform(0.05, 10.0, n), 1 if n > 7 else 3)  # rounding creates ties
        p = np.round(rng.uniform(0.05, 10.0, n), 1)
        kat.append((t.tolist(), p.tolist()))
    metrics = []
    for t, p in kat:
        t, p = np.array(t), np.array(p)
        _, m = ref.mape(t, p)
        st, thr, kept = ref.mape_thresholded(t, p, 0.3)
        st2, rho = ref.spearman(t, p)
        metrics.append({"truth": t.tolist(), "pred": p.tolist(), "mape": m, "mape_thr": thr if st == 0 else None,
                        "n_kept": kept if st == 0 else None, "rho": rho if st2 == 0 else None})
    g["metrics"] = metrics
    # 6. blur schedule selection with a reference-trained blur model
    w = combos[40]
    seed = P.combo_seed(1, 40)
    st, feats, c, rt, nf = ref.build_dataset(w, seed, 250)
    st, params, trace, norm, bad = ref.train_nn(abi.BLUR, 0, abi.NNC, feats, c, rt, (5, 5), 1e-2, 3000, seed, True)
    assert st == 0, ref.last_error()
    cands = ref.enumerate_candidates(0, 1 << 20, 1)
    sel = []
    for n_img in (1024, 4096, 32768):
        st, chosen, score = ref.select_schedule(abi.NNC, (5, 5), params, norm, True, n_img, cands)
        sel.append({"n_img": n_img, "chosen": int(chosen), "score": score})
    sub = ref.enumerate_candidates(0, 100, 3)
    g["select"] = {"params": params.tolist(), "norm": norm.tolist(), "hidden": [5, 5], "log_target": 1,
                   "lattice_sizes": {"cpu": len(cands), "gpu_style": len(ref.enumerate_candidates(1, 1 << 20, 1))},
                   "cpu_lattice_sha256": sha(cands), "choices": sel, "sample100_seed3": sub.tolist()}
    # 7. predictions of the config-1 seed-1 model on its held-out part (raw features)
    j = c1[0]
    st, feats, c, rt, nf = ref.build_dataset(j.world, 1, 500)
    _, order, ntr = ref.split_order(500, 0.5, 1)
    tr, te = order[:ntr], order[ntr:]
    st, params, trace, norm, bad = ref.train_nn(abi.MM, 1, abi.NNC, feats[tr], c[tr], rt[tr], (8,), 1e-2, 8000, 1)
    st, pred = ref.predict(abi.MM, 1, abi.NNC, (8,), params, norm, False, feats[te], c[te])
    g["predict_config1_seed1"] = {"params": params.tolist(), "norm": norm.tolist(), "pred_sha256": sha(pred),
                                  "pred_head": pred[:5].tolist(), "n": int(len(te))}
    # 8. mse_gradient KATs on random nets (mlp.cpp:75-122)
    grads = []
    rng = np.random.default_rng(11)
    for dims in ([3, 4, 1], [7, 8, 1], [6, 5, 5, 1], [2, 3, 2, 1]):
        n, params = ref.mlp_init(dims, 5)
        X = np.zeros((6, 8))
        X[:, : dims[0]] = rng.uniform(-1, 1, (6, dims[0]))
        y = rng.uniform(0, 1, 6)
        st, loss, grad = ref.mse_gradient(dims, params, X, y)
        grads.append({"dims": dims, "params": params.tolist(), "X": X.tolist(), "y": y.tolist(), "loss": loss,
                      "grad": grad.tolist()})
    g["mse_gradient"] = grads
    path = os.path.join(HERE, "golden_r01.json")
    with open(path, "w") as f:
        json.dump(g, f)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
