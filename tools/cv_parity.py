"""Config 3 at full length in both arithmetic modes on one GPU: the FP64-exact sweep (bit-identical
to the reference, tests/test_gpu_full_length.py) is the reference's answer for all 61,440 models;
the FP32 sweep is compared with it on north_star's statistic, the final test MAPE, here the test-part
MAPE of every seed's fold-mean model averaged per combination (include/lann_engine.h), plus the
population median of the held-out fold thr-MAPE. Writes gpurun_out/cv_parity.json.

  python tools/cv_parity.py [n_seeds]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import engine as E  # noqa: E402
from paper_2003_07497_b200 import population as P  # noqa: E402


def run(eng, jobs, precision):
    t0 = time.perf_counter()
    pop = E.Population(eng, jobs, precision)
    pop.run(1)
    dev_ms = eng.last_device_ms
    st, res, _, _ = pop.fetch()
    groups, ens = pop.cv()
    pop.close()
    return {"status": st, "res": res, "groups": groups, "ens": ens, "device_ms": dev_ms,
            "wall_s": time.perf_counter() - t0}


def main():
    n_seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    jobs = P.config3_jobs(root_seed=1, n_seeds=n_seeds)
    out = {"models": len(jobs), "n_seeds": n_seeds}
    with E.Engine(0) as eng:
        r64 = run(eng, jobs, abi.FP64_EXACT)
        r32 = run(eng, jobs, abi.FP32)
    me = P.model_epochs(jobs)
    for name, r in (("fp64_exact", r64), ("fp32", r32)):
        out[name] = {"status": r["status"], "device_ms": r["device_ms"], "wall_s": r["wall_s"],
                     "model_epochs_per_s": me / (r["device_ms"] / 1e3),
                     "failed_models": sum(x.status != 0 for x in r["res"]),
                     "ensembles_ok": sum(g.n_ensembles_ok for g in r["groups"])}
    d_test = [a.test_mape.mean - b.test_mape.mean for a, b in zip(r32["groups"], r64["groups"])]
    d_test_thr = [a.test_mape_thr.mean - b.test_mape_thr.mean for a, b in zip(r32["groups"], r64["groups"])]
    d_fold_thr = [a.fold_mape_thr.median - b.fold_mape_thr.median for a, b in zip(r32["groups"], r64["groups"])]
    d_fold_mean = [a.fold_mape_thr.mean - b.fold_mape_thr.mean for a, b in zip(r32["groups"], r64["groups"])]
    d_test_thr_med = [a.test_mape_thr.median - b.test_mape_thr.median for a, b in zip(r32["groups"], r64["groups"])]
    thr64 = np.array([x.mape_thr for x in r64["res"] if x.status == 0])
    thr32 = np.array([x.mape_thr for x in r32["res"] if x.status == 0])
    per_model = np.abs(np.array([a.mape_thr - b.mape_thr for a, b in zip(r32["res"], r64["res"])
                                 if a.status == 0 and b.status == 0]))
    out["gap_pp"] = {
        "fold_mean_test_mape_per_combo": {"max_abs": float(np.max(np.abs(d_test))),
                                          "median_abs": float(np.median(np.abs(d_test))),
                                          "mean_signed": float(np.mean(d_test))},
        "fold_mean_test_mape_thr_per_combo": {"max_abs": float(np.max(np.abs(d_test_thr))),
                                              "median_abs": float(np.median(np.abs(d_test_thr))),
                                              "mean_signed": float(np.mean(d_test_thr))},
        "fold_mean_test_mape_thr_median_over_seeds_per_combo": {
            "max_abs": float(np.max(np.abs(d_test_thr_med))), "median_abs": float(np.median(np.abs(d_test_thr_med))),
            "mean_signed": float(np.mean(d_test_thr_med))},
        "fold_thr_mape_median_per_combo": {"max_abs": float(np.max(np.abs(d_fold_thr))),
                                           "median_abs": float(np.median(np.abs(d_fold_thr)))},
        "fold_thr_mape_mean_per_combo": {"max_abs": float(np.max(np.abs(d_fold_mean))),
                                         "median_abs": float(np.median(np.abs(d_fold_mean)))},
        "population_median_fold_thr_mape": {"fp64": float(np.median(thr64)), "fp32": float(np.median(thr32)),
                                            "abs": float(abs(np.median(thr32) - np.median(thr64)))},
        "population_mean_fold_thr_mape": {"fp64": float(np.mean(thr64)), "fp32": float(np.mean(thr32)),
                                          "abs": float(abs(np.mean(thr32) - np.mean(thr64)))},
        "per_model_abs_thr_mape": {"median": float(np.median(per_model)), "p90": float(np.percentile(per_model, 90)),
                                   "max": float(np.max(per_model))},
    }
    out["per_combo"] = [{"combo": i, "fp64_test_mape_mean": b.test_mape.mean, "fp32_test_mape_mean": a.test_mape.mean,
                         "fp64_test_mape_thr_mean": b.test_mape_thr.mean, "fp32_test_mape_thr_mean": a.test_mape_thr.mean,
                         "fp64_test_mape_thr_median": b.test_mape_thr.median,
                         "fp32_test_mape_thr_median": a.test_mape_thr.median,
                         "fp64_fold_thr_median": b.fold_mape_thr.median, "fp32_fold_thr_median": a.fold_mape_thr.median}
                        for i, (a, b) in enumerate(zip(r32["groups"], r64["groups"]))]
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    out["note"] = ("means over seeds of the fold-mean test MAPE are heavy-tailed on the log-target blur "
                   "combinations (40-47: a diverging seed's exp() extrapolation); medians are the robust statistic")
    with open(os.path.join(ROOT, "gpurun_out", "cv_parity.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "per_combo"}, indent=1))


if __name__ == "__main__":
    main()
