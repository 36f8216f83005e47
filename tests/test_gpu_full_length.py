"""GPU parity at FULL training length against the reference's own outputs
(tests/golden/golden_r02_full.json, generated from the compiled reference by
tests/golden/make_golden_r02.py).

* FP64 exact mode: the whole config-2 population (40 prediction nets x 8000 epochs, 8 blur
  nets x 20,000 epochs) and the stratified config-3 subset (48 combos x 4 seeds x 5 folds =
  960 models) — every weight, every loss of every epoch (sha256 of the full trace), every
  metric identical (==) to the reference.
* FP32 throughput mode: population-level accuracy against the same goldens, the statistic
  north_star's "final test MAPE within 0.1 percentage points" is applied to (training is
  chaotic, SURVEY.md 7 hard part 1, so per-model FP32 parity is not defined).
"""
import hashlib

import numpy as np
import pytest

from paper_2003_07497_b200 import abi
from paper_2003_07497_b200 import engine as E
from paper_2003_07497_b200 import population as P
from golden.make_golden import job_from

pytestmark = pytest.mark.gpu

MAPE_PP = 0.1  # north_star: final test MAPE within 0.1 percentage points


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def check_metrics(r, exp, log_target):
    assert r.status == exp["status"]
    assert r.final_loss == exp["final_loss"]
    for k in ("mape", "mape_thr", "rho"):
        if log_target:  # predictions de-normalise through exp(): CUDA's exp is within 1 ulp of glibc's
            assert abs(getattr(r, k) - exp[k]) <= 1e-12 * max(1.0, abs(exp[k])), k
        else:
            assert getattr(r, k) == exp[k], k
    for k in ("n_kept", "n_inputs", "n_params", "n_train", "n_eval", "nonfinite_epoch"):
        assert getattr(r, k) == exp[k], k


def subset_jobs(golden_full):
    g = golden_full["config3_subset"]
    jobs = P.config3_jobs(root_seed=1, n_seeds=g["n_seeds"])
    assert hashlib.sha256(b"".join(bytes(j) for j in jobs)).hexdigest() == g["jobs_sha256"]
    return jobs


def test_fp64_config2_full_length_bit_exact(engine, golden_full):
    g = golden_full["config2_full"]
    jobs = [job_from(j) for j in g["jobs"]]
    assert max(j.epochs for j in jobs) == 20000
    st, res, params, traces = engine.run_population(jobs, abi.FP64_EXACT, want_params=True, want_trace=True)
    assert st == 0, engine.last_error
    for j, r, p, t, exp in zip(jobs, res, params, traces, g["results"]):
        check_metrics(r, exp, bool(j.log_target))
        assert np.array_equal(p, np.array(exp["params"]))
        assert len(t) == j.epochs
        assert sha(np.asarray(t, dtype=np.float64)) == exp["trace_sha256"]


def test_fp64_config3_subset_full_length_bit_exact(engine, golden_full):
    jobs = subset_jobs(golden_full)
    st, res, params, _ = engine.run_population(jobs, abi.FP64_EXACT, want_params=True)
    assert st == 0, engine.last_error
    for j, r, p, exp in zip(jobs, res, params, golden_full["config3_subset"]["results"]):
        check_metrics(r, exp, bool(j.log_target))
        assert sha(np.asarray(p, dtype=np.float64)) == exp["params_sha256"]


def fp32_stats(engine, jobs, golden_results):
    st, res, _, _ = engine.run_population(jobs, abi.FP32)
    assert st == 0, engine.last_error
    ref = np.array([e["mape_thr"] for e in golden_results])
    got = np.array([r.mape_thr for r in res])
    d = got - ref
    return {"n": len(jobs), "median_ref": float(np.median(ref)), "median_fp32": float(np.median(got)),
            "mean_ref": float(np.mean(ref)), "mean_fp32": float(np.mean(got)),
            "abs_diff_median": float(np.median(np.abs(d))), "abs_diff_p90": float(np.percentile(np.abs(d), 90)),
            "abs_diff_max": float(np.max(np.abs(d))), "failed": int(sum(1 for r in res if r.status))}


def test_fp32_population_thr_mape_gap(engine, golden_full):
    """The population statistic of the config-3 subset (960 models, full length) under FP32.
    Measured on a B200 (round 2): median held-out thresholded MAPE 13.284 vs the reference's
    13.070 (gap 0.21 pp), mean 16.955 vs 16.874 (0.08 pp); per model |delta| median 0.31 pp,
    p90 3.4 pp, max 92 pp (chaotic divergence). The median gap does NOT meet north_star's
    0.1 pp, which is why the headline runs the FP64 exact mode (bit-identical, above) and FP32
    is reported beside it. This test bounds the gap at what was measured (median <= 0.3 pp,
    mean <= 0.2 pp) so a regression of the FP32 trainer shows."""
    jobs = subset_jobs(golden_full)
    s = fp32_stats(engine, jobs, golden_full["config3_subset"]["results"])
    print("config-3 subset FP32 vs reference:", s)
    assert s["failed"] == 0
    assert abs(s["median_fp32"] - s["median_ref"]) <= 3 * MAPE_PP, s
    assert abs(s["mean_fp32"] - s["mean_ref"]) <= 2 * MAPE_PP, s


def test_fp32_config2_population_report(engine, golden_full):
    """Config 2 (48 models, one per combo) under FP32: no failures; the population statistics
    against the reference are reported (48 chaotic samples are too few for a 0.1 pp bar)."""
    g = golden_full["config2_full"]
    jobs = [job_from(j) for j in g["jobs"]]
    s = fp32_stats(engine, jobs, g["results"])
    print("config-2 FP32 vs reference:", s)
    assert s["failed"] == 0


def test_fp32_full_config3_population_within_0p1pp(engine, golden_full):
    """north_star's "final test MAPE within 0.1 percentage points" on the population it is about:
    the whole config-3 sweep (48 combos x 256 seeds x 5 folds = 61,440 models, full length) in
    FP32 against the FP64-exact sweep, which is the reference's answer (bit-identical: the 960
    golden models of the subset above are checked inside this very run). Measured on a B200
    (round 2, profiles/r02_cv_parity.json): population median held-out thr-MAPE 13.0828 (FP32)
    vs 13.0731 (reference): 0.0098 pp; per combination, the median over seeds of the fold-mean
    model's test thr-MAPE moves by a median 0.03 pp. ~11 s of device time."""
    jobs = P.config3_jobs(root_seed=1, n_seeds=256)
    out = {}
    for prec in (abi.FP64_EXACT, abi.FP32):
        pop = E.Population(engine, jobs, prec)
        pop.run(1)
        st, res, _, _ = pop.fetch()
        groups, _ = pop.cv()
        pop.close()
        assert st == 0 and all(r.status == 0 for r in res)
        out[prec] = (res, groups)
    res64, g64 = out[abi.FP64_EXACT]
    res32, g32 = out[abi.FP32]
    # the FP64 sweep is the reference on the golden subset (seeds 0..3 of every combination)
    g = golden_full["config3_subset"]
    n_sub = g["n_seeds"]
    sub = [r for i, r in enumerate(res64) if (i // 5) % 256 < n_sub]
    for r, exp in zip(sub, g["results"]):
        assert r.final_loss == exp["final_loss"]
    thr64 = np.array([r.mape_thr for r in res64])
    thr32 = np.array([r.mape_thr for r in res32])
    gap = abs(float(np.median(thr32)) - float(np.median(thr64)))
    per_combo = np.abs([a.test_mape_thr.median - b.test_mape_thr.median for a, b in zip(g32, g64)])
    print(f"config 3 FP32 vs reference: population median thr-MAPE {np.median(thr32):.4f} vs "
          f"{np.median(thr64):.4f} (gap {gap:.4f} pp); per-combo fold-mean test thr-MAPE median |d| "
          f"{np.median(per_combo):.4f} pp, max {per_combo.max():.3f} pp")
    assert gap <= MAPE_PP
    assert np.median(per_combo) <= MAPE_PP
