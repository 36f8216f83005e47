"""GPU: the error contract of the C ABI mirrors the reference exceptions (errors.hpp):
ParamError for configs ModelConfig::validate rejects (models.cpp:48-64), SchemaError for
feature-length mismatches, DomainError for metric domains, TrainingError(epoch)."""
import ctypes as C

import numpy as np
import pytest

from paper_2003_07497_b200 import abi
from paper_2003_07497_b200 import engine as E

pytestmark = pytest.mark.gpu


def job(**kw):
    return abi.make_job(abi.acceptance_world(), 1, count=60, epochs=kw.pop("epochs", 5), **kw)


@pytest.mark.parametrize("kw,msg", [
    ({"lr": 0.5}, "learning rate"),
    ({"hidden": (32,)}, "75-parameter budget"),
    ({"hidden": (8, 8, 8)}, None),
    ({"epochs": 0}, "epochs"),
])
def test_param_errors(engine, kw, msg):
    st, res, _, _ = engine.run_population([job(**kw)], abi.FP64_EXACT)
    assert st == abi.PARAM_ERROR and res[0].status == abi.PARAM_ERROR
    if msg:
        assert msg in engine.last_error


def test_unconstrained_lifts_budget(engine):
    st, res, _, _ = engine.run_population([job(hidden=(64,), unconstrained=True)], abi.FP64_EXACT)
    assert st == 0 and res[0].n_params == 577


def test_mixed_population_reports_per_job(engine):
    """A bad job does not poison the rest of the population."""
    st, res, _, _ = engine.run_population([job(), job(lr=0.3), job(epochs=3)], abi.FP64_EXACT)
    assert st == abi.PARAM_ERROR
    assert [r.status for r in res] == [0, abi.PARAM_ERROR, 0]


def test_schema_errors(engine):
    model = {"inputs": 7, "h1": 8, "h2": 0, "log_target": 0, "params": np.zeros(73), "norm": np.zeros(18)}
    with pytest.raises(E.SchemaError):
        engine.predict([model], np.zeros((2, 7)), np.array([0, 3], dtype=np.int32))
    with pytest.raises(E.SchemaError):  # selection needs the blur schema (selector.cpp:44-45)
        engine.select_schedule(model, 1024, np.array([[2, 2, 2, 2]], dtype=np.uint32))
    with pytest.raises(E.SchemaError):
        engine.select_variants([model], [1], abi.MV, 4, 1, 0, 10)


def test_select_needs_candidates(engine):
    model = {"inputs": 6, "h1": 5, "h2": 5, "log_target": 1, "params": np.zeros(71), "norm": np.zeros(18)}
    with pytest.raises(E.ParamError):
        engine.select_schedule(model, 1024, np.zeros((0, 4), dtype=np.uint32))


def test_training_error_in_population(engine):
    """A world whose runtimes overflow to inf: BuildAbortError-free dataset, TrainingError epoch."""
    w = abi.acceptance_world()
    w.alpha = 1e300
    st, res, _, _ = engine.run_population([abi.make_job(w, 1, count=60, epochs=5)], abi.FP64_EXACT)
    assert st in (abi.TRAINING_ERROR, abi.PARAM_ERROR, abi.BUILD_ABORT)


def test_population_wide_check_failure_is_an_error_not_a_crash(engine):
    """A failure of the checks that run after packing (hidden widths over 64, which the
    unconstrained budget lets through) comes back as PARAM_ERROR for the whole population,
    with or without good jobs beside it (a null launch plan was run)."""
    bad = job(hidden=(65,), unconstrained=True)
    st, res, _, _ = engine.run_population([bad], abi.FP64_EXACT)
    assert st == abi.PARAM_ERROR
    st, res, _, _ = engine.run_population([job(), bad], abi.FP64_EXACT)
    assert st == abi.PARAM_ERROR
    with pytest.raises(E.ParamError):
        engine.prepare([job(), bad], abi.FP64_EXACT)


def test_all_jobs_failing_keep_their_own_statuses(engine):
    """Every job fails host preparation: each result carries its own status (a DomainError for
    a one-sample evaluation set beside ParamErrors), not one aggregate code."""
    tiny = abi.make_job(abi.acceptance_world(), 1, count=3, epochs=5)  # 2 train / 1 eval sample
    st, res, _, _ = engine.run_population([job(lr=0.5), tiny, job(hidden=(32,))], abi.FP64_EXACT)
    assert st != 0
    assert [r.status for r in res] == [abi.PARAM_ERROR, abi.DOMAIN_ERROR, abi.PARAM_ERROR]


def test_large_evaluation_set(engine, oracle):
    """Evaluation sets beyond one CTA's shared memory (the reference takes any size) go
    through the global-memory metric kernels, bit-identical to the reference order."""
    rng = np.random.default_rng(5)
    n = 12000
    t = rng.uniform(1e-6, 1e-3, n)
    t[::7] = t[3]  # ties in the truth
    p = t * rng.uniform(0.8, 1.25, n)
    p[::11] = p[5]  # ties in the predictions
    mape, thr, kept, rho = engine.eval([t, t[:300]], [p, p[:300]], 0.3)
    for k, (tt, pp) in enumerate([(t, p), (t[:300], p[:300])]):
        assert mape[k] == oracle.mape(tt, pp)[1]
        _, othr, okept = oracle.mape_thresholded(tt, pp, 0.3)
        assert (thr[k], kept[k]) == (othr, okept)
        assert rho[k] == oracle.spearman(tt, pp)[1]


def test_population_with_large_evaluation_set(engine, oracle):
    """count 14000 -> 7000 held-out samples per model: runs (was 'evaluation set too large')."""
    j = abi.make_job(abi.acceptance_world(), 2, count=14000, epochs=3)
    st, res, _, _ = engine.run_population([j], abi.FP64_EXACT)
    assert st == 0, engine.last_error
    ref, _, _ = oracle.run_job(j)
    assert (res[0].mape, res[0].mape_thr, res[0].rho) == (ref.mape, ref.mape_thr, ref.rho)


@pytest.mark.gpu
def test_population_outlives_its_engine():
    """Closing an engine frees the populations prepared on it (C ABI: lann_engine_destroy frees
    them; lann_population_destroy on such a handle, or twice, is a no-op) — no use-after-free."""
    eng = E.Engine(0)
    pops = [E.Population(eng, [job(epochs=5)], abi.FP64_EXACT) for _ in range(3)]
    pops[0].run(1)
    pops[1].close()
    pops[1].close()
    eng.close()
    for p in pops:
        with pytest.raises(E.Error):
            p.run(1)
        p.close()
    # the C handles directly: the engine frees a population it still owns; destroying that handle
    # afterwards (twice) is a no-op
    eng2 = E.Engine(0)
    arr = (abi.Job * 1)(job(epochs=5))
    raw = C.c_void_p()
    assert eng2.L.lann_population_create(eng2.h, 1, arr, abi.FP64_EXACT, 0, C.byref(raw)) == 0
    assert eng2.L.lann_population_run(raw, 1) == 0
    eng2.close()
    eng2.L.lann_population_destroy(raw)
    eng2.L.lann_population_destroy(raw)
