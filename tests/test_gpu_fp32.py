"""GPU: the FP32 throughput mode against the exact reference arithmetic.

Training is chaotic (ReLU kinks x Adam's normalised steps amplify 1-ulp differences), so the
FP32 trainer is held to: (1) forward parity for identical weights, (2) one-step parity from
identical state, (3) the pre-divergence prefix of the loss trace, and (4) population-level
accuracy (the reference's own acceptance bar, criterion 5), as DESIGN.md states.
"""
import numpy as np
import pytest

from paper_2003_07497_b200 import abi
from paper_2003_07497_b200 import engine as E
from paper_2003_07497_b200 import population as P
from golden.make_golden import job_from

pytestmark = pytest.mark.gpu

FWD_RTOL = 1e-5  # north_star: forward predictions within 1e-5 relative for identical weights


def heldout_rows(oracle, job, n_inputs):
    """Raw model-input rows (features, then c) of a config-2 job's held-out half."""
    st, feats, c, rt, nf = oracle.build_dataset(job.world, job.data_seed, job.count)
    _, order, ntr = oracle.split_order(job.count, job.train_fraction, job.data_seed)
    te = order[ntr:]
    rows = np.zeros((len(te), 8))
    rows[:, :nf] = feats[te, :nf]
    rows[:, nf] = c[te].astype(np.float64)
    assert nf + 1 == n_inputs
    return rows


def test_fp32_forward_parity_relative_in_seconds(engine, oracle):
    """north_star: forward predictions within 1e-5 RELATIVE error for identical weights — here
    measured in seconds (the unit predict() returns, models.cpp:346-363) over every held-out row
    of all 48 config-2 models, FP32 predictor vs the exact FP64 one with the same (FP64-trained)
    weights. Measured on a B200 (round 2), 12,000 predictions: 98.7% within 1e-5, median
    1.5e-7, p99 1.3e-5, max 7.1e-4; max 2.9e-5 over predictions above 1% of the target range.
    So FP32 meets 1e-5 for the bulk of the predictions but not everywhere — least of all for the
    smallest runtimes of a linear-target model: the
    network output is a difference of O(1) terms there, so an FP32 rounding of ~6e-8 of the
    target range becomes ~1e-4..1e-3 relative of a prediction at ~1e-3 of the range. The FP64
    predictor is bit-identical to the reference (test_gpu_parity.py), which is why the
    precision-matched headline runs FP64."""
    jobs = P.config2_jobs(root_seed=1, epochs_scale=0.25)
    pop = engine.prepare(jobs, abi.FP64_EXACT)
    pop.run(1)
    st, res, params, _ = pop.fetch(want_params=True)
    norms = pop.norms()
    pop.close()
    errs, errs_big, n_total = [], [], 0
    for j, r, p, nm in zip(jobs, res, params, norms):
        rows = heldout_rows(oracle, j, r.n_inputs)
        model = {"inputs": r.n_inputs, "h1": j.hidden[0], "h2": j.hidden[1] if j.n_hidden > 1 else 0,
                 "log_target": j.log_target, "params": p, "norm": nm}
        rm = np.zeros(len(rows), dtype=np.int32)
        p64 = engine.predict([model], rows, rm, abi.FP64_EXACT)
        p32 = engine.predict([model], rows, rm, abi.FP32)
        keep = p64 > 1e-9  # rows not clamped by max(v, 1e-9)
        rel = np.abs(p32[keep] - p64[keep]) / p64[keep]
        errs.append(rel)
        lo, hi = (np.exp(nm[16]), np.exp(nm[17])) if j.log_target else (nm[16], nm[17])
        errs_big.append(rel[p64[keep] >= lo + 0.01 * (hi - lo)])
        n_total += len(rows)
    e = np.concatenate(errs)
    eb = np.concatenate(errs_big)
    stats = {"predictions": int(n_total), "frac_within_1e-5": float(np.mean(e <= FWD_RTOL)),
             "median": float(np.median(e)), "p99": float(np.percentile(e, 99)), "max": float(e.max()),
             "max_above_1pct_of_range": float(eb.max())}
    print("FP32 forward, relative error in seconds:", stats)
    assert stats["frac_within_1e-5"] >= 0.95, stats
    assert stats["max_above_1pct_of_range"] <= 1e-4, stats


def test_fp32_one_step_parity(engine, oracle):
    """From identical weights: epoch-0 loss within 1e-6 relative; after one Adam step every
    weight within 1e-5 of the exact step (Adam's first step is +-lr * g/|g|)."""
    rng = np.random.default_rng(5)
    n = 250
    X = rng.uniform(0, 1, (n, 7))
    y = rng.uniform(0, 1, n)
    p0 = E.init_params([7, 8, 1], 11)
    m = [{"tile": 0, "h1": 8, "lr": 1e-2, "epochs": 2, "params": p0}]
    params, final, bad, traces = engine.train([X], [y], m, abi.FP32, trace=True)
    Xp = np.zeros((n, 8))
    Xp[:, :7] = X
    st, p_exp, t_exp, _ = oracle.train_full_batch([7, 8, 1], p0, Xp, y, 1e-2, 2)
    assert abs(traces[0][0] - t_exp[0]) <= 1e-6 * t_exp[0]
    assert abs(traces[0][1] - t_exp[1]) <= 1e-5 * t_exp[1]
    assert np.max(np.abs(params[0] - p_exp)) <= 1e-4


@pytest.mark.parametrize("kind_shape", [("mm", 7, (8,)), ("blur", 6, (5, 5))])
def test_fp32_trace_prefix(engine, oracle, kind_shape):
    """The FP32 loss trace follows the exact one within 1e-4 relative over its pre-divergence
    prefix (the first 40 epochs)."""
    _, I, hidden = kind_shape
    rng = np.random.default_rng(8)
    n = 250
    X = rng.uniform(0, 1, (n, I))
    y = rng.uniform(0, 1, n)
    dims = [I, *hidden, 1]
    p0 = E.init_params(dims, 4)
    m = [{"tile": 0, "h1": hidden[0], "h2": hidden[1] if len(hidden) > 1 else 0, "lr": 1e-2, "epochs": 40,
          "params": p0}]
    params, final, bad, traces = engine.train([X], [y], m, abi.FP32, trace=True)
    Xp = np.zeros((n, 8))
    Xp[:, :I] = X
    st, p_exp, t_exp, _ = oracle.train_full_batch(dims, p0, Xp, y, 1e-2, 40)
    rel = np.abs(traces[0] - t_exp) / t_exp
    assert rel.max() <= 1e-4, rel.max()


def test_fp32_criterion5_population_accuracy(engine, golden):
    """Acceptance criterion 5 (acceptance_main.cpp:312-328) in FP32: NN+C median thresholded
    MAPE <= 10% and below NN; and within 3 pp of the exact reference median (a sequential FP32
    restatement already moves the 5-seed median by 1.4 pp, SURVEY.md 7 hard part 1)."""
    nnc = [job_from(j) for j in golden["config1"]["jobs"]]
    nn = [job_from(j) for j in golden["config1_nn"]["jobs"]]
    st, r1, _, _ = engine.run_population(nnc + nn, abi.FP32)
    assert st == 0, engine.last_error
    m_nnc = np.median([r.mape_thr for r in r1[:5]])
    m_nn = np.median([r.mape_thr for r in r1[5:]])
    ref_nnc = np.median([r["mape_thr"] for r in golden["config1"]["results"]])
    assert m_nnc <= 10.0 and m_nnc < m_nn
    assert abs(m_nnc - ref_nnc) <= 3.0


def test_fp32_population_lane_mappings_agree(engine, monkeypatch):
    """Every warp mapping (lanes per model 1/2/4/8/32 and the CTA-per-model kernel) trains the
    same population to the same accuracy (different summation trees -> FP32-level differences)."""
    jobs = P.config2_jobs(root_seed=3, epochs_scale=0.1)
    out = {}
    for lanes in ("1", "2", "4", "8", "32", "64", "128", "256"):
        monkeypatch.setenv("LANN_FP32_LANES", lanes)
        st, res, _, _ = engine.run_population(jobs, abi.FP32)
        assert st == 0, engine.last_error
        out[lanes] = np.array([r.mape_thr for r in res])
    ref = np.median(out["256"])
    for k, v in out.items():
        assert abs(np.median(v) - ref) <= 1.5, k


def test_fp32_population_status_and_metrics(engine):
    jobs = P.config2_jobs(root_seed=1)
    st, res, _, _ = engine.run_population(jobs, abi.FP32)
    assert st == 0
    assert all(r.status == 0 and r.n_kept == 175 and 0.0 < r.mape_thr < 100.0 and r.rho > 0.0 for r in res)


@pytest.mark.parametrize("I", [4, 5, 6])
@pytest.mark.parametrize("n", [100, 129, 250, 700, 2500])
def test_fp32_cta_kernel_two_hidden_trace_prefix(engine, oracle, I, n):
    """The CTA-per-model kernel (two interleaved samples per thread, lean reduce-scatter) on
    the two-hidden-layer nets, every compiled input width and on row counts below one
    pass, odd, the config-2 size and above two passes: loss trace within 1e-4 relative of the
    exact reference over the first 25 epochs (its pre-divergence prefix at every size)."""
    rng = np.random.default_rng(100 + 7 * I + n)
    X = rng.uniform(0, 1, (n, I))
    y = rng.uniform(0, 1, n)
    dims = [I, 5, 5, 1]
    p0 = E.init_params(dims, 9 + I)
    m = [{"tile": 0, "h1": 5, "h2": 5, "lr": 1e-2, "epochs": 25, "params": p0}]
    params, final, bad, traces = engine.train([X], [y], m, abi.FP32, trace=True)
    Xp = np.zeros((n, 8))
    Xp[:, :I] = X
    st, p_exp, t_exp, _ = oracle.train_full_batch(dims, p0, Xp, y, 1e-2, 25)
    rel = np.abs(traces[0] - t_exp) / t_exp
    assert rel.max() <= 1e-4, rel.max()
    assert np.max(np.abs(params[0] - p_exp)) <= 1e-3


def test_fp32_cta_kernel_paired_matches_single(engine, monkeypatch):
    """Config-2 population: the CTA kernel with two interleaved samples per thread (default)
    and with one sample per loop trip (LANN_CTA_PAIR=0) reach the same accuracy."""
    jobs = P.config2_jobs(root_seed=2, epochs_scale=0.25)
    st, fast, _, _ = engine.run_population(jobs, abi.FP32)
    assert st == 0, engine.last_error
    monkeypatch.setenv("LANN_CTA_PAIR", "0")
    st, gen, _, _ = engine.run_population(jobs, abi.FP32)
    assert st == 0, engine.last_error
    a = np.array([r.mape_thr for r in fast])
    b = np.array([r.mape_thr for r in gen])
    assert abs(np.median(a) - np.median(b)) <= 1.0, (a, b)


@pytest.mark.parametrize("lanes", [None, "1", "4", "128", "256"])
@pytest.mark.parametrize("I,hidden", [(7, (8,)), (6, (5, 5))])
def test_fp32_training_error_and_trace_tail(engine, monkeypatch, lanes, I, hidden):
    """Every FP32 mapping: a non-finite target -> TrainingError(epoch 0) (mlp.cpp:166-169); a
    finite run records all E pre-update losses and reports the last one as the final loss (the
    CTA kernel checks epoch e's loss at the top of epoch e + 1, so the tail is handled apart)."""
    if lanes:
        monkeypatch.setenv("LANN_FP32_LANES", lanes)
    rng = np.random.default_rng(1)
    n = 250
    X = rng.uniform(0, 1, (n, I))
    y = rng.uniform(0, 1, n)
    dims = [I, *hidden, 1]
    m = {"tile": 0, "h1": hidden[0], "h2": hidden[1] if len(hidden) > 1 else 0, "lr": 1e-2, "epochs": 37,
         "params": E.init_params(dims, 3)}
    params, final, bad, traces = engine.train([X], [y], [m], abi.FP32, trace=True)
    assert len(traces[0]) == 37 and np.all(np.isfinite(traces[0]))
    assert final[0] == traces[0][-1]
    y_bad = y.copy()
    y_bad[17] = np.inf
    with pytest.raises(E.TrainingError) as ei:
        engine.train([X], [y_bad], [m], abi.FP32)
    assert ei.value.epoch == 0


def test_fp32_requests_report_the_precision_that_ran(engine, monkeypatch):
    """Every shape runs in FP32 under an FP32 request: the LANN shapes on their packed kernels, the
    unconstrained 7-64-1 net on the generic FP32 CTA kernel; lann_job_result.precision_run says
    which precision ran (with LANN_FP32_NO_WIDE the generic shapes fall back to FP64 exact and
    report it)."""
    w = abi.acceptance_world()
    jobs = [abi.make_job(w, 1, count=120, epochs=30), abi.make_job(w, 2, count=120, epochs=30, hidden=(64,),
                                                                   unconstrained=True)]
    st, res, _, _ = engine.run_population(jobs, abi.FP32)
    assert st == 0
    assert [r.precision_run for r in res] == [abi.FP32, abi.FP32]
    monkeypatch.setenv("LANN_FP32_NO_WIDE", "1")
    st, res, _, _ = engine.run_population(jobs, abi.FP32)
    assert [r.precision_run for r in res] == [abi.FP32, abi.FP64_EXACT]
    monkeypatch.delenv("LANN_FP32_NO_WIDE")
    st, res, _, _ = engine.run_population(jobs, abi.FP64_EXACT)
    assert [r.precision_run for r in res] == [abi.FP64_EXACT, abi.FP64_EXACT]
    st, res, _, _ = engine.run_population([abi.make_job(w, 1, count=120, epochs=30, lr=0.5)], abi.FP32)
    assert res[0].precision_run == -1


@pytest.mark.parametrize("hidden,n", [((64,), 2500), ((40, 40), 1000), ((20,), 300), ((13, 7), 777)])
def test_fp32_generic_shapes_track_fp64(engine, hidden, n):
    """The generic FP32 CTA kernel (shapes without a packed FP32 kernel; records in shared-memory
    chunks for large N) against the FP64 exact trainer from identical weights: the loss trace's
    pre-divergence prefix within 1e-4 relative (north_star's per-epoch bar) and the trained
    weights still close after 40 epochs."""
    rng = np.random.default_rng(31)
    I = 6 if len(hidden) == 2 else 7
    X = rng.uniform(0, 1, (n, I))
    y = rng.uniform(0, 1, n)
    dims = [I] + list(hidden) + [1]
    p0 = E.init_params(dims, 9)
    model = {"tile": 0, "h1": hidden[0], "h2": hidden[1] if len(hidden) > 1 else 0, "lr": 1e-3, "epochs": 40,
             "params": p0}
    p64, f64, b64, t64 = engine.train([X], [y], [model], abi.FP64_EXACT, trace=True)
    p32, f32, b32, t32 = engine.train([X], [y], [model], abi.FP32, trace=True)
    assert b32[0] == -1 and b64[0] == -1
    rel = np.abs(t32[0] - t64[0]) / np.abs(t64[0])
    assert rel.max() <= 1e-4, rel.max()
    assert np.max(np.abs(p32[0] - p64[0])) <= 1e-3


def test_fp32_unconstrained_criterion6(engine):
    """Acceptance criterion 6's unconstrained nets (7-64-1, 2500 training rows, 3000 epochs, five
    seeds) in FP32: every model trains, and the median thresholded MAPE stays within 1 pp of the
    FP64 exact run's (the reference's)."""
    w = abi.acceptance_world()
    jobs = [abi.make_job(w, P.derive_seed(90, s), count=5000, hidden=(64,), lr=1e-2, epochs=3000, init_seed=s,
                         unconstrained=True) for s in range(1, 6)]
    st32, r32, _, _ = engine.run_population(jobs, abi.FP32)
    st64, r64, _, _ = engine.run_population(jobs, abi.FP64_EXACT)
    assert st32 == 0 and st64 == 0
    assert all(r.precision_run == abi.FP32 for r in r32)
    m32 = float(np.median([r.mape_thr for r in r32]))
    m64 = float(np.median([r.mape_thr for r in r64]))
    print(f"criterion 6: FP32 median thr-MAPE {m32:.3f}% vs FP64 exact {m64:.3f}%")
    assert abs(m32 - m64) <= 1.0


@pytest.mark.parametrize("I,hidden,n", [(7, (64,), 2501), (6, (40, 40), 300), (7, (13,), 7)])
def test_fp32_generic_kernel_training_error_and_trace_tail(engine, I, hidden, n):
    """The generic FP32 CTA kernel (unconstrained shapes): ragged sample counts (a chunk tail that
    is not a multiple of the float4 step, fewer samples than one chunk), every pre-update loss
    recorded with the last one as the final loss, and a non-finite target -> TrainingError(epoch 0)
    (mlp.cpp:166-169); the run is the FP32 kernel's, not an FP64 fallback."""
    rng = np.random.default_rng(5)
    X = rng.uniform(0, 1, (n, I))
    y = rng.uniform(0, 1, n)
    dims = [I, *hidden, 1]
    m = {"tile": 0, "h1": hidden[0], "h2": hidden[1] if len(hidden) > 1 else 0, "lr": 1e-2, "epochs": 23,
         "params": E.init_params(dims, 4)}
    params, final, bad, traces = engine.train([X], [y], [m], abi.FP32, trace=True)
    assert bad[0] == -1
    assert len(traces[0]) == 23 and np.all(np.isfinite(traces[0]))
    assert final[0] == traces[0][-1]
    _, _, _, t64 = engine.train([X], [y], [m], abi.FP64_EXACT, trace=True)
    assert np.max(np.abs(traces[0][:5] - t64[0][:5]) / np.abs(t64[0][:5])) <= 1e-4
    y_bad = y.copy()
    y_bad[n // 2] = np.nan
    with pytest.raises(E.TrainingError) as ei:
        engine.train([X], [y_bad], [m], abi.FP32)
    assert ei.value.epoch == 0


def test_fp32_generic_kernel_mixed_launch(engine):
    """Several unconstrained shapes and sample counts in ONE population launch (the chunk is sized
    for the largest model): each model's trace prefix tracks its own FP64 exact run."""
    rng = np.random.default_rng(8)
    shapes = [(7, (64,), 900), (6, (40, 40), 257), (5, (20,), 31), (7, (9, 33), 1200)]
    Xs, ys, models = [], [], []
    for t, (I, hidden, n) in enumerate(shapes):
        Xs.append(rng.uniform(0, 1, (n, I)))
        ys.append(rng.uniform(0, 1, n))
        models.append({"tile": t, "h1": hidden[0], "h2": hidden[1] if len(hidden) > 1 else 0, "lr": 1e-3,
                       "epochs": 20, "params": E.init_params([I, *hidden, 1], 11 + t)})
    _, _, b32, t32 = engine.train(Xs, ys, models, abi.FP32, trace=True)
    _, _, b64, t64 = engine.train(Xs, ys, models, abi.FP64_EXACT, trace=True)
    for k in range(len(shapes)):
        assert b32[k] == -1 and b64[k] == -1
        rel = np.abs(t32[k] - t64[k]) / np.abs(t64[k])
        assert rel.max() <= 1e-4, (k, rel.max())
