"""GPU parity: the CUDA engine (through the C ABI) against the reference's own outputs
(golden vectors from the compiled reference) and the C oracle on the same seeded inputs.

FP64 exact mode: bit-identical (==) loss traces, weights, predictions, metrics, argmins.
"""
import hashlib

import numpy as np
import pytest

from paper_2003_07497_b200 import abi
from paper_2003_07497_b200 import engine as E
from paper_2003_07497_b200 import population as P
from golden.make_golden import job_from

pytestmark = pytest.mark.gpu


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def check(r, exp, params=None, trace=None, log_target=False):
    """Training outputs (loss, weights) must be identical. Metrics too, except for log-target
    models, whose predictions de-normalise through exp(): CUDA's exp is within 1 ulp of glibc's
    (models.cpp:138), so their MAPEs agree to ~1e-15 relative, and rho exactly unless a 1-ulp
    change breaks a prediction tie."""
    assert r.status == exp["status"]
    assert r.final_loss == exp["final_loss"]
    for k in ("mape", "mape_thr", "rho"):
        if log_target:
            assert abs(getattr(r, k) - exp[k]) <= 1e-12 * max(1.0, abs(exp[k])), k
        else:
            assert getattr(r, k) == exp[k], k
    for k in ("n_kept", "n_inputs", "n_params", "n_train", "n_eval"):
        assert getattr(r, k) == exp[k], k
    if params is not None and "params" in exp:
        assert np.array_equal(params, np.array(exp["params"]))
    if trace is not None and "trace_sha256" in exp:
        assert sha(np.asarray(trace, dtype=np.float64)) == exp["trace_sha256"]


@pytest.mark.parametrize("arm", ["config1", "config1_nn"])
def test_fp64_config1_bit_exact(engine, golden, arm):
    """8000-epoch training of the acceptance model, seeds 1..5: every loss, weight, metric identical."""
    jobs = [job_from(j) for j in golden[arm]["jobs"]]
    st, res, params, traces = engine.run_population(jobs, abi.FP64_EXACT, want_params=True, want_trace=True)
    assert st == 0, engine.last_error
    for r, p, t, exp in zip(res, params, traces, golden[arm]["results"]):
        check(r, exp, p, t)


def test_fp64_population_bit_exact(engine, golden):
    """All 48 combos (one population, one launch set) with 200 epochs each."""
    jobs = [job_from(j) for j in golden["config2_short"]["jobs"]]
    st, res, params, _ = engine.run_population(jobs, abi.FP64_EXACT, want_params=True)
    assert st == 0, engine.last_error
    for j, r, p, exp in zip(jobs, res, params, golden["config2_short"]["results"]):
        check(r, exp, p, log_target=bool(j.log_target))


def test_fp64_kfold_sweep_bit_exact(engine, golden):
    jobs = [job_from(j) for j in golden["config3_kfold_short"]["jobs"]]
    st, res, params, _ = engine.run_population(jobs, abi.FP64_EXACT, want_params=True)
    assert st == 0, engine.last_error
    for j, r, p, exp in zip(jobs, res, params, golden["config3_kfold_short"]["results"]):
        check(r, exp, p, log_target=bool(j.log_target))


def test_fp64_sharded_population_identical(engine, golden):
    """Multi-GPU invariant: a population trained as 1, 2 or 4 contiguous
    shards (what ranks of bench.py / sharding.shard run) gives bit-identical results."""
    from paper_2003_07497_b200 import sharding
    jobs = [job_from(j) for j in golden["config3_kfold_short"]["jobs"]]
    st, whole, _, _ = engine.run_population(jobs, abi.FP64_EXACT)
    assert st == 0
    for world in (2, 4):
        merged = []
        for rank in range(world):
            part, off = sharding.shard(jobs, rank, world)
            st, res, _, _ = engine.run_population(part, abi.FP64_EXACT)
            assert st == 0
            merged.extend(res)
        assert [(r.final_loss, r.mape, r.mape_thr, r.rho) for r in merged] == \
               [(r.final_loss, r.mape, r.mape_thr, r.rho) for r in whole]


def random_problem(rng, I, dims_hidden, n):
    X = np.zeros((n, I))
    X[:] = rng.uniform(0, 1, (n, I))
    y = rng.uniform(0, 1, n)
    return X, y


@pytest.mark.parametrize("seed", range(4))
def test_fp64_train_random_shapes(engine, oracle, seed):
    """lann_train (train_full_batch) on random shapes / sizes / learning rates, one batched call."""
    rng = np.random.default_rng(100 + seed)
    tiles_X, tiles_y, models, expect = [], [], [], []
    for k in range(10):
        I = int(rng.integers(1, 8))
        hidden = [int(rng.integers(1, 10))] + ([int(rng.integers(1, 8))] if k % 3 == 0 else [])
        n = int(rng.integers(2, 300))
        X, y = random_problem(rng, I, hidden, n)
        dims = [I] + hidden + [1]
        p0 = E.init_params(dims, int(rng.integers(0, 1000)))
        lr = [1e-2, 1e-3, 1e-4][k % 3]
        epochs = int(rng.integers(1, 120))
        tiles_X.append(X)
        tiles_y.append(y)
        models.append({"tile": k, "h1": hidden[0], "h2": hidden[1] if len(hidden) > 1 else 0, "lr": lr,
                       "epochs": epochs, "params": p0})
        Xp = np.zeros((n, 8))
        Xp[:, :I] = X
        expect.append(oracle.train_full_batch(dims, p0, Xp, y, lr, epochs))
    params, final, bad, traces = engine.train(tiles_X, tiles_y, models, abi.FP64_EXACT, trace=True)
    for m, (st, p_exp, t_exp, b_exp) in enumerate(expect):
        assert st == 0 and bad[m] == -1
        assert np.array_equal(params[m], p_exp), m
        assert np.array_equal(traces[m], t_exp), m
        assert final[m] == t_exp[-1]


@pytest.mark.parametrize("global_records", [False, True])
def test_fp64_records_larger_than_shared_memory(engine, oracle, monkeypatch, global_records):
    """Models whose per-sample records exceed one CTA's shared memory: processed in chunks of
    samples held in shared memory, the chains carrying over between chunks (default), or in global
    scratch (LANN_FP64_GLOBAL_RECORDS=1). Compiled wide net (7-64-1, criterion 6's unconstrained
    shape), generic 1- and 2-hidden-layer shapes (6-40-40-1: eight chains per thread), a LANN
    shape on N > 256 rows, odd and even N: weights and every epoch's loss == the oracle."""
    if global_records:
        monkeypatch.setenv("LANN_FP64_GLOBAL_RECORDS", "1")
    rng = np.random.default_rng(21)
    cases = [(7, [64], 2500, 4), (6, [40, 40], 1001, 3), (3, [20], 3001, 3), (7, [8], 1999, 6),
             (4, [5, 5], 777, 6), (2, [9], 600, 5)]
    tiles_X, tiles_y, models, expect = [], [], [], []
    for k, (I, hidden, n, epochs) in enumerate(cases):
        X, y = random_problem(rng, I, hidden, n)
        dims = [I] + hidden + [1]
        p0 = E.init_params(dims, 40 + k)
        tiles_X.append(X)
        tiles_y.append(y)
        models.append({"tile": k, "h1": hidden[0], "h2": hidden[1] if len(hidden) > 1 else 0, "lr": 1e-3,
                       "epochs": epochs, "params": p0})
        Xp = np.zeros((n, 8))
        Xp[:, :I] = X
        expect.append(oracle.train_full_batch(dims, p0, Xp, y, 1e-3, epochs))
    params, final, bad, traces = engine.train(tiles_X, tiles_y, models, abi.FP64_EXACT, trace=True)
    for m, (st, p_exp, t_exp, b_exp) in enumerate(expect):
        assert st == 0 and bad[m] == -1
        assert np.array_equal(params[m], p_exp), cases[m]
        assert np.array_equal(traces[m], t_exp), cases[m]


def test_fp64_unconstrained_global_scratch(engine, oracle):
    """Unconstrained width (7->64->1, P=577) on N=2500 rows: per-sample records exceed shared
    memory (chunked shared-memory records; criterion 6 shape, acceptance_main.cpp:330-348)."""
    rng = np.random.default_rng(9)
    X, y = random_problem(rng, 7, [64], 2500)
    dims = [7, 64, 1]
    p0 = E.init_params(dims, 3)
    params, final, bad, traces = engine.train([X], [y], [{"tile": 0, "h1": 64, "lr": 1e-2, "epochs": 4,
                                                         "params": p0}], abi.FP64_EXACT, trace=True)
    Xp = np.zeros((2500, 8))
    Xp[:, :7] = X
    st, p_exp, t_exp, _ = oracle.train_full_batch(dims, p0, Xp, y, 1e-2, 4)
    assert np.array_equal(params[0], p_exp) and np.array_equal(traces[0], t_exp)


def test_training_error_epoch(engine):
    """Non-finite loss -> TrainingError naming the epoch (mlp.cpp:166-169)."""
    X = np.ones((4, 2))
    y = np.array([0.0, 1.0, np.inf, 0.5])
    p0 = E.init_params([2, 3, 1], 1)
    for prec in (abi.FP64_EXACT, abi.FP32):
        with pytest.raises(E.TrainingError) as ei:
            engine.train([X], [y], [{"tile": 0, "h1": 3, "lr": 1e-2, "epochs": 10, "params": p0}], prec)
        assert ei.value.epoch == 0


def test_predict_fp64_bit_exact(engine, oracle, golden):
    g = golden["predict_config1_seed1"]
    st, feats, c, rt, nf = oracle.build_dataset(abi.acceptance_world(), 1, 500)
    _, order, ntr = oracle.split_order(500, 0.5, 1)
    te = order[ntr:]
    rows = np.zeros((len(te), 8))
    rows[:, :6] = feats[te, :6]
    rows[:, 6] = c[te].astype(np.float64)
    model = {"inputs": 7, "h1": 8, "h2": 0, "log_target": 0, "params": np.array(g["params"]),
             "norm": np.array(g["norm"])}
    pred = engine.predict([model], rows, np.zeros(len(te), dtype=np.int32), abi.FP64_EXACT)
    assert sha(pred) == g["pred_sha256"]


def test_predict_log_target_within_one_ulp(engine, oracle, golden):
    """Log-target (blur) models de-normalise through exp: CUDA's exp is within 1 ulp of glibc's."""
    s = golden["select"]
    lat = np.array(s["sample100_seed3"], dtype=np.uint32)
    rows = np.zeros((len(lat), 8))
    rows[:, 0] = 4096.0
    rows[:, 1:5] = lat
    rows[:, 5] = 4096.0 ** 2
    model = {"inputs": 6, "h1": 5, "h2": 5, "log_target": 1, "params": np.array(s["params"]), "norm": np.array(s["norm"])}
    pred = engine.predict([model], rows, np.zeros(len(lat), dtype=np.int32), abi.FP64_EXACT)
    ref = np.array([oracle.predict_row(6, (5, 5), model["params"], model["norm"], True, r[:6]) for r in rows])
    assert np.all(np.abs(pred - ref) <= 2 * np.spacing(ref))


def test_eval_bit_exact(engine, golden):
    sets = [m for m in golden["metrics"] if m["mape_thr"] is not None and m["rho"] is not None]
    mape, thr, kept, rho = engine.eval([m["truth"] for m in sets], [m["pred"] for m in sets])
    for i, m in enumerate(sets):
        assert (mape[i], thr[i], kept[i], rho[i]) == (m["mape"], m["mape_thr"], m["n_kept"], m["rho"])


def test_eval_domain_errors(engine):
    with pytest.raises(E.DomainError):
        engine.eval([[1.0, 0.0]], [[1.0, 1.0]])  # truth must be > 0 (eval.cpp:16-22)
    with pytest.raises(E.DomainError):
        engine.eval([[1.0]], [[1.0]])  # spearman needs two samples
    with pytest.raises(E.DomainError):
        engine.eval([[1.0, 2.0]], [[1.0, 2.0]], drop=1.0)  # threshold would drop every sample


def test_select_schedule_matches_reference(engine, golden):
    s = golden["select"]
    from test_oracle_golden import lattice
    lat = lattice(0)
    model = {"inputs": 6, "h1": 5, "h2": 5, "log_target": 1, "params": np.array(s["params"]), "norm": np.array(s["norm"])}
    for ch in s["choices"]:
        i, score = engine.select_schedule(model, ch["n_img"], lat)
        assert i == ch["chosen"]
        assert abs(score - ch["score"]) <= 2 * np.spacing(ch["score"])


def test_select_schedule_tie_rule(engine):
    """Ties go to the lexicographically smaller schedule (selector.cpp:38-39,
    test_selector.cpp:66-75): a constant model scores every candidate the same."""
    from test_oracle_golden import lattice
    lat = lattice(0)[::-1].copy()  # reversed order: smallest schedule is last
    p = np.zeros(E.param_count(6, 5, 5))
    norm = np.zeros(18)
    norm[16] = norm[17] = np.log(0.5)
    model = {"inputs": 6, "h1": 5, "h2": 5, "log_target": 1, "params": p, "norm": norm}
    i, score = engine.select_schedule(model, 1024, lat)
    assert tuple(lat[i]) == (2, 2, 2, 2) and score == 0.5


def trained_variant_models(engine):
    jobs = P.config2_jobs(root_seed=1, epochs_scale=0.05)
    pop = engine.prepare(jobs, abi.FP64_EXACT)
    pop.run(1)
    st, res, params, _ = pop.fetch(want_params=True)
    norms = pop.norms()
    pop.close()
    return jobs, res, params, norms


@pytest.mark.parametrize("max_threads", [16, 12, 5000])
def test_select_variants_fp64_bit_exact(engine, oracle, max_threads):
    """Counter-generated candidates (Rng::bounded's rejection rule: power-of-two, table-driven
    exact remainder for n <= 4096, and the plain 64-bit modulo above) and exact-order scores are
    identical to the C oracle for every kernel kind."""
    jobs, res, params, norms = trained_variant_models(engine)
    for kind in (abi.MM, abi.MV, abi.MC, abi.MP):
        idx = [i for i, j in enumerate(jobs) if j.world.kind == kind]
        models = [{"inputs": res[i].n_inputs, "h1": 8, "h2": 0, "log_target": 0, "params": params[i],
                   "norm": norms[i]} for i in idx]
        thd = np.array([1 if jobs[i].world.hw_class == abi.HW_CPU else 0 for i in idx], dtype=np.int32)
        n = 4000
        gi, gs = engine.select_variants(models, thd, kind, max_threads, 7, 1000, n, precision=abi.FP64_EXACT)
        ms, keep = E._model_set(models, abi.FP64_EXACT)
        oi = np.zeros(n, dtype=np.int32)
        os_ = np.zeros(n)
        oracle.lib.or_select_variants(ms, thd, kind, max_threads, 7, 1000, n, oi, os_)
        assert np.array_equal(gi, oi) and np.array_equal(gs, os_)


def test_select_variants_fp32_argmin(engine, oracle):
    """FP32 scorer: argmin identical to the exact oracle except where the best two scores are
    within the FP32 tolerance (relative gap < 1e-4)."""
    jobs, res, params, norms = trained_variant_models(engine)
    kind = abi.MM
    idx = [i for i, j in enumerate(jobs) if j.world.kind == kind]
    models = [{"inputs": res[i].n_inputs, "h1": 8, "h2": 0, "log_target": 0, "params": params[i], "norm": norms[i]}
              for i in idx]
    thd = np.array([1 if jobs[i].world.hw_class == abi.HW_CPU else 0 for i in idx], dtype=np.int32)
    n = 20000
    gi, gs = engine.select_variants(models, thd, kind, 16, 7, 0, n, precision=abi.FP32)
    ei, es = engine.select_variants(models, thd, kind, 16, 7, 0, n, precision=abi.FP64_EXACT)
    mism = np.nonzero(gi != ei)[0]
    for i in mism:  # a flipped argmin must be a near-tie: its exact score is within tolerance
        assert abs(gs[i] - es[i]) <= 1e-4 * abs(es[i]) + 1e-9, (i, gs[i], es[i])
    assert len(mism) <= n * 1e-3
    both = gi == ei
    assert np.all(np.abs(gs[both] - es[both]) <= 1e-3 * np.abs(es[both]) + 1e-7)


def test_compact_streamed_selection_equals_the_full_outputs(engine):
    """lann_select_variants_compact (uint8 index + float score, chunked copies overlapping the
    scoring, win histogram): the same argmins and scores as lann_select_variants, into pinned
    and pageable buffers, and hist == bincount(idx)."""
    rng = np.random.default_rng(11)
    models = []
    for v in range(10):
        I = 7 if v % 2 == 0 else 6  # with / without n_thd (augmented MM nets)
        p = rng.uniform(-1, 1, (I + 1) * 8 + 9)
        nrm = np.zeros(18)
        nrm[:8] = rng.uniform(0, 10, 8)
        nrm[8:16] = nrm[:8] + rng.uniform(1, 1e3, 8)
        nrm[16], nrm[17] = -12.0, -2.0
        models.append({"inputs": I, "h1": 8, "h2": 0, "log_target": 1, "params": p, "norm": nrm})
    thd = [1 if v % 2 == 0 else 0 for v in range(10)]
    n = 3_000_001
    idx, score = engine.select_variants(models, thd, abi.MM, 4, 7, 11, n)
    pi, ps = E.Pinned(n, np.uint8), E.Pinned(n, np.float32)
    for bi, bs in [(pi.array, ps.array), (np.zeros(n, np.uint8), np.zeros(n, np.float32))]:
        ci, cs, hist = engine.select_variants_compact(models, thd, abi.MM, 4, 7, 11, n, idx=bi, score=bs)
        assert np.array_equal(ci.astype(np.int32), idx)
        assert np.array_equal(cs, score.astype(np.float32))
        assert np.array_equal(hist, np.bincount(idx, minlength=10))
    _, _, hist = engine.select_variants_compact(models, thd, abi.MM, 4, 7, 11, n)  # histogram only
    assert np.array_equal(hist, np.bincount(idx, minlength=10))
    pi.free()
    ps.free()


def test_batched_predictor_compiled_and_generic_shapes(engine, oracle):
    """lann_predict over a mixed model set: compiled shapes (I-8-1, I-5-5-1, unrolled) and
    generic ones (7-64-1, 3-12-6-1), rows interleaved across models: FP64 exact == the oracle's
    predict (models.cpp:346-363) row by row; FP32 within 1e-5 of the target range."""
    rng = np.random.default_rng(3)
    shapes = [(7, (8,), 0), (4, (8,), 0), (6, (5, 5), 1), (5, (5, 5), 0), (7, (64,), 0), (3, (12, 6), 1)]
    models = []
    for I, h, lt in shapes:
        P_ = (I + 1) * h[0] + ((h[0] + 1) * h[1] + h[1] + 1 if len(h) > 1 else h[0] + 1)
        nrm = np.zeros(18)
        nrm[:I] = rng.uniform(0, 100, I)
        nrm[8:8 + I] = nrm[:I] + rng.uniform(1, 1e4, I)
        nrm[16], nrm[17] = (-9.0, -1.0) if lt else (1e-6, 2e-3)
        models.append({"inputs": I, "h1": h[0], "h2": h[1] if len(h) > 1 else 0, "log_target": lt,
                       "params": rng.uniform(-0.6, 0.6, P_), "norm": nrm})
    n = 6000
    rm = rng.integers(0, len(models), n).astype(np.int32)
    rows = np.zeros((n, 8))
    for r in range(n):
        m = models[rm[r]]
        rows[r, : m["inputs"]] = rng.uniform(m["norm"][: m["inputs"]], m["norm"][8: 8 + m["inputs"]])
    got = engine.predict(models, rows, rm, precision=abi.FP64_EXACT)
    for r in range(0, n, 7):
        m = models[rm[r]]
        h = (m["h1"],) if m["h2"] == 0 else (m["h1"], m["h2"])
        ref = oracle.predict_row(m["inputs"], h, m["params"], m["norm"], m["log_target"], rows[r, : m["inputs"]])
        if m["log_target"]:  # exp through CUDA's libm (<= 1 ulp from glibc), DESIGN 4
            assert abs(got[r] - ref) <= 4e-16 * abs(ref)
        else:
            assert got[r] == ref
    got32 = engine.predict(models, rows, rm, precision=abi.FP32)
    for r in range(n):
        m = models[rm[r]]
        if not m["log_target"]:
            assert abs(got32[r] - got[r]) <= 1e-5 * (m["norm"][17] - m["norm"][16]) + 1e-12


@pytest.mark.parametrize("kernel", ["4", "41", "42", "43"])
def test_fp64_pipeline_kernels_edge_sizes(engine, oracle, monkeypatch, kernel):
    """The FP64 kernels of the LANN shapes — the latency pipeline (product records, 4), the
    throughput pipeline (factor records, two CTAs per SM, 41) and the pair-row latency variant
    (two rows per chain lane, a padding slot for odd row counts: 5-5-5, 42) — on sample counts around the
    32-sample blocks and producer rounds (2, 7, 31, 32, 33, 100, 129, 255, 256), one- and two-hidden
    layer shapes: weights and every epoch's loss == the oracle."""
    monkeypatch.setenv("LANN_FP64_PRODUCERS", kernel)
    rng = np.random.default_rng(77)
    tiles_X, tiles_y, models, expect, cases = [], [], [], [], []
    for k, n in enumerate((2, 7, 31, 32, 33, 100, 129, 255, 256)):
        for I, hidden in ((7, [8]), (4, [8]), (6, [5, 5]), (5, [5, 5])):
            X, y = random_problem(rng, I, hidden, n)
            dims = [I] + hidden + [1]
            p0 = E.init_params(dims, 7 * k + I)
            t = len(tiles_X)
            tiles_X.append(X)
            tiles_y.append(y)
            models.append({"tile": t, "h1": hidden[0], "h2": hidden[1] if len(hidden) > 1 else 0, "lr": 1e-2,
                           "epochs": 9, "params": p0})
            Xp = np.zeros((n, 8))
            Xp[:, :I] = X
            expect.append(oracle.train_full_batch(dims, p0, Xp, y, 1e-2, 9))
            cases.append((I, hidden, n))
    params, final, bad, traces = engine.train(tiles_X, tiles_y, models, abi.FP64_EXACT, trace=True)
    for m, (st, p_exp, t_exp, b_exp) in enumerate(expect):
        assert st == 0 and bad[m] == -1
        assert np.array_equal(params[m], p_exp), cases[m]
        assert np.array_equal(traces[m], t_exp), cases[m]
