"""CPU: the C oracle (oracle/lann_oracle.c) against golden vectors produced by the
REFERENCE ITSELF (tests/golden/make_golden.py runs the compiled reference core), and
against the compiled reference directly where it is present (oracle/_ref)."""
import hashlib

import numpy as np
import pytest

from paper_2003_07497_b200 import abi
from golden.make_golden import job_from, world_from


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def check_result(r, exp, params=None, trace=None):
    assert r.status == exp["status"]
    for k in ("final_loss", "mape", "mape_thr", "rho"):
        assert getattr(r, k) == exp[k], k  # bit-exact
    for k in ("n_kept", "n_inputs", "n_params", "n_train", "n_eval"):
        assert getattr(r, k) == exp[k], k
    if params is not None and "params" in exp:
        assert np.array_equal(params, np.array(exp["params"]))
    if trace is not None and "trace_sha256" in exp:
        assert trace[:5].tolist() == exp["trace_head"]
        assert sha(np.asarray(trace, dtype=np.float64)) == exp["trace_sha256"]


@pytest.mark.parametrize("arm", ["config1", "config1_nn"])
def test_config1_full_training_bit_exact(oracle, golden, arm):
    """Acceptance criterion 5 protocol (acceptance_main.cpp:312-328), 8000 epochs, seeds 1..5."""
    for jd, exp in zip(golden[arm]["jobs"], golden[arm]["results"]):
        r, params, trace = oracle.run_job(job_from(jd), want_params=True, want_trace=True)
        check_result(r, exp, params, trace)


def test_config1_seed1_known_values(golden):
    # SURVEY.md 7 minimum-slice numbers, from the reference run
    r = golden["config1"]["results"][0]
    assert r["trace_head"][:2] == [0.324627613197639, 0.27518962559376992]
    assert abs(r["final_loss"] - 8.87098e-05) < 1e-9
    assert round(r["mape_thr"], 4) == 6.8151 and round(r["rho"], 4) == 0.9935


def test_criterion5_augmentation_advantage(golden):
    """NN+C median thr-MAPE <= 10% and below NN (acceptance_main.cpp:326-327)."""
    nnc = np.median([r["mape_thr"] for r in golden["config1"]["results"]])
    nn = np.median([r["mape_thr"] for r in golden["config1_nn"]["results"]])
    assert nnc <= 10.0 and nnc < nn


def test_combo_datasets_and_splits(oracle, golden):
    for d in golden["combos"]:
        st, feats, c, rt, nf = oracle.build_dataset(world_from(d["world"]), d["seed"], 500)
        assert st == 0 and nf == d["n_features"]
        assert sha(feats, c, rt) == d["sha256"]
        st, order, ntr = oracle.split_order(500, 0.5, d["seed"])
        assert sha(order) == d["split_sha256"] and ntr == d["n_train"]


def test_population_short_training(oracle, golden):
    for jd, exp in zip(golden["config2_short"]["jobs"], golden["config2_short"]["results"]):
        r, params, _ = oracle.run_job(job_from(jd), want_params=True)
        check_result(r, exp, params)


def test_kfold_slice(oracle, golden):
    for jd, exp in zip(golden["config3_kfold_short"]["jobs"], golden["config3_kfold_short"]["results"]):
        r, params, _ = oracle.run_job(job_from(jd), want_params=True)
        check_result(r, exp, params)


def test_metrics(oracle, golden):
    for m in golden["metrics"]:
        t, p = np.array(m["truth"]), np.array(m["pred"])
        assert oracle.mape(t, p)[1] == m["mape"]
        st, thr, kept = oracle.mape_thresholded(t, p, 0.3)
        if m["mape_thr"] is None:
            assert st == abi.DOMAIN_ERROR
        else:
            assert (thr, kept) == (m["mape_thr"], m["n_kept"])
        st, rho = oracle.spearman(t, p)
        if m["rho"] is None:
            assert st == abi.DOMAIN_ERROR
        else:
            assert rho == m["rho"]


def test_metric_hand_examples(oracle):
    # test_eval.cpp:64-68, 92-135, 137-157
    assert oracle.mape([1.0, 2.0], [2.0, 1.0])[1] == 75.0
    assert oracle.mape([100.0], [90.0])[1] == 10.0
    assert abs(oracle.spearman([1.0, 2.0, 3.0, 4.0], [1.0, 3.0, 2.0, 4.0])[1] - 0.8) < 1e-12
    assert oracle.spearman([0.1, 0.2, 0.5, 0.9], [4.0, 3.0, 2.0, 1.0])[1] == -1.0
    t = np.arange(1, 11, dtype=float)
    st, v, k = oracle.mape_thresholded(t, t * 1.1, 0.3)
    assert k == 7 and abs(v - 10.0) < 1e-9
    assert oracle.mape([0.0], [1.0])[0] == abi.DOMAIN_ERROR
    assert oracle.mape_thresholded([1.0, 2.0], [1.0, 2.0], 1.0)[0] == abi.DOMAIN_ERROR
    assert oracle.spearman([1.0], [1.0])[0] == abi.DOMAIN_ERROR


def test_schedule_selection(oracle, golden):
    s = golden["select"]
    assert s["lattice_sizes"] == {"cpu": 2200, "gpu_style": 196}  # test_selector.cpp:15-21
    from oracle_lib import ROW  # noqa: F401
    lat = lattice(0)
    assert sha(lat) == s["cpu_lattice_sha256"]
    for ch in s["choices"]:
        i, score = oracle.select_schedule(abi.NNC, s["hidden"], np.array(s["params"]), np.array(s["norm"]),
                                          s["log_target"], ch["n_img"], lat)
        assert i == ch["chosen"] and score == ch["score"]


def lattice(gpu_style):
    """ScheduleSpace::enumerate_all (kernels.cpp:77-87), lexicographic."""
    out = []
    if gpu_style:
        for a in (2, 4, 8, 16):
            for b in (1, 2, 4, 8, 16, 32, 64):
                for c in (1, 2, 4, 8, 16, 32, 64):
                    out.append((a, b, c, 1))
    else:
        p2 = [2 ** k for k in range(1, 11)]
        for a in p2:
            for b in p2:
                for c in [x for x in p2 if x <= b]:
                    for d in [x for x in p2 if x <= c]:
                        out.append((a, b, c, d))
    return np.array(out, dtype=np.uint32)


def test_predict_rows(oracle, golden):
    g = golden["predict_config1_seed1"]
    w = abi.acceptance_world()
    st, feats, c, rt, nf = oracle.build_dataset(w, 1, 500)
    _, order, ntr = oracle.split_order(500, 0.5, 1)
    te = order[ntr:]
    pred = np.array([oracle.predict_row(7, (8,), np.array(g["params"]), np.array(g["norm"]), False,
                                        np.concatenate([feats[i][:6], [float(c[i])]])) for i in te])
    assert pred[:5].tolist() == g["pred_head"]
    assert sha(pred) == g["pred_sha256"]


def test_mse_gradient(oracle, golden):
    for g in golden["mse_gradient"]:
        st, loss, grad = oracle.mse_gradient(g["dims"], np.array(g["params"]), np.array(g["X"]), np.array(g["y"]))
        assert loss == g["loss"] and grad.tolist() == g["grad"]


# ---- directly against the compiled reference (where oracle/_ref was built) -------------

def test_oracle_matches_reference_random_nets(oracle, reference):
    rng = np.random.default_rng(3)
    for trial in range(12):
        I = int(rng.integers(1, 8))
        dims = [I, int(rng.integers(1, 9))] + ([int(rng.integers(1, 7))] if trial % 2 else []) + [1]
        n = int(rng.integers(2, 40))
        X = np.zeros((n, 8))
        X[:, :I] = rng.uniform(0, 1, (n, I))
        y = rng.uniform(0, 1, n)
        _, p0 = reference.mlp_init(dims, trial)
        a = oracle.train_full_batch(dims, p0, X, y, 1e-2, 300)
        b = reference.train_full_batch(dims, p0, X, y, 1e-2, 300)
        assert a[0] == b[0] == 0
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


def test_oracle_matches_reference_divergence(oracle, reference):
    """TrainingError(epoch) on a non-finite loss (mlp.cpp:166-169)."""
    dims = [2, 3, 1]
    _, p0 = reference.mlp_init(dims, 1)
    X = np.zeros((4, 8))
    X[:, :2] = 1.0
    y = np.array([0.0, 1.0, np.inf, 0.5])
    a = oracle.train_full_batch(dims, p0, X, y, 1e-2, 10)
    b = reference.train_full_batch(dims, p0, X, y, 1e-2, 10)
    assert a[0] == b[0] == abi.TRAINING_ERROR and a[3] == b[3] == 0


def test_oracle_matches_reference_metrics_random(oracle, reference):
    rng = np.random.default_rng(12345)
    for trial in range(300):
        n = int(rng.integers(2, 60))
        t = np.round(rng.uniform(0.05, 10.0, n), int(rng.integers(0, 3)))
        t[t <= 0] = 0.05
        p = np.round(rng.uniform(0.05, 10.0, n), int(rng.integers(0, 3)))
        assert oracle.mape(t, p) == reference.mape(t, p)
        assert oracle.mape_thresholded(t, p) == reference.mape_thresholded(t, p)
        assert oracle.spearman(t, p) == reference.spearman(t, p)


@pytest.mark.parametrize("combo", [0, 17, 40, 43])
def test_full_length_config2_model_bit_exact(oracle, golden_full, combo):
    """Config-2 models at their FULL length (8000 epochs for prediction nets, 20,000 for the
    blur selection nets): the oracle reproduces the reference's every loss (full-trace sha256),
    weight and metric (tests/golden/make_golden_r02.py)."""
    g = golden_full["config2_full"]
    jd, exp = g["jobs"][combo], g["results"][combo]
    r, params, trace = oracle.run_job(job_from(jd), want_params=True, want_trace=True)
    assert len(trace) == jd["epochs"]
    check_result(r, exp, params, trace)
    assert trace[-3:].tolist() == exp["trace_tail"]


def test_config3_subset_recipe_and_oracle(oracle, golden_full):
    """The stratified config-3 subset is population.config3_jobs(root_seed=1, n_seeds=4) byte
    for byte; two of its fold models (one per hidden-layer shape) reproduce the reference."""
    from paper_2003_07497_b200 import population as P
    g = golden_full["config3_subset"]
    jobs = P.config3_jobs(root_seed=1, n_seeds=g["n_seeds"])
    assert len(jobs) == 48 * 4 * 5 == len(g["results"])
    assert hashlib.sha256(b"".join(bytes(j) for j in jobs)).hexdigest() == g["jobs_sha256"]
    for i in (3, 40 * 20 + 7):  # an MM fold model, a blur fold model
        r, params, _ = oracle.run_job(jobs[i], want_params=True)
        check_result(r, g["results"][i])
        assert sha(np.asarray(params, dtype=np.float64)) == g["results"][i]["params_sha256"]
