"""GPU: the `perfsage` command-line caller end to end on the engine.

* train (FP64 exact) on the reference-written dataset reproduces the REFERENCE CLI's outputs: the
  model file's norm stats, weights and full loss trace bit for bit, and byte-identical
  train.csv / test.csv (fixtures from tests/golden/make_formats_golden.py).
* eval of that model on test.csv == the reference's evaluate_model_on report.
* compare trains both NN families in one batched call; its nnc row == train + eval.
* select (blur schedules) and select-variants (config 4) produce consistent choices.
* sweep (config 3 / 5 driver) rows == the C oracle's run of the same jobs (FP64 exact).
"""
import csv
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2003_07497_b200 import abi
from paper_2003_07497_b200 import engine as E
from paper_2003_07497_b200.population import derive_seed

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
CLI = os.path.join(ROOT, "paper_2003_07497_b200", "bin", "perfsage")
FMT = json.load(open(os.path.join(GOLD, "formats_r01.json")))
REF_CSV = os.path.join(GOLD, FMT["csv"])


def cli(*args):
    out = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout + out.stderr
    return out.stdout


def model_hex(path):
    m = json.load(open(path))
    n = m["norm_stats"]
    vals = n["f_min"] + n["f_max"] + [n["t_min"], n["t_max"]]
    for layer in m["payload"]["layers"]:
        vals += layer["weights"] + layer["biases"]
    vals += m["metrics"]["loss_trace"]
    return [float(v).hex() for v in vals]


def sha(path):
    import hashlib

    return hashlib.sha256(open(path, "rb").read()).hexdigest()


def read_reports(path):
    with open(path) as f:
        return list(csv.DictReader(f))


@pytest.fixture(scope="module")
def trained(tmp_path_factory):
    out = tmp_path_factory.mktemp("train")
    t = FMT["train"]
    cli("train", "--data", REF_CSV, "--seed", t["seed"], "--epochs", t["epochs"], "--family", t["family"],
        "--precision", "fp64", "--out", out)
    return out


def test_cli_train_reproduces_the_reference_cli(trained):
    assert model_hex(trained / "model_nnc.json") == FMT["model_dump_hex"]
    assert sha(trained / "train.csv") == FMT["train_csv_sha256"]
    assert sha(trained / "test.csv") == FMT["test_csv_sha256"]
    man = json.load(open(trained / "manifest.json"))
    assert man["runs"][-1]["command"] == "train" and man["runs"][-1]["inputs"] == [REF_CSV]


def test_cli_eval_matches_the_reference_report(trained, tmp_path):
    cli("eval", "--model", trained / "model_nnc.json", "--data", trained / "test.csv", "--out", tmp_path,
        "--group-by", "family")
    (row,) = read_reports(tmp_path / "eval.csv")
    ref = FMT["eval_test"]
    assert float(row["mape_full"]) == ref["mape_full"]
    assert float(row["mape_thresholded"]) == ref["mape_thresholded"]
    assert float(row["rho"]) == ref["rho"]
    assert int(row["n_kept"]) == ref["n_kept"] and int(row["n_total"]) == 250
    assert row["kernel"] == "mm" and row["model_family"] == "nnc" and row["variant"] == "dense_threaded@cpu4"


def test_cli_compare_nnc_row_is_train_plus_eval(trained, tmp_path):
    t = FMT["train"]
    out = cli("compare", "--data", REF_CSV, "--seed", t["seed"], "--epochs", t["epochs"], "--precision", "fp64",
              "--out", tmp_path)
    rows = read_reports(tmp_path / "compare.csv")
    assert [r["model_family"] for r in rows][:2] == ["nnc", "nn"]
    assert float(rows[0]["mape_thresholded"]) == FMT["eval_test"]["mape_thresholded"]
    assert "best thresholded MAPE" in out


def test_cli_select_blur_schedule(tmp_path):
    out = cli("select", "--world", 40, "--n", 1024, "--candidates", 120, "--seed", 2, "--epochs", 400,
              "--out", tmp_path)
    rep = json.load(open(tmp_path / "selection.json"))
    assert rep["regret"] >= 1.0 and rep["measured_s"] > 0 and rep["speedup_vs_default"] > 0
    with open(tmp_path / "schedules.csv") as f:
        rows = list(csv.DictReader(f))
    sched = {(int(r["s1"]), int(r["s2"]), int(r["s3"]), int(r["s4"])): float(r["runtime_s"]) for r in rows}
    ch = rep["chosen"]
    key = (ch["s1"], ch["s2"], ch["s3"], ch["s4"])
    assert sched[key] == rep["measured_s"]
    assert min(sched.values()) == rep["true_best_s"]
    assert "chosen schedule" in out
    # the measured table fed back through --data reproduces the same model and choice
    again = tmp_path / "again"
    cli("select", "--data", tmp_path / "schedules.csv", "--n", 1024, "--seed", 2, "--epochs", 400, "--out", again)
    assert json.load(open(again / "selection.json")) == rep


def test_cli_sweep_matches_the_oracle(tmp_path, oracle):
    """Two combinations x 2 seeds x 5 folds, FP64 exact, 2% of the default epochs: every sweep.csv
    row equals the C oracle's run of the identical job (training bit-exact; blur metrics to 1e-12)."""
    cli("sweep", "--combos", "0,40", "--seeds", 2, "--folds", 5, "--epochs-scale", 0.02, "--precision", "fp64",
        "--root-seed", 1, "--out", tmp_path)
    with open(tmp_path / "sweep.csv") as f:
        rows = list(csv.DictReader(f))
    assert len(rows) == 2 * 2 * 5
    worlds = E.default_combos()
    for r in rows:
        combo, s, fold = int(r["combo"]), int(r["seed_index"]), int(r["fold"])
        w = worlds[combo]
        ds = derive_seed(1, combo)
        blur = w.kind == abi.BLUR
        job = abi.make_job(w, ds, n_folds=5, fold=fold, hidden=(5, 5) if blur else (8,), lr=1e-2,
                           epochs=int((20000 if blur else 8000) * 0.02), log_target=blur,
                           init_seed=derive_seed(ds, 1 + s))
        ref, _, _ = oracle.run_job(job)
        assert int(r["status"]) == ref.status == 0
        assert float(r["final_loss"]) == ref.final_loss
        if blur:  # log-target predictions go through CUDA exp (<= 1 ulp from glibc): DESIGN.md 4
            assert float(r["mape_thresholded"]) == pytest.approx(ref.mape_thr, rel=1e-12)
            assert float(r["rho"]) == pytest.approx(ref.rho, rel=1e-12)
        else:
            assert float(r["mape_thresholded"]) == ref.mape_thr
            assert float(r["rho"]) == ref.rho
    # cv.csv: the per-combination cross-validation summary == the oracle's restatement
    jobs = []
    for combo in (0, 40):
        w = worlds[combo]
        ds = derive_seed(1, combo)
        blur = w.kind == abi.BLUR
        for s in range(2):
            for fold in range(5):
                jobs.append(abi.make_job(w, ds, n_folds=5, fold=fold, hidden=(5, 5) if blur else (8,), lr=1e-2,
                                         epochs=int((20000 if blur else 8000) * 0.02), log_target=blur,
                                         init_seed=derive_seed(ds, 1 + s)))
    runs = [oracle.run_job(j, want_params=True) for j in jobs]
    og, _ = oracle.cv_summary(jobs, [o for o, _, _ in runs], [p for _, p, _ in runs])
    with open(tmp_path / "cv.csv") as f:
        cv_rows = list(csv.DictReader(f))
    assert [int(r["combo"]) for r in cv_rows] == [0, 40]
    for r, o in zip(cv_rows, og):
        blur = int(r["combo"]) == 40
        assert int(r["n_ensembles_ok"]) == o["n_ensembles_ok"] == 2 and int(r["n_models_ok"]) == 10
        for k in ("fold_mape", "fold_mape_thr", "fold_rho", "test_mape", "test_mape_thr", "test_rho"):
            for a, b in ((float(r[k + "_mean"]), o[k][0]), (float(r[k + "_median"]), o[k][1])):
                assert (a == pytest.approx(b, rel=1e-12)) if blur else a == b, (k, a, b)


def test_cli_select_variants(tmp_path):
    """Config 4 through the CLI: two MM variant models (worlds 0 and 5: dense / sparse on the
    same host) score 200k counter-generated shapes; every candidate gets exactly one winner."""
    for w in (0, 5):
        d = tmp_path / f"w{w}"
        cli("gen", "--world", w, "--count", 500, "--seed", 1, "--out", d)
        (data,) = [p for p in d.iterdir() if p.suffix == ".csv"]
        cli("train", "--data", data, "--seed", 1, "--epochs", 500, "--precision", "fp32", "--out", d)
    out = cli("select-variants", "--model", tmp_path / "w0" / "model_nnc.json", "--model",
              tmp_path / "w5" / "model_nnc.json", "--candidates", 200000, "--max-threads", 4,
              "--precision", "fp32", "--out", tmp_path)
    with open(tmp_path / "variants.csv") as f:
        rows = list(csv.DictReader(f))
    assert sum(int(r["chosen"]) for r in rows) == 200000
    assert "predictions/s" in out


def _linear(path):
    p = json.load(open(path))["payload"]["linear"]
    return [float(w).hex() for w in p["weights"]] + [float(p["intercept"]).hex()]


@pytest.mark.parametrize("fam", ["const", "lrc"])
def test_cli_least_squares_baselines_are_the_reference(tmp_path, fam):
    """const / lrc (models.cpp:305-320) fitted on the GPU: weights and intercept bit-identical to
    the reference's model file, and its test-set report identical."""
    cli("train", "--data", REF_CSV, "--seed", 3, "--family", fam, "--out", tmp_path)
    assert _linear(tmp_path / f"model_{fam}.json") == _linear(os.path.join(GOLD, FMT["baselines"][fam]["model"]))
    cli("eval", "--model", tmp_path / f"model_{fam}.json", "--data", tmp_path / "test.csv", "--out", tmp_path / "e")
    (row,) = read_reports(tmp_path / "e" / "eval.csv")
    ref = FMT["baselines"][fam]["eval_test"]
    assert (float(row["mape_full"]), float(row["mape_thresholded"]), float(row["rho"]), int(row["n_kept"])) == (
        ref["mape_full"], ref["mape_thresholded"], ref["rho"], ref["n_kept"])


def test_cli_forest_baseline_tracks_the_reference(tmp_path):
    """nlrc (forest.cpp) on the GPU: the same bootstraps and split rule as the reference; trees
    agree node for node except where equal feature values are summed in a different order (a
    last-bit SSE difference can flip a tied split), so the report matches to tolerance."""
    cli("train", "--data", REF_CSV, "--seed", 3, "--family", "nlrc", "--out", tmp_path)
    forest = json.load(open(tmp_path / "model_nlrc.json"))["payload"]["forest"]
    counts = [len(t) for t in forest]
    ref_counts = FMT["baselines"]["nlrc"]["tree_node_counts"]
    assert len(counts) == len(ref_counts) == 100
    same = sum(a == b for a, b in zip(counts, ref_counts))
    assert same >= 90, (same, counts[:10], ref_counts[:10])
    cli("eval", "--model", tmp_path / "model_nlrc.json", "--data", tmp_path / "test.csv", "--out", tmp_path / "e")
    (row,) = read_reports(tmp_path / "e" / "eval.csv")
    ref = FMT["baselines"]["nlrc"]["eval_test"]
    assert abs(float(row["mape_thresholded"]) - ref["mape_thresholded"]) <= 0.1
    assert abs(float(row["rho"]) - ref["rho"]) <= 1e-3


def test_cli_compare_runs_all_five_families(tmp_path):
    out = cli("compare", "--data", REF_CSV, "--seed", 3, "--epochs", 300, "--precision", "fp32", "--out", tmp_path)
    rows = read_reports(tmp_path / "compare.csv")
    assert [r["model_family"] for r in rows] == ["nnc", "nn", "const", "lrc", "nlrc"]
    assert float(rows[2]["mape_thresholded"]) == FMT["baselines"]["const"]["eval_test"]["mape_thresholded"]
    assert "best thresholded MAPE" in out


def test_cli_select_mock_timer_is_the_reference_cli(tmp_path, reference):
    """`perfsage select --mock-timer` == the reference CLI's cmd_select with its mock timer
    (perfsage.cpp:307-382): same candidates, measured table, FP64 model, chosen schedule, true
    best, regret and speedups (predicted_s through CUDA exp: 1e-12)."""
    cli("select", "--mock-timer", "--n", 1024, "--candidates", 150, "--seed", 5, "--epochs", 1500, "--max-threads", 4,
        "--precision", "fp64", "--out", tmp_path)
    rep = json.load(open(tmp_path / "selection.json"))
    st, ref = reference.cli_select_mock(1024, 150, 5, 1500, 4)
    assert st == 0, reference.last_error()
    sched = lambda d: [d["s1"], d["s2"], d["s3"], d["s4"]]  # noqa: E731
    assert sched(rep["chosen"]) == list(ref[0:4])
    assert rep["predicted_s"] == pytest.approx(ref[4], rel=1e-12)
    assert rep["measured_s"] == ref[5]
    assert sched(rep["true_best"]) == list(ref[6:10])
    assert (rep["true_best_s"], rep["default_s"], rep["regret"], rep["speedup_vs_default"],
            rep["speedup_vs_random_mean"]) == tuple(ref[10:15])


def test_cli_forest_and_eval_on_large_sets(tmp_path, reference):
    """nlrc on 5000 training rows (its working set no longer fits shared memory: the forest
    kernel runs from HBM scratch) and eval on 5000 held-out rows; the report of the trained
    model equals the reference library's evaluate_model_on of the same model file."""
    cli("gen", "--world", 0, "--count", 10000, "--seed", 4, "--out", tmp_path)
    (data,) = [p for p in tmp_path.iterdir() if p.suffix == ".csv"]
    cli("train", "--data", data, "--seed", 4, "--family", "nlrc", "--out", tmp_path)
    cli("eval", "--model", tmp_path / "model_nlrc.json", "--data", tmp_path / "test.csv", "--out", tmp_path / "e")
    (row,) = read_reports(tmp_path / "e" / "eval.csv")
    st, ref = reference.eval_model(tmp_path / "model_nlrc.json", tmp_path / "test.csv")
    assert st == 0, reference.last_error()
    assert int(row["n_total"]) == 5000
    got = [float(row["mape_full"]), float(row["mape_thresholded"]), float(row["rho"])]
    np.testing.assert_allclose(got, ref[:3], rtol=1e-12)
