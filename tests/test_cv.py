"""Cross-validation summary of a k-fold sweep (BASELINE config 3: held-out fold
metrics per combination plus the test-set MAPE of the fold-mean model), computed on the device
in the population pass (lann_population_cv, include/lann_engine.h) and checked against the oracle's
restatement (oracle/lann_oracle.c or_fold_mean + tests/oracle_lib.py Oracle.cv_summary) built on
the reference's primitives: split (datagen.cpp:225-248), predict (models.cpp:346-363),
make_report (eval.cpp:98-108) and aggregate's per-group means (eval.cpp:110-146)."""
import numpy as np
import pytest

from paper_2003_07497_b200 import abi
from paper_2003_07497_b200 import engine as E
from paper_2003_07497_b200 import population as P

LOG_TOL = 1e-12  # log-target predictions de-normalise through CUDA's exp (<= 1 ulp from glibc's)


def small_sweep(n_seeds=3, epochs=150, combos=(0, 17, 33, 41)):
    worlds = P.combo_worlds()
    jobs = P.config3_jobs(root_seed=7, n_seeds=n_seeds, combos=[worlds[i] for i in combos])
    for j in jobs:
        j.epochs = epochs if not j.log_target else 2 * epochs
    return jobs


# ---- host only -----------------------------------------------------------------------------

def test_cv_layout_counts():
    """Config 3 forms 48 groups (one per combination) and 48 x 256 ensembles; config 2 none."""
    assert E.cv_layout(P.config3_jobs(root_seed=1, n_seeds=256)) == (48, 48 * 256)
    assert E.cv_layout(P.config2_jobs(root_seed=1)) == (0, 0)
    jobs = small_sweep()
    # fold and init seed are not part of the group key; every other field is
    jobs[0].learning_rate = 1e-3
    assert E.cv_layout(jobs) == (5, 12 + 1)


def test_oracle_fold_mean_is_the_mean_of_fold_predictions(oracle):
    """or_fold_mean == (p_0 + ... + p_{k-1}) / k of the per-fold models::predict on the split's
    test part, each fold model with the NormStats of its own training blocks."""
    jobs = small_sweep(n_seeds=1, epochs=20, combos=(0,))
    runs = [oracle.run_job(j, want_params=True) for j in jobs]
    pred, truth = oracle.fold_mean(jobs, [p for _, p, _ in runs])
    j0 = jobs[0]
    _, feats, c, rt, nf = oracle.build_dataset(j0.world, j0.data_seed, j0.count)
    _, order, n_train = oracle.split_order(j0.count, j0.train_fraction, j0.data_seed)
    assert len(pred) == j0.count - n_train
    acc = np.zeros(len(pred))
    I = nf + 1
    for f, (j, (r, params, _)) in enumerate(zip(jobs, runs)):
        b0, b1 = n_train * f // 5, n_train * (f + 1) // 5
        tr = [order[i] for i in range(n_train) if not b0 <= i < b1]
        X = np.zeros((len(tr), abi.ROW))
        X[:, :nf] = feats[tr, :nf]
        X[:, nf] = c[tr].astype(np.float64)
        norm = oracle.norm_fit(X, rt[tr], I)
        for s, idx in enumerate(order[n_train:]):
            x = list(feats[idx, :nf]) + [float(c[idx])]
            p = oracle.predict_row(I, [8], params, norm, False, x)
            acc[s] = p if f == 0 else acc[s] + p
    assert np.array_equal(pred, acc / 5)
    assert np.array_equal(truth, rt[order[n_train:]])


# ---- GPU ---------------------------------------------------------------------------------------

def check_against_oracle(groups, ens, og, oe, jobs):
    assert len(groups) == len(og) and len(ens) == len(oe)
    for e, o in zip(ens, oe):
        assert e.group == o["group"] and e.init_seed == o["seed"]
        assert e.status == o["status"], (e.status, o)
        if e.status:
            continue
        logt = jobs[groups[e.group].first_job].log_target
        for k in ("mape", "mape_thr", "rho"):
            a, b = getattr(e, k), o[k]
            assert (abs(a - b) <= LOG_TOL * max(1.0, abs(b))) if logt else a == b, (k, a, b)
        assert e.n_kept == o["n_kept"] and e.n_test == o["n_test"]
    for g, o in zip(groups, og):
        for k in ("first_job", "n_folds", "n_models", "n_models_ok", "n_ensembles", "n_ensembles_ok"):
            assert getattr(g, k) == o[k], (k, getattr(g, k), o[k])
        logt = jobs[g.first_job].log_target
        for k in ("fold_mape", "fold_mape_thr", "fold_rho", "test_mape", "test_mape_thr", "test_rho"):
            st = getattr(g, k)
            for a, b in ((st.mean, o[k][0]), (st.median, o[k][1])):
                assert (abs(a - b) <= LOG_TOL * max(1.0, abs(b))) if logt else a == b, (k, a, b)


@pytest.mark.gpu
def test_cv_summary_fp64_equals_oracle(engine, oracle):
    """FP64 exact: every fold-mean test metric and every group statistic equals the oracle's
    (bit for bit; 1e-12 relative on the log-target blur group)."""
    jobs = small_sweep()
    pop = E.Population(engine, jobs, abi.FP64_EXACT)
    pop.run(1)
    st, res, _, _ = pop.fetch()
    assert st == 0
    groups, ens = pop.cv()
    runs = [oracle.run_job(j, want_params=True) for j in jobs]
    assert [r.status for r in res] == [o.status for o, _, _ in runs]
    og, oe = oracle.cv_summary(jobs, [o for o, _, _ in runs], [p for _, p, _ in runs])
    check_against_oracle(groups, ens, og, oe, jobs)
    assert all(g.n_ensembles_ok == 3 and g.n_models_ok == 15 and g.n_test == 250 for g in groups)
    # a second pass of the resident population reproduces the summary
    pop.run(2)
    g2, e2 = pop.cv()
    assert [bytes(x) for x in g2] == [bytes(x) for x in groups] and [bytes(x) for x in e2] == [bytes(x) for x in ens]
    pop.close()


@pytest.mark.gpu
def test_cv_summary_incomplete_and_failed_ensembles(engine, oracle):
    """A missing fold (PARAM_ERROR) and a member that fails host preparation (its own status)
    leave their ensembles out of the test statistics; the other models still count."""
    jobs = small_sweep(n_seeds=2, epochs=60, combos=(0, 5))
    del jobs[3]                 # combo 0, seed 0: fold 3 missing
    jobs[7].hidden[0] = 0       # combo 0, seed 1, fold 3: hidden width 0 -> ParamError
    pop = E.Population(engine, jobs, abi.FP64_EXACT)
    pop.run(1)
    groups, ens = pop.cv()
    runs = [oracle.run_job(j, want_params=True) for j in jobs]
    og, oe = oracle.cv_summary(jobs, [o for o, _, _ in runs], [p for _, p, _ in runs])
    # the job with hidden 0 forms its own group (hidden is part of the key): groups in order of
    # first appearance are combo 0, the hidden-0 job, combo 5
    assert len(groups) == 3
    assert [e.status for e in ens][:3] == [abi.PARAM_ERROR] * 3
    assert groups[0].n_ensembles_ok == 0 and groups[0].n_models_ok == 8
    assert groups[1].n_models == 1 and groups[1].n_models_ok == 0
    assert groups[2].n_ensembles_ok == 2 and groups[2].n_models_ok == 10
    check_against_oracle(groups, ens, og, oe, jobs)
    pop.close()


@pytest.mark.gpu
def test_cv_summary_fp32_population(engine, oracle):
    """FP32: the same summary from the FP32 trainer and predictor; every ensemble scores, and the
    fold-mean test MAPE per group is close to the FP64-exact one at this short length."""
    jobs = small_sweep(epochs=300)
    p32 = E.Population(engine, jobs, abi.FP32)
    p32.run(1)
    g32, e32 = p32.cv()
    p64 = E.Population(engine, jobs, abi.FP64_EXACT)
    p64.run(1)
    g64, _ = p64.cv()
    assert all(e.status == 0 for e in e32)
    for a, b in zip(g32, g64):
        assert a.n_ensembles_ok == b.n_ensembles_ok == 3
        assert np.isfinite(a.test_mape.mean) and abs(a.test_mape_thr.mean - b.test_mape_thr.mean) < 5.0
    p32.close()
    p64.close()


@pytest.mark.gpu
def test_cv_group_equals_single_engine(engine):
    """lann_group_run_cv over two shards (one B200 listed twice) == the single-engine summary, bit
    for bit in FP64, also for a job list whose ensembles are interleaved (sorted by fold: the group
    places each ensemble's jobs together before cutting); lann_cv_summarize over the single
    engine's host results reproduces its on-device group statistics."""
    base = small_sweep(n_seeds=3, epochs=80)
    for jobs in (base, sorted(base, key=lambda j: j.fold)):
        pop = E.Population(engine, jobs, abi.FP64_EXACT)
        pop.run(1)
        st, res, _, _ = pop.fetch()
        groups, ens = pop.cv()
        assert st == 0
        again = engine.cv_summarize(jobs, res, ens)
        assert [bytes(x) for x in again] == [bytes(x) for x in groups]
        for n_dev in (2, 4):  # identical outputs for any device count
            with E.Group([0] * n_dev) as g:
                b = g.shard_bounds(jobs)
                assert 0 < b[1] < len(jobs)
                gst, gres, ggroups, gens = g.run_cv(jobs)
            assert gst == 0, g.last_error
            assert [bytes(x) for x in gres] == [bytes(x) for x in res]
            assert [bytes(x) for x in gens] == [bytes(x) for x in ens]
            assert [bytes(x) for x in ggroups] == [bytes(x) for x in groups]
        pop.close()


@pytest.mark.gpu
def test_cv_summary_other_fold_counts_and_shapes(engine, oracle):
    """Fold counts 2, 3 and 10 side by side in one population (different groups), ragged test
    parts (count 301: 150 test rows) and an unconstrained 7-64-1 net (the generic predictor path of
    fold_mean_kernel and the phased FP64 trainer): FP64 summary == the oracle's."""
    w = P.combo_worlds()[0]
    jobs = []
    for k, count in ((2, 301), (3, 120), (10, 400)):
        ds = P.derive_seed(11, k)
        for s in range(2):
            for f in range(k):
                jobs.append(abi.make_job(w, ds, count=count, n_folds=k, fold=f, hidden=(8,), lr=1e-2, epochs=40,
                                         init_seed=P.derive_seed(ds, 1 + s)))
    ds = P.derive_seed(11, 99)
    for f in range(3):
        jobs.append(abi.make_job(w, ds, count=200, n_folds=3, fold=f, hidden=(64,), lr=1e-3, epochs=15,
                                 init_seed=5, unconstrained=True))
    pop = E.Population(engine, jobs, abi.FP64_EXACT)
    pop.run(1)
    st, res, _, _ = pop.fetch()
    assert st == 0, engine.last_error
    groups, ens = pop.cv()
    runs = [oracle.run_job(j, want_params=True) for j in jobs]
    og, oe = oracle.cv_summary(jobs, [o for o, _, _ in runs], [p for _, p, _ in runs])
    assert [g.n_folds for g in groups] == [2, 3, 10, 3]
    assert [g.n_test for g in groups] == [150, 60, 200, 100]
    check_against_oracle(groups, ens, og, oe, jobs)


@pytest.mark.gpu
def test_cv_summary_large_group_and_bad_folds(engine, oracle):
    """A group of 2,100 fold models (more than one CTA's register-held compaction: the sequential
    gather path of cv_stats_kernel) == the oracle; a job whose fold index is out of range
    (ParamError) forms an ensemble with no valid member, through the single engine and the group."""
    w = P.combo_worlds()[3]
    ds = P.derive_seed(5, 3)
    jobs = [abi.make_job(w, ds, n_folds=5, fold=f, hidden=(8,), lr=1e-2, epochs=3, init_seed=P.derive_seed(ds, 1 + s))
            for s in range(420) for f in range(5)]
    pop = E.Population(engine, jobs, abi.FP64_EXACT)
    pop.run(1)
    st, res, _, _ = pop.fetch()
    groups, ens = pop.cv()
    pop.close()
    assert st == 0 and len(groups) == 1 and groups[0].n_models_ok == 2100 and groups[0].n_ensembles_ok == 420
    runs = [oracle.run_job(j, want_params=True) for j in jobs]
    og, oe = oracle.cv_summary(jobs, [o for o, _, _ in runs], [p for _, p, _ in runs])
    check_against_oracle(groups, ens, og, oe, jobs)
    bad = jobs[:10] + [abi.make_job(w, ds, n_folds=5, fold=7, hidden=(8,), lr=1e-2, epochs=3, init_seed=99)]
    p2 = E.Population(engine, bad, abi.FP64_EXACT)
    p2.run(1)
    g1, e1 = p2.cv()
    p2.close()
    assert [e.status for e in e1] == [abi.OK, abi.OK, abi.PARAM_ERROR]
    with E.Group([0, 0]) as g:
        gst, gres, g2, e2 = g.run_cv(bad)
    assert gres[-1].status == abi.PARAM_ERROR
    assert [e.status for e in e2] == [abi.OK, abi.OK, abi.PARAM_ERROR]
    assert [bytes(x) for x in g2] == [bytes(x) for x in g1]
