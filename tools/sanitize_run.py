"""Small end-to-end exercise of every kernel family, for compute-sanitizer (developer tool):
  compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import engine as E  # noqa: E402
from paper_2003_07497_b200 import population as P  # noqa: E402

eng = E.Engine(0)
small = P.config2_jobs(root_seed=1, epochs_scale=0.005)
for prec in (abi.FP32, abi.FP64_EXACT):
    st, res, params, _ = eng.run_population(small, prec, want_params=True, want_trace=True)
    print("config2 tiny", prec, st)
sweep = P.config3_jobs(root_seed=1, n_seeds=2, combos=E.default_combos()[::6])
for lanes in ("1", "2", "8", "32"):
    os.environ["LANN_FP32_LANES"] = lanes
    st, res, _, _ = eng.run_population([j for j in sweep], abi.FP32)
    print("sweep lanes", lanes, st)
os.environ.pop("LANN_FP32_LANES")
pop = eng.prepare(P.config2_jobs(root_seed=1, epochs_scale=0.005), abi.FP32)
pop.run(1)
st, res, params, _ = pop.fetch(want_params=True)
norms = pop.norms()
jobs = P.config2_jobs(root_seed=1)
idx = [i for i, j in enumerate(jobs) if j.world.kind == abi.MM]
models = [{"inputs": res[i].n_inputs, "h1": 8, "h2": 0, "log_target": 0, "params": params[i], "norm": norms[i]}
          for i in idx]
thd = [1 if jobs[i].world.hw_class == abi.HW_CPU else 0 for i in idx]
for prec in (abi.FP32, abi.FP64_EXACT):
    gi, gs = eng.select_variants(models, thd, abi.MM, 12, 7, 0, 5000, precision=prec)
    print("select", prec, int(gi.max()))
# round 2: k-fold populations with the cross-validation summary (fold_mean_kernel, cv_stats_kernel),
# the compact config-4 scorer, the batched predictor's 4-row path, the mlp.hpp batch operations
cv_jobs = P.config3_jobs(root_seed=3, n_seeds=2, combos=E.default_combos()[::12])
for j in cv_jobs:
    j.epochs = 20
for prec in (abi.FP32, abi.FP64_EXACT):
    p = E.Population(eng, cv_jobs, prec)
    p.run(1)
    groups, ens = p.cv()
    print("cv", prec, len(groups), sum(g.n_ensembles_ok for g in groups))
    p.close()
print("cv summarize", len(eng.cv_summarize(cv_jobs, eng.run_population(cv_jobs, abi.FP64_EXACT)[1],
                                           [E.abi.CvEnsemble() for _ in range(E.cv_layout(cv_jobs)[1])])))
ci, cs = np.zeros(5000, dtype=np.uint8), np.zeros(5000, dtype=np.float32)
eng.select_variants_compact(models, thd, abi.MM, 12, 7, 0, 5000, idx=ci, score=cs)
print("select compact", int(ci.max()))
rows = np.random.default_rng(0).random((4096, abi.ROW))
row_model = np.repeat(np.arange(len(models), dtype=np.int32), 4096 // len(models) + 1)[:4096]
for prec in (abi.FP32, abi.FP64_EXACT):
    out = eng.predict(models, rows, row_model, precision=prec)
    print("predict", prec, float(out[0]))
dims, w = [7, 8, 1], np.linspace(-0.5, 0.5, 73)
Xs, ys = rows[:100, :7].copy(), rows[:100, 7].copy()
fwd, loss, grad = eng.mlp_forward([(dims, w, Xs)]), eng.mse_loss([(dims, w, Xs, ys)]), eng.mse_gradient([(dims, w, Xs, ys)])
print("mlp ops", np.ravel(fwd)[:1], np.ravel(loss)[:1], len(grad))
print("done")
# late round 2: unconstrained shapes (FP64 exact with chunked shared-memory records, the generic
# FP32 kernel) and the throughput-regime FP64 factor kernel (>= 2 models per SM)
wide = [abi.make_job(abi.acceptance_world(), P.derive_seed(90, s), count=5000, hidden=h, lr=1e-2, epochs=3,
                     init_seed=s, unconstrained=True) for s, h in ((1, (64,)), (2, (40, 40)))]
for prec in (abi.FP32, abi.FP64_EXACT):
    st, res, _, _ = eng.run_population(wide, prec)
    print("unconstrained", prec, st, [r.precision_run for r in res])
big = P.config3_jobs(root_seed=5, n_seeds=8)  # >= 2 models per SM per shape bucket
for j in big:
    j.epochs = 3
print("fp64 sweep (factor kernel)", eng.run_population(big, abi.FP64_EXACT)[0])
print("done (late round 2)")
