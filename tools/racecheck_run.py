import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_2003_07497_b200 import abi, engine as E, population as P
eng = E.Engine(0)
jobs = [j for j in P.config2_jobs(root_seed=1, epochs_scale=0.002)][::6]
print(eng.run_population(jobs, abi.FP32)[0], eng.run_population(jobs, abi.FP64_EXACT)[0])
# round 2: the pipelined FP64 trainer (mbarrier producer/chain) is in the FP64 run above; the
# cross-validation kernels (fold_mean_kernel, cv_stats_kernel) on a tiny k-fold population
cv = P.config3_jobs(root_seed=3, n_seeds=2, combos=E.default_combos()[::24])
for j in cv:
    j.epochs = 10
for prec in (abi.FP32, abi.FP64_EXACT):
    p = E.Population(eng, cv, prec)
    p.run(1)
    print("cv", prec, [g.n_ensembles_ok for g in p.cv()[0]])
    p.close()
# late round 2: unconstrained shapes (chunked FP64 records, generic FP32 kernel), the factor kernel
wide = [abi.make_job(abi.acceptance_world(), P.derive_seed(90, s), count=5000, hidden=h, lr=1e-2, epochs=2,
                     init_seed=s, unconstrained=True) for s, h in ((1, (64,)), (2, (40, 40)))]
print("unconstrained", eng.run_population(wide, abi.FP32)[0], eng.run_population(wide, abi.FP64_EXACT)[0])
big = P.config3_jobs(root_seed=5, n_seeds=8)  # >= 2 models per SM per shape bucket
for j in big:
    j.epochs = 2
print("fp64 sweep (factor kernel)", eng.run_population(big, abi.FP64_EXACT)[0])
