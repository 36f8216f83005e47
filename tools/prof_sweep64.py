"""Profiling driver: a config-3-shaped FP64 exact population (every combination x n_seeds x 5 folds,
epochs scaled) so the pipelined trainer runs in the throughput regime (more models than SMs).
usage: prof_sweep64.py [n_seeds] [epochs_scale]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import engine as E  # noqa: E402
from paper_2003_07497_b200 import population as P  # noqa: E402

n_seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 16
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.05
jobs = P.config3_jobs(root_seed=1, n_seeds=n_seeds)
for j in jobs:
    j.epochs = max(1, int(j.epochs * scale))
with E.Engine(0) as eng:
    pop = eng.prepare(jobs, abi.FP64_EXACT)
    pop.run(1)
    print(f"{len(jobs)} models: {eng.last_device_ms:.2f} ms, {pop.flop / (eng.last_train_ms / 1e3) / 1e12:.2f} TFLOP/s")
    pop.close()
