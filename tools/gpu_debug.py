"""Developer probe: run individual engine entry points (for compute-sanitizer)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import engine as E  # noqa: E402
from paper_2003_07497_b200 import population as P  # noqa: E402

which = sys.argv[1:] or ["onestep", "random64", "select"]
eng = E.Engine(0)
rng = np.random.default_rng(5)
if "onestep" in which:
    X = rng.uniform(0, 1, (250, 7))
    y = rng.uniform(0, 1, 250)
    p0 = E.init_params([7, 8, 1], 11)
    out = eng.train([X], [y], [{"tile": 0, "h1": 8, "lr": 1e-2, "epochs": 2, "params": p0}], abi.FP32, trace=True)
    print("onestep ok", out[3][0])
if "random64" in which:
    X = rng.uniform(0, 1, (50, 3))
    y = rng.uniform(0, 1, 50)
    p0 = E.init_params([3, 4, 2, 1], 1)
    out = eng.train([X], [y], [{"tile": 0, "h1": 4, "h2": 2, "lr": 1e-3, "epochs": 5, "params": p0}],
                    abi.FP64_EXACT, trace=True)
    print("random64 ok", out[3][0])
if "select" in which:
    jobs = P.config2_jobs(root_seed=1, epochs_scale=0.002)
    pop = eng.prepare(jobs, abi.FP32)
    pop.run(1)
    st, res, params, _ = pop.fetch(want_params=True)
    norms = pop.norms()
    idx = [i for i, j in enumerate(jobs) if j.world.kind == abi.MM]
    models = [{"inputs": res[i].n_inputs, "h1": 8, "h2": 0, "log_target": 0, "params": params[i], "norm": norms[i]}
              for i in idx]
    thd = [1 if jobs[i].world.hw_class == abi.HW_CPU else 0 for i in idx]
    gi, gs = eng.select_variants(models, thd, abi.MM, 16, 7, 0, 1000, precision=abi.FP32)
    print("select ok", gi[:10], gs[:3])
