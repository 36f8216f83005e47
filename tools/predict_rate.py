"""Developer tool: batched predictor kernel rate (48 config-2-shaped models x rows, FP32/FP64)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import engine as E  # noqa: E402
from paper_2003_07497_b200 import population as P  # noqa: E402

rows_per_model = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
eng = E.Engine(0)
jobs = P.config2_jobs(root_seed=1, epochs_scale=0.01)
st, res, params, _ = eng.run_population(jobs, abi.FP32, want_params=True)
pop = eng.prepare(jobs, abi.FP32)
norms = pop.norms()
pop.close()
models = [{"inputs": r.n_inputs, "h1": j.hidden[0], "h2": j.hidden[1] if j.n_hidden > 1 else 0,
           "log_target": j.log_target, "params": p, "norm": n} for j, r, p, n in zip(jobs, res, params, norms)]
base = []
for j in jobs:
    f, c, _, nf = E.build_dataset(j.world, j.data_seed, 500)
    if j.family == abi.NNC:
        f[:, nf] = c.astype(np.float64)
    base.append(f)
rows = np.concatenate([np.resize(b, (rows_per_model, abi.ROW)) for b in base])
rm = np.repeat(np.arange(len(jobs), dtype=np.int32), rows_per_model)
n = len(rm)
for prec, name in ((abi.FP32, "fp32"), (abi.FP64_EXACT, "fp64")):
    ks = []
    for _ in range(4):
        eng.predict(models, rows, rm, precision=prec)
        ks.append(eng.last_train_ms)
    k = float(np.median(ks[1:]))
    print(f"{name}: {k:.3f} ms  {n / k / 1e6:.2f} G pred/s  {76 * n / k / 1e6:.0f} GB/s")
