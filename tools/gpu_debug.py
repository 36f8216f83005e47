"""Developer probe: FP64 exact one/two-epoch comparisons against the oracle (prints diffs)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_lib import Oracle  # noqa: E402
from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import engine as E  # noqa: E402

o = Oracle()
eng = E.Engine(0)
rng = np.random.default_rng(5)
for dims, n, ep in [([1, 1, 1], 3, 1), ([2, 3, 1], 20, 1), ([7, 8, 1], 250, 1), ([7, 8, 1], 250, 2), ([6, 5, 5, 1], 250, 1)]:
    I = dims[0]
    X = rng.uniform(0, 1, (n, I))
    y = rng.uniform(0, 1, n)
    p0 = E.init_params(dims, 3)
    m = {"tile": 0, "h1": dims[1], "h2": dims[2] if len(dims) > 3 else 0, "lr": 1e-2, "epochs": ep, "params": p0}
    params, final, bad, traces = eng.train([X], [y], [m], abi.FP64_EXACT, trace=True)
    Xp = np.zeros((n, 8))
    Xp[:, :I] = X
    st, p_exp, t_exp, _ = o.train_full_batch(dims, p0, Xp, y, 1e-2, ep)
    _, l0, g0 = o.mse_gradient(dims, p0, Xp, y)
    dp = params[0] - p_exp
    print(dims, n, ep, "trace eq", np.array_equal(traces[0], t_exp), traces[0][:2], t_exp[:2],
          "param diff idx", np.nonzero(dp)[0][:12], "max", np.abs(dp).max())
