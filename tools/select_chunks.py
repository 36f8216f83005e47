"""Developer tool: config-4 scorer kernel / end-to-end time by chunk count and outputs."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import engine as E  # noqa: E402

rng = np.random.default_rng(1)
models = []
for v in range(10):
    I = 7 if v % 2 == 0 else 6
    nrm = np.zeros(18)
    nrm[8:16] = 1e3
    nrm[16], nrm[17] = -12.0, -2.0
    models.append({"inputs": I, "h1": 8, "h2": 0, "log_target": 1, "params": rng.uniform(-1, 1, (I + 1) * 8 + 9),
                   "norm": nrm})
thd = [1 if v % 2 == 0 else 0 for v in range(10)]
n = 10_000_000
eng = E.Engine(0)
pi, ps = E.Pinned(n, np.uint8), E.Pinned(n, np.float32)
for chunks in ("1", "2", "4", "8"):
    os.environ["LANN_SELECT_CHUNKS"] = chunks
    for hist in (False, True):
        ks, ws = [], []
        for _ in range(5):
            t0 = time.perf_counter()
            eng.select_variants_compact(models, thd, abi.MM, 16, 7, 0, n, idx=pi.array, score=ps.array, want_hist=hist)
            ws.append((time.perf_counter() - t0) * 1e3)
            ks.append(eng.last_train_ms)
        print(f"chunks {chunks} hist {hist}: kernel {np.median(ks):.3f} ms  e2e {np.median(ws):.3f} ms")
ks = []
for _ in range(5):
    eng.select_variants(models, thd, abi.MM, 16, 7, 0, n)
    ks.append(eng.last_train_ms)
print(f"full-width call: kernel {np.median(ks):.3f} ms")
