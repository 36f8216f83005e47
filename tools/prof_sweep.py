"""Profiling driver: one pass of a config-3 sweep slice (48 combos x S seeds x 5 folds) in FP32,
for `ncu -k regex:train_fp32_kernel` (the many-models warp kernel)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import engine as E  # noqa: E402
from paper_2003_07497_b200 import population as P  # noqa: E402

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 32
eng = E.Engine(0)
jobs = P.config3_jobs(root_seed=1, n_seeds=seeds)
pop = eng.prepare(jobs, abi.FP32)
pop.run(1)
print(f"{len(jobs)} models, {eng.last_device_ms:.1f} ms, train {eng.last_train_ms:.1f} ms, "
      f"{pop.flop / (eng.last_train_ms / 1e3) / 1e12:.2f} TFLOP/s")
