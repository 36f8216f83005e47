"""Profiling driver: one device pass of the config-2 population.
usage: prof_pop.py fp32|fp64 [lanes] [epochs_scale]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import engine as E  # noqa: E402
from paper_2003_07497_b200 import population as P  # noqa: E402

prec = abi.FP32 if sys.argv[1] == "fp32" else abi.FP64_EXACT
if len(sys.argv) > 2:
    os.environ["LANN_FP32_LANES"] = sys.argv[2]
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
eng = E.Engine(0)
jobs = P.config2_jobs(root_seed=1, epochs_scale=scale)
pop = eng.prepare(jobs, prec)
pop.run(1)
cold = eng.last_device_ms
pop.run(1)
print(f"{eng.last_device_ms:.2f} ms (first pass {cold:.2f} ms)")
