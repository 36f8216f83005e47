"""Split the e2e (lann_run_population) time of the config-2 population into host preparation +
upload, device pass, fetch and teardown (developer tool)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import engine as E  # noqa: E402
from paper_2003_07497_b200 import population as P  # noqa: E402

eng = E.Engine(0)
jobs = P.config2_jobs(root_seed=1)
for it in range(6):
    t0 = time.perf_counter()
    pop = eng.prepare(jobs, abi.FP32)
    t1 = time.perf_counter()
    pop.run(1)
    t2 = time.perf_counter()
    pop.fetch()
    t3 = time.perf_counter()
    pop.close()
    t4 = time.perf_counter()
    t5 = time.perf_counter()
    eng.run_population(jobs, abi.FP32)
    t6 = time.perf_counter()
    print(f"prepare {1e3*(t1-t0):.2f} ms  run {1e3*(t2-t1):.2f} (device {eng.last_device_ms:.2f})  fetch {1e3*(t3-t2):.2f}"
          f"  close {1e3*(t4-t3):.2f}  | run_population {1e3*(t6-t5):.2f} ms")
