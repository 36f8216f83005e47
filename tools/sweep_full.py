"""Time the whole config-3 sweep (all 61,440 models in one population, buckets concurrent)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import engine as E  # noqa: E402
from paper_2003_07497_b200 import population as P  # noqa: E402

eng = E.Engine(0)
jobs = P.config3_jobs(root_seed=1, n_seeds=int(sys.argv[1]) if len(sys.argv) > 1 else 256)
pop = eng.prepare(jobs, abi.FP32)
pop.run(1)
pop.run(1)
ms = eng.last_device_ms
print(f"{os.environ.get('LANN_FP32_LANES', 'auto')}: {len(jobs)} models {ms:.1f} ms, "
      f"{pop.flop / (eng.last_train_ms / 1e3) / 1e12:.2f} TFLOP/s", flush=True)
