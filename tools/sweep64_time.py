"""Developer tool: the full config-3 sweep in the FP64 exact mode, device time of one pass."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import engine as E  # noqa: E402
from paper_2003_07497_b200 import population as P  # noqa: E402

jobs = P.config3_jobs(root_seed=1, n_seeds=int(sys.argv[1]) if len(sys.argv) > 1 else 256)
with E.Engine(0) as eng:
    pop = eng.prepare(jobs, abi.FP64_EXACT)
    pop.run(1)
    st, res, _, _ = pop.fetch()
    print(f"{len(jobs)} models: {eng.last_device_ms:.1f} ms, {P.model_epochs(jobs) / eng.last_device_ms / 1e3:.1f} M model-epochs/s, "
          f"median thr {sorted(r.mape_thr for r in res)[len(res) // 2]!r}")
    pop.close()
