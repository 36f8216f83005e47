"""Developer tool: time the config-2 population (device-only passes) under each FP32 mapping
and in FP64 exact mode; optional config-3 sweep mappings."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import engine as E  # noqa: E402
from paper_2003_07497_b200 import population as P  # noqa: E402

eng = E.Engine(0)
jobs = P.config2_jobs(root_seed=1)
me = P.model_epochs(jobs)
for lanes in sys.argv[1].split(",") if len(sys.argv) > 1 else ["32", "64", "128", "256"]:
    os.environ["LANN_FP32_LANES"] = lanes
    pop = eng.prepare(jobs, abi.FP32)
    pop.run(1)
    pop.run(2)
    ms = eng.last_device_ms / 2
    st, res, _, _ = pop.fetch()
    import numpy as np
    print(f"fp32 lanes={lanes}: {ms:.2f} ms/step, {me / ms * 1e3:.3e} model-epochs/s, "
          f"median thr {np.median([r.mape_thr for r in res]):.3f}", flush=True)
    pop.close()
os.environ.pop("LANN_FP32_LANES", None)
pop = eng.prepare(jobs, abi.FP64_EXACT)
pop.run(1)
pop.run(1)
ms = eng.last_device_ms
print(f"fp64 exact: {ms:.2f} ms/step, {me / ms * 1e3:.3e} model-epochs/s", flush=True)
pop.close()
if len(sys.argv) > 2:
    sweep = P.config3_jobs(root_seed=1, n_seeds=int(sys.argv[2]))
    me3 = P.model_epochs(sweep)
    for lanes in ["1", "2", "4"]:
        os.environ["LANN_FP32_LANES"] = lanes
        pop = eng.prepare(sweep, abi.FP32)
        pop.run(1)
        ms, tms = eng.last_device_ms, eng.last_train_ms
        print(f"sweep lanes={lanes}: {len(sweep)} models {ms:.1f} ms, {me3 / ms * 1e3:.3e} model-epochs/s, "
              f"{pop.flop / tms * 1e3 / 1e12:.2f} TFLOP/s", flush=True)
        pop.close()
