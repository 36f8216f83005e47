"""Developer tool: time the config-3 sweep split into its prediction-net part (40 combos,
7/6/...-8-1) and its blur part (8 combos, 6-5-5-1), to see which kernel bounds the sweep."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import engine as E  # noqa: E402
from paper_2003_07497_b200 import population as P  # noqa: E402

eng = E.Engine(0)
combos = E.default_combos()
seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 256
for name, sub in (("pred", combos[:40]), ("blur", combos[40:])):
    jobs = P.config3_jobs(root_seed=1, n_seeds=seeds, combos=sub)
    pop = eng.prepare(jobs, abi.FP32)
    pop.run(1)
    ms, tms = eng.last_device_ms, eng.last_train_ms
    print(f"{name}: {len(jobs)} models {ms:.1f} ms, {P.model_epochs(jobs) / ms * 1e3:.3e} model-epochs/s, "
          f"{pop.flop / tms * 1e3 / 1e12:.2f} TFLOP/s ({100 * pop.flop / tms * 1e3 / 1e12 / 74.12:.1f}% of FP32 peak)",
          flush=True)
    pop.close()
