"""Quick GPU sanity/parity probe (developer tool): config-1 job and the 48-combo
population through the engine in both precisions, against the oracle."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_lib import Oracle  # noqa: E402
from paper_2003_07497_b200 import engine as E  # noqa: E402
from paper_2003_07497_b200.abi import *  # noqa: E402,F401,F403
from paper_2003_07497_b200 import population as pop  # noqa: E402

o = Oracle()
eng = E.Engine(0)
j = make_job(acceptance_world(), 1)
t0 = time.time()
st, res, params, traces = eng.run_population([j], FP64_EXACT, want_params=True, want_trace=True)
print("fp64 job", st, time.time() - t0, eng.last_device_ms, res[0].final_loss, res[0].mape_thr, res[0].rho)
ro, po, to = o.run_job(j, True, True)
print("oracle   ", ro.final_loss, ro.mape_thr, ro.rho)
print("trace bit-exact:", np.array_equal(traces[0], to), "params bit-exact:", np.array_equal(params[0], po),
      "mape:", res[0].mape == ro.mape, res[0].mape_thr == ro.mape_thr, res[0].rho == ro.rho)
if not np.array_equal(traces[0], to):
    d = np.nonzero(traces[0] != to)[0]
    print("first diff epoch", d[0], traces[0][d[0]], to[d[0]])
st, res32, _, tr32 = eng.run_population([j], FP32, want_trace=True)
print("fp32 job", st, eng.last_device_ms, res32[0].final_loss, res32[0].mape_thr, "trace[0:3]", tr32[0][:3], to[:3])

jobs = pop.config2_jobs(root_seed=1)
for prec in (FP64_EXACT, FP32):
    st, rr, _, _ = eng.run_population(jobs, prec)
    ms = eng.last_device_ms
    st, rr, _, _ = eng.run_population(jobs, prec)
    ms = eng.last_device_ms
    me = sum(x.epochs for x in jobs)
    print("config2 prec", prec, "status", st, "ms", ms, "model-epochs/s %.3e" % (me / ms * 1e3),
          "median thr-MAPE", np.median([x.mape_thr for x in rr]))
ro = [o.run_job(jj)[0] for jj in jobs[:3]]
print("oracle first 3 thr", [x.mape_thr for x in ro], "gpu fp32", [x.mape_thr for x in rr[:3]])
