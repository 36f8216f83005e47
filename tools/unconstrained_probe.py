import sys, time
sys.path.insert(0, '/root/repo')
from paper_2003_07497_b200 import abi, engine as E, population as P
jobs = []
for s in range(1, 6):
    ds = P.derive_seed(90, s)
    jobs.append(abi.make_job(abi.acceptance_world(), ds, count=5000, hidden=(64,), lr=1e-2, epochs=3000,
                             init_seed=s, unconstrained=True))
with E.Engine(0) as eng:
    for prec in (abi.FP64_EXACT, abi.FP32):
        p = eng.prepare(jobs, prec); p.run(1); p.run(1)
        st, res, _, _ = p.fetch()
        print(prec, st, "device ms", eng.last_device_ms, [round(r.mape_thr, 3) for r in res], [r.precision_run for r in res])
