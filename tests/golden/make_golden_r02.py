"""Generate tests/golden/golden_r02_full.json from the REFERENCE ITSELF, at FULL length.

The round-1 goldens pinned the config-2 population at 200 epochs only; this file pins it at
the lengths BASELINE config 2 trains (prediction nets 8000 epochs, blur selection nets 20,000
epochs, models::default_config, models.cpp:66-85) and adds the stratified config-3 subset
SURVEY.md 8(d) prescribes for the CPU baseline (every combo x 4 init seeds x 5 folds = 960
models, full epochs) for the population-level FP32-vs-reference statistics.

Source: the unmodified reference core compiled from /root/reference (oracle/_ref/
libperfsage_ref.so, built by oracle/Makefile) through oracle/ref_driver.cpp — the stock
build_dataset -> split -> train_nn -> predict_dataset -> make_report pipeline per model.
/root/reference is not needed at test time. Regenerate with:
    make -C oracle && python tests/golden/make_golden_r02.py        (~2-3 min on 8 cores)
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_lib import Reference  # noqa: E402
from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import population as P  # noqa: E402
from golden.make_golden import job_dict, result_dict, sha  # noqa: E402


def one_with_trace(ref, j):
    arr = (abi.Job * 1)(j)
    res = (abi.JobResult * 1)()
    params = np.zeros(4096)
    po = np.zeros(1, dtype=np.int64)
    trace = np.zeros(j.epochs)
    to = np.zeros(1, dtype=np.int64)
    ref.lib.ref_run_population(1, arr, res, params.ctypes.data, po.ctypes.data, trace.ctypes.data,
                               to.ctypes.data, 1)
    r = res[0]
    d = result_dict(r, params[: r.n_params], trace)
    d["trace_tail"] = [float(x) for x in trace[-3:]]
    return d


def main():
    ref = Reference()
    threads = os.cpu_count() or 1
    g = {"generator": "tests/golden/make_golden_r02.py",
         "source": "reference core compiled from /root/reference (oracle/_ref/libperfsage_ref.so) via "
                   "oracle/ref_driver.cpp (build_dataset -> split -> train_nn -> predict_dataset -> make_report)"}
    # 1. config 2 at full length: every model's weights, full-trace sha256, metrics
    c2 = P.config2_jobs(root_seed=1)
    with cf.ThreadPoolExecutor(threads) as ex:
        res = list(ex.map(lambda j: one_with_trace(ref, j), c2))
    g["config2_full"] = {"jobs": [job_dict(j) for j in c2], "results": res}
    # 2. config-3 stratified subset: 48 combos x 4 seeds x 5 folds, full length (metrics + params sha)
    c3 = P.config3_jobs(root_seed=1, n_seeds=4)
    secs, rr, params = ref.run_population(c3, threads=threads, want_params=True)
    out = []
    for i, r in enumerate(rr):
        d = result_dict(r)
        d["params_sha256"] = sha(params[i * 4096:i * 4096 + r.n_params])
        out.append(d)
    # the job list is the recipe population.config3_jobs(root_seed=1, n_seeds=4); its bytes are pinned
    g["config3_subset"] = {"recipe": "population.config3_jobs(root_seed=1, n_seeds=4)", "n_seeds": 4, "n_folds": 5,
                           "jobs_sha256": hashlib.sha256(b"".join(bytes(j) for j in c3)).hexdigest(),
                           "seconds": secs, "threads": threads, "results": out}
    path = os.path.join(HERE, "golden_r02_full.json")
    with open(path, "w") as f:
        json.dump(g, f)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
