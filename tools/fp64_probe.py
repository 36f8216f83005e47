"""FP64 exact trainer probe (developer tool): config-2 device time and the phase split for the
phased kernel and the pipelined one at several producer-warp counts; bit-identity of the
pipelined results against the phased kernel's on the same population.
usage: fp64_probe.py [epochs_scale]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if len(sys.argv) > 2:  # child: one configuration
    import numpy as np
    from paper_2003_07497_b200 import abi
    from paper_2003_07497_b200 import engine as E
    from paper_2003_07497_b200 import population as P
    scale = float(sys.argv[1])
    eng = E.Engine(0)
    jobs = P.config2_jobs(root_seed=1, epochs_scale=scale)
    pop = eng.prepare(jobs, abi.FP64_EXACT)
    pop.run(1)
    pop.run(1)
    ms = eng.last_device_ms
    st, res, params, _ = pop.fetch(want_params=True)
    np.save(sys.argv[2], np.concatenate([np.concatenate(params), [r.final_loss for r in res]]))
    print(f"{os.environ.get('TAG')}: {ms:.2f} ms  ({P.model_epochs(jobs) / ms / 1e3:.3f} M model-epochs/s)", flush=True)
    sys.exit(0)

import numpy as np  # noqa: E402
scale = sys.argv[1] if len(sys.argv) > 1 else "1.0"
out = {}
CONFIGS = [("phased", {"LANN_FP64_PHASED": "1"}), ("pipe2", {"LANN_FP64_PRODUCERS": "2"}),
           ("pipe3", {"LANN_FP64_PRODUCERS": "3"}), ("pipe4", {"LANN_FP64_PRODUCERS": "4"}), ("pipe8", {"LANN_FP64_PRODUCERS": "8"}),
           ]
only = os.environ.get("PROBE_ONLY")
for tag, env in CONFIGS:
    if only and tag not in only.split(",") and tag != "phased":
        continue
    for prof in (0, 1):
        e = dict(os.environ, TAG=tag + (" (profiled)" if prof else ""), **env)
        if prof:
            e["LANN_PHASE_PROFILE"] = "1"
        f = f"/tmp/fp64probe_{tag}.npy"
        subprocess.run([sys.executable, __file__, scale, f], env=e, check=False)
        if not prof:
            out[tag] = np.load(f)
for tag, v in out.items():
    print(tag, "bit-identical to phased:", np.array_equal(v, out["phased"]))
