import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_2003_07497_b200 import abi, engine as E, population as P
eng = E.Engine(0)
jobs = [j for j in P.config2_jobs(root_seed=1, epochs_scale=0.002)][::6]
print(eng.run_population(jobs, abi.FP32)[0], eng.run_population(jobs, abi.FP64_EXACT)[0])
