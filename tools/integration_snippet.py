# the Python snippet of INTEGRATION.md, run as-is (developer check)
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.chdir(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
from paper_2003_07497_b200.abi import Job, JobResult, make_job, acceptance_world, FP64_EXACT

lib = C.CDLL("paper_2003_07497_b200/lib/libperfsage_b200.so")
eng = C.c_void_p()
assert lib.lann_engine_create(0, C.byref(eng)) == 0          # 7 = LANN_NO_DEVICE
jobs = (Job * 1)(make_job(acceptance_world(), 1))             # acceptance criterion 5, seed 1
res = (JobResult * 1)()
lib.lann_run_population.argtypes = [C.c_void_p, C.c_int32, C.POINTER(Job), C.c_int32,
                                    C.POINTER(JobResult)] + [C.c_void_p] * 4
st = lib.lann_run_population(eng, 1, jobs, FP64_EXACT, res, None, None, None, None)
print(st, res[0].final_loss, res[0].mape_thr)                # 0 8.870984881723841e-05 6.815...
lib.lann_engine_destroy(eng)
