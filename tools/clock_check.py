"""Sample SM clocks while the config-2 population runs back to back (developer tool)."""
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import engine as E  # noqa: E402
from paper_2003_07497_b200 import population as P  # noqa: E402

eng = E.Engine(0)
pop = eng.prepare(P.config2_jobs(root_seed=1), abi.FP32)
pop.run(1)
samples = []
stop = threading.Event()


def sampler():
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True).stdout.strip()
        samples.append(out)
        time.sleep(0.05)


t = threading.Thread(target=sampler)
t.start()
t0 = time.time()
n = 0
while time.time() - t0 < 4.0:
    pop.run(10)
    n += 10
stop.set()
t.join()
print(f"{n} passes, last device ms per 10 passes {eng.last_device_ms:.2f}")
print(samples)
