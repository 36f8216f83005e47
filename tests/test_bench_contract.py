"""CPU: bench.py's reference arm prints the contract's JSON line (the GPU arm is exercised by the
driver on the B200; its keys are pinned by the same list in the GPU-side smoke)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    from oracle_lib import Reference

    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.workload_config("fp64")  # the GPU arm prints the same dict
    assert d["config"]["model_epochs_per_gpu_step"] == 480000 and d["dtype"] == "f64"


def test_reference_arm_never_maps_the_engine_library():
    """The reference arm times the reference alone: the engine's .so must not even be loaded."""
    from oracle_lib import Reference

    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    code = ("import atexit, runpy, sys\n"
            "atexit.register(lambda: print('MAPS', 'libperfsage_b200' in open('/proc/self/maps').read()))\n"
            "sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '1']\n"
            "runpy.run_path('bench.py', run_name='__main__')\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert "MAPS False" in out.stdout, out.stdout + out.stderr
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    assert d["warmup"] == 1
