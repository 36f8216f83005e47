"""GPU: the multi-GPU product path (lann_group_*, `perfsage sweep --devices`) on one B200 by
listing device 0 twice: two engines, two host threads, two contiguous cost-balanced shards,
results gathered on the host in job order (no collective). The FP64-exact results
must equal the unsharded population's bit for bit."""
import csv
import os
import subprocess

import numpy as np
import pytest

from paper_2003_07497_b200 import abi
from paper_2003_07497_b200 import engine as E
from paper_2003_07497_b200 import population as P

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2003_07497_b200", "bin", "perfsage")


@pytest.mark.parametrize("n_dev", [2, 4, 8])
def test_group_of_shards_equals_one_engine(engine, n_dev):
    """SURVEY 8(e)'s determinism invariant: identical outputs for G = 1, 2, 4, 8 shards."""
    jobs = P.config2_jobs(root_seed=3, epochs_scale=0.05)
    st1, res1, par1, _ = engine.run_population(jobs, abi.FP64_EXACT, want_params=True)
    assert st1 == 0
    with E.Group([0] * n_dev) as g:
        b = g.shard_bounds(jobs)
        assert len(b) == n_dev + 1 and b[0] == 0 and b[-1] == len(jobs)
        assert all(b[k] < b[k + 1] for k in range(n_dev))
        st2, res2, par2 = g.run_population(jobs, abi.FP64_EXACT, want_params=True)
        assert st2 == 0, g.last_error
        assert g.last_device_ms > 0 and g.last_wall_ms > 0
    for a, c, pa, pc in zip(res1, res2, par1, par2):
        assert (a.status, a.final_loss, a.mape, a.mape_thr, a.rho, a.n_kept) == \
            (c.status, c.final_loss, c.mape, c.mape_thr, c.rho, c.n_kept)
        assert np.array_equal(pa, pc)


def test_group_reports_a_failing_shard():
    jobs = P.config2_jobs(root_seed=3, epochs_scale=0.01)
    jobs[-1].learning_rate = 0.5  # ParamError in the last shard only
    with E.Group([0, 0]) as g:
        st, res, _ = g.run_population(jobs, abi.FP64_EXACT)
    assert st == abi.PARAM_ERROR
    assert res[-1].status == abi.PARAM_ERROR and res[0].status == 0


def _sweep(tmp, *dev):
    out = subprocess.run([CLI, "sweep", "--seeds", "2", "--folds", "5", "--epochs-scale", "0.02", "--precision",
                          "fp64", "--combos", "0,7,40", "--out", str(tmp), *dev],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    with open(tmp / "sweep.csv") as f:
        return list(csv.DictReader(f)), out.stdout


def test_cli_sweep_over_devices_equals_one_device(tmp_path):
    one, _ = _sweep(tmp_path / "a", "--device", "0")
    two, log = _sweep(tmp_path / "b", "--devices", "0,0")
    assert one == two and len(one) == 3 * 2 * 5
    assert "on 2 device(s)" in log and "shards" in log
