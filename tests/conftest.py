import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the engine's kernels")


@pytest.fixture(scope="session")
def oracle():
    from oracle_lib import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle_lib import Reference

    if not Reference.available():
        pytest.skip("oracle/_ref/libperfsage_ref.so not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def engine():
    """The CUDA engine on device 0. No fallback: a GPU test without a device errors."""
    from paper_2003_07497_b200 import engine as E

    eng = E.Engine(0)
    yield eng
    eng.close()


@pytest.fixture(scope="session")
def golden():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "golden_r01.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_full():
    """Full-length reference goldens (tests/golden/make_golden_r02.py): config 2 at 8000 / 20,000
    epochs and the stratified config-3 subset (48 combos x 4 seeds x 5 folds)."""
    import json

    with open(os.path.join(ROOT, "tests", "golden", "golden_r02_full.json")) as f:
        return json.load(f)
