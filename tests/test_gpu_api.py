"""GPU: models::train_full_batch through the C++ API (mlp.cpp:156-175) — the engine's FP64
exact-order trainer behind the reference's host signature — against the reference's own
train_full_batch on the same Glorot-initialised net and rows: loss trace and final parameters bit
for bit; a diverging learning rate raises TrainingError at the reference's epoch."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2003_07497_b200", "lib")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tool(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("api") / "formats_tool")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "formats_tool.cpp"), "-L", LIB, "-lperfsage_b200",
                    f"-Wl,-rpath,{LIB}", "-o", exe], check=True)
    return exe


def api_train(tool, seed, epochs, lr, n, dims):
    out = subprocess.run([tool, "api-train", str(seed), str(epochs), repr(lr), str(n), *map(str, dims)],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    rows = {}
    for line in out.stdout.splitlines():
        key, *vals = line.split()
        rows[key] = vals
    return rows


def fromhex(vals):
    return np.array([float.fromhex(v) for v in vals])


@pytest.mark.parametrize("dims,n,epochs", [([4, 8, 1], 250, 300), ([6, 5, 5, 1], 250, 300), ([7, 8, 8, 1], 97, 120),
                                           ([2, 3, 1], 5, 50), ([6, 5, 5, 1], 249, 80), ([5, 8, 1], 3, 40),
                                           ([7, 8, 1], 256, 60)])
def test_train_full_batch_is_the_reference(tool, reference, dims, n, epochs):
    r = api_train(tool, 7, epochs, 1e-2, n, dims)
    X = np.zeros((n, 8))
    X[:, :dims[0]] = fromhex(r["X"]).reshape(n, dims[0])
    y = fromhex(r["y"])
    st, p_ref, trace_ref, bad = reference.train_full_batch(dims, fromhex(r["p0"]), X, y, 1e-2, epochs)
    assert st == 0 and bad == -1, reference.last_error()
    assert [v.hex() for v in fromhex(r["trace"])] == [float(v).hex() for v in trace_ref]
    assert [v.hex() for v in fromhex(r["p1"])] == [float(v).hex() for v in p_ref]


def test_train_full_batch_divergence_is_the_reference_epoch(tool, reference):
    dims, n, epochs, lr = [4, 8, 1], 64, 50, 1e100
    r = api_train(tool, 3, epochs, lr, n, dims)
    assert "TrainingError" in r, r.keys()
    X = np.zeros((n, 8))
    X[:, :4] = fromhex(r["X"]).reshape(n, 4)
    st, _, _, bad = reference.train_full_batch(dims, fromhex(r["p0"]), X, fromhex(r["y"]), lr, epochs)
    assert st != 0 and bad >= 0
    assert int(r["TrainingError"][0]) == bad
