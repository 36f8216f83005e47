"""CPU: the engine's C-ABI library loads and exports every symbol include/lann_engine.h
declares; the engine's host-side domain code (datagen, split, init, combos) matches the
reference golden vectors; compute entry points refuse to run without a device (no fallback)."""
import hashlib
import os
import re

import numpy as np
import pytest

from paper_2003_07497_b200 import abi
from paper_2003_07497_b200 import engine as E
from paper_2003_07497_b200 import population as P
from golden.make_golden import world_from

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "lann_engine.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lann_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = E.load_library()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(E.EXPORTS) == syms


def test_struct_layouts_match_header():
    import ctypes as C
    assert C.sizeof(abi.World) == 4 * 4 + 6 * 8 + 8 * 8
    assert C.sizeof(abi.JobResult) == 6 * 4 + 4 * 8 + 2 * 4
    assert abi.Job.hidden.offset % 4 == 0 and abi.Job.learning_rate.offset % 8 == 0


def test_host_datagen_matches_reference(golden):
    for d in golden["combos"]:
        feats, c, rt, nf = E.build_dataset(world_from(d["world"]), d["seed"], 500)
        h = hashlib.sha256()
        for a in (feats, c, rt):
            h.update(np.ascontiguousarray(a).tobytes())
        assert h.hexdigest() == d["sha256"] and nf == d["n_features"]


def test_default_combos_are_the_golden_worlds(golden):
    combos = E.default_combos()
    assert len(combos) == 48
    kinds = [w.kind for w in combos]
    assert kinds.count(abi.BLUR) == 8 and all(kinds.count(k) == 10 for k in range(4))
    for w, d in zip(combos, golden["combos"]):
        assert bytes(w) == bytes(world_from(d["world"]))
    # combo 0 is the acceptance world bit for bit (acceptance_main.cpp:271-279)
    assert bytes(combos[0]) == bytes(abi.acceptance_world())


def test_python_world_table_is_the_engine_table():
    """population.combo_worlds() (used by job lists, incl. bench.py's reference arm, which must
    not load the engine library) is byte-identical to the engine's lann_default_combos."""
    py, eng = P.combo_worlds(), E.default_combos()
    assert len(py) == len(eng) == 48
    for a, b in zip(py, eng):
        assert bytes(a) == bytes(b)


def test_init_matches_reference(golden):
    for g in golden["mse_gradient"]:
        assert E.init_params(g["dims"], 5).tolist() == g["params"]


def test_population_recipes():
    c2 = P.config2_jobs(root_seed=1)
    assert len(c2) == 48 and P.model_epochs(c2) == 40 * 8000 + 8 * 20000
    blur = [j for j in c2 if j.world.kind == abi.BLUR]
    assert all(j.n_hidden == 2 and j.hidden[0] == 5 and j.log_target and j.epochs == 20000 for j in blur)
    c3 = P.config3_jobs(root_seed=1, n_seeds=256)
    assert len(c3) == 48 * 256 * 5 == 61440
    assert P.flop_per_model_epoch(7, (8,), 250) == 70272
    assert P.flop_per_model_epoch(7, (8,), 200) == 56422
    assert P.flop_per_model_epoch(6, (8,), 250) == 62160
    assert P.flop_per_model_epoch(6, (5, 5), 250) == 78494


def test_param_budget_and_counts():
    # test_models.cpp:76-103
    assert E.param_count(7, 8) == 73 and E.param_count(6, 5, 5) == 71
    for kind in range(5):
        for fam in (abi.NNC, abi.NN):
            I = {0: 5, 1: 3, 2: 4, 3: 5, 4: 5}[kind] + (1 if kind != 4 else 0) + (1 if fam == abi.NNC else 0)
            hidden, *_ = P.default_model(abi.World(kind=kind), fam)
            assert E.param_count(I, *hidden) <= 75


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    with pytest.raises(E.NoDeviceError):
        E.Engine(0)


def test_derive_seed_matches_oracle(oracle):
    for r, s in [(0, 0), (1, 0x9015E), (2 ** 64 - 1, 0xA11CE), (12345, 7)]:
        assert P.derive_seed(r, s) == oracle.lib.or_derive_seed(r, s)


def test_seqrng_bounded_fast_paths_are_exact(tmp_path):
    """The host sampler's bounded() fast paths (mask for powers of two, cached exact remainder
    for n <= 4096) draw exactly what Rng::bounded (rng.hpp) draws: 10 M draws over n = 1..5000
    and four large n."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "seqrng_check")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(root, "paper_2003_07497_b200", "csrc"),
                    os.path.join(root, "tests", "cpp", "seqrng_bounded_check.cpp"), "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and " 0 mismatches" in out.stdout, out.stdout
