"""CPU: the on-disk formats and the `perfsage gen` caller, against the
reference's own writers and readers.

* datagen::save_csv / load_csv (csv.cpp:43-102): `perfsage gen` writes byte-for-byte the CSV the
  reference writes for the same dataset; CSV round trips are byte-identical in both directions.
* models::save_model / load_model (model_io.cpp:114-173): every double (norm stats, weights, loss
  trace) survives engine -> reference -> engine and reference -> engine -> reference bit for bit.
* LoadError behaviour on malformed files mirrors csv.cpp / model_io.cpp.
Pinned by fixtures written by the reference itself (tests/golden/make_formats_golden.py), and
cross-checked live against oracle/_ref/libperfsage_ref.so where it was built.
"""
import hashlib
import json
import os
import subprocess

import pytest

from paper_2003_07497_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
CLI = os.path.join(ROOT, "paper_2003_07497_b200", "bin", "perfsage")
LIB = os.path.join(ROOT, "paper_2003_07497_b200", "lib")


def sha_file(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


@pytest.fixture(scope="module")
def fmt():
    return json.load(open(os.path.join(GOLD, "formats_r01.json")))


@pytest.fixture(scope="module")
def tool(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("fmt") / "formats_tool")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "formats_tool.cpp"), "-L", LIB, "-lperfsage_b200",
                    f"-Wl,-rpath,{LIB}", "-o", exe], check=True)
    return exe


def run(*args):
    out = subprocess.run(list(args), capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    return out.stdout


def dump_hex(tool, path):
    return [float.fromhex(x).hex() for x in run(tool, "model-dump", str(path)).split()]


def test_gen_csv_is_the_reference_csv(tmp_path, fmt):
    """`perfsage gen --world 0 --seed 1 --count 500` == the reference's build_dataset + save_csv
    of the acceptance world, byte for byte (sha256 of the reference-written fixture)."""
    run(CLI, "gen", "--world", "0", "--count", "500", "--seed", "1", "--out", str(tmp_path))
    ours = tmp_path / "dataset_mm_dense_threaded_cpu4.csv"
    assert sha_file(ours) == fmt["csv_sha256"]
    man = json.load(open(tmp_path / "manifest.json"))
    assert man["runs"][0]["command"] == "gen" and man["runs"][0]["seed"] == 1
    assert man["runs"][0]["outputs"] == [str(ours)]


@pytest.mark.parametrize("world", [3, 12, 27, 40, 46])
def test_gen_csv_matches_live_reference(tmp_path, reference, world):
    """Every kind of world (GPU-class without n_thd, MV, MP, both blur lattices): our CSV bytes ==
    the reference's save_csv of its own build_dataset with the same probe."""
    from paper_2003_07497_b200 import engine as E

    run(CLI, "gen", "--world", str(world), "--count", "64", "--seed", "5", "--out", str(tmp_path))
    (ours,) = [p for p in tmp_path.iterdir() if p.suffix == ".csv"]
    vid = open(ours).read().split("\n")[1].split(",")[1]
    ref = tmp_path / "ref.csv"
    assert reference.save_dataset_csv(E.default_combos()[world], 5, 64, vid, ref) == 0, reference.last_error()
    assert open(ours, "rb").read() == open(ref, "rb").read()


def test_csv_round_trips_are_byte_identical(tmp_path, tool, reference):
    src = os.path.join(GOLD, "ref_dataset_w0_s1.csv")
    run(tool, "csv-roundtrip", src, str(tmp_path / "ours.csv"))
    assert open(tmp_path / "ours.csv", "rb").read() == open(src, "rb").read()
    assert reference.csv_roundtrip(tmp_path / "ours.csv", tmp_path / "back.csv") == 0
    assert open(tmp_path / "back.csv", "rb").read() == open(src, "rb").read()


def test_reference_model_file_loads_bit_exact(tmp_path, tool, fmt):
    """The reference-written model (nlohmann formatting) loads here with every double identical to
    the reference's own load_model; re-saving and re-loading changes nothing."""
    src = os.path.join(GOLD, fmt["model"])
    assert dump_hex(tool, src) == fmt["model_dump_hex"]
    run(tool, "model-roundtrip", src, str(tmp_path / "m.json"))
    assert dump_hex(tool, tmp_path / "m.json") == fmt["model_dump_hex"]


def test_model_round_trip_through_the_reference(tmp_path, tool, reference):
    """Awkward doubles (subnormals, -0, DBL_MAX, 0.1, a u64 seed of 2^64-1) written by the engine
    load bit-exact in the reference, and the reference's re-save loads bit-exact here."""
    ours = tmp_path / "synth.json"
    run(tool, "model-synth", str(ours), "17")
    mine = dump_hex(tool, ours)
    assert [float(x).hex() for x in reference.model_dump(ours)] == mine
    back = tmp_path / "back.json"
    assert reference.model_roundtrip(ours, back) == 0, reference.last_error()
    assert dump_hex(tool, back) == mine
    assert json.load(open(back))["config"]["seed"] == 2**64 - 1


def test_csv_load_errors(tmp_path, tool):
    """csv.cpp:62-100: LoadError for a bad header, unknown schema, wrong field count, bad numbers,
    a kernel column that disagrees with the schema, negative c, runtime <= 0."""
    head = "kernel,variant,m,n,k,d1,d2,n_thd,c,runtime_s\n"
    good = "mm,v,1,2,3,1,1,1,6,0.5\n"
    cases = {
        "header": "kernel,variant,c\n",
        "schema": "kernel,variant,a,b,c,runtime_s\nmm,v,1,2,3,0.5\n",
        "fields": head + "mm,v,1,2,3,1,1,1,6\n",
        "number": head + "mm,v,1,x,3,1,1,1,6,0.5\n",
        "kernel": head + "mv,v,1,2,3,1,1,1,6,0.5\n",
        "neg_c": head + "mm,v,1,2,3,1,1,1,-6,0.5\n",
        "runtime": head + "mm,v,1,2,3,1,1,1,6,0\n",
    }
    for name, text in cases.items():
        p = tmp_path / f"{name}.csv"
        p.write_text(text)
        assert run(tool, "csv-load", str(p)).startswith("LoadError"), name
    p = tmp_path / "ok.csv"
    p.write_text(head + good + "\r\n" + good.replace("\n", "\r\n"))
    assert run(tool, "csv-load", str(p)).strip() == "ok 2"


def test_model_load_errors(tmp_path, tool, fmt):
    src = json.load(open(os.path.join(GOLD, fmt["model"])))
    bad = {
        "not_json": "{",
        "format": json.dumps({**src, "format": "other"}),
        "version": json.dumps({**src, "version": 2}),
        "missing": json.dumps({k: v for k, v in src.items() if k != "norm_stats"}),
        "shape": json.dumps({**src, "payload": {"layers": [{"rows": 2, "cols": 2, "weights": [1.0], "biases": [0.0, 0.0]}]}}),
        "family": json.dumps({**src, "config": {**src["config"], "family": "svm"}}),
    }
    for name, text in bad.items():
        p = tmp_path / f"{name}.json"
        p.write_text(text)
        assert run(tool, "model-load", str(p)).startswith("LoadError"), name


def test_cli_gpu_commands_fail_loudly_without_a_device(tmp_path):
    """No CPU fallback: on a machine without a GPU the training commands exit 1 with an error."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    out = subprocess.run([CLI, "train", "--data", os.path.join(GOLD, "ref_dataset_w0_s1.csv"), "--out",
                          str(tmp_path)], capture_output=True, text=True)
    assert out.returncode == 1 and "no CUDA device" in out.stderr


def test_cli_argument_errors(tmp_path):
    for args in (["frobnicate"], ["gen", "--world"], ["gen", "--count", "x"], ["gen", "--world", "99"],
                 ["sweep", "--family", "svm"]):
        out = subprocess.run([CLI, *args, "--out", str(tmp_path)] if len(args) > 1 else [CLI, *args],
                             capture_output=True, text=True)
        assert out.returncode == 1 and out.stderr.startswith("error:"), args


@pytest.mark.parametrize("kind,gpu_class", [(abi.MM, False), (abi.MV, True), (abi.MP, False), (abi.BLUR, False)])
def test_gen_external_protocol_matches_reference(tmp_path, reference, kind, gpu_class):
    """`perfsage gen --external-cmd CMD` (external.cpp protocol: one line of %.17g features on
    stdin, one runtime on stdout) builds the CSV the reference builds with the same command."""
    name = {abi.MM: "mm", abi.MV: "mv", abi.MP: "mp", abi.BLUR: "blur"}[kind]
    cmd = "awk '{s=1; for(i=1;i<=NF;i++) s+=$i; printf \"%.17g\\n\", s*1e-9}'"
    args = ["gen", "--external-cmd", cmd, "--kernel", name, "--count", "12", "--seed", "9", "--max-threads", "4",
            "--external-id", "ext", "--out", str(tmp_path)]
    if gpu_class:
        args.append("--gpu-class")
    run(CLI, *args)
    ours = tmp_path / f"dataset_{name}_ext.csv"
    ref = tmp_path / "ref.csv"
    assert reference.save_external_csv(kind, gpu_class, 4, cmd, "ext", 12, 9, ref) == 0, reference.last_error()
    assert open(ours, "rb").read() == open(ref, "rb").read()


def test_gen_external_protocol_errors(tmp_path):
    for cmd, what in (("exit 3", "exited with status 3"), ("echo abc", "non-numeric"), ("echo -1", "non-positive"),
                      ("true", "no runtime")):
        out = subprocess.run([CLI, "gen", "--external-cmd", cmd, "--kernel", "mm", "--count", "2", "--out",
                              str(tmp_path)], capture_output=True, text=True)
        assert out.returncode == 1 and what in out.stderr, (cmd, out.stderr)


def _payload_hex(path):
    p = json.load(open(path))["payload"]
    if "linear" in p:
        return [float(x).hex() for x in p["linear"]["weights"] + [p["linear"]["intercept"]]]
    return [(n["feature"], float(n["threshold"]).hex(), n["left"], n["right"], float(n["value"]).hex())
            for t in p["forest"] for n in t]


@pytest.mark.parametrize("kind", ["linear", "forest"])
def test_baseline_model_files_round_trip_through_the_reference(tmp_path, tool, reference, kind):
    """const/lrc (payload.linear) and nlrc (payload.forest) model files: engine -> reference ->
    engine leaves every weight, threshold and leaf value bit-identical."""
    ours = tmp_path / "m.json"
    run(tool, f"model-synth-{kind}", str(ours), "5")
    back = tmp_path / "back.json"
    assert reference.model_roundtrip(ours, back) == 0, reference.last_error()
    assert _payload_hex(back) == _payload_hex(ours)
    again = tmp_path / "again.json"
    run(tool, "model-roundtrip", str(back), str(again))
    assert _payload_hex(again) == _payload_hex(ours)
    assert json.load(open(again))["metrics"] is None


@pytest.mark.parametrize("fam", ["const", "lrc"])
def test_reference_baseline_files_load(tmp_path, tool, fam):
    src = os.path.join(GOLD, f"ref_model_w0_s3_{fam}.json")
    run(tool, "model-roundtrip", src, str(tmp_path / "m.json"))
    assert _payload_hex(tmp_path / "m.json") == _payload_hex(src)


@pytest.mark.parametrize("kernel,kind,variant,extra,sides,gpu", [
    ("mm", abi.MM, "dense_threaded", [], [1024], False),
    ("mm", abi.MM, "tiled_threaded", ["--dim-max", "4096"], [1024], False),
    ("mv", abi.MV, "sparse_single", [], [1024], False),
    ("mc", abi.MC, "dense_single", ["--dim-max", "300"], [1024], False),
    ("mp", abi.MP, "dense_threaded", [], [1024], False),
    ("blur", abi.BLUR, "tiled", ["--blur-n", "512", "--blur-n", "2048"], [512, 2048], False),
    ("blur", abi.BLUR, "tiled", ["--blur-space", "gpu"], [1024], True),
])
def test_gen_mock_timer_is_the_reference_cli(tmp_path, reference, kernel, kind, variant, extra, sides, gpu):
    """`perfsage gen --mock-timer` (perfsage.cpp:71-84 probe, :197-248 body) writes the dataset the
    reference CLI writes, byte for byte, for every builtin variant class and parameter-space option."""
    run(CLI, "gen", "--mock-timer", "--kernel", kernel, "--variant", variant, "--count", "80", "--seed", "4",
        "--max-threads", "6", *extra, "--out", str(tmp_path))
    ours = tmp_path / f"dataset_{kernel}_{variant}.csv"
    ref = tmp_path / "ref.csv"
    dim_max = int(extra[extra.index("--dim-max") + 1]) if "--dim-max" in extra else 1024
    assert reference.cli_gen_mock(kind, variant, 6, dim_max, sides, gpu, 80, 4, ref) == 0, reference.last_error()
    assert open(ours, "rb").read() == open(ref, "rb").read()


@pytest.mark.parametrize("kernel,kind,variant,dim_max,sides,gpu", [
    ("mm", abi.MM, "dense_threaded", 1024, [1024], False),
    ("mm", abi.MM, "tiled_threaded", 4096, [1024], False),
    ("mv", abi.MV, "sparse_single", 1024, [1024], False),
    ("mc", abi.MC, "dense_single", 300, [1024], False),
    ("mp", abi.MP, "dense_threaded", 1024, [1024], False),
    ("blur", abi.BLUR, "tiled", 1024, [512, 2048], False),
    ("blur", abi.BLUR, "tiled", 1024, [1024], True),
])
def test_api_build_dataset_is_the_reference(tmp_path, tool, reference, kernel, kind, variant, dim_max, sides, gpu):
    """The C++ API path a reference user calls — ParamSpace::defaults, VariantDescriptor,
    datagen::build_dataset(variant, space, count, seed, {probe}) (datagen.cpp:177-223, sample_params
    :60-110, featurize, complexity, Rng) — writes the reference's dataset byte for byte."""
    ours = tmp_path / "api.csv"
    run(tool, "api-gen", kernel, variant, "6", str(dim_max), str(int(gpu)), "80", "4", str(ours), *map(str, sides))
    ref = tmp_path / "ref.csv"
    assert reference.cli_gen_mock(kind, variant, 6, dim_max, sides, gpu, 80, 4, ref) == 0, reference.last_error()
    assert open(ours, "rb").read() == open(ref, "rb").read()


@pytest.mark.parametrize("kernel,kind", [("mm", abi.MM), ("mv", abi.MV), ("mc", abi.MC), ("mp", abi.MP),
                                         ("blur", abi.BLUR)])
def test_api_sample_params_is_the_reference(tool, reference, kernel, kind):
    """datagen::sample_params draws (defaults space, max_threads 8) featurize to the reference's
    values bit for bit over 300 draws of one Rng stream."""
    rows = [[float.fromhex(x) for x in line.split()] for line in run(tool, "api-params", kernel, "11", "300").splitlines()]
    nf, ref = reference.sample_features(kind, 11, 300)
    assert nf > 0, reference.last_error()
    assert [[v.hex() for v in r] for r in rows] == [[float(v).hex() for v in r] for r in ref]


@pytest.mark.parametrize("dims", [[4, 8, 1], [6, 5, 5, 1], [7, 1], [1, 1], [3, 16, 16, 1]])
def test_api_mlp_init_is_the_reference(tool, reference, dims):
    """models::Mlp::init(dims, Rng) (mlp.cpp: Glorot-uniform weights, zero biases) draws the
    reference's parameters bit for bit."""
    ours = [float.fromhex(x) for x in run(tool, "api-init", "2024", *map(str, dims)).split()]
    n, ref = reference.mlp_init(dims, 2024, raw=True)
    assert n == len(ours)
    assert [v.hex() for v in ours] == [float(v).hex() for v in ref]


@pytest.mark.parametrize("dims", [["4"], ["4", "0", "1"]])
def test_api_mlp_init_rejects_bad_dims(tool, dims):
    assert run(tool, "api-init", "1", *dims).startswith("ParamError")


def test_api_build_dataset_errors(tool):
    """datagen.cpp:177-223: ParamError before sampling (count < 2, kind mismatch); a probe
    failure or a runtime <= 0 aborts with BuildAbortError carrying the completed count and the
    reference's message; without a probe the engine (which times no CPU kernel) refuses."""
    out = dict(line.split(" ", 1) for line in run(tool, "api-gen-errors").splitlines())
    assert out["count1"] == "ParamError build_dataset needs count >= 2"
    assert out["kind"] == "ParamError variant kernel does not match the parameter space"
    assert out["noprobe"].startswith("ParamError ")
    assert out["zero"] == "BuildAbortError 2 dataset build aborted after 2/5 samples: measured runtime must be > 0"
    assert out["throws"] == "BuildAbortError 0 dataset build aborted after 0/5 samples: probe failed"


def test_api_instance_params_validate_and_complexity(tool):
    """kernels.cpp:149-206: InstanceParams::validate domain rules and the complexity formulas;
    datagen::median_of, density_ladder and eval::speedup."""
    out = dict(line.split(" ", 1) for line in run(tool, "api-validate").splitlines())
    assert out["mm-ok"] == "60" and out["mv-ok"] == "63" and out["mc-ok"] == str(7 * 6 * 9)
    assert out["mp-ok"] == str(4 * 5 * 4) and out["blur-ok"] == str(1024 * 1024)
    for bad in ("mm-zero-dim", "mm-density", "mc-small", "mp-small", "blur-npow2", "blur-small", "n_thd0"):
        assert out[bad] == "ParamError", bad
    assert [float.fromhex(x) for x in out["median"].split()] == [2.0, 2.5]
    assert float.fromhex(out["speedup"]) == 4.0
    assert [float.fromhex(x) for x in out["ladder"].split()] == [0.5, 0.25, 0.125]


def test_gen_rejects_unknown_native_variant(tmp_path):
    out = subprocess.run([CLI, "gen", "--mock-timer", "--kernel", "blur", "--variant", "dense_single", "--out",
                          str(tmp_path)], capture_output=True, text=True)
    assert out.returncode == 1 and "no variant" in out.stderr
