"""Generate the on-disk-format fixtures under tests/golden/ from the REFERENCE ITSELF.

Uses the unmodified reference core (oracle/_ref/libperfsage_ref.so, built by oracle/Makefile from
/root/reference) through the ref_driver.cpp shim:
  * ref_dataset_w0_s1.csv   datagen::save_csv of build_dataset(world 0 = the acceptance world,
                            seed 1, 500 samples), variant id "dense_threaded@cpu4"
  * ref_model_w0_s3.json    the body of the reference CLI's `train` (perfsage.cpp:250-278) on that
                            CSV: split(derive_seed(3, 0x5b11)) -> default nnc config, seed 3,
                            200 epochs -> models::save_model (nlohmann json formatting)
  * ref_model_w0_s3_{const,lrc}.json  the same `train` body for the least-squares baselines
  * formats_r01.json        sha256 of the reference's train.csv / test.csv of that run, the
                            reference's load_model dump of the model (norm stats, weights, loss
                            trace as %a hex) and its evaluate_model_on report on test.csv
Regenerate with:  make -C oracle && python tests/golden/make_formats_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_lib import Reference  # noqa: E402
from paper_2003_07497_b200 import abi  # noqa: E402

CSV = os.path.join(HERE, "ref_dataset_w0_s1.csv")
MODEL = os.path.join(HERE, "ref_model_w0_s3.json")
SEED, EPOCHS = 3, 200


def sha_file(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def main():
    ref = Reference()
    assert ref.save_dataset_csv(abi.acceptance_world(), 1, 500, "dense_threaded@cpu4", CSV) == 0, ref.last_error()
    with tempfile.TemporaryDirectory() as d:
        tr, te = os.path.join(d, "train.csv"), os.path.join(d, "test.csv")
        assert ref.cli_train(CSV, SEED, "nnc", EPOCHS, MODEL, tr, te) == 0, ref.last_error()
        st, rep = ref.eval_model(MODEL, te, 0.3)
        assert st == 0
        out = {
            "csv": os.path.basename(CSV), "csv_sha256": sha_file(CSV),
            "model": os.path.basename(MODEL), "train": {"seed": SEED, "epochs": EPOCHS, "family": "nnc"},
            "train_csv_sha256": sha_file(tr), "test_csv_sha256": sha_file(te),
            "model_dump_hex": [float(x).hex() for x in ref.model_dump(MODEL)],
            "eval_test": {"mape_full": rep[0], "mape_thresholded": rep[1], "rho": rep[2], "n_kept": int(rep[3])},
            "baselines": {},
        }
        # the baseline families (models.cpp:305-333): const / lrc files are small enough to commit;
        # the 100-tree forest (5 MB) is pinned by its per-tree node counts and its report
        for fam in ("const", "lrc", "nlrc"):
            path = os.path.join(HERE if fam != "nlrc" else d, f"ref_model_w0_s3_{fam}.json")
            assert ref.cli_train(CSV, SEED, fam, 0, path, tr, te) == 0, ref.last_error()
            st, rep = ref.eval_model(path, te, 0.3)
            assert st == 0
            entry = {"eval_test": {"mape_full": rep[0], "mape_thresholded": rep[1], "rho": rep[2],
                                   "n_kept": int(rep[3])}}
            if fam == "nlrc":
                with open(path) as f:
                    forest = json.load(f)["payload"]["forest"]
                entry["tree_node_counts"] = [len(t) for t in forest]
            else:
                entry["model"] = os.path.basename(path)
            out["baselines"][fam] = entry
    with open(os.path.join(HERE, "formats_r01.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", CSV, MODEL, "formats_r01.json")


if __name__ == "__main__":
    main()
