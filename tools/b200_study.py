"""The paper's comparison on REAL B200 runtimes (SURVEY.md 8(f) row 3 end to end): for every
GPU-class kernel variant of measure.cu, measure a dataset on this B200 (`perfsage gen --measure`,
sample_params draws, median of reps, CUDA events), then train and evaluate the five model
families on it (`perfsage compare`, 50/50 split) and print one table.

usage: python tools/b200_study.py [count] [out_dir]    (developer tool; needs a GPU)
"""
import csv
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2003_07497_b200", "bin", "perfsage")
count = int(sys.argv[1]) if len(sys.argv) > 1 else 500
out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "b200_study")
VARIANTS = [("mm", "gemm_tiled"), ("mm", "cublas_sgemm"), ("mm", "spmm_csr"), ("mv", "gemv_dense"),
            ("mv", "spmv_csr"), ("mc", "conv_direct"), ("mp", "maxpool"), ("blur", "blur_sched")]

rows = []
for kind, variant in VARIANTS:
    d = os.path.join(out, f"{kind}_{variant}")
    t0 = time.time()
    subprocess.run([CLI, "gen", "--measure", "--kernel", kind, "--variant", variant, "--count", str(count),
                    "--seed", "1", "--reps", "5", "--out", d], check=True, capture_output=True)
    t_meas = time.time() - t0
    data = os.path.join(d, f"dataset_{kind}_{variant}_b200.csv")
    with open(data) as f:
        rt = [float(r["runtime_s"]) for r in csv.DictReader(f)]
    t0 = time.time()
    subprocess.run([CLI, "compare", "--data", data, "--seed", "1", "--precision", "fp32", "--out", d], check=True,
                   capture_output=True)
    t_cmp = time.time() - t0
    with open(os.path.join(d, "compare.csv")) as f:
        rep = {r["model_family"]: r for r in csv.DictReader(f)}
    rows.append((kind, variant, min(rt), max(rt), t_meas, t_cmp, rep))

fams = ["nnc", "nn", "const", "lrc", "nlrc"]
print(f"B200 measured datasets: {count} sample_params draws per variant, median of 5 CUDA-event timings, "
      f"50/50 split, thresholded MAPE % (30% smallest runtimes dropped) / Spearman rho on the test half")
print(f"{'kernel':6} {'variant':13} {'runtime range (us)':>20} " + " ".join(f"{f:>13}" for f in fams) +
      "   measure_s compare_s")
for kind, variant, lo, hi, tm, tc, rep in rows:
    cells = " ".join(f"{float(rep[f]['mape_thresholded']):6.1f}/{float(rep[f]['rho']):5.3f}" for f in fams)
    print(f"{kind:6} {variant:13} {lo * 1e6:9.1f}-{hi * 1e6:9.1f} {cells}   {tm:9.1f} {tc:9.1f}")
