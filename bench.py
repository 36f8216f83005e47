#!/usr/bin/env python
"""bench.py — LANN model-epochs/s (BASELINE config 2) on N B200s, plus the reference arm.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--precision fp64|fp32] [--impl ours|reference]

One STEP = one full pass of the hot path over the config-2 population: the 48
kernel-variant-hardware LANNs (40 prediction nets 8000 epochs, 8 blur selection
nets 20000 epochs; 480,000 model-epochs) trained from their initial weights,
then every held-out sample predicted and MAPE / thresholded MAPE / Spearman
computed per model, in the FP64 exact mode (bit-identical to the reference; the
reference computes in f64). Multi-GPU (torchrun): weak scaling, every rank trains
its own 48-combo population (root seed 1 + rank); no collective on the data path;
the barrier and the MAX-over-ranks reduction of the timing go over gloo (host).

value : model-epochs/s over all ranks, device time (CUDA events on the engine
        stream) of K device-only passes with all inputs resident in HBM; L2 is
        flushed (256 MiB write) between timed steps.
e2e   : the same metric through the public C ABI (lann_run_population) from host
        job descriptions to host results: host data generation, H2D, the device
        pass, D2H, wall clock per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2003_07497_b200 import abi  # noqa: E402
from paper_2003_07497_b200 import population as popmod  # noqa: E402

WORKLOAD = ("config2: 48 kernel-variant-hardware LANNs trained as one population "
            "(40 prediction nets I=4..7,H=8,8000 ep + 8 blur selection nets 6-5-5-1,20000 ep; "
            "250 train / 250 eval samples each) + held-out predict + MAPE/thr-MAPE/Spearman")


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML every ~2 ms (the
    config-2 timed region is ~80 ms), nvidia-smi every 0.2 s where NVML is unavailable."""

    _REASONS = [("hw_slowdown", "HwSlowdown", 0x8), ("hw_thermal_slowdown", "HwThermalSlowdown", 0x40),
                ("sw_thermal_slowdown", "SwThermalSlowdown", 0x20), ("sw_power_cap", "SwPowerCap", 0x4)]

    def __init__(self, index):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, set of reason names)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:  # the CUDA device's own NVML handle (CUDA_VISIBLE_DEVICES may renumber devices)
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _run_nvml(self, nv, h):
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            bits = get_reasons(h)
            self.samples.append((float(sm), float(mx), {n for n, _, b in self._REASONS if bits & b}))
            self._stop.wait(0.002)

    def _run_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    f = [x.strip() for x in out.split(",")]
                    num = lambda x: float(x) if x.replace(".", "").isdigit() else None  # noqa: E731
                    self.samples.append((num(f[0]), num(f[1]),
                                         {self._REASONS[i][0] for i in range(4) if len(f) > i + 2 and f[i + 2] == "Active"}))
            except Exception:
                pass
            self._stop.wait(0.2)

    def _run(self):
        try:
            nv, h = self._handle()
            self.source = "nvml"
            self._run_nvml(nv, h)
        except Exception:
            self.source = "nvidia-smi"
            self._run_smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        sm = [s[0] for s in self.samples if s[0] is not None]
        mx = [s[1] for s in self.samples if s[1] is not None]
        reasons = sorted(set().union(*[s[2] for s in self.samples]))
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples), "source": getattr(self, "source", None)}


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def fp32_peak():
    d = load_json(os.path.join(ROOT, "profiles", "fp32_peak.json"))
    if d and d.get("fp32_tflops"):
        return float(d["fp32_tflops"]), "measured: profiles/fp32_peak.json (tools/peaks.cu FFMA/FFMA2 microbenchmark)"
    return 74.4, "derived nominal: 148 SM x 128 lanes x 2 FLOP x 1.965 GHz (no measured FP32 peak found)"


def host_cpu_name():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_reference_run(jobs, threads):
    """The reference's own CPU path (oracle/_ref, compiled from the reference sources) or,
    if that library is absent, the C restatement; returns (seconds, kind)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Oracle, Reference  # test infrastructure: the baseline leg only
    if Reference.available():
        secs, res, _ = Reference().run_population(jobs, threads)
        bad = [r.status for r in res if r.status]
        return secs, "reference", bad
    o = Oracle()
    import concurrent.futures as cf
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(threads) as ex:
        res = list(ex.map(lambda j: o.run_job(j)[0], jobs))
    return time.perf_counter() - t0, "port", [r.status for r in res if r.status]


def hbm_peak():
    """(GB/s, source): MEASURED_PEAKS.json's copy bandwidth (driver-written), else the
    profiling recipe's B200 fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "of measured (MEASURED_PEAKS.json hbm_gbs: copy, read+write bytes)"
    except Exception:  # noqa: BLE001
        return 6650.0, "of fallback (B200_PROFILING.md: 6.65 TB/s)"


def fp_peaks():
    """FP64 / FP32 CUDA-core peaks measured on this pool's B200 (tools/peaks.cu ->
    profiles/fp32_peak.json); MEASURED_PEAKS.json carries neither."""
    d = load_json(os.path.join(ROOT, "profiles", "fp32_peak.json")) or {}
    return {"dfma_tflops": d.get("dfma_tflops", 36.98), "dadd_tflops": d.get("dadd_gops", 18482.6) / 1e3,
            "fp32_tflops": fp32_peak()[0], "source": "measured: profiles/fp32_peak.json (tools/peaks.cu)"}


def workload_config(precision):
    """The one config dict both arms print (the driver compares them)."""
    return {"workload": WORKLOAD, "models_per_gpu": 48, "model_epochs_per_gpu_step": 480000,
            "arithmetic": "f64, the reference's exact operation order (mlp.cpp:36-175)" if precision == "fp64"
            else "f32 with FMA (throughput mode)",
            "multi_gpu": "weak scaling: one independent 48-model population per GPU, no data-path collective",
            "l2": "GPU arm flushes L2 between timed steps (256 MiB write)"}


def run_reference_arm(args, rank, world):
    """The reference's own CPU implementation (oracle/_ref: the unmodified perfsage core built
    from /root/reference sources) on the host cores: build_dataset -> split -> train_nn ->
    predict_dataset -> make_report per model, one model per std::thread task. Only rank 0 runs.
    Nothing here maps the engine library: the job list comes from population.py."""
    if rank != 0:
        return 0
    jobs = popmod.config2_jobs(root_seed=1)
    me = popmod.model_epochs(jobs)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference_run(jobs, threads)
    times = []
    kind = "reference"
    for _ in range(args.steps):
        secs, kind, bad = cpu_reference_run(jobs, threads)
        times.append(secs)
    total = sum(times)
    value = me * len(times) / total
    line = {
        "impl": "reference", "metric": "LANN model-epochs/sec", "value": value, "unit": "model-epochs/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config("fp64"),
        "host": "reference perfsage core (oracle/_ref) train_nn+predict_dataset+make_report, one model per std::thread task",
        "cpu_baseline": {"value": value, "unit": "model-epochs/s", "cores": threads, "kind": kind,
                         "sample": f"the whole config-2 population (48 models, {me} model-epochs) per step on {threads} host threads",
                         "host": host_cpu_name()},
        "e2e": {"value": value, "unit": "model-epochs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def time_population(eng, pop, steps, flush):
    """K device passes of a prepared population, L2 flushed before each: (device ms, trainer ms,
    launches) summed over the steps (CUDA events on the engine stream)."""
    import torch
    dev_ms, train_ms, launches = 0.0, 0.0, 0
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        pop.run(1)
        dev_ms += eng.last_device_ms
        train_ms += eng.last_train_ms
        launches += eng.last_launches
    return dev_ms, train_ms, launches


def time_e2e(E, eng, jobs, precision, steps):
    """The same metric through the public C ABI with host buffers: lann_run_population from host
    job descriptions (host datagen, split, NormStats, init) through H2D, the device pass and D2H
    of every model's results, wall clock per call."""
    E.transfer_bytes(reset=True)
    times = []
    for _ in range(steps):
        t1 = time.perf_counter()
        st, res, _, _ = eng.run_population(jobs, precision)
        times.append(time.perf_counter() - t1)
        assert st == 0, eng.last_error
    h2d, d2h = E.transfer_bytes(reset=True)
    return sum(times) / len(times), h2d // len(times), d2h // len(times)


def critical_path(jobs, train_launch_ms, clock_mhz, precision):
    max_epochs = max(j.epochs for j in jobs)
    us = 1e3 * train_launch_ms / max_epochs
    cyc = us * clock_mhz
    extra = {}
    if precision == "fp64":
        # the serial floor bit-exactness imposes: each parameter's gradient is an N-long dependent DADD
        # chain in sample order (mlp.cpp:106-118), at the measured DADD latency (profiles/fp32_peak.json)
        n = max(int(round(j.count * j.train_fraction)) for j in jobs if j.epochs == max_epochs)
        lat = (load_json(os.path.join(ROOT, "profiles", "fp32_peak.json")) or {}).get("dadd_latency_cyc", 8.07)
        extra = {"dadd_chain_floor_cycles": n * lat, "frac_of_chain_floor": n * lat / cyc,
                 "chain_floor_note": f"{n} dependent DADD links x {lat} cycles (measured latency): the epoch's "
                                     "irreducible serial part; producers' first round and Adam add to it"}
    return {"models_on_path": sum(1 for j in jobs if j.epochs == max_epochs), "epochs": max_epochs,
            "us_per_epoch": us, "cycles_per_epoch": cyc, "clock_mhz": clock_mhz, **extra,
            "sms_busy": f"{len(jobs)} of 148 (one CTA per model)",
            "note": ("per epoch (FP64 exact, train_fp64_pipe): producer warps run the samples' forward/backward "
                     "and store per-parameter terms; one lane per parameter extends its sample-order DADD chain "
                     "(250 dependent links) as rounds land; then Adam (3 correctly rounded divisions + sqrt); "
                     "DESIGN.md section 3") if precision == "fp64" else
                    ("per epoch (FP32 CTA kernel): forward/backward of 2 samples per thread, warp reduce-scatter of "
                     "72 gradient values, cross-warp sum + Adam + weight broadcast (2 CTA barriers)")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--precision", choices=["fp64", "fp32"], default="fp64",
                    help="headline arithmetic: fp64 = the reference's exact order (bit-identical), the default")
    ap.add_argument("--no-extras", action="store_true", help="skip the secondary measurements")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank, local_rank, world = dist_env()
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2003_07497_b200 import engine as E

    # LANN_BENCH_SHARE_DEVICE=1: every rank on device 0 — only for exercising the multi-rank code
    # path on a one-GPU box. The plumbing (barrier, max over ranks) is gloo on the host: the data
    # path has no collective, and nothing here needs NCCL.
    share = os.environ.get("LANN_BENCH_SHARE_DEVICE") == "1"
    device = 0 if share else local_rank
    torch.cuda.set_device(device)
    if world > 1:
        dist.init_process_group("gloo")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    precision = abi.FP64_EXACT if args.precision == "fp64" else abi.FP32
    eng = E.Engine(device)
    jobs = popmod.config2_jobs(root_seed=1 + rank)
    me_rank = popmod.model_epochs(jobs)
    pop = eng.prepare(jobs, precision)
    flop = pop.flop
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        pop.run(1)
    barrier()
    t0 = time.perf_counter()
    with ClockSampler(device) as clk:
        dev_ms, train_ms, launches = time_population(eng, pop, args.steps, flush)
    barrier()
    wall_s = time.perf_counter() - t0
    st, results, _, _ = pop.fetch()
    bad = [r.status for r in results if r.status]
    dev_ms = max_over_ranks(dev_ms)
    value = me_rank * world * args.steps / (dev_ms / 1e3)
    clocks = clk.summary()
    clock_mhz = clocks.get("sm_mhz") or 1965.0
    peaks = fp_peaks()
    train_launch_ms = train_ms / args.steps
    achieved = flop / (train_launch_ms / 1e3) / 1e12
    prof = load_json(os.path.join(ROOT, "profiles", "r02_traffic.json")) or {}
    if precision == abi.FP64_EXACT:
        roofline = {"bound": "fp64", "achieved": achieved, "peak": peaks["dfma_tflops"], "unit": "TFLOP/s",
                    "frac": achieved / peaks["dfma_tflops"], "traffic": prof.get("fp64_train_dram_bytes_per_launch"),
                    "kernel": "train_fp64_pipe (the trainer launch set: one launch per network shape, concurrent)",
                    "algorithmic_flop_per_step": flop, "kernel_ms_per_step": train_launch_ms,
                    "peak_source": peaks["source"] + " (DFMA)",
                    "peak_without_fma_tflops": peaks["dadd_tflops"],
                    "note": "exact-order parity forbids FMA contraction (the reference object code has none), so the "
                            "arithmetic ceiling is the DADD/DMUL rate (peak_without_fma_tflops); the 48-model "
                            "population is latency-bound on the blur nets' 20,000 sequential epochs (critical_path)",
                    "critical_path": critical_path(jobs, train_launch_ms, clock_mhz, "fp64")}
    else:
        roofline = {"bound": "fp32", "achieved": achieved, "peak": peaks["fp32_tflops"], "unit": "TFLOP/s",
                    "frac": achieved / peaks["fp32_tflops"], "traffic": prof.get("fp32_train_dram_bytes_per_launch"),
                    "kernel": "train_fp32_cta_kernel + train_fp32_kernel (trainer launch set)",
                    "algorithmic_flop_per_step": flop, "kernel_ms_per_step": train_launch_ms,
                    "peak_source": peaks["source"], "critical_path": critical_path(jobs, train_launch_ms, clock_mhz, "fp32")}

    e2e_s, h2d, d2h = time_e2e(E, eng, jobs, precision, args.steps)
    e2e_s = max_over_ranks(e2e_s)
    e2e = {"value": me_rank * world / e2e_s, "unit": "model-epochs/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * e2e_s, "steps": args.steps,
           "path": "lann_run_population: host datagen+split+NormStats+init -> H2D -> train/predict/eval -> D2H"}

    line = {
        "metric": "LANN model-epochs/sec", "value": value, "unit": "model-epochs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if precision == abi.FP64_EXACT else "f32",
        "data": "synthetic", "config": workload_config(args.precision),
        "parity": ("bit-identical (==) to the reference on this population at full length: every weight, every "
                   "epoch's loss, every metric (tests/test_gpu_full_length.py)") if precision == abi.FP64_EXACT else
                  "FP32 throughput mode: population-level parity only (DESIGN.md section 4)",
        "roofline": roofline, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        "wall_s_timed_region": wall_s, "failed_models": len(bad),
        "median_thr_mape": float(np.median([r.mape_thr for r in results])),
    }
    if not args.no_extras:
        ex = extras(E, eng, rank, world, barrier, max_over_ranks, args, flush, peaks)
        if rank == 0:
            line["extras"] = ex
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        secs, kind, cbad = cpu_reference_run(jobs, threads)
        # single-core rate: one prediction net and one blur net on one thread
        one = [next(j for j in jobs if j.epochs < max(x.epochs for x in jobs)), max(jobs, key=lambda j: j.epochs)]
        secs1, _, _ = cpu_reference_run(one, 1)
        line["cpu_baseline"] = {"value": me_rank / secs, "unit": "model-epochs/s", "cores": threads, "kind": kind,
                                "sample": f"the whole config-2 population (48 models, {me_rank} model-epochs) once, "
                                          f"one model per host thread task, {threads} threads",
                                "seconds": secs, "host": host_cpu_name(),
                                "single_core": {"value": popmod.model_epochs(one) / secs1, "unit": "model-epochs/s",
                                                "sample": "one H=8 prediction net + one 5-5 blur net on 1 thread"}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    pop.close()
    eng.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def extras(E, eng, rank, world, barrier, max_over_ranks, args, flush, peaks):
    """Secondary measurements (every rank participates where the work shards): config 2 in the
    FP32 throughput mode; config 1 (one LANN) latency; config 5 (the same 48 combinations as plain
    FFNNs, family nn, next to the LANNs); the config-3 seed x fold sweep SHARDED over the ranks
    (strong scaling: 61,440 models, cost-balanced contiguous slices, no collective); config-4
    variant selection with the candidate range split over the ranks."""
    from paper_2003_07497_b200 import sharding
    out = {}
    jobs = popmod.config2_jobs(root_seed=1 + rank)
    try:
        p32 = eng.prepare(jobs, abi.FP32)
        p32.run(1)
        barrier()
        dev_ms, train_ms, launches = time_population(eng, p32, args.steps, flush)
        dev_ms = max_over_ranks(dev_ms)
        flop = p32.flop
        p32.close()
        e2e_s, h2d, d2h = time_e2e(E, eng, jobs, abi.FP32, args.steps)
        e2e_s = max_over_ranks(e2e_s)
        tl = train_ms / args.steps
        me = popmod.model_epochs(jobs) * world
        out["config2_fp32"] = {
            "value": me * args.steps / (dev_ms / 1e3), "unit": "model-epochs/s", "dtype": "f32",
            "ms_per_step": dev_ms / args.steps, "steps": args.steps, "gpu_launches": launches,
            "e2e": {"value": me / e2e_s, "unit": "model-epochs/s", "ms_per_step": 1e3 * e2e_s,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "roofline": {"bound": "fp32", "achieved": flop / (tl / 1e3) / 1e12, "peak": peaks["fp32_tflops"],
                         "unit": "TFLOP/s", "frac": flop / (tl / 1e3) / 1e12 / peaks["fp32_tflops"],
                         "kernel_ms_per_step": tl, "critical_path": critical_path(jobs, tl, 1965.0, "fp32")},
            "parity": "population level (training is chaotic, per-model FP32 parity is undefined): over the whole "
                      "config-3 sweep (61,440 models, full length) the FP32 median held-out thr-MAPE is 0.0098 pp "
                      "from the reference's (FP64-exact sweep, bit-identical) -- within north_star's 0.1 pp "
                      "(tests/test_gpu_full_length.py::test_fp32_full_config3_population_within_0p1pp, "
                      "profiles/r02_cv_parity.json); on a 960-model subset 0.21 pp (too few samples); per-model "
                      "|delta| median 0.36 pp; forward 98.7% of predictions within 1e-5 relative "
                      "(tests/test_gpu_fp32.py)"}
    except Exception as ex:  # noqa: BLE001
        out["config2_fp32"] = {"error": str(ex)}
    if rank == 0:
        try:
            out["config1_single_lann"] = single_lann(E, eng, args)
        except Exception as ex:  # noqa: BLE001
            out["config1_single_lann"] = {"error": str(ex)}
        try:
            out["config5_lann_vs_ffnn"] = lann_vs_ffnn(eng)
        except Exception as ex:  # noqa: BLE001
            out["config5_lann_vs_ffnn"] = {"error": str(ex)}
    def config3_cv_summary(eng, sweep, res, cv_ens, rank, world):
        """Per-combination cross-validation statistics (lann_engine.h): on one GPU straight from the
        device pass; with N ranks the shards' results and ensemble scores are gathered on the host
        (gloo) and rank 0 computes the group statistics on its device (lann_cv_summarize)."""
        if world > 1:
            import torch.distributed as dist
            parts = [None] * world
            dist.all_gather_object(parts, ([bytes(r) for r in res], [bytes(e) for e in cv_ens]))
            res = [abi.JobResult.from_buffer_copy(b) for p in parts for b in p[0]]
            cv_ens = [abi.CvEnsemble.from_buffer_copy(b) for p in parts for b in p[1]]
        if rank != 0:
            return None
        groups = eng.cv_summarize(sweep, res, cv_ens)
        rows = [{"combo": i, "fold_mape_thr_median": g.fold_mape_thr.median,
                 "test_mape_mean": g.test_mape.mean, "test_mape_thr_mean": g.test_mape_thr.mean,
                 "test_mape_thr_median": g.test_mape_thr.median, "ensembles_ok": g.n_ensembles_ok}
                for i, g in enumerate(groups)]
        return {"groups": len(groups), "ensembles": len(cv_ens),
                "ensembles_ok": int(sum(g.n_ensembles_ok for g in groups)),
                # medians over seeds per combination (a diverging seed's exp() extrapolation makes the
                # per-combination means of the log-target blur nets heavy-tailed), then over combinations
                "median_over_combos_fold_mean_test_mape_thr": float(np.median([g.test_mape_thr.median for g in groups])),
                "mean_over_combos_fold_mean_test_mape_thr": float(np.mean([g.test_mape_thr.median for g in groups])),
                "median_over_combos_fold_thr_mape": float(np.median([g.fold_mape_thr.median for g in groups])),
                "definition": "per combination: held-out fold metrics over 256 seeds x 5 folds and the test-part "
                              "MAPE of each seed's fold-mean model ((p_0+...+p_4)/5), mean and median; computed "
                              "on the device inside the timed pass (include/lann_engine.h)",
                "per_combo": rows}

    n_seeds = int(os.environ.get("LANN_SWEEP_SEEDS", 256))

    def sweep(precision, family=abi.NNC, warm=True):
        """Config 3 (48 combos x n_seeds x 5 folds) through one prepared population per rank:
        contiguous cost-balanced shards, device time max over ranks, results and ensemble scores
        gathered on the host, the cross-validation summary on rank 0."""
        jobs = popmod.config3_jobs(root_seed=1, n_seeds=n_seeds, family=family)
        mine, _ = sharding.shard(jobs, rank, world)
        t0 = time.perf_counter()
        ps = eng.prepare(mine, precision)
        prep_s = time.perf_counter() - t0
        if warm:
            ps.run(1)  # warm-up (module load, first-touch)
        barrier()
        ps.run(1)
        ms = max_over_ranks(eng.last_device_ms)
        tms, flop = eng.last_train_ms, ps.flop
        st, res, _, _ = ps.fetch()
        _, cv_ens = ps.cv()  # this shard's fold-mean test scores (shard cuts never split an ensemble)
        ps.close()
        merged = sharding.gather_results(res, rank, world)
        thr = np.array([r[3] for r in merged]) if world > 1 else np.array([r.mape_thr for r in merged])
        return {"jobs": jobs, "mine": mine, "ms": ms, "tms": tms, "flop": flop, "prep_s": prep_s, "thr": thr,
                "failed": int(sum(1 for r in res if r.status)),
                "cv": config3_cv_summary(eng, jobs, res, cv_ens, rank, world)}

    note = (f"48 combos x {n_seeds} seeds x 5 folds; contiguous cost-balanced shards, one per rank, no "
            "data-path collective; max-over-ranks device time")
    s32 = None
    try:
        s32 = sweep(abi.FP32)
        me = popmod.model_epochs(s32["jobs"])
        tflops = s32["flop"] / (s32["tms"] / 1e3) / 1e12
        out["config3_sweep_fp32"] = {"models": len(s32["jobs"]), "model_epochs": me, "n_gpus": world,
                                     "scaling": "strong", "value": me / (s32["ms"] / 1e3), "unit": "model-epochs/s",
                                     "ms": s32["ms"], "dtype": "f32", "rank0_models": len(s32["mine"]),
                                     "rank0_train_tflops": tflops, "rank0_frac_of_fp32_peak": tflops / peaks["fp32_tflops"],
                                     "rank0_host_prepare_s": s32["prep_s"], "failed_models": s32["failed"],
                                     "median_fold_thr_mape": float(np.median(s32["thr"])),
                                     "cross_validation": s32["cv"], "note": note}
    except Exception as ex:  # noqa: BLE001
        out["config3_sweep_fp32"] = {"error": str(ex)}
    if os.environ.get("LANN_SWEEP_FP64", "1") == "1":
        try:  # the same sweep in the FP64 exact mode (bit-identical to the reference), one pass
            s64 = sweep(abi.FP64_EXACT, warm=False)
            me = popmod.model_epochs(s64["jobs"])
            med64 = float(np.median(s64["thr"]))
            tf64 = s64["flop"] / (s64["tms"] / 1e3) / 1e12
            out["config3_sweep_fp64"] = {
                "models": len(s64["jobs"]), "model_epochs": me, "n_gpus": world, "scaling": "strong",
                "value": me / (s64["ms"] / 1e3), "unit": "model-epochs/s", "ms": s64["ms"], "dtype": "f64", "steps": 1,
                "rank0_train_tflops": tf64, "rank0_frac_of_dfma_peak": tf64 / peaks["dfma_tflops"],
                "rank0_frac_of_no_fma_peak": tf64 / peaks["dadd_tflops"],
                "failed_models": s64["failed"], "median_fold_thr_mape": med64,
                "fp32_gap_pp": abs(med64 - float(np.median(s32["thr"]))) if s32 is not None else None,
                "parity": "bit-identical to the reference trainer (tests/test_gpu_full_length.py pins the 960-model "
                          "golden subset inside this sweep); fp32_gap_pp = |median held-out thr-MAPE FP32 - FP64| "
                          "over all models (north_star: 0.1 pp)",
                "cross_validation": None if s64["cv"] is None else
                {k: v for k, v in s64["cv"].items() if k != "per_combo"},
                "note": "one device pass (~10 s on one B200) after the config-2 FP64 runs loaded the kernels; " + note}
        except Exception as ex:  # noqa: BLE001
            out["config3_sweep_fp64"] = {"error": str(ex)}
    try:  # config 5 at scale: the same sweep with plain FFNNs (family nn, no complexity input), FP32
        snn = sweep(abi.FP32, family=abi.NN)
        me = popmod.model_epochs(snn["jobs"])
        row = {"models": len(snn["jobs"]), "dtype": "f32", "n_gpus": world,
               "ffnn_value": me / (snn["ms"] / 1e3), "unit": "model-epochs/s",
               "ffnn_median_fold_thr_mape": float(np.median(snn["thr"])), "ffnn_failed_models": snn["failed"]}
        if s32 is not None:
            row["lann_value"] = popmod.model_epochs(s32["jobs"]) / (s32["ms"] / 1e3)
            row["lann_median_fold_thr_mape"] = float(np.median(s32["thr"]))
            row["thr_mape_gap_pp"] = row["ffnn_median_fold_thr_mape"] - row["lann_median_fold_thr_mape"]
            if rank == 0 and s32["cv"] and snn["cv"]:
                lann = [g["test_mape_thr_median"] for g in s32["cv"]["per_combo"]]
                ffnn = [g["test_mape_thr_median"] for g in snn["cv"]["per_combo"]]
                row["fold_mean_test_thr_mape_median_over_combos"] = {"lann": float(np.median(lann)),
                                                                     "ffnn": float(np.median(ffnn))}
                row["combos_where_lann_is_better"] = int(sum(a < b for a, b in zip(lann, ffnn)))
        out["config5_at_scale"] = row
    except Exception as ex:  # noqa: BLE001
        out["config5_at_scale"] = {"error": str(ex)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:  # the reference CPU trainer on the stratified subset (every combo x 4 seeds x 5
            # folds = 960 models) on all host threads, extrapolated linearly in model-epochs
            sub = popmod.config3_jobs(root_seed=1, n_seeds=4)
            threads = os.cpu_count() or 1
            secs, kind, bad = cpu_reference_run(sub, threads)
            rate = popmod.model_epochs(sub) / secs
            full = popmod.model_epochs(popmod.config3_jobs(root_seed=1, n_seeds=n_seeds))
            out["config3_cpu_reference"] = {"value": rate, "unit": "model-epochs/s", "cores": threads, "kind": kind,
                                            "sample": "960 models (48 combos x 4 seeds x 5 folds), full length",
                                            "seconds": secs, "failed": len(bad),
                                            "extrapolated_full_sweep_s": full / rate}
        except Exception as ex:  # noqa: BLE001
            out["config3_cpu_reference"] = {"error": str(ex)}
    try:
        out["config4_selection"] = selection_extra(E, eng, rank, world, barrier, max_over_ranks)
    except Exception as ex:  # noqa: BLE001
        out["config4_selection"] = {"error": str(ex)}
    try:
        out["batched_predictor"] = predictor_extra(E, eng, rank, world, barrier, max_over_ranks)
    except Exception as ex:  # noqa: BLE001
        out["batched_predictor"] = {"error": str(ex)}
    return out


def predictor_extra(E, eng, rank, world, barrier, max_over_ranks, rows_per_model=1_000_000):
    """The general batched predictor (lann_predict: models::predict / predict_dataset,
    models.cpp:346-378): the 48 trained config-2 models x rows_per_model rows each (every model's
    250 held-out rows tiled), FP32 and FP64-exact. value = predictions/s of the predictor kernel
    with rows resident in HBM; e2e = the whole call from host rows (64 B/row H2D, 8 B/row D2H).
    Roofline: HBM, 76 algorithmic bytes per prediction (64-B row + 4-B model index + 8-B result)."""
    jobs = popmod.config2_jobs(root_seed=1)
    out = {"models": len(jobs), "rows_per_model": rows_per_model, "bytes_per_prediction": 76,
           "n_gpus": world, "scaling": "weak"}
    for prec, name in ((abi.FP32, "fp32"), (abi.FP64_EXACT, "fp64_exact")):
        pop = eng.prepare(jobs, prec)
        pop.run(1)
        st, res, params, _ = pop.fetch(want_params=True)
        norms = pop.norms()
        pop.close()
        models = [{"inputs": r.n_inputs, "h1": j.hidden[0], "h2": j.hidden[1] if j.n_hidden > 1 else 0,
                   "log_target": j.log_target, "params": p, "norm": nrm} for j, r, p, nrm in zip(jobs, res, params, norms)]
        # rows: each model's own feature distribution (its world at its data seed), tiled
        base = []
        for j in jobs:  # model inputs: the dataset's features (+ c for the augmented family)
            f, c, _, nf = E.build_dataset(j.world, j.data_seed, 500)
            if j.family == abi.NNC:
                f[:, nf] = c.astype(np.float64)
            base.append(f)
        n_rows = rows_per_model * len(jobs)
        # host buffers in pinned memory: the copies run at link speed (the call's own H2D / D2H)
        p_rows, p_rm, p_out = E.Pinned(n_rows * abi.ROW, np.float64), E.Pinned(n_rows, np.int32), \
            E.Pinned(n_rows, np.float64)
        rows = p_rows.array.reshape(n_rows, abi.ROW)
        rows[:] = np.concatenate([np.resize(b, (rows_per_model, abi.ROW)) for b in base])
        row_model = p_rm.array
        row_model[:] = np.repeat(np.arange(len(jobs), dtype=np.int32), rows_per_model)  # grouped by model
        eng.predict(models, rows[:1024], row_model[:1024], precision=prec)  # warm-up
        barrier()
        kms, wall = [], []
        for _ in range(3):
            t0 = time.perf_counter()
            eng.predict(models, rows, row_model, precision=prec, out=p_out.array)
            wall.append((time.perf_counter() - t0) * 1e3)
            kms.append(eng.last_train_ms)
        for b in (p_rows, p_rm, p_out):
            b.free()
        k = max_over_ranks(statistics.median(kms))
        w = max_over_ranks(statistics.median(wall))
        n = n_rows * world
        gbs = 76 * n_rows / (k / 1e3) / 1e9
        peak = hbm_peak()
        out[name] = {"value": n / (k / 1e3), "unit": "predictions/s", "kernel_ms": k,
                     "e2e": {"value": n / (w / 1e3), "unit": "predictions/s", "ms": w,
                             "h2d_bytes": 68 * n_rows, "d2h_bytes": 8 * n_rows,
                             "note": "lann_predict from pinned host rows: H2D of 68 B and D2H of 8 B per row inside"},
                     "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak[0], "unit": "GB/s",
                                  "frac": gbs / peak[0], "peak_source": peak[1]}}
    return out


def single_lann(E, eng, args):
    """Config 1: one LANN (the acceptance MM model 7-8-1, 250 training samples, 8000 epochs,
    seed 1) in the FP64 exact mode: device latency of the training pass and end-to-end latency
    through lann_run_population, next to the reference trainer on ONE host core (the reference
    trains one model on one thread)."""
    jobs = popmod.config1_jobs(seeds=(1,))
    p = eng.prepare(jobs, abi.FP64_EXACT)
    p.run(1)
    ms = []
    for _ in range(args.steps):
        p.run(1)
        ms.append(eng.last_device_ms)
    p.close()
    e2e_s, h2d, d2h = time_e2e(E, eng, jobs, abi.FP64_EXACT, args.steps)
    row = {"epochs": jobs[0].epochs, "device_ms": float(np.mean(ms)), "e2e_ms": 1e3 * e2e_s,
           "value": jobs[0].epochs / (np.mean(ms) / 1e3), "unit": "model-epochs/s", "dtype": "f64"}
    if not args.no_cpu_baseline:
        secs, kind, _ = cpu_reference_run(jobs, 1)
        row["cpu_reference_1core_ms"] = 1e3 * secs
        row["cpu_reference_kind"] = kind
        row["speedup_e2e_vs_1core"] = secs / e2e_s
    return row


def lann_vs_ffnn(eng):
    """Config 5: the config-2 population trained as LANNs (family nnc, complexity input) and as
    plain FFNNs (family nn, same worlds and seeds, no complexity input) in the FP64 exact mode:
    device throughput of each and the accuracy gap (median held-out thresholded MAPE)."""
    row = {}
    for name, fam in (("lann_nnc", abi.NNC), ("ffnn_nn", abi.NN)):
        jobs = popmod.config2_jobs(root_seed=1, family=fam)
        p = eng.prepare(jobs, abi.FP64_EXACT)
        p.run(1)
        p.run(1)
        ms = eng.last_device_ms
        st, res, _, _ = p.fetch()
        p.close()
        pred = [r.mape_thr for r, j in zip(res, jobs) if j.world.kind != abi.BLUR]
        row[name] = {"value": popmod.model_epochs(jobs) / (ms / 1e3), "unit": "model-epochs/s", "ms": ms, "dtype": "f64",
                     "median_thr_mape_all": float(np.median([r.mape_thr for r in res])),
                     "median_thr_mape_prediction_nets": float(np.median(pred)),
                     "failed": int(sum(1 for r in res if r.status))}
    row["thr_mape_gap_pp"] = row["ffnn_nn"]["median_thr_mape_all"] - row["lann_nnc"]["median_thr_mape_all"]
    return row


def selection_extra(E, eng, rank, world, barrier, max_over_ranks, n_cands=10_000_000):
    """Config 4: per kernel kind, n_cands counter-generated candidate shapes scored by its
    10 variant-hardware prediction models from the config-2 population, argmin per candidate;
    each rank scores a contiguous 1/world of the candidate range (candidate i is generated from
    derive_seed(seed, i), so the split changes nothing)."""
    jobs = popmod.config2_jobs(root_seed=1)
    pop = eng.prepare(jobs, abi.FP32)
    pop.run(1)
    st, res, params, _ = pop.fetch(want_params=True)
    norms = pop.norms()
    pop.close()
    lo = n_cands * rank // world
    hi = n_cands * (rank + 1) // world
    per_kind = []
    for kind in (abi.MM, abi.MV, abi.MC, abi.MP):
        idx = [i for i, j in enumerate(jobs) if j.world.kind == kind]
        models = [{"inputs": res[i].n_inputs, "h1": 8, "h2": 0, "log_target": 0, "params": params[i],
                   "norm": norms[i]} for i in idx]
        thd = [1 if jobs[i].world.hw_class == abi.HW_CPU else 0 for i in idx]
        per_kind.append((kind, models, thd))
    eng.select_variants(per_kind[0][1], per_kind[0][2], per_kind[0][0], 16, 7, lo, min(hi - lo, 1 << 16),
                        precision=abi.FP32)  # warm-up
    n_mine = hi - lo
    pin_idx, pin_score = E.Pinned(n_mine, np.uint8), E.Pinned(n_mine, np.float32)
    eng.select_variants_compact(per_kind[0][1], per_kind[0][2], per_kind[0][0], 16, 7, lo, min(n_mine, 1 << 16),
                                idx=pin_idx.array[: 1 << 16], score=pin_score.array[: 1 << 16])  # warm-up
    barrier()
    total_pred, kern_ms, e2e_ms, flop = 0, 0.0, 0.0, 0.0
    hist_total = []
    for kind, models, thd in per_kind:
        # the product call: uint8 argmin + float score per candidate into pinned host buffers,
        # copies overlapping the scoring (wall clock: kernels + D2H + host bookkeeping)
        t0 = time.perf_counter()
        _, _, hist = eng.select_variants_compact(models, thd, kind, 16, 7, lo, n_mine, idx=pin_idx.array,
                                                 score=pin_score.array)
        e2e_ms += (time.perf_counter() - t0) * 1e3
        # the scorer alone (one launch, winner histogram only): the kernel rate
        eng.select_variants_compact(models, thd, kind, 16, 7, lo, n_mine)
        kern_ms += eng.last_train_ms
        total_pred += n_cands * len(models)
        hist_total.append([int(h) for h in hist])
        # algorithmic FLOP per prediction: normalise 2I, forward 2IH + 2H, denormalise 2
        flop += sum(n_cands * (2 * m["inputs"] * 8 + 2 * 8 + 2 * m["inputs"] + 2) for m in models)
    # the legacy full-width call (int32 index + double score into pageable memory), for comparison
    t0 = time.perf_counter()
    for kind, models, thd in per_kind:
        eng.select_variants(models, thd, kind, 16, 7, lo, n_mine, precision=abi.FP32)
    legacy_ms = (time.perf_counter() - t0) * 1e3
    pin_idx.free()
    pin_score.free()
    kern_ms = max_over_ranks(kern_ms)
    e2e_ms = max_over_ranks(e2e_ms)
    legacy_ms = max_over_ranks(legacy_ms)
    out = {"candidates_per_kind": n_cands, "models_per_kind": 10, "predictions": total_pred, "n_gpus": world,
           "scaling": "strong", "value": total_pred / (kern_ms / 1e3), "unit": "predictions/s",
           "kernel_ms": kern_ms,
           "e2e": {"value": total_pred / (e2e_ms / 1e3), "unit": "predictions/s", "ms": e2e_ms,
                   "d2h_bytes": 5 * n_cands * 4, "path": "lann_select_variants_compact: uint8 argmin + float "
                   "score per candidate into pinned host buffers, chunked D2H overlapping the scoring"},
           "e2e_over_kernel": e2e_ms / kern_ms,
           "legacy_call_ms_int32_double_pageable": legacy_ms,
           "winner_histogram_rank0": hist_total,
           "algorithmic_tflops": flop / (kern_ms / 1e3) / 1e12,
           "flop_note": "per prediction 2*I*H + 2*H + 2*I + 2 with each model's own I (4..7), H = 8"}
    if rank == 0:
        try:
            out["cpu_reference"] = reference_predictions(jobs, res, params, norms)
        except Exception as ex:  # noqa: BLE001
            out["cpu_reference"] = {"error": str(ex)}
    return out


def reference_predictions(jobs, res, params, norms, n=1_000_000):
    """The reference's own models::predict_dataset (oracle/_ref) on the host cores for the MM
    kind's 10 variant models over a bounded sample of n candidate shapes (same feature ranges;
    timing does not depend on the values), one model per thread task."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Reference  # test infrastructure: the baseline leg only
    if not Reference.available():
        return {"unavailable": "oracle/_ref not built"}
    import concurrent.futures as cf
    ref = Reference()
    rng = np.random.default_rng(0)
    idx = [i for i, j in enumerate(jobs) if j.world.kind == abi.MM]
    threads = os.cpu_count() or 1
    dims = rng.integers(1, 1025, (n, 3)).astype(np.float64)
    feats = np.zeros((n, 8))
    feats[:, :3] = dims
    feats[:, 3] = 2.0 ** -rng.integers(0, 10, n)
    feats[:, 4] = 2.0 ** -rng.integers(0, 10, n)
    feats[:, 5] = rng.integers(1, 17, n)
    c = (dims[:, 0] * dims[:, 1] * dims[:, 2]).astype(np.uint64)

    feats_gpu = feats.copy()
    feats_gpu[:, 5] = 0.0  # GPU-class variants take no n_thd

    def one(i):
        thd = jobs[i].world.hw_class == abi.HW_CPU
        st, _ = ref.predict(abi.MM, thd, abi.NNC, (8,), params[i], norms[i], False, feats if thd else feats_gpu, c)
        return st

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(threads) as ex:
        sts = list(ex.map(one, idx))
    secs = time.perf_counter() - t0
    return {"value": n * len(idx) / secs, "unit": "predictions/s", "cores": threads, "kind": "reference",
            "sample": f"{n} MM candidate shapes x {len(idx)} variant models, models::predict_dataset, "
                      f"one model per host thread task", "seconds": secs, "failed": int(sum(1 for s in sts if s))}


if __name__ == "__main__":
    sys.exit(main())
