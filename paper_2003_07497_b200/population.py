"""Population recipes for the BASELINE configs (host-side job lists, no compute).

* config 1: the acceptance-criterion-5 model (acceptance_main.cpp:283-328), one job per seed.
* config 2: the 48 kernel-variant-hardware combinations trained as one population,
  each with models::default_config (models.cpp:66-85): prediction nets {8}, lr 1e-2,
  8000 epochs; blur selection nets {5,5}, lr 1e-2, 20000 epochs, log target.
* config 3: 48 combos x S init seeds x 5-fold CV over each combo's training split.
* config 5: the same populations with family=nn (no complexity input).
"""
from __future__ import annotations

from . import abi
from .abi import make_job

MASK = (1 << 64) - 1


def splitmix64(state: int):
    """rng.hpp:10-15 -> (output, new state)"""
    state = (state + 0x9E3779B97F4A7C15) & MASK
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31), state


def derive_seed(root: int, stream: int) -> int:
    """rng.hpp:18-22"""
    s = (root ^ ((0x9E3779B97F4A7C15 * (stream + 1)) & MASK)) & MASK
    _, s = splitmix64(s)
    out, _ = splitmix64(s)
    return out


def default_model(world, family=abi.NNC, unconstrained=False):
    """models::default_config (models.cpp:66-85) -> (hidden, lr, epochs, log_target)."""
    if world.kind == abi.BLUR:
        hidden, lr, epochs, logt = (5, 5), 1e-2, 20000, True
    else:
        hidden, lr, epochs, logt = (8,), 1e-2, 8000, False
    if unconstrained:
        hidden = tuple(h * 8 for h in hidden)
    return hidden, lr, epochs, logt


def combo_worlds():
    """The 48 synthetic kernel-variant-hardware worlds (SURVEY 7 hard part 8), restated from the
    engine's table (csrc/domain.cpp:401-456, exported as lann_default_combos) so that job lists
    can be built without loading the engine library (the reference arm of bench.py must not map
    it); tests/test_host.py checks the two tables are identical. 4 kernels x {dense, sparse} x
    {3 CPU hosts with n_thd, 2 GPU-class black boxes without} = 40 prediction worlds (combo 0 is
    the acceptance world, acceptance_main.cpp:271-279), then 8 blur selection worlds."""
    kind_alpha = (3e-9, 2e-9, 1.5e-9, 1e-9)
    hws = ((abi.HW_CPU, 4, 1.0, 0.25, 0.75, 0.0), (abi.HW_CPU, 8, 0.7, 0.15, 0.85, 0.0),
           (abi.HW_CPU, 16, 1.3, 0.10, 0.90, 0.0), (abi.HW_GPU, 1, 0.02, 1.0, 0.0, 5e-6),
           (abi.HW_GPU, 1, 0.05, 1.0, 0.0, 2e-5))
    out = []
    for kind in range(4):
        for variant in range(2):
            for cls, threads, mult, g0, g1, beta in hws:
                out.append(abi.World(kind=kind, hw_class=cls, max_threads=threads, blur_lattice=0,
                                     alpha=kind_alpha[kind] * (2.5 if variant else 1.0) * mult, g0=g0, g1=g1,
                                     delta=0.9 if variant else 0.0, beta=beta, noise=0.02))
    blurs = ((0, 1.0e-9, 0.0, (3, 8, 7, 3), (0.05, 0.02, 0.03, 0.04)),
             (0, 0.7e-9, 0.0, (4, 7, 6, 2), (0.04, 0.03, 0.02, 0.05)),
             (0, 1.3e-9, 0.0, (2, 9, 8, 4), (0.06, 0.01, 0.04, 0.03)),
             (1, 1e-11, 1e-5, (2, 4, 4, 0), (0.20, 0.10, 0.10, 0.0)),
             (1, 2e-11, 2e-5, (3, 3, 5, 0), (0.15, 0.12, 0.08, 0.0)),
             (0, 2.0e-9, 0.0, (5, 6, 5, 3), (0.03, 0.05, 0.05, 0.02)),   # FFT stand-ins
             (0, 1.5e-9, 0.0, (6, 10, 9, 5), (0.02, 0.04, 0.06, 0.01)),
             (0, 0.9e-9, 0.0, (1, 5, 3, 1), (0.08, 0.02, 0.02, 0.06)))
    for lattice, alpha, beta, mu, kappa in blurs:
        w = abi.World(kind=abi.BLUR, hw_class=abi.HW_CPU, max_threads=1, blur_lattice=lattice, alpha=alpha,
                      g0=1.0, g1=0.0, delta=0.0, beta=beta, noise=0.02)
        for j in range(4):
            w.mu[j] = float(mu[j])
            w.kappa[j] = kappa[j]
        out.append(w)
    return out


def combo_seed(root_seed: int, combo: int) -> int:
    return derive_seed(root_seed, combo)


def config1_jobs(seeds=(1, 2, 3, 4, 5), family=abi.NNC):
    w = abi.acceptance_world()
    return [make_job(w, s, family=family) for s in seeds]


def config2_jobs(root_seed=1, family=abi.NNC, combos=None, epochs_scale=1.0):
    worlds = combos if combos is not None else combo_worlds()
    jobs = []
    for i, w in enumerate(worlds):
        hidden, lr, epochs, logt = default_model(w, family)
        ds = combo_seed(root_seed, i)
        jobs.append(make_job(w, ds, family=family, hidden=hidden, lr=lr,
                             epochs=max(1, int(epochs * epochs_scale)), log_target=logt, init_seed=ds))
    return jobs


def config3_jobs(root_seed=1, n_seeds=256, n_folds=5, family=abi.NNC, combos=None, seed_offset=0):
    """48 combos x n_seeds init seeds x n_folds folds; fold f holds out block f of the
    combo's 250-sample training split (contiguous blocks of the split permutation)."""
    worlds = combos if combos is not None else combo_worlds()
    jobs = []
    for i, w in enumerate(worlds):
        hidden, lr, epochs, logt = default_model(w, family)
        ds = combo_seed(root_seed, i)
        for s in range(seed_offset, seed_offset + n_seeds):
            init = derive_seed(ds, 1 + s)
            for f in range(n_folds):
                jobs.append(make_job(w, ds, n_folds=n_folds, fold=f, family=family, hidden=hidden, lr=lr,
                                     epochs=epochs, log_target=logt, init_seed=init))
    return jobs


def model_epochs(jobs) -> int:
    return int(sum(j.epochs for j in jobs))


def flop_per_model_epoch(n_inputs: int, hidden, n_train: int) -> int:
    """N * F_s + 14 P (2 FLOP per FMA; Adam 14 FLOP per parameter)."""
    if len(hidden) == 1:
        h = hidden[0]
        fs = 4 * n_inputs * h + 6 * h + 5
        p = (n_inputs + 1) * h + h + 1
    else:
        h1, h2 = hidden
        fs = 4 * n_inputs * h1 + 6 * h1 * h2 + 6 * h2 + h1 + 5
        p = (n_inputs + 1) * h1 + (h1 + 1) * h2 + h2 + 1
    return n_train * fs + 14 * p
