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


def combo_seed(root_seed: int, combo: int) -> int:
    return derive_seed(root_seed, combo)


def config1_jobs(seeds=(1, 2, 3, 4, 5), family=abi.NNC):
    w = abi.acceptance_world()
    return [make_job(w, s, family=family) for s in seeds]


def config2_jobs(root_seed=1, family=abi.NNC, combos=None, epochs_scale=1.0):
    from .engine import default_combos
    worlds = combos if combos is not None else default_combos()
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
    from .engine import default_combos
    worlds = combos if combos is not None else default_combos()
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
