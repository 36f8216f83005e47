"""Multi-GPU partitioning of a model population (one process per GPU).

The population shards as independent models: there is no exchange step on the data path
(SURVEY.md 8(e)). Ranks get contiguous, cost-balanced slices of the job list (cost = epochs x
train rows x parameters), which keeps all seeds/folds of a combination together so their
training tile is staged once per CTA. Results are merged on the host in job order; the only
collectives are the timing barrier / max and an optional host-side gather of results.
"""
from __future__ import annotations

from typing import List, Sequence

from . import abi


def job_cost(j) -> float:
    n_train = int(round(j.count * j.train_fraction))
    if j.n_folds >= 2:
        n_train -= n_train // j.n_folds
    base = {abi.MM: 5, abi.MV: 3, abi.MC: 4, abi.MP: 5, abi.BLUR: 5}[j.world.kind]
    I = base + (1 if (j.world.hw_class == abi.HW_CPU and j.world.kind != abi.BLUR) else 0) + (1 if j.family == abi.NNC else 0)
    h = list(j.hidden)[: j.n_hidden]
    p = (I + 1) * h[0] + ((h[0] + 1) * h[1] + h[1] + 1 if len(h) > 1 else h[0] + 1)
    return float(j.epochs) * n_train * p


def _ensemble_key(j):
    """A job's cross-validation ensemble (include/lann_engine.h): every field except fold."""
    return (bytes(j.world), j.data_seed, j.count, j.train_fraction, j.n_folds, j.family, j.n_hidden,
            j.hidden[0], j.hidden[1], j.learning_rate, j.epochs, j.log_target, j.unconstrained, j.init_seed)


def shard_bounds(jobs: Sequence, world: int) -> List[int]:
    """Contiguous split points [b0=0, b1, ..., bW=len] balancing cumulative cost; each cut is then
    moved forward past adjacent jobs of one cross-validation ensemble (k-fold jobs that differ only
    in fold), so a shard scores its ensembles' fold-mean models itself (lann_shard_bounds)."""
    costs = [job_cost(j) for j in jobs]
    total = sum(costs)
    bounds, acc, r = [0], 0.0, 1
    for i, c in enumerate(costs):
        acc += c
        while r < world and acc >= total * r / world:
            bounds.append(i + 1)
            r += 1
    while len(bounds) < world:
        bounds.append(len(jobs))
    bounds.append(len(jobs))
    for w in range(1, world):
        c = max(bounds[w], bounds[w - 1])
        while 0 < c < len(jobs) and jobs[c - 1].n_folds >= 2 and jobs[c].n_folds >= 2 and \
                _ensemble_key(jobs[c - 1]) == _ensemble_key(jobs[c]):
            c += 1
        bounds[w] = c
    return bounds


def shard(jobs: Sequence, rank: int, world: int):
    """This rank's contiguous slice (and its offset in the global job list)."""
    b = shard_bounds(jobs, world)
    return list(jobs[b[rank]:b[rank + 1]]), b[rank]


def gather_results(results, rank: int, world: int):
    """Host-side merge of per-rank results into global job order (rank 0 gets the list)."""
    if world == 1:
        return list(results)
    import torch.distributed as dist
    out = [None] * world
    payload = [(r.status, r.final_loss, r.mape, r.mape_thr, r.rho, r.n_kept) for r in results]
    dist.all_gather_object(out, payload)
    merged = []
    for part in out:
        merged.extend(part)
    return merged
