"""CPU, world_size 2 over gloo: the N>1 path of the population engine.

Ranks shard the config-3 job list (contiguous, cost-balanced, disjoint, exhaustive), prepare
their share on the host exactly as a single process would (datasets / tiles are deterministic
per job, independent of the rank), and merge results in global job order. The GPU data path
has no collective; only the timing barrier / max and this host-side gather use one."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2003_07497_b200 import abi
from paper_2003_07497_b200 import population as P
from paper_2003_07497_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    from oracle_lib import Oracle
    jobs = P.config3_jobs(root_seed=1, n_seeds=2, combos=None)[:60]
    for j in jobs:
        j.epochs = 20
    mine, off = sharding.shard(jobs, rank, world)
    o = Oracle()
    res = [o.run_job(j)[0] for j in mine]  # the host-side checker stands in for the device pass
    merged = sharding.gather_results(res, rank, world)
    ids = [None] * world
    dist.all_gather_object(ids, list(range(off, off + len(mine))))
    # timing reduction used by bench.py: MAX over ranks
    import torch
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        np.save(os.path.join(out_dir, "merged.npy"), np.array([m[3] for m in merged]))
        np.save(os.path.join(out_dir, "ids.npy"), np.concatenate([np.array(x, dtype=np.int64) for x in ids]))
        np.save(os.path.join(out_dir, "tmax.npy"), t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_matches_single_process(tmp_path, oracle):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    ids = np.load(tmp_path / "ids.npy")
    assert np.array_equal(ids, np.arange(60))  # disjoint + exhaustive, in order
    assert float(np.load(tmp_path / "tmax.npy")[0]) == 2.0
    jobs = P.config3_jobs(root_seed=1, n_seeds=2)[:60]
    for j in jobs:
        j.epochs = 20
    single = np.array([oracle.run_job(j)[0].mape_thr for j in jobs])
    assert np.array_equal(np.load(tmp_path / "merged.npy"), single)


def test_shard_bounds_balance():
    jobs = P.config3_jobs(root_seed=1, n_seeds=8)
    for world in (1, 2, 4, 8):
        b = sharding.shard_bounds(jobs, world)
        assert b[0] == 0 and b[-1] == len(jobs) and len(b) == world + 1
        assert all(b[i] <= b[i + 1] for i in range(world))
        costs = [sum(sharding.job_cost(j) for j in jobs[b[i]:b[i + 1]]) for i in range(world)]
        assert max(costs) <= 1.05 * sum(costs) / world + max(sharding.job_cost(j) for j in jobs)


def test_weak_scaling_populations_are_distinct():
    """bench.py N>1: rank r trains the config-2 population with root seed 1 + r."""
    a = P.config2_jobs(root_seed=1)
    b = P.config2_jobs(root_seed=2)
    assert [j.data_seed for j in a] != [j.data_seed for j in b]
    assert [bytes(j.world) for j in a] == [bytes(j.world) for j in b]
    assert all(j.world.kind == abi.BLUR for j in a[40:])


def test_engine_shard_bounds_match_the_python_rule():
    """lann_shard_bounds (the C++ cut behind lann_group_run_population and `perfsage sweep
    --devices`) == sharding.shard_bounds on the config-2 / config-3 / config-5 job lists."""
    from paper_2003_07497_b200 import engine as E

    lists = [P.config2_jobs(root_seed=1), P.config3_jobs(root_seed=1, n_seeds=4),
             P.config3_jobs(root_seed=1, n_seeds=2, family=abi.NN) + P.config3_jobs(root_seed=1, n_seeds=2)]
    for jobs in lists:
        for w in (1, 2, 3, 4, 8):
            b = E.shard_bounds(jobs, w)
            assert b == sharding.shard_bounds(jobs, w)
            assert b[0] == 0 and b[-1] == len(jobs) and all(x <= y for x, y in zip(b, b[1:]))
