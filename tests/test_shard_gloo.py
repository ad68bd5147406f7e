"""CPU, world_size 2 over gloo: the multi-rank host logic of the sharded search
(shard ranges + all-gather + lexicographic reduction) reproduces the full search.
Each rank's range scan uses the oracle here (no GPU); on B200 boxes bench.py runs
the same logic over NCCL with the engine."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, ids, window, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from common import problem
    from oracles import Oracle
    from paper_2511_00796_b200.shard import gather_winner, shard_range
    orc = Oracle(problem("c3_64gpu"))
    total = orc.train_space(ids)
    lo, hi = shard_range(total, rank, world)
    r = orc.constrained_search(ids, window, lo=lo, hi=hi)
    w = gather_winner(r["found"], r.get("cost", 0.0), r.get("rank", -1), r["feasible"])
    out[rank] = w
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_search_gloo(world):
    from common import problem
    from oracles import Oracle
    ids = list(range(0, 6)) + list(range(24, 30)) + list(range(48, 52))
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), ids, 4, out), nprocs=world, join=True)
    full = Oracle(problem("c3_64gpu")).constrained_search(ids, 4)
    for rank in range(world):
        cost, r, feas = out[rank]
        assert (cost, r, feas) == (full["cost"], full["rank"], full["feasible"])
