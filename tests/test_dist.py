"""CPU (gloo, world_size 2) tests of the ciphertext-sharded multi-GPU path:
partitioning, max-over-ranks timing and the gather to rank 0. The per-pair
compute here is the test oracle (this only exercises the host-side logic;
the GPU path is the same code with the CUDA library as compute)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2003_04510_b200.dist import shard

CFG = (30, 4, 10)


def test_shard_partition_is_contiguous_and_complete():
    for total in (0, 1, 7, 8, 64, 65):
        for world in (1, 2, 3, 4, 8):
            shards = [shard(total, r, world) for r in range(world)]
            assert sum(s.count for s in shards) == total
            pos = 0
            for s in shards:
                assert s.start == pos
                pos += s.count
            assert max(s.count for s in shards) - min(s.count for s in shards) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(total, n, q):
    from oracle_lib import random_poly

    rng = np.random.default_rng(123)
    evk = (random_poly(rng, n, 2 * q), random_poly(rng, n, 2 * q))
    pairs = [((random_poly(rng, n, q), random_poly(rng, n, q)),
              (random_poly(rng, n, q), random_poly(rng, n, q))) for _ in range(total)]
    return evk, pairs


def _worker(rank, world, port, total, q_out):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "tests")]
    import torch.distributed as dist

    from oracle_lib import Restated
    from paper_2003_04510_b200.dist import max_over_ranks, run_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Restated()
    log_p, depth, log_n = CFG
    q = log_p * depth
    n = 1 << log_n
    evk, pairs = _inputs(total, n, q)

    def compute(start, count):
        res = []
        for c1, c2 in pairs[start:start + count]:
            st, oa, ob = orc.he_mul(log_n, log_p, q, q, c1, c2, evk)
            assert st == 0
            res.append(orc.digest(q - log_p, n, oa, ob))
        return res

    out = run_sharded(total, rank, world, compute)
    slowest = max_over_ranks(float(rank + 1))
    if rank == 0:
        q_out.put((out, slowest))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [5, 4])
def test_gloo_two_ranks_match_single_process(total, restated):
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q_out)) for r in range(2)]
    for p in procs:
        p.start()
    out, slowest = q_out.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    log_p, depth, log_n = CFG
    q, n = log_p * depth, 1 << log_n
    evk, pairs = _inputs(total, n, q)
    want = []
    for c1, c2 in pairs:
        st, oa, ob = restated.he_mul(log_n, log_p, q, q, c1, c2, evk)
        want.append(restated.digest(q - log_p, n, oa, ob))
    assert out == want
    assert slowest == 2.0
