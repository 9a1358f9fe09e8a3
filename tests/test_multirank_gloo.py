"""N>1 host logic on CPU with the gloo backend (world_size 2): cell sharding
partitions the batch, each rank's generated shard is byte-identical to the
same cells of the single-rank batch (SPEC.md:290 determinism), and the
counter / time reductions are SUM / MAX."""
import os

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1905_01141_b200 import shard
from paper_1905_01141_b200 import workload as wlmod


def test_cells_partition():
    for n in (1, 100, 256):
        for w in (1, 2, 3, 4, 8):
            got = sum((shard.cells_for_rank(r, w, n) for r in range(w)), [])
            assert got == list(range(n))
            sizes = [len(shard.cells_for_rank(r, w, n)) for r in range(w)]
            assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cells = shard.cells_for_rank(rank, world, 100)
    wl = wlmod.make_workload(3, seed=5, cells=cells, scale=0.2)
    bits = sum(int(p.sum()) for p in wl.payload)
    c, t = shard.reduce_counters([wl.n_tb, bits, int(wl.tbs.sum()), 0, rank + 1], 10.0 * (rank + 1), dist)
    q.put((rank, cells, [p.numpy().tobytes() for p in wl.payload], wl.tb_ebn0_db.tolist(), c, t))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_shard_invariance_and_reductions():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=120) for _ in ps], key=lambda x: x[0])
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = wlmod.make_workload(3, seed=5, scale=0.2)
    pay = [p.numpy().tobytes() for p in full.payload]
    merged = res[0][2] + res[1][2]
    assert merged == pay
    assert res[0][3] + res[1][3] == full.tb_ebn0_db.tolist()
    for r in res:
        c, t = r[4], r[5]
        assert c["n_cb"] == full.n_tb and c["info_bits"] == int(full.tbs.sum())
        assert c["counted_ops"] == 3 and t == 20.0
