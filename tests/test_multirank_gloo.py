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


def _fake_outputs(cells, per_cell=3, K=(40, 6144, 1056)):
    """A dense output layout for the given cells with deterministic per-CB words
    (a function of (cell, CB) only) -- stands in for the decoder's outputs."""
    import numpy as np
    from paper_1905_01141_b200 import crn
    n = len(cells) * per_cell
    d = np.zeros(n, crn.DESC_DTYPE)
    d["K"] = [K[i % len(K)] for i in range(n)]
    nw = (d["K"].astype(np.int64) + 31) // 32
    d["bit_off"] = np.concatenate([[0], np.cumsum(nw)[:-1]])
    cb_cell = np.repeat(np.array(cells, np.int32), per_cell)
    words = np.zeros(int(nw.sum()), np.uint32)
    ok = np.zeros(n, np.uint8)
    for i in range(n):
        rng = np.random.default_rng(int(cb_cell[i]) * 1000 + i % per_cell)
        words[d["bit_off"][i]:d["bit_off"][i] + nw[i]] = rng.integers(0, 2**32, nw[i], dtype=np.uint32)
        ok[i] = (cb_cell[i] + i % per_cell) % 2
    return d, cb_cell, words, ok


def _digest_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cells = shard.cells_for_rank(rank, world, 10)
    local = shard.cell_digests(*_fake_outputs(cells))
    merged = shard.gather_digests(local, dist)
    q.put((rank, merged, shard.combined_digest(merged)))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_cell_digests_do_not_depend_on_rank_count():
    """bench.py's per-cell output digests: every rank digests the cells it
    decoded, the gather gives all ranks the union, and the combined digest over
    10 cells is the same at world size 1, 2 and 3 (SPEC.md:290 determinism
    evidence for the strong split; SURVEY.md §8(e) test line)."""
    one = shard.cell_digests(*_fake_outputs(list(range(10))))
    ref = shard.combined_digest(one)
    assert len(one) == 10
    for world in (2, 3):
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = 29600 + world * 7 + os.getpid() % 500
        ps = [ctx.Process(target=_digest_worker, args=(r, world, port, q)) for r in range(world)]
        for p in ps:
            p.start()
        res = [q.get(timeout=120) for _ in ps]
        for p in ps:
            p.join(timeout=60)
            assert p.exitcode == 0
        for _, merged, comb in res:
            assert merged == one and comb == ref
    # a flipped word in one CB changes exactly its cell's digest
    d, cc, w, ok = _fake_outputs(list(range(10)))
    w[int(d["bit_off"][7])] ^= 1
    two = shard.cell_digests(d, cc, w, ok)
    assert [c for c in one if one[c] != two[c]] == [int(cc[7])]
    assert shard.combined_digest(two) != ref
