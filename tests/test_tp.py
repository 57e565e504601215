"""CPU: TP head-sharding host logic with a real 2-process gloo group —
shard geometry, rank-independent chunk keys (every rank derives the same
plan), the MIN agreement of delivered prefixes, max-over-ranks timing."""
import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def test_shard_geometry():
    from paper_2510_09665_b200.tp import head_range, shard_bpt
    assert [shard_bpt(4096, t) for t in (1, 2, 4, 8)] == [4096, 2048, 1024, 512]
    assert [head_range(8, 8, r) for r in range(8)] == [(r, r + 1) for r in range(8)]
    assert head_range(8, 2, 1) == (4, 8)
    with pytest.raises(ValueError):
        shard_bpt(4096, 3)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np

        import oracle
        from paper_2510_09665_b200.tp import agree_loaded, max_over_ranks, shard_bpt
        C = oracle.C()
        prompt = np.random.default_rng(7).integers(0, 128256, size=2000, dtype=np.uint32)
        keys = C.chunk_keys(prompt, 256, "llama-3.1-70b")  # same on every rank
        gathered = [None] * world
        dist.all_gather_object(gathered, [k.hex() for k in keys])
        # rank 1's tier lost a chunk: its safe prefix is shorter
        loaded = {5: 1999 if rank == 0 else 512, 6: 256}
        agreed = agree_loaded(loaded)
        t = max_over_ranks(1.5 + rank)
        q.put((rank, gathered[0] == gathered[1], agreed, t, shard_bpt(4096, world)))
    finally:
        dist.destroy_process_group()


def test_tp_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(60)
    for rank, same_keys, agreed, t, bpt in out:
        assert same_keys
        assert agreed == {5: 512, 6: 256}
        assert t == 2.5
        assert bpt == 2048
