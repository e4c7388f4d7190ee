"""Multi-GPU host logic on CPU (gloo, world_size 2 and 3): deterministic chunk
sharding in equal slots, the in-place all-gather of the partials slots (the one
data-path collective) and the MIN merge of the device error words."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2108_03076_b200.distributed import gather_partials_, merge_error_word, shard, slice_chunks


def test_shards_tile_the_chunk_space():
    for n in (0, 1, 7, 31, 1000, 1 << 20):
        for world in (1, 2, 3, 4, 8):
            cover = []
            for r in range(world):
                lo, hi = shard(n, r, world)
                assert lo <= hi
                cover.extend(range(lo, hi)) if n < 5000 else None
                if r > 0:
                    assert shard(n, r - 1, world)[1] == lo
            assert shard(n, 0, world)[0] == 0 and shard(n, world - 1, world)[1] == n
            if n < 5000:
                assert cover == list(range(n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(7)
        n_chunks, n_out = 1001, 3
        slots = slice_chunks(n_chunks, world) * world
        full = torch.randn(slots * n_out * 3, generator=g, dtype=torch.float64)
        full[::5] = -0.0  # signed zeros are moved, not summed: bits survive
        lo, hi = shard(n_chunks, rank, world)
        mine = torch.full_like(full, float("nan"))  # other slots: garbage until gathered
        mine[lo * n_out * 3:hi * n_out * 3] = full[lo * n_out * 3:hi * n_out * 3]
        gather_partials_(mine)
        live = n_chunks * n_out * 3
        ok_parts = bool(torch.equal(mine[:live].view(torch.int64), full[:live].view(torch.int64)))
        words = [2**64 - 1, (12345 << 24) | 7, 2**64 - 1]  # only rank 1 fails: path 12345
        w = merge_error_word(words[rank])
        words2 = [(2**38 << 24) | 3, (5 << 24) | 9, (6 << 24) | 1]  # lowest path wins
        w2 = merge_error_word(words2[rank])
        w3 = merge_error_word(2**64 - 1)                 # nobody fails
        out[rank] = (ok_parts, w, w2, w3)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_world_merges(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        ok_parts, w, w2, w3 = out[r]
        assert ok_parts
        assert w == (12345 << 24) | 7
        assert w2 == (5 << 24) | 9
        assert w3 == 2**64 - 1


def test_shard_slots_are_equal_and_ordered():
    for n in (1, 2, 5, 999, 1000, 1001):
        for world in (1, 2, 3, 8):
            s = slice_chunks(n, world)
            for r in range(world):
                lo, hi = shard(n, r, world)
                assert lo == min(n, r * s) and hi == min(n, (r + 1) * s)
                assert hi - lo <= s
