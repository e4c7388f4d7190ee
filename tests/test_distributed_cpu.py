"""Multi-GPU host logic on CPU (gloo, world_size 2): deterministic chunk
sharding, the exact SUM merge of the partials buffer (the one data-path
collective) and the MIN merge of the device error words."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2108_03076_b200.distributed import merge_error_word, merge_partials_, shard


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
        full = torch.randn(n_chunks * n_out * 3, generator=g, dtype=torch.float64)
        full[::5] = -0.0  # signed zeros survive as zeros
        lo, hi = shard(n_chunks, rank, world)
        mine = torch.zeros_like(full)
        mine[lo * n_out * 3:hi * n_out * 3] = full[lo * n_out * 3:hi * n_out * 3]
        merge_partials_(mine)
        ok_parts = bool(torch.equal(mine, full + 0.0))
        words = [2**64 - 1, (12345 << 24) | 7]          # rank 0: none; rank 1: path 12345
        w = merge_error_word(words[rank % 2])
        words2 = [(2**38 << 24) | 3, (5 << 24) | 9]      # both fail: lowest path wins
        w2 = merge_error_word(words2[rank % 2])
        w3 = merge_error_word(2**64 - 1)                 # nobody fails
        out[rank] = (ok_parts, w, w2, w3)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_merges():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        ok_parts, w, w2, w3 = out[r]
        assert ok_parts
        assert w == (12345 << 24) | 7
        assert w2 == (5 << 24) | 9
        assert w3 == 2**64 - 1
