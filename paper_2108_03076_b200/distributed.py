"""Multi-GPU pricing: one process per GPU (torch.distributed, NCCL over
NVLink/NVSwitch for the plumbing).

The path index space is cut into the plan's deterministic chunks
(``Plan.chunking``, a function of the path count only); rank g prices the
contiguous chunk range [g*C/G, (g+1)*C/G) into its slice of a full-size
partials buffer (zeros elsewhere), then ONE ``all_reduce(SUM)`` over NVLink
assembles the buffer on every rank -- exact, since each element has a single
non-zero contributor -- and every rank runs the same fixed-order combine.
Prices are therefore bit-identical for any GPU count, the analogue of the
reference's thread-count invariance (proj/src/pricing.cpp:268-286,
proj/tests/test_pricing.cpp:110-117).  A second tiny all_reduce(MIN) merges
the device error words so every rank raises the reference's error for the
lowest failing path.
"""
from __future__ import annotations

from typing import Sequence

import torch
import torch.distributed as dist

from . import Kernel, Plan


def shard(n_chunks: int, rank: int, world: int) -> tuple[int, int]:
    return n_chunks * rank // world, n_chunks * (rank + 1) // world


class DistributedPricer:
    """A compiled plan bound to this rank's GPU plus its partials buffer."""

    def __init__(self, kernels: Sequence[Kernel] | Kernel, model, days: Sequence[int] = (0,),
                 tenv: dict | None = None, device: int | None = None, rewrite: bool = True):
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        if device is None:
            device = torch.cuda.current_device()
        self.device = device
        self.plan = Plan(kernels, model, days, tenv, device=device, rewrite=rewrite)
        self._parts = None
        self._paths = None

    def partials(self, paths: int) -> torch.Tensor:
        _, nc = self.plan.chunking(paths)
        need = nc * max(1, self.plan.n_outputs) * 3
        if self._parts is None or self._parts.numel() < need:
            self._parts = torch.zeros(need, dtype=torch.float64, device=f"cuda:{self.device}")
        return self._parts[:need]

    def launch(self, paths: int, seed: int) -> torch.Tensor:
        """Zero the buffer, price this rank's chunk range, all-reduce (async on
        the current stream).  Returns the partials tensor."""
        _, nc = self.plan.chunking(paths)
        parts = self.partials(paths)
        parts.zero_()
        c0, c1 = shard(nc, self.rank, self.world)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self.plan.launch(paths, seed, c0, c1, parts.data_ptr(), stream)
        if self.world > 1:
            dist.all_reduce(parts, op=dist.ReduceOp.SUM)
        return parts

    def finalize(self, paths: int, seed: int, parts: torch.Tensor) -> list[dict]:
        stream = torch.cuda.current_stream(self.device).cuda_stream
        if self.world > 1:
            word = torch.tensor([self.plan.error_word(stream)], dtype=torch.int64,
                                device=f"cuda:{self.device}")
            # error words are unsigned; flip the sign bit so signed MIN orders them
            word ^= torch.tensor([-(2**63)], dtype=torch.int64, device=word.device)
            dist.all_reduce(word, op=dist.ReduceOp.MIN)
            w = int(word.item()) ^ -(2**63)
            self.plan.set_error_word(w & (2**64 - 1), stream)
        return self.plan.finalize(paths, seed, parts.data_ptr(), stream)

    def price(self, paths: int, seed: int) -> list[dict]:
        return self.finalize(paths, seed, self.launch(paths, seed))


def price(kernel: Kernel | Sequence[Kernel], model, paths: int = 100000, seed: int = 0,
          days: Sequence[int] = (0,), tenv: dict | None = None) -> list[dict]:
    """priceAcrossTime over every rank of the default process group."""
    return DistributedPricer(kernel, model, days, tenv).price(paths, seed)
