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
    """Contiguous chunk range of ``rank``: the ranges tile [0, n_chunks)."""
    return n_chunks * rank // world, n_chunks * (rank + 1) // world


_SIGN = -(2**63)


def merge_partials_(parts: torch.Tensor, group=None) -> torch.Tensor:
    """The single data-path collective: every element of the full-size
    partials buffer has exactly one non-zero contributor (its chunk's owner),
    so the SUM all-reduce reproduces it exactly on every rank."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(parts, op=dist.ReduceOp.SUM, group=group)
    return parts


def merge_error_word(word: int, device: torch.device | str = "cpu", group=None) -> int:
    """MIN over ranks of the unsigned device error words (path << 24 | site;
    2^64-1 = no error): the lowest failing path wins on every rank, as it
    would in a single-GPU run."""
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return word
    signed = (word & (2**64 - 1)) - 2**64 if word >= 2**63 else word
    t = torch.tensor([signed ^ _SIGN], dtype=torch.int64, device=device)  # order-preserving
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return (int(t.item()) ^ _SIGN) & (2**64 - 1)


class DistributedPricer:
    """A compiled plan bound to this rank's GPU plus its partials buffer."""

    def __init__(self, kernels: Sequence[Kernel] | Kernel, model, days: Sequence[int] = (0,),
                 tenv: dict | None = None, device: int | None = None, rewrite: bool = True,
                 literals=None, rng: str = "philox", jit=False):
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        if device is None:
            device = torch.cuda.current_device()
        self.device = device
        self.plan = Plan(kernels, model, days, tenv, device=device, rewrite=rewrite,
                         literals=literals, rng=rng, jit=jit)
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
        return merge_partials_(parts)

    def finalize(self, paths: int, seed: int, parts: torch.Tensor) -> list[dict]:
        stream = torch.cuda.current_stream(self.device).cuda_stream
        if self.world > 1:
            w = merge_error_word(self.plan.error_word(stream), f"cuda:{self.device}")
            self.plan.set_error_word(w, stream)
        return self.plan.finalize(paths, seed, parts.data_ptr(), stream)

    def price(self, paths: int, seed: int) -> list[dict]:
        return self.finalize(paths, seed, self.launch(paths, seed))


def price(kernel: Kernel | Sequence[Kernel], model, paths: int = 100000, seed: int = 0,
          days: Sequence[int] = (0,), tenv: dict | None = None, literals=None,
          rng: str = "philox", jit=False) -> list[dict]:
    """priceAcrossTime over every rank of the default process group."""
    return DistributedPricer(kernel, model, days, tenv, literals=literals, rng=rng,
                             jit=jit).price(paths, seed)
