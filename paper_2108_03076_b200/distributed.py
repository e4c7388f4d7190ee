"""Multi-GPU pricing, one process per GPU (torch.distributed; NCCL over
NVLink/NVSwitch for the plumbing).

The path index space is cut into the plan's deterministic chunks
(``Plan.chunking``, a function of the path count and output count only --
never of the GPU count).  With S = ceil(C / G), rank g prices the contiguous
chunk slice [g*S, min(C, (g+1)*S)) into its slot of a G*S-chunk partials
buffer, then ONE all-gather (``all_gather_into_tensor``, in place: each rank
sends only its S-chunk slice) assembles the buffer on every rank, and every
rank runs the same fixed-order combine -> identical bits for any G, the
analogue of the reference's thread-count invariance
(proj/src/pricing.cpp:268-286, proj/tests/test_pricing.cpp:110-117).  A
second tiny all_reduce(MIN) merges the device error words so every rank
raises the reference's error for the lowest failing path.

The same sharding runs inside one process over several GPUs through the C
ABI (``price(..., devices=[...])``, ``cltk_options.devices``: one NCCL
communicator per device list, ncclAllGather in a group).
"""
from __future__ import annotations

from typing import Sequence

import torch
import torch.distributed as dist

from . import Kernel, Plan


def slice_chunks(n_chunks: int, world: int) -> int:
    """Chunks per rank slot: S = ceil(C / G)."""
    return (n_chunks + world - 1) // world


def shard(n_chunks: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous chunk range of ``rank``: [r*S, min(C, (r+1)*S)); the ranges
    tile [0, n_chunks) (trailing ranks may be short or empty)."""
    s = slice_chunks(n_chunks, world)
    return min(n_chunks, rank * s), min(n_chunks, (rank + 1) * s)


_SIGN = -(2**63)


def _world(group=None) -> int:
    return dist.get_world_size(group) if dist.is_initialized() else 1


def gather_partials_(parts: torch.Tensor, group=None) -> torch.Tensor:
    """The single data-path collective: ``parts`` holds world equal slots
    (S chunks x outputs x 3 doubles each); this rank's slot is filled, the
    all-gather fills the others in place on every rank.  Over gloo (CPU tests)
    the collective runs on a host copy."""
    world = _world(group)
    if world <= 1:
        return parts
    rank = dist.get_rank(group)
    slot = parts.numel() // world
    if dist.get_backend(group) == "gloo" and parts.is_cuda:
        host = parts.cpu()
        outs = list(host.split(slot))
        dist.all_gather(outs, host[rank * slot:(rank + 1) * slot].clone(), group=group)
        parts.copy_(torch.cat(outs))
        return parts
    if parts.is_cuda:
        dist.all_gather_into_tensor(parts, parts[rank * slot:(rank + 1) * slot], group=group)
    else:
        outs = list(parts.split(slot))
        dist.all_gather(outs, parts[rank * slot:(rank + 1) * slot].clone(), group=group)
        parts.copy_(torch.cat(outs))
    return parts


def merge_error_word(word: int, device: torch.device | str = "cpu", group=None) -> int:
    """MIN over ranks of the unsigned device error words (path << 24 | site;
    2^64-1 = no error): the lowest failing path wins on every rank, as it
    would in a single-GPU run."""
    if _world(group) <= 1:
        return word
    signed = (word & (2**64 - 1)) - 2**64 if word >= 2**63 else word
    dev = "cpu" if dist.get_backend(group) == "gloo" else device
    t = torch.tensor([signed ^ _SIGN], dtype=torch.int64, device=dev)  # order-preserving
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return (int(t.item()) ^ _SIGN) & (2**64 - 1)


class DistributedPricer:
    """A compiled plan bound to this rank's GPU plus its partials buffer."""

    def __init__(self, kernels: Sequence[Kernel] | Kernel, model, days: Sequence[int] = (0,),
                 tenv: dict | None = None, device: int | None = None, rewrite: bool = True,
                 literals=None, rng: str = "philox", jit=False, group=None, fault: bool = False):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = _world(group)
        if device is None:
            device = torch.cuda.current_device()
        self.device = device
        self.plan = Plan(kernels, model, days, tenv, device=device, rewrite=rewrite,
                         literals=literals, rng=rng, jit=jit, fault=fault)
        self._parts = None

    def partials(self, paths: int) -> torch.Tensor:
        """World equal slots of S chunks (zeroed by ``launch``)."""
        _, nc = self.plan.chunking(paths)
        need = slice_chunks(nc, self.world) * self.world * max(1, self.plan.n_outputs) * 3
        if self._parts is None or self._parts.numel() < need:
            self._parts = torch.zeros(need, dtype=torch.float64, device=f"cuda:{self.device}")
        return self._parts[:need]

    def shard(self, paths: int) -> tuple[int, int]:
        _, nc = self.plan.chunking(paths)
        return shard(nc, self.rank, self.world)

    def launch_local(self, paths: int, seed: int, stream_ptr: int | None = None) -> torch.Tensor:
        """Price this rank's chunk slice into its slot (asynchronous)."""
        parts = self.partials(paths)
        c0, c1 = self.shard(paths)
        if stream_ptr is None:
            stream_ptr = torch.cuda.current_stream(self.device).cuda_stream
        self.plan.launch(paths, seed, c0, c1, parts.data_ptr(), stream_ptr)
        return parts

    def launch(self, paths: int, seed: int) -> torch.Tensor:
        """Price this rank's slice, then the all-gather (async on the current
        stream for NCCL).  Returns the assembled partials tensor."""
        return gather_partials_(self.launch_local(paths, seed), self.group)

    def finalize(self, paths: int, seed: int, parts: torch.Tensor) -> list[dict]:
        stream = torch.cuda.current_stream(self.device).cuda_stream
        if self.world > 1:
            w = merge_error_word(self.plan.error_word(stream), f"cuda:{self.device}", self.group)
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
