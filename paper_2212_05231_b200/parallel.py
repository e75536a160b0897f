"""Ray-sharded data parallelism.

One process per GPU (torchrun / NCCL over NVLink).  Every rank draws the SAME global
ray batch from the shared seeded generator (so the N-GPU step equals the 1-GPU and
oracle steps) and keeps the rays r = rank, rank + N, rank + 2N, ... of it.  The global
batch is [foreground | background] (`scene_io.py:129-172`) and a background ray keeps
~17 samples against ~107 for a foreground ray, so contiguous slices would hand the
last rank all the cheap rays; the interleaved shard gives every rank the same
foreground/background mix and per-rank sample counts within ~0.1 % at 2^18 rays per
rank (`tests/test_parallel.py::test_interleaved_shards_balance_samples`).  With a
`scene_io.DeviceSampler` only the shard's picks go to the device and only its rays are
built.  The exchanges are:

  1. all-reduce(SUM) of the kept-sample count P after marching — the Eikonal mean
     divides by the global P (`trainer.py:229-235`);
  2. all-reduce(SUM) of the flat gradient prefix [MLP | tables[:lambda]] and of the
     fp64 step scalars (Huber sum, dL/ds_log, squared error, Eikonal sum).

Adam then runs replicated on identical reduced gradients, so parameters stay
bit-identical across ranks without a broadcast.  The helpers only use
torch.distributed, so the same code runs on `gloo` (CPU tests) and `nccl` (GPU).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import torch
import torch.distributed as dist


def shard_bounds(m: int, rank: int, world: int):
    """Contiguous [lo, hi) ray slice of rank `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(int(m), int(world))
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def shard_slice(m: int, rank: int, world: int) -> slice:
    """Rays rank, rank + world, ... of an m-ray global batch (interleaved shard)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return slice(rank, int(m), world)


def shard_size(m: int, rank: int, world: int) -> int:
    """Number of rays in `shard_slice(m, rank, world)`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return max(0, (int(m) - rank + world - 1) // world)


@dataclass
class DataParallel:
    rank: int = 0
    world: int = 1
    group: object = None

    @classmethod
    def from_env(cls):
        if dist.is_available() and dist.is_initialized():
            return cls(dist.get_rank(), dist.get_world_size(), None)
        return cls(0, 1, None)

    @property
    def active(self):
        return self.world > 1

    def shard(self, m):
        """This rank's interleaved slice of an m-ray global batch."""
        return shard_slice(m, self.rank, self.world)

    def shard_size(self, m):
        return shard_size(m, self.rank, self.world)

    def allreduce_(self, t: torch.Tensor):
        """In-place SUM all-reduce (no-op on one rank)."""
        if self.active:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def allreduce_count(self, local_count: int, device) -> int:
        if not self.active:
            return int(local_count)
        t = torch.tensor([int(local_count)], dtype=torch.int64, device=device)
        self.allreduce_(t)
        return int(t.item())

    def max_(self, t: torch.Tensor):
        if self.active:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t


def init_from_env(backend=None):
    """Initialise torch.distributed from torchrun's environment (127.0.0.1 rendezvous)."""
    if "RANK" not in os.environ or dist.is_initialized():
        return DataParallel.from_env()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group(backend=backend)
    return DataParallel.from_env()
