"""Multi-GPU plumbing (host side only): one process per GPU, contiguous observation shards
(SPEC.md:397-405), the ncclUniqueId bootstrap over torch.distributed and the
max-over-ranks of device timings.  The per-iteration exchange itself — ONE ncclAllReduce of the
[statistics, l, underflow flag] vector — runs inside libcfust (cfust_estep / the iteration graph),
not here.  bench.py drives exactly these functions; tests/test_dist_gloo.py drives them with the
gloo backend on CPU (world_size 2)."""
from __future__ import annotations

import dataclasses
import os


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [j0, j1) of rank `rank`: contiguous blocks whose sizes differ by at most one."""
    if world < 1 or not (0 <= rank < world) or n < 0:
        raise ValueError("bad shard arguments")
    base, rem = divmod(n, world)
    j0 = rank * base + min(rank, rem)
    return j0, j0 + base + (1 if rank < rem else 0)


def env_rank() -> tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment (1 process when absent)."""
    r = int(os.environ.get("RANK", "0"))
    w = int(os.environ.get("WORLD_SIZE", "1"))
    lr = int(os.environ.get("LOCAL_RANK", str(r)))
    return r, w, lr


def broadcast_unique_id(dist, rank: int, device="cuda", make_id=None) -> bytes:
    """Rank 0 creates the 128-byte ncclUniqueId (libcfust's cfust_nccl_unique_id unless make_id
    is given) and broadcasts it over the default process group."""
    import torch
    buf = torch.zeros(128, dtype=torch.uint8, device=device)
    if rank == 0:
        if make_id is None:
            from . import nccl_unique_id
            make_id = nccl_unique_id
        raw = make_id()
        assert len(raw) == 128
        buf.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))
    dist.broadcast(buf, 0)
    return bytes(buf.cpu().numpy().tobytes())


def max_over_ranks(dist, value: float, device="cuda") -> float:
    """Device timings are reported as the max over ranks."""
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


@dataclasses.dataclass
class Ranks:
    """This process's place in the job and the communicator bootstrap for libcfust."""
    rank: int
    world: int
    local: int
    device: str          # torch device of the process-group tensors ("cuda" or "cpu")
    dist: object = None  # torch.distributed when world > 1

    def shard(self, n: int) -> tuple[int, int]:
        return shard_range(n, self.rank, self.world)

    def nccl_id(self, make_id=None) -> bytes | None:
        """A fresh ncclUniqueId shared by all ranks (None for one rank: no communicator)."""
        if self.world == 1:
            return None
        return broadcast_unique_id(self.dist, self.rank, self.device, make_id)

    def barrier(self):
        if self.device == "cuda":
            import torch
            torch.cuda.synchronize()
        if self.world > 1:
            self.dist.barrier()
        if self.device == "cuda":
            import torch
            torch.cuda.synchronize()

    def max(self, value: float) -> float:
        return max_over_ranks(self.dist, value, self.device) if self.world > 1 else float(value)

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def bootstrap(backend: str = "nccl") -> Ranks:
    """Join the torchrun job (env://, MASTER_ADDR 127.0.0.1 by the launcher) with `backend`
    ("nccl": one GPU per process, device = LOCAL_RANK; "gloo": CPU tests)."""
    rank, world, local = env_rank()
    device = "cuda" if backend == "nccl" else "cpu"
    if device == "cuda":
        import torch
        torch.cuda.set_device(local)
    d = None
    if world > 1:
        import torch.distributed as d
        d.init_process_group(backend, init_method="env://", rank=rank, world_size=world)
    return Ranks(rank, world, local, device, d)
