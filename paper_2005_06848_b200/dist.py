"""Multi-GPU plumbing (host side only): contiguous observation shards (
SPEC.md:397-405) and the ncclUniqueId bootstrap over torch.distributed.  The per-iteration
exchange itself — one ncclAllReduce of the (g*K+1)-double statistics vector — runs inside
libcfust (cfust_estep), not here."""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [j0, j1) of rank `rank`: contiguous blocks whose sizes differ by at most one."""
    if world < 1 or not (0 <= rank < world) or n < 0:
        raise ValueError("bad shard arguments")
    base, rem = divmod(n, world)
    j0 = rank * base + min(rank, rem)
    return j0, j0 + base + (1 if rank < rem else 0)


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
