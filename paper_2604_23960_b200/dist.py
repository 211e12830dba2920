"""Motion-index data parallelism.

Motions are independent (no state is shared between motions; the scene is
read-only), so G ranks -- one process per GPU -- each validate a contiguous block
of ceil(M/G) motions and one NCCL all-gather of the per-motion results (uint8
validity, uint32 FFC keys) assembles the whole batch on every rank.  The kernels
write straight into their rank's slice of the gathered buffer, so the
all-gather runs in place.  There is no other collective on the data path.
"""
from __future__ import annotations

import os


def shard(M: int, rank: int, world: int):
    """Contiguous block [lo, hi) of rank ``rank``; every rank gets ``per = ceil(M/G)``
    slots (the tail of the last rank is padding)."""
    per = (M + world - 1) // world
    lo = min(M, rank * per)
    hi = min(M, lo + per)
    return lo, hi, per


def init_from_env(backend: str = "nccl"):
    """(rank, world, local_rank) from torchrun's env; initialises the process group if world > 1."""
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend, rank=rank, world_size=world)
    return rank, world, local


def gather_inplace(buf, per: int, rank: int, world: int):
    """All-gather in place: ``buf`` holds world*per results and this rank has filled
    buf[rank*per:(rank+1)*per].  Returns buf (now complete on every rank)."""
    if world == 1:
        return buf
    import torch.distributed as dist
    dist.all_gather_into_tensor(buf, buf[rank * per:(rank + 1) * per])
    return buf


def pad_rows(x, per: int):
    """Pad a local shard (first dim) up to ``per`` rows by repeating row 0 (results discarded)."""
    import torch
    n = x.shape[0]
    if n == per:
        return x
    if n == 0:
        raise ValueError("empty shard cannot be padded")
    reps = torch.zeros(per - n, dtype=torch.long, device=x.device)
    return torch.cat([x, x[reps]], 0).contiguous()


def max_over_ranks(value: float, world: int, device=None) -> float:
    """Max of a float over ranks (timings are reported as the max over ranks)."""
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_ranks(value: float, world: int, device=None) -> list:
    """Every rank's value of a float (per-rank timings: load imbalance)."""
    if world == 1:
        return [value]
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    out = torch.empty(world, dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(out, t)
    return [float(x) for x in out.tolist()]


# --------------------------------------------------------------------------- time split
def time_window(T: int, rank: int, world: int, align: int = 32):
    """[t0, t1) of rank ``rank`` when one long horizon T is split across ``world`` ranks
    (boundaries aligned to ``align`` timesteps so no warp batch straddles two ranks)."""
    per = -(-T // world)
    per = -(-per // align) * align
    t0 = min(T, rank * per)
    return t0, min(T, t0 + per)


def allreduce_min_keys(keys, world: int):
    """Element-wise minimum over ranks of uint32 FFC keys held in an int32 tensor
    (0xFFFFFFFF = no conflict must compare as the largest key, so reduce in int64).
    Keys encode t * P + rank(i, j), so the minimum over disjoint time windows is the
    first conflict of the whole horizon."""
    if world == 1:
        return keys
    import torch
    import torch.distributed as dist
    k64 = keys.to(torch.int64) & 0xFFFFFFFF
    dist.all_reduce(k64, op=dist.ReduceOp.MIN)
    return (k64 - (k64 >= 2 ** 31).to(torch.int64) * 2 ** 32).to(torch.int32)


def allreduce_and_valid(valid, world: int):
    """MotVal over disjoint time windows: a motion is valid iff valid in every window."""
    if world == 1:
        return valid
    import torch.distributed as dist
    v = valid.clone()
    dist.all_reduce(v, op=dist.ReduceOp.MIN)
    return v
