"""Multi-GPU sharding for the batched path (one process per GPU).

The batch is embarrassingly parallel (batch.hpp:77-81: every state is
independent, bitwise equal to serial evaluation), so each rank takes the
contiguous shard [begin, end) of the global batch (vd_shard_range, the
partition rule of batch_eval, batch.hpp:109-119) and runs the kernels on it.
There is no data-path collective; torch.distributed is used only for the
barrier around the timed region, the max-over-ranks time reduction and the
optional result gather used by tests.
"""
import torch
import torch.distributed as dist

from . import shard_range


def rank_world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def local_shard(N):
    r, w = rank_world()
    return shard_range(N, w, r)


def max_over_ranks(value, device=None):
    """Max of a float across ranks (timing rule: the slowest rank defines the step)."""
    r, w = rank_world()
    if w == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local, N):
    """Concatenate per-rank (rows, K) shards into the global (N, K) array in
    rank order (validation only; not on the timed path)."""
    r, w = rank_world()
    if w == 1:
        return local
    parts = [None] * w
    dist.all_gather_object(parts, local.cpu() if torch.is_tensor(local) else local)
    out = torch.cat([torch.as_tensor(p) for p in parts], dim=0)
    assert out.shape[0] == N
    return out
