"""Multi-GPU plumbing: candidates shard across ranks by contiguous S* ranges (no
data-path collective); the single exchange is an all-reduce MIN of the packed
per-budget (cost << idx_bits | idx) keys.  torch.distributed
supplies the process group (NCCL over NVLink on GPUs, gloo in CPU tests)."""
from __future__ import annotations


def shard_range(n_sstar_total: int, rank: int, world: int):
    """Rank r owns S* [floor(r N / P), floor((r+1) N / P))."""
    lo = (rank * n_sstar_total) // world
    hi = ((rank + 1) * n_sstar_total) // world
    return lo, hi


def global_best(best_key, group=None):
    """In-place all-reduce MIN of the int64 keys; equal keys cannot come from two ranks
    because the index field is global, so the result is the global (cost, idx) argmin."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(best_key, op=dist.ReduceOp.MIN, group=group)
    return best_key


def decode_keys(best_key, idx_bits: int):
    """Host decode of a key vector -> list of (cost, idx); (-1, -1) for 'none feasible'."""
    out = []
    for k in best_key.tolist():
        if k == (1 << 63) - 1:
            out.append((-1, -1))
        else:
            out.append((k >> idx_bits, k & ((1 << idx_bits) - 1) if idx_bits else 0))
    return out
