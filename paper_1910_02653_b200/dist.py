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
    because the index field is global, so the result is the global (cost, idx) argmin.
    The max-batch keys ((2^31-1 - B_max) << idx_bits | idx) reduce the same way."""
    import torch
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        with torch.cuda.nvtx.range("cm_allreduce_min"):
            dist.all_reduce(best_key, op=dist.ReduceOp.MIN, group=group)
    return best_key


def gather_winner_masks(best_key, idx_bits: int, index_base: int, r_mask, s_mask, group=None):
    """Winners' R / S masks on every rank: after global_best, the rank owning
    budget b's winner (global index in [index_base, index_base + local count)) copies its
    rows into slot b of a zero [n_budget][2][n][W] int64 buffer; an all-reduce SUM (one
    contributor per slot) leaves every rank with all winners' masks, e.g. for cm_emit_plan.
    r_mask / s_mask: this rank's [local candidates][n][W] int64 tensors (round_and_evaluate
    with masks=True).  Slots of budgets with no feasible candidate stay zero."""
    import torch
    import torch.distributed as dist
    nb = best_key.numel()
    n, W = r_mask.shape[1], r_mask.shape[2]
    out = torch.zeros((nb, 2, n, W), dtype=torch.int64, device=r_mask.device)
    for b, k in enumerate(best_key.tolist()):
        if k == (1 << 63) - 1:
            continue
        idx = k & ((1 << idx_bits) - 1) if idx_bits else 0
        local = idx - index_base
        if 0 <= local < r_mask.shape[0]:
            out[b, 0] = r_mask[local]
            out[b, 1] = s_mask[local]
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        with torch.cuda.nvtx.range("cm_gather_winner_masks"):
            dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


def decode_keys(best_key, idx_bits: int):
    """Host decode of a key vector -> list of (cost, idx); (-1, -1) for 'none feasible'."""
    out = []
    for k in best_key.tolist():
        if k == (1 << 63) - 1:
            out.append((-1, -1))
        else:
            out.append((k >> idx_bits, k & ((1 << idx_bits) - 1) if idx_bits else 0))
    return out
