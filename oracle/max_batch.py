"""CPU ORACLE: the max-batch epilogue.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares no code with the CUDA path.

PAPER.md:498-511 (§6.3, Eq. 13): the largest batch B a schedule supports, with every M_i
replaced by B·M_i, subject to the cost constraint
    sum_t sum_i C_i R_{t,i} <= 2 sum_{v in G_fwd} C_i + sum_{v in G_bwd} C_i      (Eq. 13).
A fixed schedule's peak is affine in the activation sizes (SURVEY §8(c) invariant 8:
peak(B·M) - ovh = B·(peak(M) - ovh), the overhead M_input + 2 M_param held fixed -- DESIGN.md
reading R2), so for a candidate with cost within the limit
    B_max(c, b) = floor((b - ovh) / (peak_c - ovh))      (peak_c > ovh; capped at B_CAP)
is the largest B with peak(B·M) <= b.  Per budget the result is the candidate with the largest
B_max >= 1 (ties: lowest index), or none.
"""
from __future__ import annotations

B_CAP = (1 << 31) - 1


def b_max(peak: int, budget: int, ovh: int) -> int:
    """Largest B >= 0 with ovh + B (peak - ovh) <= budget (B_CAP when peak == ovh)."""
    if budget < ovh:
        return 0
    if peak <= ovh:
        return B_CAP
    return min(B_CAP, (budget - ovh) // (peak - ovh))


def max_batch_per_budget(peaks, costs, budgets, ovh: int, cost_limit: int, index_base: int = 0):
    """[(B_max, idx)] per budget; (0, -1) when no candidate within the cost limit fits B >= 1."""
    out = []
    for b in budgets:
        best = (0, -1)
        for c, (p, q) in enumerate(zip(peaks, costs)):
            if q > cost_limit:
                continue
            bm = b_max(int(p), int(b), ovh)
            if bm >= 1 and (bm > best[0] or (bm == best[0] and index_base + c < best[1])):
                best = (bm, index_base + c)
        out.append(best)
    return out
