"""Independent cross-checks for the oracle (TEST INFRASTRUCTURE ONLY; see
checkmate_oracle.py header for who may import this).

  generate_plan      Alg. 1 "Generate execution plan": row-major scan of
                     R with deallocations from FREE, virtual registers REGS[1..|V|].
  simulate_plan      Interpret a plan with explicit register bookkeeping.  Stage-boundary
                     semantics (SURVEY §8(c) invariant 6 and its caveat): at the start of
                     stage t the resident set is exactly S_t (values kept by constraint (3));
                     peak is recorded after each compute and before the deallocations that
                     follow it (Fig. 4 caption).  With drop_at_boundary=False
                     nothing is dropped between stages (SPEC.md:468-476 plain simulate).
  simulate_greedy    A set-based re-statement of the accounting, no FREE matrix: in stage t
                     start with S_t resident; compute R_t in topological order; after computing
                     v_k, release every value whose last use in the stage is v_k (a computed
                     user, or itself when no user is computed) unless it is kept for stage t+1.
  hoisted_plan       Alg. 1 plus the code motion of PAPER.md:328: a
                     checkpoint resident at the start of stage t (S_t) that no computation of
                     stage t uses and that is not kept for stage t+1 is deallocated at the start
                     of the stage instead of staying resident until the boundary.
  brute_force_min_R  Enumerate every R (lower triangular, R_{t,t} = 1) satisfying (2) and (3)
                     for a fixed S and return the cheapest (tiny n only).
"""
from __future__ import annotations

import itertools

import numpy as np


def generate_plan(inst, R, FREE):
    """Alg. 1.  Statements: ("compute", t, k, reg) or ("dealloc", t, reg, i)."""
    n = inst.n
    REGS = [-1] * (n + 1)
    r = 0
    P = []
    for t in range(1, n + 1):
        for k in range(1, n + 1):
            if R[t, k]:
                P.append(("compute", t, k, r))
                REGS[k] = r
                r += 1
            for i in inst.DEPS[k] + [k]:
                if FREE[(i, k)][t - 1]:
                    P.append(("dealloc", t, REGS[i], i))
    return P


def spurious_checkpoints(inst, R, S, t):
    """Checkpoints of stage t that are 'unused in a stage' and not kept:
    i in S_t, no k with R_{t,k} and i in DEPS(k), S_{t+1,i} = 0."""
    n = inst.n
    used = set()
    for k in range(1, n + 1):
        if R[t, k]:
            used.update(inst.DEPS[k])
    return [i for i in range(1, n + 1) if S[t, i] and i not in used and not S[t + 1, i]]


def hoisted_plan(inst, R, S, FREE):
    """Alg. 1 with the spurious checkpoints of every stage deallocated at its start.
    The register of such a checkpoint is the one of its last computation (REGS[i])."""
    n = inst.n
    REGS = [-1] * (n + 1)
    r = 0
    P = []
    for t in range(1, n + 1):
        for i in spurious_checkpoints(inst, R, S, t):
            P.append(("dealloc", t, REGS[i], i))
        for k in range(1, n + 1):
            if R[t, k]:
                P.append(("compute", t, k, r))
                REGS[k] = r
                r += 1
            for i in inst.DEPS[k] + [k]:
                if FREE[(i, k)][t - 1]:
                    P.append(("dealloc", t, REGS[i], i))
    return P


def simulate_plan(inst, plan, S, drop_at_boundary=True):
    """Returns (peak, cost).  Raises AssertionError on use of a non-resident value,
    double free, or a checkpoint that is not resident when its stage starts."""
    n = inst.n
    resident = {}                     # reg -> node
    holder = {}                       # node -> reg currently holding it
    stage = 0
    mem = inst.ovh
    peak = None
    cost = 0

    def begin_stage(t):
        nonlocal mem
        if t > 1:
            for i in range(1, n + 1):
                if S[t, i]:
                    assert i in holder and holder[i] in resident, \
                        f"checkpoint {i} not resident entering stage {t} (constraint (3))"
        if drop_at_boundary:
            for reg in list(resident):
                node = resident[reg]
                if not S[t, node]:
                    del resident[reg]
                    if holder.get(node) == reg:
                        del holder[node]
                    mem -= int(inst.M[node])

    for st in plan:
        t = st[1]
        while stage < t:
            stage += 1
            begin_stage(stage)
        if st[0] == "compute":
            _, _, k, reg = st
            for i in inst.DEPS[k]:
                assert i in holder and holder[i] in resident, f"stage {t}: v{k} needs v{i}"
            resident[reg] = k
            holder[k] = reg
            mem += int(inst.M[k])
            cost += int(inst.C[k])
            peak = mem if peak is None else max(peak, mem)
        else:
            _, _, reg, i = st
            assert reg in resident, f"stage {t}: double free / unknown register {reg}"
            node = resident.pop(reg)
            if holder.get(node) == reg:
                del holder[node]
            mem -= int(inst.M[node])
    return peak, cost


def simulate_greedy(inst, R, S):
    """Returns (peak, cost) from R, S alone (no FREE)."""
    n = inst.n
    peak = None
    cost = 0
    for t in range(1, n + 1):
        live = {i for i in range(1, n + 1) if S[t, i]}
        mem = inst.ovh + sum(int(inst.M[i]) for i in live)
        computed = [k for k in range(1, n + 1) if R[t, k]]
        for pos, k in enumerate(computed):
            assert all(i in live for i in inst.DEPS[k]), (t, k)
            live.add(k)
            mem += int(inst.M[k])
            cost += int(inst.C[k])
            peak = mem if peak is None else max(peak, mem)
            later = computed[pos + 1:]
            for v in sorted(set(inst.DEPS[k]) | {k}):
                if v not in live or S[t + 1, v]:
                    continue
                users_here = [j for j in inst.USERS[v] if R[t, j]]
                last_use = max(users_here) if users_here else v
                if last_use == k and not any(j in later for j in users_here):
                    live.discard(v)
                    mem -= int(inst.M[v])
    return peak, cost


def constraints_hold(inst, R, S) -> bool:
    n = inst.n
    for t in range(1, n + 1):
        for (i, j) in inst.E:                                  # (2)
            if R[t, j] and not (R[t, i] or S[t, i]):
                return False
        if t >= 2:
            for i in range(1, n + 1):                          # (3)
                if S[t, i] and not (R[t - 1, i] or S[t - 1, i]):
                    return False
        if not R[t, t]:                                        # (12a)
            return False
        if R[t, t + 1:].any() or S[t, t:].any():               # (12b), (12c)
            return False
    return True


def brute_force_min_R(inst, S):
    """Cheapest R (by sum C R, ties broken by fewest ones) satisfying (2), (3), (12a-c)."""
    n = inst.n
    free_pos = [(t, i) for t in range(1, n + 1) for i in range(1, t)]
    best = None
    for bits in itertools.product((False, True), repeat=len(free_pos)):
        R = np.zeros((n + 2, n + 1), bool)
        for t in range(1, n + 1):
            R[t, t] = True
        for (t, i), b in zip(free_pos, bits):
            R[t, i] = b
        if not constraints_hold(inst, R, S):
            continue
        key = (int((R[1:n + 1, 1:].astype(np.int64) * inst.C[1:]).sum()), int(R.sum()))
        if best is None or key < best[0]:
            best = (key, R.copy())
    return best[1]
