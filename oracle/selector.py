"""Algorithm 1 step by step, plus brute force (TEST INFRASTRUCTURE).

Inputs are per-layer costs t[pi], m[pi] of each enabled strategy at the current
(b, s) — the layers are homogeneous (R-31), so a plan's cost is
sum_l t[pi_l] and its memory sum_l m[pi_l] (Eqs. 5-6).
Feasibility is Eq. 6's strict "< OOM" (R-23), evaluated layer by
layer with the OOM short-circuit of PAPER.md:275.  Reading R-22: the plan also
needs one workspace, the largest of its own strategies' w[pi] (the transient
buffers are reused layer after layer), so a plan is feasible iff
sum_l m[pi_l] + max_l w[pi_l] < cap.  w = None (all zero) is the paper's Eq. 6.

Readings: R-17 the inner loop resets `strategies` to [P_i] x L for
every k (``literal=True`` keeps the listing's in-place mutation); R-18 the
early termination returns [P_0] x L at once; R-19 smoothing keeps the previous
plan when it is feasible and t_prev <= (1 + gamma) t_best; R-20
`pop_useless` = Pareto prune then sort by (t, m, enum id); R-24 ties keep the
first plan in generation order; least-memory fallback ties go to enum order.

Pins (tests/test_oracle_selector.py): SPEC.md:396 worked example [A,A,B];
SPEC.md:387 pop_useless example; SPEC.md:400 smoothing; SPEC.md:407 strict
equality; the R-17 / R-18 discriminators of SURVEY Q-17 / Q-18; |P| = 2 equals
brute force exactly; the result is the least-time member of the independently
enumerated candidate space.
"""
from __future__ import annotations

import itertools


class Counters:
    def __init__(self):
        self.layer_checks = 0     # per-layer memory-model lookups (OOM checks)
        self.plans = 0            # candidate plans generated
        self.cache_hits = 0


def _w(w, pi):
    return 0.0 if w is None else w[pi]


def pop_useless(t, m, enabled, w=None):
    """Pareto prune (drop pi if some pi' has t' <= t, m' <= m and w' <= w, one
    strict), then sort ascending by (t, m, id)."""
    keep = []
    for a in enabled:
        dom = any((t[b] <= t[a] and m[b] <= m[a] and _w(w, b) <= _w(w, a))
                  and (t[b] < t[a] or m[b] < m[a] or _w(w, b) < _w(w, a))
                  for b in enabled if b != a)
        if not dom:
            keep.append(a)
    return sorted(keep, key=lambda a: (t[a], m[a], a))


def feasible(plan, m, cap, ctr=None, w=None):
    acc = 0.0
    ws = 0.0
    for pi in plan:
        acc += m[pi]
        ws = max(ws, _w(w, pi))
        if ctr is not None:
            ctr.layer_checks += 1
        if acc + ws >= cap:       # short-circuit: the prefix already breaks Eq. 6
            return False
    return acc + ws < cap


def plan_time(plan, t):
    acc = 0.0
    for pi in plan:
        acc += t[pi]
    return acc


def plan_mem(plan, m):
    acc = 0.0
    for pi in plan:
        acc += m[pi]
    return acc


def candidates(L, order, m, cap, literal=False, ctr=None, w=None):
    """Lines 5-21 of Algorithm 1 without line 8's early exit: the generated
    feasible plans in generation order."""
    opts = []
    for i in range(len(order)):
        strategies = [order[i]] * L
        if ctr is not None:
            ctr.plans += 1
        if feasible(strategies, m, cap, ctr, w):
            opts.append(list(strategies))
        else:
            for k in range(i + 1, len(order)):
                if not literal:
                    strategies = [order[i]] * L
                for _ in range(L):
                    strategies.pop(0)
                    strategies.append(order[k])
                    if ctr is not None:
                        ctr.plans += 1
                    if feasible(strategies, m, cap, ctr, w):
                        opts.append(list(strategies))
    return opts


def alg1(L, t, m, enabled, cap, cache=None, key=None, literal=False, ctr=None, w=None):
    """Algorithm 1.  Returns (plan, infeasible_flag)."""
    if L <= 0:
        raise ValueError("L must be >= 1 (SPEC.md:394)")
    if not enabled:
        raise ValueError("no enabled strategy")
    if cache is not None and key in cache:                 # lines 2-4
        if ctr is not None:
            ctr.cache_hits += 1
        return list(cache[key][0]), cache[key][1]
    order = pop_useless(t, m, enabled, w)                  # line 1
    opts = []
    result = None
    for i in range(len(order)):                            # line 6
        strategies = [order[i]] * L                        # line 7
        if ctr is not None:
            ctr.plans += 1
        ok = feasible(strategies, m, cap, ctr, w)
        if i == 0 and ok:                                  # lines 8-10 (R-18)
            result = list(strategies)
            break
        if ok:                                             # lines 12-13
            opts.append(list(strategies))
        else:                                              # lines 14-21
            for k in range(i + 1, len(order)):
                if not literal:
                    strategies = [order[i]] * L            # R-17 reset
                for _ in range(L):
                    strategies.pop(0)
                    strategies.append(order[k])
                    if ctr is not None:
                        ctr.plans += 1
                    if feasible(strategies, m, cap, ctr, w):
                        opts.append(list(strategies))
    infeasible = False
    if result is None:
        if opts:                                           # lines 24-25
            best = None
            for p in opts:
                tp = plan_time(p, t)
                if best is None or tp < best[0]:
                    best = (tp, p)
            result = best[1]
        else:                                              # lines 26-27
            least = min(order, key=lambda a: (m[a], a))        # R-24 (per-layer m decides)
            result = [least] * L
            infeasible = True
    if cache is not None:                                  # line 29
        cache[key] = (list(result), infeasible)
    return result, infeasible


def smooth(plan, prev, t, m, cap, gamma, enabled=None, w=None):
    """Smoothing (R-19): retain prev if feasible and within gamma.
    A previous plan using a strategy that is no longer enabled is never retained."""
    if prev is None or len(prev) != len(plan):
        return plan, False
    if list(prev) == list(plan):
        return plan, False
    if enabled is not None and any(p not in enabled for p in prev):
        return plan, False
    if feasible(prev, m, cap, None, w) and plan_time(prev, t) <= (1.0 + gamma) * plan_time(plan, t):
        return list(prev), True
    return plan, False


def brute_force(L, t, m, enabled, cap, w=None):
    """Exhaustive argmin over all |P|^L assignments satisfying Eq. 6."""
    best = None
    for plan in itertools.product(sorted(enabled), repeat=L):
        if feasible(plan, m, cap, None, w):
            tp = plan_time(plan, t)
            if best is None or tp < best[0]:
                best = (tp, list(plan))
    return best


def multiset_best(L, t, m, enabled, cap, w=None):
    """Exact optimum for any L by enumerating strategy multisets (costs are
    permutation invariant for homogeneous layers): C(L+|P|-1, |P|-1) cases."""
    en = sorted(enabled)
    best = None
    for combo in itertools.combinations_with_replacement(en, L):
        if plan_mem(combo, m) + max(_w(w, p) for p in combo) < cap:
            tp = plan_time(combo, t)
            if best is None or tp < best[0]:
                best = (tp, list(combo))
    return best
