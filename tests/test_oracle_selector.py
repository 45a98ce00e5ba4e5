"""Pins for oracle/selector.py (Algorithm 1)."""
import itertools

import numpy as np
import pytest

from oracle import selector as A


def test_pop_useless_example():
    # {A:(1,10), B:(2,4), C:(3,5)} -> [A, B] (C dominated by B)
    t = {0: 1, 1: 2, 2: 3}
    m = {0: 10, 1: 4, 2: 5}
    assert A.pop_useless(t, m, [0, 1, 2]) == [0, 1]
    assert A.pop_useless(t, m, [2]) == [2]
    # duplicate costs: deterministic order by id
    assert A.pop_useless({0: 1, 1: 1}, {0: 1, 1: 1}, [1, 0]) == [0, 1]


def test_spec_worked_example():
    # A(1,10), B(2,4), L=3, cap 25 -> [A,A,B]
    t = {0: 1.0, 1: 2.0}
    m = {0: 10.0, 1: 4.0}
    plan, inf = A.alg1(3, t, m, [0, 1], 25.0)
    assert plan == [0, 0, 1] and not inf
    opts = A.candidates(3, [0, 1], m, 25.0)
    assert opts == [[0, 0, 1], [0, 1, 1], [1, 1, 1], [1, 1, 1]]


def test_early_termination_and_cache_counters():
    t = {0: 1.0, 1: 2.0, 2: 3.0}
    m = {0: 1.0, 1: 0.5, 2: 0.1}
    ctr = A.Counters()
    cache = {}
    L = 32
    plan, _ = A.alg1(L, t, m, [0, 1, 2], 1e9, cache=cache, key=(1, 4096), ctr=ctr)
    assert plan == [0] * L
    assert ctr.layer_checks == L and ctr.plans == 1          # O(L) best case
    ctr2 = A.Counters()
    plan2, _ = A.alg1(L, t, m, [0, 1, 2], 1e9, cache=cache, key=(1, 4096), ctr=ctr2)
    assert plan2 == plan and ctr2.layer_checks == 0 and ctr2.cache_hits == 1   # O(1)


def test_short_circuit_and_worst_case_bound():
    # OOM short-circuit: an infeasible uniform plan stops at the first failing prefix
    ctr = A.Counters()
    assert not A.feasible([0] * 10, {0: 3.0}, 7.0, ctr)
    assert ctr.layer_checks == 3
    # worst case O(|P|^2 L^2) checks
    rng = np.random.default_rng(0)
    for _ in range(50):
        k, L = 4, 16
        t = dict(enumerate(np.sort(rng.random(k))))
        m = dict(enumerate(np.sort(rng.random(k))[::-1]))
        ctr = A.Counters()
        A.alg1(L, t, m, list(range(k)), 0.3 * L, ctr=ctr)
        assert ctr.layer_checks <= k * k * L * L


def test_strict_inequality():
    # sum of memory exactly equal to capacity is infeasible (Eq. 6 "<")
    assert not A.feasible([0, 0], {0: 5.0}, 10.0)
    assert A.feasible([0, 0], {0: 5.0}, 10.0 + 1e-9)


def test_smoothing_example():
    # gamma = 0.05, prev 4.1 vs optimum 4.0 -> prev retained
    t = {0: 4.0, 1: 4.1}
    m = {0: 1.0, 1: 1.0}
    plan, kept = A.smooth([0], [1], t, m, 10.0, 0.05)
    assert plan == [1] and kept
    plan, kept = A.smooth([0], [1], {0: 4.0, 1: 4.3}, m, 10.0, 0.05)
    assert plan == [0] and not kept


def test_reset_reading_discriminator():
    # SURVEY Q-17: A(0,10), B(2.9,6), C(3,0), L=2, cap 11: reset -> [A,C] t=3,
    # literal in-place mutation -> [B,C] t=5.9
    t = {0: 0.0, 1: 2.9, 2: 3.0}
    m = {0: 10.0, 1: 6.0, 2: 0.0}
    assert A.alg1(2, t, m, [0, 1, 2], 11.0)[0] == [0, 2]
    assert A.alg1(2, t, m, [0, 1, 2], 11.0, literal=True)[0] == [1, 2]


def test_fallback_when_nothing_feasible():
    t = {0: 1.0, 1: 2.0}
    m = {0: 10.0, 1: 5.0}
    plan, inf = A.alg1(3, t, m, [0, 1], 1.0)
    assert plan == [1, 1, 1] and inf                # least-memory uniform
    assert A.brute_force(3, t, m, [0, 1], 1.0) is None


def test_two_strategies_equal_brute_force():
    # |P| = 2: Algorithm 1's prefix mixes cover every multiset -> optimal
    rng = np.random.default_rng(1)
    n_feas = 0
    for _ in range(500):
        L = int(rng.integers(1, 7))
        t = {0: float(rng.random()), 1: float(rng.random())}
        m = {0: float(rng.random()), 1: float(rng.random())}
        cap = float(rng.random() * L)
        plan, inf = A.alg1(L, t, m, [0, 1], cap)
        bf = A.brute_force(L, t, m, [0, 1], cap)
        if bf is None:
            assert inf
            continue
        n_feas += 1
        assert abs(A.plan_time(plan, t) - bf[0]) < 1e-12
    assert n_feas > 100


def test_candidate_space_optimality_and_gap():
    # result == least-time member of the enumerated candidate space;
    # brute force <= Alg. 1 (gap reported, not bounded)
    rng = np.random.default_rng(2)
    gaps = 0
    for _ in range(300):
        k = int(rng.integers(1, 6))
        L = int(rng.integers(1, 7))
        t = {i: float(rng.random()) for i in range(k)}
        m = {i: float(rng.random()) for i in range(k)}
        cap = float(rng.random() * L * 0.8 + 0.05)
        plan, inf = A.alg1(L, t, m, list(range(k)), cap)
        order = A.pop_useless(t, m, list(range(k)))
        opts = A.candidates(L, order, m, cap)
        bf = A.brute_force(L, t, m, list(range(k)), cap)
        if inf:
            assert not opts
            continue
        if A.feasible([order[0]] * L, m, cap):
            assert plan == [order[0]] * L
        else:
            best = min(opts, key=lambda p: A.plan_time(p, t))
            assert A.plan_time(plan, t) == A.plan_time(best, t)
        assert bf[0] <= A.plan_time(plan, t) + 1e-12
        gaps += bf[0] < A.plan_time(plan, t) - 1e-12
    # multiset search is exact: equals brute force
    for _ in range(100):
        k, L = 3, int(rng.integers(1, 6))
        t = {i: float(rng.random()) for i in range(k)}
        m = {i: float(rng.random()) for i in range(k)}
        cap = float(rng.random() * L)
        bf = A.brute_force(L, t, m, [0, 1, 2], cap)
        ms = A.multiset_best(L, t, m, [0, 1, 2], cap)
        assert (bf is None) == (ms is None)
        if bf:
            assert abs(bf[0] - ms[0]) < 1e-12


def test_heuristic_gap_example():
    # SURVEY: A(0,10), B(1,6), C(3,0), L=3, cap 16.5 -> Alg. 1 t=5 vs optimum [A,B,C] t=4
    t = {0: 0.0, 1: 1.0, 2: 3.0}
    m = {0: 10.0, 1: 6.0, 2: 0.0}
    plan, _ = A.alg1(3, t, m, [0, 1, 2], 16.5)
    assert A.plan_time(plan, t) == 5.0
    assert A.brute_force(3, t, m, [0, 1, 2], 16.5)[0] == 4.0


def test_workspace_reading_two_strategies_equal_brute_force():
    # R-22: one workspace per plan (max over its strategies).  Feasibility stays
    # permutation invariant, so |P| = 2 prefix mixes still cover every multiset
    rng = np.random.default_rng(11)
    n_feas = 0
    for _ in range(500):
        L = int(rng.integers(1, 7))
        t = {0: float(rng.random()), 1: float(rng.random())}
        m = {0: float(rng.random()), 1: float(rng.random())}
        w = {0: float(rng.random()), 1: float(rng.random())}
        cap = float(rng.random() * L + 0.5)
        plan, inf = A.alg1(L, t, m, [0, 1], cap, w=w)
        bf = A.brute_force(L, t, m, [0, 1], cap, w=w)
        ms = A.multiset_best(L, t, m, [0, 1], cap, w=w)
        assert (bf is None) == (ms is None)
        if bf is None:
            assert inf
            continue
        n_feas += 1
        assert abs(A.plan_time(plan, t) - bf[0]) < 1e-12 and abs(ms[0] - bf[0]) < 1e-12
        assert A.plan_mem(plan, m) + max(w[p] for p in plan) < cap
    assert n_feas > 100


def test_workspace_reading_example():
    # A fast strategy with a huge workspace (UZ-like) must not shrink the budget of
    # plans that do not use it: T (t 1, m 4, w 1), U (t 1.1, m 4.5, w 10), M (t 2, m 2, w 1)
    t, m, w = {0: 1.0, 1: 1.1, 2: 2.0}, {0: 4.0, 1: 4.5, 2: 2.0}, {0: 1.0, 1: 10.0, 2: 1.0}
    # cap 13: [T,T,T] = 12 + 1 = 13 (not < 13); [T,T,M] = 10 + 1 < 13 -> feasible
    plan, inf = A.alg1(3, t, m, [0, 1, 2], 13.0, w=w)
    assert not inf and sorted(plan) == [0, 0, 2]
    # the enabled-max reading (cap - max w = 3) would have found nothing feasible
    plan2, inf2 = A.alg1(3, t, m, [0, 1, 2], 13.0 - 10.0)
    assert inf2
