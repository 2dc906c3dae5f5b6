"""Pins of the oracle's Alg. 2 and segment plan (reading C-2)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import topology as T


def _is_derangement(src, n):
    return sorted(src) == list(range(n)) and all(src[i] != i for i in range(n))


@pytest.mark.parametrize("n", [2, 3, 4, 5, 7, 8, 16, 33, 64, 100])
def test_every_topology_is_a_derangement(n):
    # P2: "every worker sends and receives exactly one copy" (load balance)
    for step in range(6):
        for seg in range(4):
            src = T.alg2(0xC0FFEE, step, seg, n)
            assert _is_derangement(src, n)
            send_to = T.inverse(src)
            assert all(src[send_to[r]] == r for r in range(n))


def test_n2_is_forced_swap_for_every_seed():
    # the unique derangement of two ranks
    for seed in (0, 1, 2**40 + 3, 2**64 - 1):
        for step in range(5):
            assert T.alg2(seed, step, 0, 2) == [1, 0]


def test_world_below_two_is_an_error():
    with pytest.raises(ValueError):
        T.alg2(0, 0, 0, 1)


def _exact_law(n):
    """Brute force: enumerate every branch of Alg. 2 with uniform rows (exact Fractions);
    restart on dead end = renormalise over the non-dead-end outcomes."""
    law, dead = {}, Fraction(0)

    def rec(i, avail, src, p):
        nonlocal dead
        if i == n:
            law[tuple(src)] = law.get(tuple(src), Fraction(0)) + p
            return
        cand = [r for r in avail if r != i]
        if not cand:
            dead += p
            return
        for c in cand:
            rec(i + 1, [r for r in avail if r != c], src + [c], p / len(cand))

    rec(0, list(range(n)), [], Fraction(1))
    ok = 1 - dead
    return {k: v / ok for k, v in law.items()}, dead


def test_exact_law_matches_golden():
    gold = json.load(open(os.path.join(GOLDEN, "alg2_exact_law.json")))
    for n in (3, 4):
        law, dead = _exact_law(n)
        want = {tuple(int(v) for v in k.split(",")): Fraction(p) for k, p in gold[str(n)].items()}
        assert law == want
        assert dead == Fraction(gold["dead_end_probability"][str(n)])
    assert _exact_law(5)[1] == Fraction(gold["dead_end_probability"]["5"])
    # every derangement reachable: !3=2, !4=9, !5=44
    assert [len(_exact_law(n)[0]) for n in (3, 4, 5)] == [2, 9, 44]


@pytest.mark.parametrize("n,draws,crit", [(3, 20000, 10.83), (4, 20000, 26.12)])
def test_oracle_follows_exact_law(n, draws, crit):
    # P3: chi^2 goodness of fit at p = 0.001 (df = #derangements - 1)
    law, _ = _exact_law(n)
    counts = {k: 0 for k in law}
    for t in range(draws // 8):
        for s in range(8):
            counts[tuple(T.alg2(11, t, s, n))] += 1
    chi2 = sum((counts[k] - draws * float(p)) ** 2 / (draws * float(p)) for k, p in law.items())
    assert chi2 < crit, (chi2, counts)


@pytest.mark.parametrize("n,expect", [(3, 1 / 3), (4, 5 / 31)])
def test_restart_rate(n, expect):
    # P4: restarts per accepted topology = p_dead / (1 - p_dead)
    N = 20000
    restarts = sum(T.alg2(3, t, s, n, return_attempts=True)[1] - 1 for t in range(N // 4) for s in range(4))
    rate = restarts / N
    sd = np.sqrt(expect * (1 + expect) / N)  # geometric count std
    assert abs(rate - expect) < 5 * sd


def test_determinism_and_segment_independence():
    # P5 + "different random network topologies for each segment"
    a = T.topology(42, 9, 16, 8)
    b = T.topology(42, 9, 16, 8)
    assert np.array_equal(a, b)
    assert len({tuple(r) for r in a}) > 1
    assert not np.array_equal(T.topology(42, 10, 16, 8), a)
    assert not np.array_equal(T.topology(43, 9, 16, 8), a)
    assert not np.array_equal(T.topology(42, 9, 16, 8, T.TAG_HIER), a)


def test_survey_prototype_goldens():
    gold = json.load(open(os.path.join(GOLDEN, "topology_seed0_n8.json")))
    for t, rows in gold["src"].items():
        assert T.topology(gold["seed"], int(t), gold["n"], len(rows), gold["tag"]).tolist() == rows


@pytest.mark.parametrize("d,k", [(1_000_000, 4), (11_689_512, 8), (25_557_032, 8), (25_557_032, 16),
                                 (100_000_000, 32), (64, 2), (33, 2), (1, 1), (97, 4)])
def test_segment_plan(d, k):
    b = T.segment_bounds(d, k)
    assert b[0] == 0 and b[-1] == d and len(b) == k + 1
    sizes = np.diff(b)
    assert np.all(sizes > 0)
    assert np.all(b[:-1] % 32 == 0)
    assert sizes.max() - sizes.min() <= 32 + (d % 32)


def test_segment_plan_config_sizes():
    # SURVEY.md §8(a) a1 sizes follow from reading C-2
    assert set(np.diff(T.segment_bounds(1_000_000, 4)).tolist()) == {249_984, 250_016}
    s = np.diff(T.segment_bounds(11_689_512, 8))
    assert s.min() == 1_461_184 and s.max() == 1_461_216


def test_segment_plan_rejects_too_many_segments():
    with pytest.raises(ValueError):
        T.segment_bounds(64, 3)
    with pytest.raises(ValueError):
        T.segment_bounds(100, 0)


def test_segment_of_columns():
    b = T.segment_bounds(1000, 4)
    cols = np.arange(1000)
    seg = T.segment_of_columns(b, cols)
    for s in range(4):
        assert np.all(seg[b[s]:b[s + 1]] == s)
