"""Pins for oracle/planner.py (Eq. 4 / Eq. 5) and oracle/schedule.py (Alg. 1).

Pinned against: hand-checkable golden cases (tests/golden/*.json, cited),
brute-force min-makespan enumeration, closed-form counts, L310's statement of
which occupancy pairs trigger temporal adaptation, and Theorem 2's grid
alignment.  No GPU.
"""
import itertools
import json
import os
import random
from fractions import Fraction

import pytest

from oracle import planner, schedule

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _gold("planner_appA.json")["cases"], ids=lambda c: c["name"])
def test_golden_cases(case):
    p = planner.plan(case["speed"], case["m_base"], case["m_warmup"], case["p_total"])
    assert p["steps"] == case["steps"]
    assert p["units"] == case["units"]
    q = planner.plan(case["speed"], case["m_base"], case["m_warmup"], case["p_total"],
                     flags=planner.SIZER_INTERVAL)
    assert q["units"] == case["units_interval"]


def _brute_min_makespan(speed, steps, p_total):
    """Enumerate every integer split (>=1 per included GPU) and return the
    minimal max_i M_i P_i / v_i — Eq. 5's objective "all GPUs finish ... within
    similar latency" (L198) made exact."""
    inc = [i for i in range(len(speed)) if steps[i] > 0]
    best = None
    for split in itertools.product(range(1, p_total + 1), repeat=len(inc)):
        if sum(split) != p_total:
            continue
        ms = max(Fraction(steps[i] * s, speed[i]) for i, s in zip(inc, split))
        best = ms if best is None or ms < best else best
    return best


def test_dhondt_is_min_makespan():
    rng = random.Random(7)
    for _ in range(400):
        n = rng.randint(1, 4)
        speed = [rng.randint(1, 1 << 16) for _ in range(n)]
        mb = rng.choice([10, 20, 50, 100])
        mw = rng.choice([2, 4])
        P = rng.randint(n, 12)
        try:
            p = planner.plan(speed, mb, mw, P)
        except planner.PlanError:
            continue
        assert p["makespan"] == _brute_min_makespan(speed, p["steps"], P)


def test_invariants_random():
    rng = random.Random(11)
    for _ in range(2000):
        n = rng.randint(1, 16)
        speed = [rng.randint(1, 1 << 40) for _ in range(n)]
        P = rng.randint(n, 256)
        for flags in (0, planner.NO_TA, planner.NO_SA, planner.NO_TA | planner.NO_SA,
                      planner.SIZER_INTERVAL):
            try:
                p = planner.plan(speed, 50, 4, P, rows_per_unit=2, flags=flags)
            except planner.PlanError:
                continue
            assert sum(p["units"]) == P
            for i in range(n):
                assert (p["tier"][i] == 0) == (p["units"][i] == 0)
                assert p["rows"][i] == 2 * p["units"][i]
            assert p["row_begin"][0] == 0
            for i in range(1, n):
                assert p["row_begin"][i] == p["row_begin"][i - 1] + p["rows"][i - 1]
            # the fastest GPU is always tier 1 (Eq. 4: a*v_max < v_max)
            assert p["tier"][speed.index(max(speed))] == 1
            if flags & planner.NO_TA:
                assert all(t == 1 for t in p["tier"])
            if flags & planner.NO_SA:
                u = [x for x in p["units"] if x]
                assert max(u) - min(u) <= 1
            # scale invariance: Eq. 4/5 depend only on speed ratios
            k = rng.randint(2, 1000)
            p2 = planner.plan([v * k for v in speed], 50, 4, P, rows_per_unit=2, flags=flags)
            assert p2["units"] == p["units"] and p2["tier"] == p["tier"]


def test_eq4_boundaries_exact():
    # R2: v = a*v_max exactly is NOT tier 1 (needs a*v_max < v); v = b*v_max is excluded.
    p = planner.plan([4, 3, 1], 100, 4, 8)
    assert p["tier"] == [1, 2, 0] and p["steps"] == [100, 52, 0]
    p = planner.plan([400, 301, 101], 100, 4, 8)
    assert p["tier"] == [1, 1, 2]


def test_l310_trigger_pattern():
    # "[0%, 20%] and [35%, 45%] ... load balancing is achieved solely
    # by adjusting the patch size"; the other Fig. 8 pairs trigger TA (Table III +TA).
    def speeds(occ):
        return [round((100 - o) * 65536 / 100) for o in occ]
    no_ta = [(0, 20), (35, 45)]
    ta = [(0, 40), (0, 60), (30, 50), (25, 55)]
    for occ in no_ta:
        assert 2 not in planner.plan(speeds(occ), 100, 4, 32)["tier"]
    for occ in ta:
        assert 2 in planner.plan(speeds(occ), 100, 4, 32)["tier"]


def test_eq4_m_i_value():
    # Eq. 4 second case: 1/2 M_base + 1/2 M_warmup (L183)
    p = planner.plan([10, 6], 100, 4, 32)
    assert p["steps"] == [100, 52]
    p = planner.plan([10, 6], 50, 4, 32)
    assert p["steps"] == [50, 27]


def test_eq5_continuous_consistency():
    # With divisible totals the integer split equals Eq. 5 exactly:
    # v/M = [1/10, 1/10, 1/5] -> P = [1/4, 1/4, 1/2] * 16 = [4, 4, 8].
    p = planner.plan([1, 1, 2], 10, 2, 16, flags=planner.NO_TA)
    assert p["units"] == [4, 4, 8]


def test_plan_errors():
    bad = [
        dict(speed=[], m_base=10, m_warmup=2, p_total=8),
        dict(speed=[0, 1], m_base=10, m_warmup=2, p_total=8),
        dict(speed=[1, 1], m_base=10, m_warmup=11, p_total=8),
        dict(speed=[1, 1], m_base=10, m_warmup=0, p_total=8),
        dict(speed=[1, 1, 1], m_base=10, m_warmup=2, p_total=2),
    ]
    for kw in bad:
        with pytest.raises(planner.PlanError):
            planner.plan(**kw)
    with pytest.raises(planner.PlanError):
        planner.plan([1, 1], 10, 2, 8, a=(1, 4), b=(3, 4))
    with pytest.raises(planner.PlanError):
        planner.plan([1, 1], 10, 2, 8, flags=planner.FORCE_UNITS, forced_units=[3, 4])


def test_forced_units():
    # Table II splits 24:8 / 16:16 / 8:24 of P_total = 32 (L294-L308)
    for split in ([24, 8], [16, 16], [8, 24]):
        p = planner.plan([10, 6], 100, 4, 32, flags=planner.FORCE_UNITS, forced_units=split)
        assert p["units"] == split


# ---------------------------------------------------------------- schedule
def test_schedule_c1_golden():
    g = _gold("schedule_C1.json")
    p = planner.plan([65536, 32768], 10, 2, 8)
    for r in (0, 1):
        got = [[s.m, s.t, s.t_prev, s.kind, s.read_ver, s.pub_ver]
               for s in schedule.schedule(p, r)]
        assert got == g[f"rank{r}"]


def test_fast_grid_leading_spacing():
    assert schedule.fast_grid(10) == [901, 801, 701, 601, 501, 401, 301, 201, 101, 1]
    assert schedule.fast_grid(50)[:3] == [981, 961, 941] and schedule.fast_grid(50)[-1] == 1
    assert schedule.fast_grid(20)[0] == 951


@pytest.mark.parametrize("mb,mw,n", [(10, 2, 2), (50, 4, 2), (100, 4, 2), (20, 4, 2),
                                     (11, 2, 3), (27, 2, 5), (51, 4, 47), (9, 2, 7)])
def test_schedule_counts_and_alignment(mb, mw, n):
    """Eq. 4 counts, exchange rounds and Thm 2 grid alignment for the slow stride n
    (2 for an even K = M_base - M_warmup; R32: smallest prime factor of an odd K)."""
    p = planner.plan([100, 60, 100, 30], mb, mw, 16)
    assert p["tier"] == [1, 2, 1, 2]
    assert p["sync_period"] == n == planner.slow_stride(mb, mw)
    assert (mb - mw) % n == 0
    fast = schedule.schedule(p, 0)
    slow = schedule.schedule(p, 1)
    # Eq. 4 step counts: tier 2 = M_warmup + K / n ((M_base + M_warmup) / 2 for n = 2)
    assert len(fast) == mb and len(slow) == mw + (mb - mw) // n == p["steps"][1]
    if n == 2:
        assert p["steps"][1] == (mb + mw) // 2
    # exchange rounds: M_warmup + K/n
    pubs = {s.pub_ver for s in fast if s.pub_ver >= 0}
    assert len(pubs) == mw + (mb - mw) // n == p["n_exchange_rounds"]
    # Thm 2 (L234-L238): slow grid is a subsample of the fast grid, both end at final
    fast_t = [s.t for s in fast]
    assert all(s.t in fast_t for s in slow)
    assert fast[-1].t_prev == slow[-1].t_prev == schedule.FINAL
    # every slow step spans exactly the n fast steps starting at the same t
    for s in slow:
        if s.kind == schedule.SLOW:
            i = fast_t.index(s.t)
            assert fast[i].kind == schedule.FAST_EVEN
            assert all(fast[i + q].kind == schedule.FAST_ODD for q in range(1, n))
            assert s.t_prev == fast[i + n - 1].t_prev
            assert s.read_ver == fast[i].read_ver and s.pub_ver == fast[i].pub_ver
    # non-publishing steps read the version the last publishing step published
    last = None
    for b in fast:
        if b.kind == schedule.FAST_ODD:
            assert b.pub_ver == schedule.NONE and b.read_ver == last
        elif b.pub_ver >= 0:
            last = b.pub_ver


def test_slow_stride_r32():
    """R32: n = 2 for even K, else the smallest prime factor of K (K = 1: n = 1)."""
    assert [planner.slow_stride(2 + k, 2) for k in range(0, 12)] == \
        [2, 1, 2, 3, 2, 5, 2, 7, 2, 3, 2, 11]
    assert planner.slow_stride(4 + 91, 4) == 7 and planner.slow_stride(4 + 121, 4) == 11
    for K in range(2, 300):                      # brute-force definition
        n = planner.slow_stride(K + 3, 3)
        if K % 2 == 0:
            assert n == 2
        else:
            assert K % n == 0 and all(n % d for d in range(2, n))
            assert all(K % d for d in range(2, n))
    # K = 1: no stride can skip a point: tier 2 runs every step, nobody is slow
    p = planner.plan([100, 60], 5, 4, 8)
    assert p["tier"] == [1, 2] and p["sync_period"] == 1 and p["steps"] == [5, 5]


def test_schedule_uniform_and_excluded():
    p = planner.plan([100, 90, 10], 10, 2, 8)        # third GPU excluded (v <= b v_max)
    assert p["tier"] == [1, 1, 0] and p["sync_period"] == 1
    assert schedule.schedule(p, 2) == []
    s = schedule.schedule(p, 0)
    assert [x.kind for x in s] == [schedule.WARMUP] * 2 + [schedule.UNIFORM] * 8
    assert all(x.read_ver == x.pub_ver - 1 for x in s[2:])
    assert p["n_exchange_rounds"] == 10


# ------------------------------------------------------------ R30 affine sizer
def _affine(speed, mb, mw, pt, alpha, beta):
    return planner.plan(speed, mb, mw, pt, 1, flags=planner.SIZER_AFFINE, alpha=alpha, beta=beta)


def test_affine_sizer_reduces_to_dhondt():
    """alpha = 0, beta_i = L / v_i (exact): the affine sizer is Eq. 5 / D'Hondt."""
    rng = random.Random(11)
    for _ in range(300):
        n = rng.randint(1, 6)
        speed = [rng.choice([1, 2, 3, 4, 5, 6, 8, 10, 12]) for _ in range(n)]
        L = 120 * 7 * 11
        beta = [L // v for v in speed]
        pt = rng.randint(n, 40)
        mb, mw = rng.choice([(10, 2), (20, 4), (50, 4)])
        a = _affine(speed, mb, mw, pt, [0] * n, beta)
        d = planner.plan(speed, mb, mw, pt, 1)
        assert a["units"] == d["units"], (speed, pt)


def test_affine_sizer_is_min_makespan_bruteforce():
    """Greedy == the minimum of max_i M_i (alpha_i + beta_i P_i) over every split
    with P_i >= 1 on the included GPUs (tiny inputs, exhaustive)."""
    rng = random.Random(5)
    for _ in range(150):
        n = rng.randint(1, 4)
        speed = [rng.randint(1, 9) for _ in range(n)]
        alpha = [rng.randint(0, 50) for _ in range(n)]
        beta = [rng.randint(1, 20) for _ in range(n)]
        pt = rng.randint(n, 9)
        p = _affine(speed, 10, 2, pt, alpha, beta)
        inc = [i for i in range(n) if p["tier"][i]]
        if len(inc) > pt:
            continue
        best = None
        for split in itertools.product(range(1, pt + 1), repeat=len(inc)):
            if sum(split) != pt:
                continue
            ms = max(p["steps"][i] * (alpha[i] + beta[i] * u) for i, u in zip(inc, split))
            best = ms if best is None else min(best, ms)
        assert p["makespan"] == best
        assert sum(p["units"]) == pt and all(p["units"][i] >= 1 for i in inc)


def test_affine_fixed_overhead_moves_units():
    """A fixed per-step overhead on a GPU never gives it more units (monotone),
    and with equal speeds a large one moves units to the other GPUs."""
    base = _affine([1, 1], 10, 10, 20, [0, 0], [10, 10])
    assert base["units"] == [10, 10]
    prev = 10
    for a0 in (0, 10, 40, 100, 400):
        u = _affine([1, 1], 10, 10, 20, [a0, 0], [10, 10])["units"][0]
        assert u <= prev
        prev = u
    assert prev < 10


def test_affine_errors():
    with pytest.raises(planner.PlanError):
        planner.plan([1, 1], 10, 2, 8, 1, flags=planner.SIZER_AFFINE)
    with pytest.raises(planner.PlanError):
        _affine([1, 1], 10, 2, 8, [0, 0], [1, 0])


# ------------------------------------------------------------ R33 CFG batch split
def test_cfg_split_pairing_bruteforce():
    """R33: consecutive GPUs in speed order are paired (the odd slowest one out is
    excluded), a pair runs at its slower member's speed, both members share the
    pair's tier / steps / band, the lower index computes branch 0."""
    import itertools
    rng = __import__("random").Random(5)
    for _ in range(300):
        n = rng.randint(2, 9)
        speed = [rng.randint(1, 100) for _ in range(n)]
        sp = planner.plan_cfg_split(speed, 10, 2, 16, 2)
        order = sorted(range(n), key=lambda i: (-speed[i], i))
        want = sorted(tuple(sorted(order[2 * k:2 * k + 2])) for k in range(n // 2))
        assert sorted(sp["pairs"]) == want
        if n % 2:
            assert sp["tier"][order[-1]] == 0 and sp["rows"][order[-1]] == 0
        pp = sp["pair_plan"]
        assert pp["n_gpus"] == n // 2
        for k, (i, j) in enumerate(sp["pairs"]):
            assert sp["branch"][i] == 0 and sp["branch"][j] == 1 and i < j
            assert sp["partner"][i] == j and sp["partner"][j] == i
            for key in ("tier", "steps", "rows", "row_begin"):
                assert sp[key][i] == sp[key][j] == pp[key][k]
        # the pair plan is the ordinary plan of the pairs' min speeds
        ref = planner.plan([min(speed[i], speed[j]) for i, j in sp["pairs"]], 10, 2, 16, 2)
        assert {k: ref[k] for k in ("tier", "steps", "units")} == \
            {k: pp[k] for k in ("tier", "steps", "units")}
        # pairing consecutive speeds maximises the slowest pair speed (brute force, n <= 6)
        if n <= 6 and n % 2 == 0:
            best = 0
            for perm in itertools.permutations(range(n)):
                best = max(best, min(min(speed[perm[2 * k]], speed[perm[2 * k + 1]])
                                     for k in range(n // 2)))
            assert min(min(speed[i], speed[j]) for i, j in sp["pairs"]) == best
    with pytest.raises(planner.PlanError):
        planner.plan_cfg_split([1], 10, 2, 8)
    with pytest.raises(planner.PlanError):
        planner.plan_cfg_split([1, 1], 10, 2, 8, flags=planner.FORCE_UNITS)
