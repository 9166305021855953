"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol the headers declare, and its planner / schedule / weight manifest are
bit-exact against the oracle / synth."""
import os
import random
import re

import pytest

from oracle import planner as OP
from oracle import schedule as OS
from synth import configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def S():
    from paper_2509_04719_b200 import stadi
    return stadi


def _declared_symbols():
    names = set()
    for h in ("stadi.h", "stadi_kernels.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(stadi_[a-z0-9_]+)\s*\(", src))
    return names


def test_exports_every_declared_symbol(S):
    declared = _declared_symbols()
    assert "stadi_plan" in declared and "stadi_run" in declared
    for name in declared:
        assert hasattr(S.lib, name), name
    assert declared <= set(S.EXPORTS)
    assert S.lib.stadi_abi_version() == 3


def _oracle_plan(speed, mb, mw, P, rpu, flags, forced=None):
    return OP.plan(speed, mb, mw, P, rpu, flags=flags, forced_units=forced)


def test_plan_bit_exact_random(S):
    rng = random.Random(1234)
    n_checked = 0
    for _ in range(20000):
        n = rng.randint(1, 12)
        scale = rng.choice([1 << 8, 1 << 20, 1 << 40, (1 << 62)])
        speed = [rng.randint(1, scale) for _ in range(n)]
        if rng.random() < 0.3:   # ties and exact threshold hits
            speed = [rng.choice([4, 3, 1, 2, 8]) * (1 << rng.randint(0, 20)) for _ in range(n)]
        mb = rng.choice([10, 20, 50, 100, 11, 7])
        mw = rng.choice([1, 2, 4, mb])
        P = rng.randint(1, 160)
        rpu = rng.choice([1, 2, 4, 8])
        flags = rng.choice([0, 0, OP.NO_TA, OP.NO_SA, OP.NO_TA | OP.NO_SA, OP.SIZER_INTERVAL])
        try:
            ref = _oracle_plan(speed, mb, mw, P, rpu, flags)
        except OP.PlanError:
            with pytest.raises(S.StadiError) as e:
                S.plan(speed, mb, mw, P, rpu, flags=flags)
            assert e.value.status == 1
            continue
        got = S.plan(speed, mb, mw, P, rpu, flags=flags).to_dict()
        for k in ("tier", "steps", "units", "row_begin", "rows", "sync_period",
                  "n_exchange_rounds"):
            assert got[k] == ref[k], (k, speed, mb, mw, P, flags)
        assert got["makespan"] == (ref["makespan"].numerator, ref["makespan"].denominator)
        n_checked += 1
    assert n_checked > 10000


def test_plan_affine_bit_exact_random(S):
    """R30 affine sizer: C++ == oracle bit for bit (units, rows, integer makespan),
    including huge alpha / beta (128-bit products) and errors."""
    rng = random.Random(4321)
    n_checked = 0
    for _ in range(5000):
        n = rng.randint(1, 10)
        speed = [rng.randint(1, 1 << 20) for _ in range(n)]
        big = rng.choice([100, 1 << 20, 1 << 40])
        alpha = [rng.randint(0, big) for _ in range(n)]
        beta = [rng.randint(0 if rng.random() < 0.02 else 1, big) for _ in range(n)]
        mb = rng.choice([10, 20, 50, 100])
        mw = rng.choice([2, 4, mb])
        P = rng.randint(1, 128)
        flags = OP.SIZER_AFFINE | rng.choice([0, 0, OP.NO_TA, OP.SIZER_INTERVAL])
        try:
            ref = OP.plan(speed, mb, mw, P, 1, flags=flags, alpha=alpha, beta=beta)
        except OP.PlanError:
            with pytest.raises(S.StadiError):
                S.plan(speed, mb, mw, P, 1, flags=flags, alpha=alpha, beta=beta)
            continue
        got = S.plan(speed, mb, mw, P, 1, flags=flags, alpha=alpha, beta=beta).to_dict()
        for k in ("tier", "steps", "units", "row_begin", "rows"):
            assert got[k] == ref[k], (k, speed, alpha, beta, P, flags)
        assert got["makespan"] == (ref["makespan"].numerator, ref["makespan"].denominator)
        n_checked += 1
    assert n_checked > 3000
    with pytest.raises(S.StadiError):
        S.plan([1, 1], 10, 2, 8, flags=S.SIZER_AFFINE)


def test_plan_forced_and_errors(S):
    p = S.plan([10, 6], 100, 4, 32, flags=S.FORCE_UNITS, forced_units=[24, 8]).to_dict()
    assert p["units"] == [24, 8]
    for kw in [dict(speed=[0, 1], m_base=10, m_warmup=2, p_total=8),
               dict(speed=[1, 1], m_base=10, m_warmup=11, p_total=8)]:
        with pytest.raises(S.StadiError):
            S.plan(**kw)
    # R32: an odd K with a tier-2 GPU is planned with stride spf(K), not rejected
    p = S.plan([10, 6], 11, 2, 8).to_dict()
    assert p["sync_period"] == 3 and p["steps"] == [11, 5]
    with pytest.raises(S.StadiError):
        S.plan([1, 1], 10, 2, 8, a=(1, 4), b=(3, 4))


def test_schedule_bit_exact(S):
    rng = random.Random(99)
    for _ in range(500):
        n = rng.randint(1, 6)
        speed = [rng.randint(1, 1000) for _ in range(n)]
        mb = rng.choice([10, 20, 50, 100, 11, 27, 9, 51])
        mw = rng.choice([2, 4])
        try:
            ref = OP.plan(speed, mb, mw, 64, 2)
        except OP.PlanError:
            continue
        p = S.plan(speed, mb, mw, 64, 2)
        for r in range(n):
            want = [(s.m, s.t, s.t_prev, s.kind, s.read_ver, s.pub_ver)
                    for s in OS.schedule(ref, r)]
            assert S.schedule(p, r) == want


@pytest.mark.parametrize("name,kw,depth", [
    ("tiny_dit", {}, 0), ("dit_xl2", {}, 0), ("pixart_alpha", {}, 0),
    ("dit_xl2", dict(depth=2), 2), ("pixart_alpha", dict(depth=3), 3),
    ("tiny_unet", {}, 0), ("sd15", {}, 0), ("sdxl", {}, 0),
    ("sdxl", dict(tdepth=[0, 1, 1], mid_depth=1), 1), ("sd15", dict(latent_h=32), 0)])
def test_weight_manifest_matches_synth(S, name, kw, depth):
    cfg = configs.model(name, **kw)
    desc = S.model_desc(name, depth=depth)
    got = S.weight_manifest(desc)
    want = [(n, int(__import__("numpy").prod(shape))) for n, shape, _ in configs.manifest(cfg)]
    assert got == want


def test_cfg_split_plan_bit_exact(S):
    """R33 CFG batch split: C++ == oracle (pairs, pair plan expansion, branches)."""
    rng = random.Random(77)
    for _ in range(2000):
        n = rng.randint(2, 12)
        speed = [rng.randint(1, 1 << 20) for _ in range(n)]
        if rng.random() < 0.3:
            speed = [rng.choice([1, 2, 3, 4]) << 16 for _ in range(n)]
        mb = rng.choice([10, 20, 50, 11])
        flags = rng.choice([0, OP.NO_TA, OP.NO_SA, OP.SIZER_INTERVAL])
        P = rng.randint(1, 64)
        try:
            ref = OP.plan_cfg_split(speed, mb, 2, P, 2, flags=flags)
        except OP.PlanError:
            with pytest.raises(S.StadiError):
                S.plan(speed, mb, 2, P, 2, flags=flags | S.CFG_SPLIT)
            continue
        got = S.plan(speed, mb, 2, P, 2, flags=flags | S.CFG_SPLIT).to_dict()
        for k in ("tier", "steps", "units", "row_begin", "rows", "branch", "partner",
                  "sync_period", "n_exchange_rounds"):
            assert got[k] == ref[k], (k, speed, flags)
        assert got["cfg_split"] == 1
