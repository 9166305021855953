"""Oracle planner: Temporal Adaptation (Eq. 4) + Spatial Adaptation (Eq. 5).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md L179-185 (§III-C, Eq. 4):
    M_i = M_base                         if a*v_max <  v_i <= v_max
    M_i = 1/2 M_base + 1/2 M_warmup      if b*v_max <  v_i <= a*v_max
    (excluded)                           if v_i <= b*v_max
PAPER.md L187-198 (§III-D, Eq. 5):
    P_i = (v_i/M_i) / sum_j (v_j/M_j) * P_total
Alg. 1 L114-119 apply them per GPU.  L284: M_base=100, M_warmup=4,
P_total=32, a=0.75, b=0.25.

Readings:
  R2  Eq. 4 boundaries as printed (v <= b*v_max is excluded), exact
      rational comparisons.
  R3  (round 1: (M_base - M_warmup) must be even with a tier-2 GPU; superseded by R32)
  R32 tier-2 stride n: K = M_base - M_warmup post-warmup intervals; n = 2 when K is
      even (Eq. 4: M_warmup + K/2 = (M_base + M_warmup)/2 steps), else the smallest
      prime factor of K, so the slow grid still lands on every n-th
      fast-grid point (Thm 2 with n M_i = M, L234-L238) and the "lowest common
      multiple of inference step sizes" (L185) is n; K = 1: n = 1 (no reduction
      possible: tier 2 runs every step).  Tier-2 steps = M_warmup + K / n.
  R4  "LCM-minimising": tier 2 runs stride 2 after warmup; sync_period =
      lcm of post-warmup strides (1 or 2).
  R5  Eq. 5 integerised by the D'Hondt divisor method on weights v_i/M_i,
      >= 1 unit per included GPU, ties to the lowest rank.
  R6  one unit = rows_per_unit latent rows.
  R7  Eq. 5 uses M_i of Eq. 4 (flag SIZER_INTERVAL: per-round step counts).
  R8  rank order, top to bottom.
  R30 (flag SIZER_AFFINE; L333: "the single-step delay no longer maintains a
      linear relationship with the patch size due to some fixed overhead")
      per-step latency of GPU i on P units modelled as alpha_i + beta_i P
      (integer time units); Eq. 5 is replaced by minimising the makespan
      max_i M_i (alpha_i + beta_i P_i): one unit per included GPU, then each
      further unit to argmin_i M_i (alpha_i + beta_i (P_i + 1)), ties to the
      lowest rank.  With alpha = 0 and beta_i = L / v_i this is R5's D'Hondt.
  R33 (flag CFG_SPLIT; DistriFusion's "batch splitting" of the CFG batch, L284 names
      it as an acceleration technique): the GPUs are PAIRED and each
      member of a pair computes one CFG branch (B = 1) of the pair's band; the two
      eps bands are combined every step, so a pair advances at its slower member's
      speed.  Pairing: GPUs sorted by speed (descending, ties to the lower index),
      consecutive ones paired; an odd GPU out (the slowest) is excluded.  Eq. 4/5
      then plan the pairs with pair speed min(v_a, v_b); the pairs' bands go top to
      bottom in the order of each pair's lower GPU index (R8).  Both members take the
      pair's tier, steps and rows; the lower index computes branch 0 (uncond).
      FORCE_UNITS / SIZER_AFFINE (per-GPU inputs) are not combined with it.
Written with plain Python integers and fractions.Fraction (exact).
"""
from __future__ import annotations

from fractions import Fraction

NO_TA = 1
NO_SA = 2
SIZER_INTERVAL = 4
FORCE_UNITS = 8
SIZER_AFFINE = 16
CFG_SPLIT = 32


class PlanError(ValueError):
    """Invalid parameters (maps to STADI_EINVAL at the C boundary)."""


def tiers(speed, a=(3, 4), b=(1, 4), flags=0):
    """Eq. 4 tier per GPU: 1 = M_base, 2 = reduced, 0 = excluded (R2)."""
    vmax = max(speed)
    out = []
    for v in speed:
        if flags & NO_TA:
            out.append(1)
        elif Fraction(v) > Fraction(a[0], a[1]) * vmax:       # a*v_max < v_i
            out.append(1)
        elif Fraction(v) > Fraction(b[0], b[1]) * vmax:       # b*v_max < v_i <= a*v_max
            out.append(2)
        else:                                                 # v_i <= b*v_max
            out.append(0)
    return out


def smallest_prime_factor(k):
    """Smallest prime p dividing k >= 2 (trial division)."""
    p = 2
    while p * p <= k:
        if k % p == 0:
            return p
        p += 1
    return k


def slow_stride(m_base, m_warmup):
    """R32: the tier-2 DDIM stride n for K = M_base - M_warmup post-warmup intervals."""
    K = m_base - m_warmup
    if K % 2 == 0:
        return 2
    return 1 if K == 1 else smallest_prime_factor(K)


def steps_of(tier, m_base, m_warmup):
    """Eq. 4 right-hand sides (L183): tier 2 = M_warmup + K/n (= (M_base+M_warmup)/2
    for n = 2, R32)."""
    if tier == 1:
        return m_base
    if tier == 2:
        return m_warmup + Fraction(m_base - m_warmup, slow_stride(m_base, m_warmup))
    return 0


def plan(speed, m_base, m_warmup, p_total, rows_per_unit=1, a=(3, 4), b=(1, 4),
         flags=0, forced_units=None, alpha=None, beta=None):
    """Return the assignment (M_i, P_i) per GPU plus derived schedule facts."""
    n = len(speed)
    if n < 1 or n > 64:
        raise PlanError("n_gpus out of range")
    if any(int(v) <= 0 for v in speed):
        raise PlanError("speed must be > 0")
    if not (0 < b[0] * a[1] < a[0] * b[1] and a[0] < a[1] and b[0] > 0):
        raise PlanError("need 0 < b < a < 1")
    if not (1 <= m_warmup <= m_base):
        raise PlanError("need 1 <= M_warmup <= M_base")
    if p_total < 1 or rows_per_unit < 1:
        raise PlanError("bad p_total / rows_per_unit")

    tier = tiers(speed, a, b, flags)
    any_slow = any(t == 2 for t in tier)
    stride = slow_stride(m_base, m_warmup) if any_slow else 1
    steps = [steps_of(t, m_base, m_warmup) for t in tier]
    assert all(Fraction(s).denominator == 1 for s in steps)
    steps = [int(s) for s in steps]
    inc = [i for i in range(n) if tier[i] > 0]
    if p_total < len(inc):
        raise PlanError("P_total < number of included GPUs")

    units = [0] * n
    if flags & FORCE_UNITS:
        if forced_units is None or len(forced_units) != n:
            raise PlanError("forced units missing")
        if sum(forced_units) != p_total:
            raise PlanError("forced units must sum to P_total")
        for i in range(n):
            if (tier[i] == 0) != (forced_units[i] == 0):
                raise PlanError("forced units: included GPUs need >= 1, excluded 0")
        units = list(forced_units)
    elif flags & NO_SA:
        q, r = divmod(p_total, len(inc))
        for k, i in enumerate(inc):
            units[i] = q + (1 if k < r else 0)
    elif flags & SIZER_AFFINE:
        if alpha is None or beta is None or len(alpha) != n or len(beta) != n:
            raise PlanError("SIZER_AFFINE needs alpha and beta")
        if any(int(beta[i]) <= 0 for i in inc):
            raise PlanError("beta must be > 0")
        for i in inc:
            units[i] = 1
        for _ in range(p_total - len(inc)):          # R30: greedy min-makespan
            best = min(inc, key=lambda i: (steps[i] * (int(alpha[i]) + int(beta[i]) * (units[i] + 1)), i))
            units[best] += 1
    else:
        # Eq. 5 weights w_i = v_i / M'_i.  D'Hondt: every included GPU starts
        # with one unit; each further unit goes to argmax w_i/(P_i+1), i.e.
        # argmin (P_i+1) * M'_i / v_i, ties to the smallest rank (R5).
        if flags & SIZER_INTERVAL:
            mprime = [(stride if (tier[i] == 1 and any_slow) else 1) for i in range(n)]
        else:
            mprime = steps
        for i in inc:
            units[i] = 1
        for _ in range(p_total - len(inc)):
            best = None
            best_val = None
            for i in inc:
                val = Fraction((units[i] + 1) * mprime[i], int(speed[i]))
                if best_val is None or val < best_val:
                    best, best_val = i, val
            units[best] += 1

    row_begin, rows = [0] * n, [0] * n
    acc = 0
    for i in range(n):                       # R8: rank order, top to bottom
        row_begin[i] = acc * rows_per_unit
        rows[i] = units[i] * rows_per_unit
        acc += units[i]
    if flags & SIZER_AFFINE and not flags & (FORCE_UNITS | NO_SA):
        makespan = Fraction(max(steps[i] * (int(alpha[i]) + int(beta[i]) * units[i]) for i in inc))
    else:
        makespan = max(Fraction(steps[i] * units[i], int(speed[i])) for i in inc)
    sync_period = stride
    return dict(
        n_gpus=n, m_base=m_base, m_warmup=m_warmup, p_total=p_total,
        rows_per_unit=rows_per_unit, tier=tier, steps=steps, units=units,
        row_begin=row_begin, rows=rows, sync_period=sync_period,
        n_exchange_rounds=m_warmup + (m_base - m_warmup) // sync_period,
        makespan=makespan,
    )


def plan_cfg_split(speed, m_base, m_warmup, p_total, rows_per_unit=1, a=(3, 4), b=(1, 4),
                   flags=0):
    """R33: per-GPU plan of the CFG batch split plus the pair plan it expands."""
    n = len(speed)
    if flags & (FORCE_UNITS | SIZER_AFFINE):
        raise PlanError("CFG_SPLIT does not combine with FORCE_UNITS / SIZER_AFFINE")
    if n < 2:
        raise PlanError("CFG_SPLIT needs >= 2 GPUs")
    order = sorted(range(n), key=lambda i: (-int(speed[i]), i))
    pairs = [tuple(sorted(order[2 * k:2 * k + 2])) for k in range(n // 2)]
    pairs.sort(key=lambda pr: pr[0])                      # R8 on the pairs' lower index
    pspeed = [min(int(speed[i]), int(speed[j])) for i, j in pairs]
    pp = plan(pspeed, m_base, m_warmup, p_total, rows_per_unit, a, b, flags & ~CFG_SPLIT)
    out = dict(pp, n_gpus=n, tier=[0] * n, steps=[0] * n, units=[0] * n, row_begin=[0] * n,
               rows=[0] * n, branch=[0] * n, partner=[-1] * n, pairs=pairs, pair_plan=pp)
    for k, (i, j) in enumerate(pairs):
        for g, br, other in ((i, 0, j), (j, 1, i)):
            for key in ("tier", "steps", "units", "row_begin", "rows"):
                out[key][g] = pp[key][k]
            out["branch"][g] = br
            out["partner"][g] = other
    return out
