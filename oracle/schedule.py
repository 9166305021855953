"""Oracle schedule expander: per-rank step table.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows Algorithm 1 lines 8-24 and Theorem 2's aligned
grids (L234-L238: for n*M_i = M_j, t^i_m = t^j_m = s and
t^i_{m+1} = t^j_{m+n} = t).

Readings:
  R9   warmup steps exchange fresh activations layer-synchronously; the last
       warmup step's activations seed version V_{-1}.
  R10  a fast GPU's odd step reads the newest complete version V_k and
       publishes nothing ("No update for buffer", L144).
  R11  the slow grid is the warmup prefix plus every n-th fast-grid point (n = 2,
       or R32's smallest prime factor of an odd K; a fast GPU publishes on the
       slow grid's points only).
  R13  with no slow GPU every GPU exchanges every step (DistriFusion).
  R18  fast grid: "leading" spacing, steps_offset 1:
       tau_m = (T // M_base) * (M_base - 1 - m) + 1,  T = 1000.
  R25  "for m = M_warmup to M_i" read as the half-open range.

Versions are numbered by exchange round e: warmup step m is round m (read ==
publish == e means "fresh"); post-warmup round j is e = M_warmup + j.
"""
from __future__ import annotations

from dataclasses import dataclass

T_TRAIN = 1000
FINAL = -1                    # t_prev of the last step: the "final" alpha (alpha_bar_0)

WARMUP, UNIFORM, FAST_EVEN, FAST_ODD, SLOW = 0, 1, 2, 3, 4
KIND_NAMES = {WARMUP: "warmup", UNIFORM: "uniform", FAST_EVEN: "fast-even",
              FAST_ODD: "fast-odd", SLOW: "slow"}
NONE = -1                     # pub_ver of a step that publishes nothing


@dataclass(frozen=True)
class Step:
    m: int          # fast-grid index of the step
    t: int          # timestep denoised from
    t_prev: int     # timestep denoised to (FINAL = alpha_bar_0)
    kind: int
    read_ver: int   # exchange version read at every site
    pub_ver: int    # exchange version published (NONE = no publish)


def fast_grid(m_base: int, T: int = T_TRAIN) -> list[int]:
    """R18: DDIM 'leading' timesteps with steps_offset = 1."""
    ratio = T // m_base
    return [ratio * (m_base - 1 - m) + 1 for m in range(m_base)]


def schedule(plan: dict, rank: int) -> list[Step]:
    """Step table of one GPU (Alg. 1)."""
    tier = plan["tier"][rank]
    if tier == 0:
        return []                                  # excluded (Eq. 4 third case)
    mb, mw = plan["m_base"], plan["m_warmup"]
    grid = fast_grid(mb)

    def nxt(i):
        return grid[i] if i < mb else FINAL

    out = []
    for m in range(mw):                            # Alg. 1: warmup
        out.append(Step(m, grid[m], nxt(m + 1), WARMUP, m, m))
    K = mb - mw
    if plan["sync_period"] == 1:                   # R13: nobody is slow
        for j in range(K):
            m, e = mw + j, mw + j
            out.append(Step(m, grid[m], nxt(m + 1), UNIFORM, e - 1, e))
        return out
    n = plan["sync_period"]                        # slow stride (2, or R32's spf(K))
    for k in range(K // n):                        # Alg. 1
        m, e = mw + n * k, mw + k
        if tier == 1:                              # fast GPU (L134-L146)
            out.append(Step(m, grid[m], nxt(m + 1), FAST_EVEN, e - 1, e))
            for q in range(1, n):                  # "no update for buffer" steps
                out.append(Step(m + q, grid[m + q], nxt(m + q + 1), FAST_ODD, e, NONE))
        else:                                      # slow GPU (L148-L152), stride n
            out.append(Step(m, grid[m], nxt(m + n), SLOW, e - 1, e))
    return out
