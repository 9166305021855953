// STADI planner: Temporal Adaptation (Eq. 4) + Spatial Adaptation (Eq. 5)
// and the per-rank schedule expander.  Host C++17, integer arithmetic only.
//
// PAPER.md L179-L185 (§III-C, Eq. 4), L187-L198 (§III-D, Eq. 5), Alg. 1
// L108-L155, Thm 2, hyper-parameters L284.  Readings R2-R8, R9-R13,
// R18, R25 of SURVEY.md §8(c) (restated in DESIGN.md §3).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>

#include "common.h"

namespace stadi {
std::string &tls_error() {
  static thread_local std::string s;
  return s;
}
}  // namespace stadi

using stadi::fail;
using u128 = unsigned __int128;

namespace {

constexpr int32_t kTrainT = 1000;

uint64_t gcd_u64(uint64_t a, uint64_t b) {
  while (b) {
    uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// Eq. 4 tier of speed v against v_max:  tier 1 iff a*v_max < v  (a = an/ad),
// tier 2 iff b*v_max < v <= a*v_max, else excluded (R2, exact).
int tier_of(uint64_t v, uint64_t vmax, uint32_t an, uint32_t ad, uint32_t bn, uint32_t bd) {
  if ((u128)ad * v > (u128)an * vmax) return 1;
  if ((u128)bd * v > (u128)bn * vmax) return 2;
  return 0;
}

}  // namespace

extern "C" uint32_t stadi_abi_version(void) { return STADI_ABI_VERSION; }

extern "C" const char *stadi_status_str(stadi_status s) {
  switch (s) {
    case STADI_OK: return "ok";
    case STADI_EINVAL: return "invalid argument";
    case STADI_ENOMEM: return "out of memory";
    case STADI_ECUDA: return "CUDA error";
    case STADI_ENCCL: return "NCCL error";
    case STADI_ESTATE: return "bad state (poisoned context or call order)";
    case STADI_EUNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

extern "C" stadi_status stadi_plan(const stadi_plan_params *in, stadi_plan_t *out) {
  if (!in || !out) return fail(nullptr, STADI_EINVAL, "stadi_plan: NULL argument");
  const uint32_t n = in->n_gpus;
  if (n < 1 || n > STADI_MAX_GPUS || !in->speed)
    return fail(nullptr, STADI_EINVAL, "stadi_plan: n_gpus %u out of range", n);
  for (uint32_t i = 0; i < n; ++i)
    if (in->speed[i] == 0) return fail(nullptr, STADI_EINVAL, "stadi_plan: speed[%u] == 0", i);
  const uint32_t an = in->a_num, ad = in->a_den, bn = in->b_num, bd = in->b_den;
  // 0 < b < a < 1
  if (!(ad > 0 && bd > 0 && bn > 0 && an < ad && (uint64_t)bn * ad < (uint64_t)an * bd))
    return fail(nullptr, STADI_EINVAL, "stadi_plan: need 0 < b < a < 1");
  if (!(in->m_warmup >= 1 && in->m_warmup <= in->m_base))
    return fail(nullptr, STADI_EINVAL, "stadi_plan: need 1 <= M_warmup <= M_base");
  if (in->m_base > 1000)
    return fail(nullptr, STADI_EINVAL, "stadi_plan: M_base > T = 1000");
  if (in->p_total < 1 || in->rows_per_unit < 1)
    return fail(nullptr, STADI_EINVAL, "stadi_plan: bad p_total / rows_per_unit");
  if ((uint64_t)in->p_total * in->rows_per_unit > 0xFFFFFFFFull)
    return fail(nullptr, STADI_EINVAL, "stadi_plan: p_total * rows_per_unit overflows");

  if (in->flags & STADI_CFG_SPLIT) {  // R33: plan the speed-ordered pairs, then expand
    if (in->flags & (STADI_FORCE_UNITS | STADI_SIZER_AFFINE))
      return fail(nullptr, STADI_EINVAL, "stadi_plan: CFG_SPLIT with FORCE_UNITS / SIZER_AFFINE");
    if (n < 2) return fail(nullptr, STADI_EINVAL, "stadi_plan: CFG_SPLIT needs >= 2 GPUs");
    uint32_t order[STADI_MAX_GPUS];
    for (uint32_t i = 0; i < n; ++i) order[i] = i;
    std::stable_sort(order, order + n, [&](uint32_t x, uint32_t y) {
      return in->speed[x] > in->speed[y];  // descending, ties keep the lower index first
    });
    uint32_t npair = n / 2, pa[STADI_MAX_GPUS / 2], pb[STADI_MAX_GPUS / 2];
    for (uint32_t k = 0; k < npair; ++k) {
      pa[k] = std::min(order[2 * k], order[2 * k + 1]);
      pb[k] = std::max(order[2 * k], order[2 * k + 1]);
    }
    uint32_t idx[STADI_MAX_GPUS / 2];  // pairs in the order of their lower index (R8)
    for (uint32_t k = 0; k < npair; ++k) idx[k] = k;
    std::sort(idx, idx + npair, [&](uint32_t x, uint32_t y) { return pa[x] < pa[y]; });
    uint64_t psp[STADI_MAX_GPUS / 2];
    for (uint32_t k = 0; k < npair; ++k)
      psp[k] = std::min(in->speed[pa[idx[k]]], in->speed[pb[idx[k]]]);
    stadi_plan_params q = *in;
    q.n_gpus = npair;
    q.speed = psp;
    q.flags &= ~STADI_CFG_SPLIT;
    stadi_plan_t pp;
    const stadi_status st = stadi_plan(&q, &pp);
    if (st != STADI_OK) return st;
    stadi_plan_t p = pp;
    p.n_gpus = n;
    std::memset(p.tier, 0, sizeof(p.tier));
    std::memset(p.steps, 0, sizeof(p.steps));
    std::memset(p.units, 0, sizeof(p.units));
    std::memset(p.row_begin, 0, sizeof(p.row_begin));
    std::memset(p.rows, 0, sizeof(p.rows));
    std::memset(p.branch, 0, sizeof(p.branch));
    std::memset(p.partner, -1, sizeof(p.partner));
    for (uint32_t k = 0; k < npair; ++k) {
      const uint32_t a = pa[idx[k]], b = pb[idx[k]];
      for (uint32_t g : {a, b}) {
        p.tier[g] = pp.tier[k];
        p.steps[g] = pp.steps[k];
        p.units[g] = pp.units[k];
        p.row_begin[g] = pp.row_begin[k];
        p.rows[g] = pp.rows[k];
      }
      p.branch[a] = 0;
      p.branch[b] = 1;
      p.partner[a] = (int8_t)b;
      p.partner[b] = (int8_t)a;
    }
    p.cfg_split = 1;
    *out = p;
    return STADI_OK;
  }

  stadi_plan_t p;
  std::memset(&p, 0, sizeof(p));
  std::memset(p.partner, -1, sizeof(p.partner));
  p.n_gpus = n;
  p.m_base = in->m_base;
  p.m_warmup = in->m_warmup;
  p.p_total = in->p_total;
  p.rows_per_unit = in->rows_per_unit;

  // ---- Step 1: temporal adaptation, Eq. 4 (Alg. 1 lines 1-3)
  uint64_t vmax = 0;
  for (uint32_t i = 0; i < n; ++i) vmax = std::max(vmax, in->speed[i]);
  bool any_slow = false;
  uint32_t n_inc = 0;
  for (uint32_t i = 0; i < n; ++i) {
    int t = (in->flags & STADI_NO_TA) ? 1 : tier_of(in->speed[i], vmax, an, ad, bn, bd);
    p.tier[i] = (uint8_t)t;
    any_slow |= (t == 2);
    n_inc += (t > 0);
  }
  // R32: tier-2 stride n over the K post-warmup intervals: 2 for even K (Eq. 4's
  // (M_base + M_warmup) / 2), else the smallest prime factor of K (K = 1: 1)
  const uint32_t K = in->m_base - in->m_warmup;
  uint32_t stride = 1;
  if (any_slow) {
    if (K % 2 == 0) {
      stride = 2;
    } else if (K > 1) {
      stride = K;
      for (uint32_t d = 3; d * d <= K; d += 2)
        if (K % d == 0) {
          stride = d;
          break;
        }
    }
  }
  for (uint32_t i = 0; i < n; ++i)
    p.steps[i] = p.tier[i] == 1 ? in->m_base
               : p.tier[i] == 2 ? in->m_warmup + K / stride : 0;
  if (in->p_total < n_inc)
    return fail(nullptr, STADI_EINVAL, "stadi_plan: P_total %u < %u included GPUs",
                in->p_total, n_inc);

  // ---- Step 2: spatial adaptation, Eq. 5 (Alg. 1 lines 4-6)
  if (in->flags & STADI_FORCE_UNITS) {
    if (!in->forced_units) return fail(nullptr, STADI_EINVAL, "stadi_plan: forced_units NULL");
    uint64_t s = 0;
    for (uint32_t i = 0; i < n; ++i) {
      if ((p.tier[i] == 0) != (in->forced_units[i] == 0))
        return fail(nullptr, STADI_EINVAL,
                    "stadi_plan: forced units: included GPUs need >= 1, excluded 0");
      p.units[i] = in->forced_units[i];
      s += in->forced_units[i];
    }
    if (s != in->p_total)
      return fail(nullptr, STADI_EINVAL, "stadi_plan: forced units must sum to P_total");
  } else if (in->flags & STADI_NO_SA) {
    const uint32_t q = in->p_total / n_inc, r = in->p_total % n_inc;
    uint32_t k = 0;
    for (uint32_t i = 0; i < n; ++i)
      if (p.tier[i]) p.units[i] = q + (k++ < r ? 1u : 0u);
  } else if (in->flags & STADI_SIZER_AFFINE) {
    // R30: greedy min-makespan of max_i M_i (alpha_i + beta_i P_i)
    if (!in->alpha || !in->beta)
      return fail(nullptr, STADI_EINVAL, "stadi_plan: SIZER_AFFINE needs alpha and beta");
    for (uint32_t i = 0; i < n; ++i) {
      if (p.tier[i] && in->beta[i] == 0)
        return fail(nullptr, STADI_EINVAL, "stadi_plan: beta[%u] == 0", i);
      if (p.tier[i]) p.units[i] = 1;
    }
    auto cost = [&](uint32_t i, uint64_t units) {
      return (u128)p.steps[i] * ((u128)in->alpha[i] + (u128)in->beta[i] * units);
    };
    for (uint32_t u = n_inc; u < in->p_total; ++u) {
      int best = -1;
      for (uint32_t i = 0; i < n; ++i) {
        if (!p.tier[i]) continue;
        if (best < 0 || cost(i, p.units[i] + 1) < cost((uint32_t)best, p.units[best] + 1))
          best = (int)i;
      }
      p.units[best] += 1;
    }
  } else {
    // D'Hondt on weights v_i / M'_i (R5); M'_i = M_i, or the per-round step
    // count with SIZER_INTERVAL (R7 variant).
    uint64_t mp[STADI_MAX_GPUS];
    for (uint32_t i = 0; i < n; ++i) {
      if (in->flags & STADI_SIZER_INTERVAL)
        mp[i] = (p.tier[i] == 1 && any_slow) ? stride : 1;
      else
        mp[i] = p.steps[i];
      if (p.tier[i]) p.units[i] = 1;
    }
    for (uint32_t u = n_inc; u < in->p_total; ++u) {
      int best = -1;
      for (uint32_t i = 0; i < n; ++i) {
        if (!p.tier[i]) continue;
        if (best < 0) {
          best = (int)i;
          continue;
        }
        // (P_i+1) M_i / v_i < (P_b+1) M_b / v_b  <=>  (P_i+1) M_i v_b < (P_b+1) M_b v_i
        u128 lhs = (u128)((uint64_t)(p.units[i] + 1) * mp[i]) * in->speed[best];
        u128 rhs = (u128)((uint64_t)(p.units[best] + 1) * mp[best]) * in->speed[i];
        if (lhs < rhs) best = (int)i;
      }
      p.units[best] += 1;
    }
  }
  uint32_t acc = 0;
  for (uint32_t i = 0; i < n; ++i) {  // R8: rank order, top to bottom
    p.row_begin[i] = acc * in->rows_per_unit;
    p.rows[i] = p.units[i] * in->rows_per_unit;
    acc += p.units[i];
  }
  // makespan = max_i M_i P_i / v_i over included GPUs, reduced
  // (SIZER_AFFINE: max_i M_i (alpha_i + beta_i P_i), an integer)
  uint64_t bn_ = 0, bd_ = 1;
  const bool affine = (in->flags & STADI_SIZER_AFFINE) &&
                      !(in->flags & (STADI_FORCE_UNITS | STADI_NO_SA));
  if (affine) {
    u128 mx = 0;
    for (uint32_t i = 0; i < n; ++i)
      if (p.tier[i])
        mx = std::max(mx, (u128)p.steps[i] * ((u128)in->alpha[i] + (u128)in->beta[i] * p.units[i]));
    if (mx >> 64) return fail(nullptr, STADI_EINVAL, "stadi_plan: affine makespan overflows");
    bn_ = (uint64_t)mx;
  }
  for (uint32_t i = 0; i < n && !affine; ++i) {
    if (!p.tier[i]) continue;
    uint64_t num = (uint64_t)p.steps[i] * p.units[i], den = in->speed[i];
    if ((u128)num * bd_ > (u128)bn_ * den) {
      bn_ = num;
      bd_ = den;
    }
  }
  uint64_t g = gcd_u64(bn_, bd_);
  p.makespan_num = bn_ / g;
  p.makespan_den = bd_ / g;
  p.sync_period = stride;
  p.n_exchange_rounds = in->m_warmup + (in->m_base - in->m_warmup) / p.sync_period;
  *out = p;
  return STADI_OK;
}

extern "C" stadi_status stadi_schedule(const stadi_plan_t *plan, uint32_t rank,
                                       stadi_step_t *buf, uint32_t cap, uint32_t *n_out) {
  if (!plan || !n_out) return fail(nullptr, STADI_EINVAL, "stadi_schedule: NULL argument");
  if (rank >= plan->n_gpus) return fail(nullptr, STADI_EINVAL, "stadi_schedule: bad rank");
  const int32_t mb = (int32_t)plan->m_base, mw = (int32_t)plan->m_warmup;
  if (mb < 1 || mw < 1 || mw > mb || mb > kTrainT || plan->sync_period < 1 ||
      (mb - mw) % (int32_t)plan->sync_period)
    return fail(nullptr, STADI_EINVAL, "stadi_schedule: bad plan");
  const int32_t ratio = kTrainT / mb;
  auto grid = [&](int32_t i) { return i < mb ? ratio * (mb - 1 - i) + 1 : STADI_T_FINAL; };
  uint32_t n = 0;
  auto emit = [&](int32_t m, int32_t t, int32_t tp, int32_t kind, int32_t rv, int32_t pv) {
    if (buf && n < cap) buf[n] = stadi_step_t{m, t, tp, kind, rv, pv};
    ++n;
  };
  const int tier = plan->tier[rank];
  if (tier != 0) {
    for (int32_t m = 0; m < mw; ++m)  // Alg. 1, R9
      emit(m, grid(m), grid(m + 1), STADI_STEP_WARMUP, m, m);
    const int32_t K = mb - mw;
    if (plan->sync_period == 1) {  // R13
      for (int32_t j = 0; j < K; ++j) {
        const int32_t m = mw + j, e = mw + j;
        emit(m, grid(m), grid(m + 1), STADI_STEP_UNIFORM, e - 1, e);
      }
    } else {
      const int32_t sn = (int32_t)plan->sync_period;  // slow stride (R11, R32)
      for (int32_t k = 0; k < K / sn; ++k) {  // Alg. 1, R10, R11
        const int32_t m = mw + sn * k, e = mw + k;
        if (tier == 1) {
          emit(m, grid(m), grid(m + 1), STADI_STEP_FAST_EVEN, e - 1, e);
          for (int32_t q = 1; q < sn; ++q)
            emit(m + q, grid(m + q), grid(m + q + 1), STADI_STEP_FAST_ODD, e, STADI_VER_NONE);
        } else {
          emit(m, grid(m), grid(m + sn), STADI_STEP_SLOW, e - 1, e);
        }
      }
    }
  }
  *n_out = n;
  return STADI_OK;
}
