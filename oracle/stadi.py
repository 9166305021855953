"""Oracle STADI run: Algorithm 1 end to end, all GPUs simulated in one process.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md Alg. 1 (L108-L155): Step 1 temporal adaptation (Eq. 4) ->
Step 2 spatial adaptation (Eq. 5) -> Step 3 inference: warmup steps with the
buffer updated synchronously (L122-L128), then per GPU: fast GPUs alternate
"update buffer asynchronously + all-gather" (even) and "no update for buffer"
(odd); slow GPUs update asynchronously every (stride-2) step (L130-L152).
Each GPU denoises only its patch p_i (L125, L171, DistriFusion-style stale
activations, L80).

Protocol (SURVEY §8(c) O5/O6 and readings R9-R17):
* "buffer" = per attention site, the K/V rows each GPU published for an
  exchange version.  A step reads version ``read_ver`` for every *other* GPU's
  rows and its own rows fresh (R14); it publishes its fresh K/V as
  ``pub_ver``.  read_ver == pub_ver (warmup) is a layer-synchronous fresh
  exchange (R9).
* Steps are processed grouped by fast-grid index m ("phases"); inside a phase
  every participating GPU runs in lock-step per layer: all publish, then all
  read.  Only warmup phases depend on the lock-step; stale phases read only
  versions published in earlier phases.
* R12 owner-computes: each GPU updates only its own rows with its own grid;
  the final (synchronous) all-gather concatenates the bands.  Intermediate
  "Get x by synchronous All-Gather" lines do not change any band.
"""
from __future__ import annotations

from . import diffusion, dit, planner, schedule, unet


def _group_phases(plan):
    """All ranks' schedule entries grouped by fast-grid index m."""
    phases = {}
    for r in range(plan["n_gpus"]):
        for st in schedule.schedule(plan, r):
            phases.setdefault(st.m, []).append((r, st))
    return [phases[m] for m in sorted(phases)]


def _update(abar, x, eps, st, ddpm_z, r0, hist=None):
    """Sampler update of one band (rows [r0, r0 + len(x)) of the image): Eq. 3
    DDIM, the R19 DDPM step with the band's rows of z_m when ddpm_z (a callable
    m -> full-image z_m, an input) is given, or (hist a dict: the band's history)
    the R34 multistep DPM-Solver-2."""
    if hist is not None:
        out = diffusion.dpm2m_step(abar, x, eps, st.t, st.t_prev, hist.get("h"))
        hist["h"] = (eps, st.t)
        return out
    if ddpm_z is None:
        return diffusion.ddim_step(abar, x, eps, st.t, st.t_prev)
    z = ddpm_z(st.m)[r0:r0 + x.shape[0]]
    return diffusion.ddpm_step(abar, x, eps, st.t, st.t_prev, z)


def run(cfg, weights, x_T, cond, plan, return_trace=False, ddpm_z=None, sampler="ddim"):
    """Execute STADI for one request.  x_T: full noise [H, W, C] (any float).
    ddpm_z: None (DDIM, Eq. 3) or m -> z_m [H, W, C] (DDPM, R19); sampler="dpm2m":
    the R34 multistep DPM-Solver-2 (each band keeps its own history).

    Returns the final latent [H, W, C] (float64) assembled from the bands.
    """
    hist = {r: {} for r in range(plan["n_gpus"])} if sampler == "dpm2m" else {}
    if cfg["family"] == "unet":
        return run_unet(cfg, weights, x_T, cond, plan, return_trace, ddpm_z, hist)
    model = dit.DiT(cfg, weights)
    abar = diffusion.alpha_bar("linear" if cfg["schedule"] == "linear" else "scaled_linear")
    B = dit.batch_of(cfg)
    y = model.caption(cond)
    p = cfg["patch"]
    inc = [r for r in range(plan["n_gpus"]) if plan["tier"][r] > 0]
    band = {r: x_T[plan["row_begin"][r]:plan["row_begin"][r] + plan["rows"][r]].astype("float64")
            for r in inc}
    store = {}                                   # (version, layer, rank) -> (k, v)
    trace = []
    for phase in _group_phases(plan):
        parts = []
        for r, st in phase:
            mods, fin = model.modulations(st.t, cond)
            h = model.embed(band[r], plan["row_begin"][r] // p, B)
            parts.append(dict(r=r, st=st, mods=mods, fin=fin, h=h))
        for l in range(model.depth):
            fresh = {}
            for P in parts:                      # everyone computes + publishes first
                q, k, v = model.block_qkv(l, P["h"], P["mods"][l])
                fresh[P["r"]] = (q, k, v)
                if P["st"].pub_ver != schedule.NONE:
                    store[(P["st"].pub_ver, l, P["r"])] = (k, v)
            for P in parts:                      # then reads version read_ver
                r, st = P["r"], P["st"]
                ks, vs = [], []
                for j in inc:                    # full image K/V in row order
                    if j == r:
                        kj, vj = fresh[r][1], fresh[r][2]      # R14: own rows fresh
                    else:
                        kj, vj = store[(st.read_ver, l, j)]
                    ks.append(kj)
                    vs.append(vj)
                P["h"] = model.block_rest(l, P["h"], fresh[r][0],
                                          _cat(ks), _cat(vs), P["mods"][l], y)
        for P in parts:                          # eps on own band + Eq. 3 on own rows
            r, st = P["r"], P["st"]
            eps = dit.guided_eps(cfg, model.final(P["h"], P["fin"], band[r].shape[0]))
            band[r] = _update(abar, band[r], eps, st, ddpm_z, plan["row_begin"][r], hist.get(r))
            if return_trace:
                trace.append((st.m, r, st.kind, band[r].copy()))
    import numpy as np
    out = np.concatenate([band[r] for r in inc], axis=0)   # final synchronous all-gather
    return (out, trace) if return_trace else out


def _assemble(kind, r, inc, own, stale):
    """Answer one exchange request of rank r: own payload
    fresh, every other included rank's payload of the read version (`stale`:
    rank -> payload).  Ranks are in row order top to bottom (R8)."""
    import numpy as np
    if kind == "kv":
        ks = [own[0] if j == r else stale[j][0] for j in inc]
        vs = [own[1] if j == r else stale[j][1] for j in inc]
        return np.concatenate(ks, axis=1), np.concatenate(vs, axis=1)
    if kind == "halo":
        i = inc.index(r)
        above = stale[inc[i - 1]][1] if i > 0 else np.zeros_like(own[0])       # its last row
        below = stale[inc[i + 1]][0] if i + 1 < len(inc) else np.zeros_like(own[1])
        return above, below
    if kind == "gn":
        tot = [a.copy() for a in own]
        for j in inc:
            if j != r:
                for t, a in zip(tot, stale[j]):
                    t += a
        return tuple(tot)
    raise ValueError(kind)


def run_unet(cfg, weights, x_T, cond, plan, return_trace=False, ddpm_z=None, hist=None):
    """Algorithm 1 for the U-Net family: every rank's band forward is a
    generator (oracle/unet.py) that yields at each exchange site; ranks of a
    phase advance in lock-step site by site: all publish (pub_ver), then all
    read (read_ver; fresh when read_ver == pub_ver, R9)."""
    import numpy as np
    model = unet.UNet(cfg, weights)
    abar = diffusion.alpha_bar(cfg["schedule"])
    inc = [r for r in range(plan["n_gpus"]) if plan["tier"][r] > 0]
    band = {r: x_T[plan["row_begin"][r]:plan["row_begin"][r] + plan["rows"][r]].astype("float64")
            for r in inc}
    store = {}                                   # (version, site, rank) -> payload
    trace = []
    for phase in _group_phases(plan):
        gens = {r: model.band_forward(band[r], st.t, cond) for r, st in phase}
        steps = {r: st for r, st in phase}
        reqs = {r: next(g) for r, g in gens.items()}
        eps = {}
        site = 0
        while reqs:
            kinds = {k for k, _ in reqs.values()}
            assert len(kinds) == 1, "ranks out of lock-step"
            for r, (kind, pay) in reqs.items():          # everyone publishes first
                if steps[r].pub_ver != schedule.NONE:
                    store[(steps[r].pub_ver, site, r)] = pay
            nxt = {}
            for r, (kind, pay) in reqs.items():          # then reads read_ver
                rv = steps[r].read_ver
                stale = {j: store[(rv, site, j)] for j in inc if j != r}
                try:
                    nxt[r] = gens[r].send(_assemble(kind, r, inc, pay, stale))
                except StopIteration as e:
                    eps[r] = e.value
            reqs = nxt
            site += 1
        for r, st in phase:                      # eps on own band + Eq. 3 on own rows
            band[r] = _update(abar, band[r], unet.guided_eps(cfg, eps[r]), st, ddpm_z,
                              plan["row_begin"][r], (hist or {}).get(r))
            if return_trace:
                trace.append((st.m, r, st.kind, band[r].copy()))
    out = np.concatenate([band[r] for r in inc], axis=0)   # final synchronous all-gather
    return (out, trace) if return_trace else out


def _cat(xs):
    import numpy as np
    return np.concatenate(xs, axis=1)


def sequential(cfg, weights, x_T, cond, m_base, ddpm_z=None, sampler="ddim"):
    """Non-distributed DDIM (or R19 DDPM, or R34 DPM-Solver-2M) with M_base steps on
    the fast grid (the "Origin" method of Table II)."""
    hist = {}

    def upd(abar, x, eps, m, t, t_prev):
        if sampler == "dpm2m":
            out = diffusion.dpm2m_step(abar, x, eps, t, t_prev, hist.get("h"))
            hist["h"] = (eps, t)
            return out
        if ddpm_z is None:
            return diffusion.ddim_step(abar, x, eps, t, t_prev)
        return diffusion.ddpm_step(abar, x, eps, t, t_prev, ddpm_z(m))

    if cfg["family"] == "unet":
        model = unet.UNet(cfg, weights)
        abar = diffusion.alpha_bar(cfg["schedule"])
        x = x_T.astype("float64")
        grid = schedule.fast_grid(m_base)
        for m, t in enumerate(grid):
            t_prev = grid[m + 1] if m + 1 < m_base else schedule.FINAL
            eps = unet.guided_eps(cfg, model.forward_full(x, t, cond))
            x = upd(abar, x, eps, m, t, t_prev)
        return x
    model = dit.DiT(cfg, weights)
    abar = diffusion.alpha_bar("linear" if cfg["schedule"] == "linear" else "scaled_linear")
    y = model.caption(cond)
    x = x_T.astype("float64")
    grid = schedule.fast_grid(m_base)
    for m, t in enumerate(grid):
        t_prev = grid[m + 1] if m + 1 < m_base else schedule.FINAL
        eps = dit.guided_eps(cfg, model.forward_full(x, t, cond, y))
        x = upd(abar, x, eps, m, t, t_prev)
    return x


def plan_for(cfg, speed, m_base, m_warmup, flags=0, forced_units=None):
    """Planner call with the model's unit (R6: one unit = one row of the coarsest
    feature map: p latent rows for a DiT, 2^(levels-1) for a U-Net)."""
    from synth.configs import rows_per_unit
    u = rows_per_unit(cfg)
    return planner.plan(speed, m_base, m_warmup, cfg["latent_h"] // u, u,
                        flags=flags, forced_units=forced_units)


def run_cfg_split(cfg, weights, x_T, cond, splan, return_trace=False):
    """R33 CFG batch split (DiT family): every included GPU runs ONE CFG branch
    (B = 1 conditioning) on its pair's band, exchanges K/V with the GPUs of its own
    branch only (versions as in Alg. 1), and combines its eps band with its
    partner's every step (R20) before the identical Eq. 3 update on both members.
    Equal to run(cfg, ..., splan["pair_plan"]) -- the pin that the split changes
    nothing but the placement (tests/test_oracle_model.py)."""
    import numpy as np
    assert cfg["family"] == "dit" and dit.batch_of(cfg) == 2
    model = dit.DiT(cfg, weights)
    abar = diffusion.alpha_bar("linear" if cfg["schedule"] == "linear" else "scaled_linear")
    p = cfg["patch"]
    inc = [r for r in range(splan["n_gpus"]) if splan["tier"][r] > 0]
    br = splan["branch"]
    cond_b = [{k: np.asarray(v)[b:b + 1] for k, v in cond.items() if k in ("labels", "text")}
              for b in (0, 1)]
    y_b = [model.caption(cond_b[b]) for b in (0, 1)]
    band = {r: x_T[splan["row_begin"][r]:splan["row_begin"][r] + splan["rows"][r]].astype("float64")
            for r in inc}
    store = {}                                   # (version, layer, rank) -> (k, v)
    trace = []
    for phase in _group_phases(splan):
        parts = []
        for r, st in phase:
            mods, fin = model.modulations(st.t, cond_b[br[r]])
            h = model.embed(band[r], splan["row_begin"][r] // p, 1)
            parts.append(dict(r=r, st=st, mods=mods, fin=fin, h=h))
        for l in range(model.depth):
            fresh = {}
            for P in parts:
                q, k, v = model.block_qkv(l, P["h"], P["mods"][l])
                fresh[P["r"]] = (q, k, v)
                if P["st"].pub_ver != schedule.NONE:
                    store[(P["st"].pub_ver, l, P["r"])] = (k, v)
            for P in parts:
                r, st = P["r"], P["st"]
                same = [j for j in inc if br[j] == br[r]]          # own branch, row order
                ks = [fresh[r][1] if j == r else store[(st.read_ver, l, j)][0] for j in same]
                vs = [fresh[r][2] if j == r else store[(st.read_ver, l, j)][1] for j in same]
                P["h"] = model.block_rest(l, P["h"], fresh[r][0], _cat(ks), _cat(vs),
                                          P["mods"][l], y_b[br[r]])
        eps_b = {P["r"]: model.final(P["h"], P["fin"], band[P["r"]].shape[0])[0] for P in parts}
        for P in parts:                          # pair exchange of eps, CFG, Eq. 3
            r, st = P["r"], P["st"]
            e_u = eps_b[r] if br[r] == 0 else eps_b[splan["partner"][r]]
            e_c = eps_b[r] if br[r] == 1 else eps_b[splan["partner"][r]]
            eps = diffusion.cfg_combine(e_u, e_c, cfg["guidance"])
            band[r] = diffusion.ddim_step(abar, band[r], eps, st.t, st.t_prev)
            if return_trace:
                trace.append((st.m, r, st.kind, band[r].copy()))
    out = np.concatenate([band[r] for r in inc if br[r] == 0], axis=0)
    return (out, trace) if return_trace else out
