"""bench.py — per-image latency / images/s of STADI on N B200s vs uniform patch
parallelism built from the same kernels (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c5|c2] [--occupancy half50|zero|<p0,p1,...>]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU)

A "step" is one whole STADI request (SURVEY §8(a) a1..a9 minus the one-off
profiling): begin (per-request conditioning) -> every denoising step of the
rank's schedule (patch-local DiT forward with stale K/V exchange + Eq. 3
sampler) -> final latent all-gather.  One step = one image, so
``value`` = images/s of the whole job and ``ms_per_step`` = per-image latency.

Workload: BASELINE configs[4] = C5, the PixArt-alpha-shaped DiT
at 2048^2 (256x256x4 latent, 16384 tokens, d 1152, 16 heads, depth 28, T5 text
120x4096, CFG 4.5), 20 DDIM steps, M_warmup 4, a = 3/4, b = 1/4; the 1/2/4/8
GPU scaling sweep with 50% emulated occupancy on the upper half of the GPUs
(0% at N = 1).  Random-init weights and seeded synthetic inputs (synth/).

JSON keys beyond the base contract: ``uniform_pp`` (the same-kernel uniform
patch-parallel baseline, NO_TA|NO_SA plan, timed the same way), ``roofline``
(dominant kernel = self-attention, CUDA events around every launch inside the
timed region), ``cpu_baseline`` (the fp64 oracle on a bounded sample,
extrapolated by FLOP count), ``e2e`` (stadi_run with pinned HOST buffers),
``clocks`` (nvidia-smi sampled during the timed region), ``gpu_launches``.

The oracle (oracle/) is executed only by the cpu_baseline leg and by
``--impl reference``; the timed path is libstadi.so through its C ABI.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from synth import configs, gen  # noqa: E402

WORKLOADS = {
    "c5": dict(model="pixart_alpha", m_base=20, m_warmup=4, name=(
        "C5 PixArt-alpha-shaped DiT 2048^2 (256x256x4 latent, 16384 tokens, d1152 h16 "
        "depth28, T5 120x4096, CFG 4.5), 20 DDIM steps, M_warmup 4")),
    "c2": dict(model="dit_xl2", m_base=50, m_warmup=4, name=(
        "C2 DiT-XL/2-shaped 256^2 (32x32x4 latent, 256 tokens, d1152 h16 depth28, "
        "class cond, CFG 4.0), 50 DDIM steps, M_warmup 4")),
    "c3": dict(model="sd15", m_base=50, m_warmup=4, name=(
        "C3 SD-1.5-shaped U-Net 512^2 (64x64x4 latent, channels 320/640/1280/1280, 8 heads, "
        "text 77x768, CFG 7.5), 50 DDIM steps, M_warmup 4")),
    "c4": dict(model="sdxl", m_base=50, m_warmup=4, name=(
        "C4 SDXL-shaped U-Net 1024^2 (128x128x4 latent, channels 320/640/1280, transformer "
        "depth 0/2/10, text 77x2048 + pooled, CFG 5.0), 50 DDIM steps, M_warmup 4")),
}
PAPER_CONTEXT = ("paper: up to 45% lower latency than patch parallelism (SDXL 1024^2, "
                 "M_base=100, 2x RTX 4090 over PCIe, occupancy [0,60]%; Table III / L11)")


# --------------------------------------------------------------------- helpers
def dit_flops(cfg, n_q, n_kv, B):
    """Algorithmic FLOPs of one DiT block on n_q own tokens against n_kv keys
    (2 per multiply-add): qkv 3d^2 + proj d^2 + fc1/fc2 8d^2 (+ xq/xproj 2d^2
    for text presets), self-attention 4 n_q n_kv d, cross-attention 4 n_q L d."""
    d = cfg["hidden"]
    text = cfg["cond"] == "text"
    lin = 2.0 * n_q * B * d * d * (12 + (2 if text else 0))
    att = 4.0 * n_q * n_kv * d * B
    xatt = 4.0 * n_q * cfg.get("text_len", 0) * d * B if text else 0.0
    return lin + att + xatt


def unet_flops(cfg, rows, kv_rows=None):
    """Algorithmic FLOPs of one U-Net forward (B = 2) on the full-width latent cut
    to `rows` rows, attention against kv_rows rows (default: the same tokens):
    conv 2*9*Cin*Cout per output pixel, linear 2*K*N per token, attention
    4*n_q*n_kv*C, cross 4*n_q*L*C."""
    B = configs.batch(cfg)
    kv_rows = rows if kv_rows is None else kv_rows
    W0, L = cfg["latent_w"], len(cfg["channels"])
    f = 0.0

    def conv(h, w, cin, cout):
        return 2.0 * 9 * cin * cout * h * w * B

    def res(h, w, cin, cout):
        return conv(h, w, cin, cout) + conv(h, w, cout, cout) + \
            (2.0 * cin * cout * h * w * B if cin != cout else 0.0)

    def tr(h, w, c, depth):
        n = h * w
        n_kv = n * kv_rows // max(rows, 1)
        per = 2.0 * n * B * c * c * (4 + 2 + 8 + 4) + 4.0 * n * n_kv * c * B + \
            4.0 * n * cfg["text_len"] * c * B
        return 2.0 * 2 * n * B * c * c + depth * per

    lv = configs.unet_levels(cfg)
    f += conv(rows, W0, cfg["c_in"], cfg["channels"][0])
    prev = cfg["channels"][0]
    for i, (c, att, depth, _) in enumerate(lv):
        h, w = rows >> i, W0 >> i
        for j in range(cfg["layers_per_block"]):
            f += res(h, w, prev if j == 0 else c, c) + (tr(h, w, c, depth) if att else 0.0)
        if i < L - 1:
            f += conv(h // 2, w // 2, c, c)
        prev = c
    h, w = rows >> (L - 1), W0 >> (L - 1)
    cm = cfg["channels"][-1]
    f += 2 * res(h, w, cm, cm) + tr(h, w, cm, cfg["mid_depth"])
    for i, io in enumerate(configs.unet_up_io(cfg)):
        l = L - 1 - i
        c, att, depth, _ = lv[l]
        h, w = rows >> l, W0 >> l
        for rin, sk, oc in io:
            f += res(h, w, rin + sk, oc) + (tr(h, w, oc, depth) if att else 0.0)
        if i < L - 1:
            f += conv(2 * h, 2 * w, c, c)
    f += conv(rows, W0, cfg["channels"][0], cfg["c_out"])
    return f


def image_flops(cfg, m_base):
    if cfg["family"] == "unet":
        return m_base * unet_flops(cfg, cfg["latent_h"])
    hp, wp = configs.tokens_hw(cfg)
    n = hp * wp
    B = configs.batch(cfg)
    return m_base * cfg["depth"] * dit_flops(cfg, n, n, B)


def step_flops(cfg, rows):
    """Algorithmic FLOPs of one denoising step of a band of `rows` latent rows
    (own queries x full-image K/V, SURVEY §8(d) 'Method')."""
    H = cfg["latent_h"]
    if cfg["family"] == "unet":
        return unet_flops(cfg, rows, kv_rows=H)
    hp, wp = configs.tokens_hw(cfg)
    nq = rows // cfg["patch"] * wp
    return cfg["depth"] * dit_flops(cfg, nq, hp * wp, configs.batch(cfg))


def kv_bytes_per_round(cfg):
    """Full-image K/V bytes of one exchange round: sum over self-attention sites
    of 2 (K, V) * B * N_tokens * C * 2 bytes (bf16) (SURVEY §8(d) 'Bytes per round')."""
    B = configs.batch(cfg)
    if cfg["family"] != "unet":
        hp, wp = configs.tokens_hw(cfg)
        return cfg["depth"] * 2 * B * hp * wp * cfg["hidden"] * 2
    tot, H, W = 0, cfg["latent_h"], cfg["latent_w"]
    lv = configs.unet_levels(cfg)
    for i, (c, att, depth, _) in enumerate(lv):
        if att:
            n = (H >> i) * (W >> i)
            sites = depth * (2 * cfg["layers_per_block"] + 1)   # down + up blocks
            tot += sites * 2 * B * n * c * 2
    L = len(lv) - 1
    tot += cfg["mid_depth"] * 2 * B * (H >> L) * (W >> L) * lv[-1][0] * 2
    return tot


NVLINK_GBS = 900.0   # NVLink 5 per direction per GPU (B200_PROFILING.md / SURVEY App. B)


def path_lower_bound(cfg, plan_d, occ, peak_tflops):
    """SURVEY §8(d) end-to-end lower bound of one image under a plan:
    LB = max(sum_i W_i / sum_i (1 - rho_i) peak,  max_i inbound_i rounds / BW_NVL,
             max_i W_i / ((1 - rho_i) peak)),
    W_i = M_i * step_flops(rows_i) (algorithmic, fewer steps on tier-2 ranks),
    inbound_i = (1 - rows_i / H) * K/V bytes per round."""
    H = cfg["latent_h"]
    inc = [i for i, t in enumerate(plan_d["tier"]) if t > 0]
    Wi = {i: plan_d["steps"][i] * step_flops(cfg, plan_d["rows"][i]) for i in inc}
    free = {i: max(1e-6, 1.0 - occ[i] / 100.0) for i in inc}
    pk = peak_tflops * 1e12
    t_total = sum(Wi.values()) / (sum(free.values()) * pk)
    t_rank = max(Wi[i] / (free[i] * pk) for i in inc)
    kvb = kv_bytes_per_round(cfg) if len(inc) > 1 else 0
    t_comm = max((1.0 - plan_d["rows"][i] / H) * kvb * plan_d["n_exchange_rounds"]
                 for i in inc) / (NVLINK_GBS * 1e9)
    lb = max(t_total, t_rank, t_comm)
    return {"lb_ms": lb * 1e3, "compute_ms": max(t_total, t_rank) * 1e3, "nvlink_ms": t_comm * 1e3,
            "flops_per_image": sum(Wi.values()), "kv_bytes_per_round": kvb,
            "peak_tflops": peak_tflops, "nvlink_gbs": NVLINK_GBS,
            "bound": "tensor" if max(t_total, t_rank) >= t_comm else "nvlink"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return dict(tflops=float(j["bf16_tflops_sustained"]), tflops_burst=float(j["bf16_tflops"]),
                    hbm=float(j["hbm_gbs"]), src="measured (MEASURED_PEAKS.json)")
    except Exception:
        return dict(tflops=1590.0, tflops_burst=1590.0, hbm=6650.0,
                    src="fallback (B200_PROFILING.md)")


def occupancy_list(spec, n):
    if spec == "zero":
        return [0] * n
    if spec == "half50":
        return [0] * n if n == 1 else [0 if r < n // 2 else 50 for r in range(n)]
    v = [int(x) for x in spec.split(",")]
    assert len(v) == n, "occupancy list must have one entry per GPU"
    return v


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for k, v in zip(names, r[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(k)
            except (ValueError, IndexError):
                continue
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------- oracle legs
def oracle_sample(cfg, rows_lat, seconds_hint=None):
    """Run the fp64 oracle (as it stands) on a bounded sample: the full-width
    latent cut to `rows_lat` rows, depth 1, ONE sequential DDIM step.  Returns
    (seconds, sample FLOPs, threads)."""
    from oracle import stadi as OR
    if cfg["family"] == "unet":
        scfg = configs.model(cfg["name"], latent_h=rows_lat)
        fl = unet_flops(scfg, rows_lat)
    else:
        scfg = configs.model(cfg["name"], depth=1, latent_h=rows_lat)
        hp, wp = configs.tokens_hw(scfg)
        n = hp * wp
        fl = dit_flops(scfg, n, n, configs.batch(scfg))
    W = gen.weights(scfg)
    x = gen.noise(scfg)
    c = gen.cond(scfg)
    t0 = time.perf_counter()
    OR.sequential(scfg, W, x, c, 1)
    dt = time.perf_counter() - t0
    return dt, fl, _blas_threads()


def _sample_rows(cfg):
    """Latent rows of the bounded oracle sample: the smallest legal band."""
    if cfg["family"] == "unet":
        return configs.rows_per_unit(cfg)
    return 32 if cfg["latent_h"] >= 32 else cfg["latent_h"]


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        th = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(th) if th else 1
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(cfg, wl, target_s=15.0):
    """Oracle throughput on a bounded sample, extrapolated per image by FLOPs."""
    rows = _sample_rows(cfg)
    total_t, total_f, reps, th = 0.0, 0.0, 0, 1
    while total_t < target_s and reps < 20:
        dt, fl, th = oracle_sample(cfg, rows)
        total_t += dt
        total_f += fl
        reps += 1
    rate = total_f / total_t                              # fp64 FLOP/s on the host
    ms_img = image_flops(cfg, wl["m_base"]) / rate * 1e3
    return {"value": 1e3 / ms_img, "unit": "images/s", "ms_per_image": ms_img, "cores": th,
            "kind": "oracle",
            "sample": (f"{reps} x oracle.stadi.sequential on a {rows}x{cfg['latent_w']} latent, "
                       f"{'full depth' if cfg['family'] == 'unet' else 'depth 1'}, 1 DDIM step "
                       f"({total_t:.1f} s, {total_f / 1e9:.0f} GFLOP fp64); "
                       f"per-image latency extrapolated by FLOP count to the full workload "
                       f"({image_flops(cfg, wl['m_base']) / 1e12:.0f} TFLOP/image)")}


def run_reference(args, cfg, wl, rank, world):
    """--impl reference: the oracle, as it stands, on this host's cores."""
    if rank != 0:
        return
    rows = _sample_rows(cfg)
    for _ in range(args.warmup):
        oracle_sample(cfg, rows)
    ts, fls, th = [], [], 1
    for _ in range(args.steps):
        dt, fl, th = oracle_sample(cfg, rows)
        ts.append(dt)
        fls.append(fl)
    rate = sum(fls) / sum(ts)
    ms_img = image_flops(cfg, wl["m_base"]) / rate * 1e3
    val = 1e3 / ms_img
    sample = (f"each step = oracle.stadi.sequential on a {rows}x{cfg['latent_w']} latent, depth 1, "
              f"1 DDIM step ({np.mean(ts):.2f} s); per-image latency extrapolated by FLOP count")
    out = {"impl": "reference", "metric": args.metric, "value": val, "unit": "images/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_img,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": wl["name"], "n_gpus": world},
           "cpu_baseline": {"value": val, "unit": "images/s", "cores": th, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": val, "unit": "images/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# --------------------------------------------------------------------- method modes
# PAPER.md §V: Table III ablation (None / +SA / +TA / +TA+SA, L316-L323), Fig. 8 occupancy
# pairs (L292, L310), Fig. 9 forced patch ratios (L325-L333), and the alpha/beta probe of
# the affine sizer (R30).  On ONE physical GPU the ranks are VIRTUAL GPUs: green-context
# SM partitions computing concurrently (paper_2509_04719_b200/vgpu.py), with the
# occupancy emulator holding rho of each partition's SMs -- HBM, L2 and copy engines are
# shared, there is no NVLink hop.  Latency of a request = max over ranks
# of its device time (stadi_run_stats.ms_total), averaged over the timed requests.
FLAGS_ABLATION = [("none", 1 | 2), ("+SA", 1), ("+TA", 2), ("+TA+SA", 0)]
FIG8_PAIRS = [[0, 20], [0, 40], [0, 60], [35, 45], [30, 50], [25, 55]]


class _Group:
    """The ranks of a method run: virtual GPUs on this device (world == 1)."""

    def __init__(self, S, desc, weights, n, sms):
        from paper_2509_04719_b200.vgpu import VirtualGpus
        self.vg = VirtualGpus(desc, n, sms, weights)
        self.n = n

    def call(self, *a, **kw):
        return self.vg.call(*a, **kw)

    def close(self):
        self.vg.close()


def _time_plan(S, grp, plan, x, c, k, w):
    outs = [np.zeros_like(x) for _ in range(grp.n)]
    for _ in range(w):
        grp.call("run", plan, x, c, per_rank=lambda r: {"out": outs[r]})
    lat = []
    for _ in range(k):
        st = grp.call("run", plan, x, c, per_rank=lambda r: {"out": outs[r]})
        lat.append(max(t.ms_total for t in st))
    return float(np.mean(lat)), [float(v) for v in lat]


def run_method(args, cfg, wl, mode=None, pairs=None, steps=None):
    """Returns the method-mode JSON object (see the block comment above)."""
    from paper_2509_04719_b200 import stadi as S
    mode = mode or args.mode
    steps = steps or args.steps
    if pairs is None:
        pairs = ([[int(v) for v in args.occupancy.split(",")]] if "," in args.occupancy
                 else (FIG8_PAIRS if mode == "fig8" else FIG8_PAIRS[:3]))
    n = len(pairs[0])
    sms = args.vgpu_sms or max(8, (112 // n) // 8 * 8)
    mb = args.m_base or wl["m_base"]
    mw = wl["m_warmup"]
    p = configs.rows_per_unit(cfg)
    P = cfg["latent_h"] // p
    x, c = gen.noise(cfg), gen.cond(cfg)
    W = gen.weights(cfg)
    desc = S.model_desc(wl["model"], S.DTYPE_BF16)
    grp = _Group(S, desc, [W[k] for k, _, _ in configs.manifest(cfg)], n, sms)
    del W
    grp.call("profile_warmup", 1, n)        # loads every kernel before any emulator
    rows = []
    t0 = time.time()
    if mode == "replan":
        # SURVEY §8(f)4 dynamic re-planning: the occupancy changes between requests;
        # a static plan (profiled once, under the first setting) vs re-profiling (a
        # 1-step probe) and re-planning before every request
        seq = pairs if len(pairs) > 1 else [[0, 50], [50, 0], [0, 0], [0, 60]][: max(2, len(pairs))]
        static = None
        try:
            for occ in seq:
                grp.call("emulator_start", per_rank=lambda r: {"pct": occ[r]})
                try:
                    tp = time.time()
                    ms, speed = grp.call("profile_warmup", 1, n)[0]
                    t_prof = (time.time() - tp) * 1e3
                    pl = S.plan(speed, mb, mw, P, p)
                    if static is None:
                        static = pl
                    lat_s, _ = _time_plan(S, grp, static, x, c, steps, 1)
                    lat_r, _ = _time_plan(S, grp, pl, x, c, steps, 1)
                    rows.append({"occupancy_pct": occ, "speed_q20": [int(v) for v in speed],
                                 "static": {"plan": _plan_json(static), "ms_per_image": lat_s},
                                 "replanned": {"plan": _plan_json(pl), "ms_per_image": lat_r,
                                               "probe_overhead_ms": t_prof},
                                 "replan_latency_reduction": 1.0 - lat_r / lat_s})
                finally:
                    grp.call("emulator_stop")
        finally:
            grp.close()
        pairs = []
    try:
        for occ in pairs:
            grp.call("emulator_start", per_rank=lambda r: {"pct": occ[r]})
            try:
                ms, speed = grp.call("profile_warmup", 3, n)[0]
                row = {"occupancy_pct": occ, "speed_q20": [int(v) for v in speed],
                       "probe_ms": ms}
                if mode in ("ablation", "fig8", "cfgsplit"):
                    fl = (FLAGS_ABLATION if mode == "ablation" else
                          [("none", 3), ("+TA+SA", 0)] if mode == "fig8" else
                          [("none", 3), ("+TA+SA", 0), ("cfg_split+TA+SA", 32)])
                    for name, f in fl:
                        pl = S.plan(speed, mb, mw, P, p, flags=f)
                        lat, all_ = _time_plan(S, grp, pl, x, c, steps, 1)
                        row[name] = {"ms_per_image": lat, "runs_ms": all_,
                                     "plan": _plan_json(pl)}
                    base = row["none"]["ms_per_image"]
                    for name, _ in fl[1:]:
                        row[name]["speedup_vs_none"] = base / row[name]["ms_per_image"]
                        row[name]["latency_reduction"] = 1.0 - row[name]["ms_per_image"] / base
                elif mode == "fig9":
                    sweep = []
                    for k8 in range(1, 8):   # rank 0 share k/8 of the rows (2 ranks), TA off
                        u0 = max(1, min(P - 1, round(P * k8 / 8)))
                        fu = [u0, P - u0] if n == 2 else None
                        if fu is None:
                            break
                        pl = S.plan(speed, mb, mw, P, p, flags=1 | 8, forced_units=fu)
                        lat, _ = _time_plan(S, grp, pl, x, c, steps, 1)
                        sweep.append({"units": fu, "ms_per_image": lat})
                    pl_sa = S.plan(speed, mb, mw, P, p, flags=1)
                    lat_sa, _ = _time_plan(S, grp, pl_sa, x, c, steps, 1)
                    pl_pp = S.plan(speed, mb, mw, P, p, flags=3)
                    lat_pp, _ = _time_plan(S, grp, pl_pp, x, c, steps, 1)
                    row.update(sweep=sweep, stadi_sa={"units": _plan_json(pl_sa)["units"],
                                                      "ms_per_image": lat_sa},
                               uniform_pp_ms=lat_pp)
                elif mode == "alphabeta":
                    # two probe band heights per rank (complementary forced splits)
                    a_u = [max(1, P // (4 * n)) if r % 2 == 0 else 0 for r in range(n)]
                    rest = P - sum(a_u)
                    odd = [r for r in range(n) if r % 2 == 1] or [n - 1]
                    for r in odd:
                        a_u[r] += rest // len(odd)
                    a_u[odd[-1]] += P - sum(a_u)
                    b_u = list(reversed(a_u)) if n == 2 else a_u[1:] + a_u[:1]
                    ms_a = grp.call("profile_band", 3, a_u)[0]
                    ms_b = grp.call("profile_band", 3, b_u)[0]
                    alpha, beta = [], []
                    for r in range(n):
                        if a_u[r] == b_u[r]:
                            bt = ms_a[r] / a_u[r]
                        else:
                            bt = (ms_b[r] - ms_a[r]) / (b_u[r] - a_u[r])
                        bt = max(bt, 1e-6)
                        alpha.append(max(0.0, ms_a[r] - bt * a_u[r]))
                        beta.append(bt)
                    ns = 1e6  # ms -> integer ns for the C ABI
                    pl_aff = S.plan(speed, mb, mw, P, p, flags=16,
                                    alpha=[int(v * ns) for v in alpha],
                                    beta=[max(1, int(v * ns)) for v in beta])
                    pl_dh = S.plan(speed, mb, mw, P, p)
                    lat_aff, _ = _time_plan(S, grp, pl_aff, x, c, steps, 1)
                    lat_dh, _ = _time_plan(S, grp, pl_dh, x, c, steps, 1)
                    row.update(probe_units=[a_u, b_u], probe_ms=[ms_a, ms_b],
                               alpha_ms=alpha, beta_ms_per_unit=beta,
                               affine={"plan": _plan_json(pl_aff), "ms_per_image": lat_aff},
                               dhondt={"plan": _plan_json(pl_dh), "ms_per_image": lat_dh})
                rows.append(row)
            finally:
                grp.call("emulator_stop")
    finally:
        grp.close()
    out = {"mode": mode, "metric": args.metric, "unit": "ms/image", "n_gpus": 1,
           "virtual_gpus": n, "vgpu_sms": sms, "steps": steps, "m_base": mb,
           "m_warmup": mw, "workload": wl["name"], "results": rows,
           "wall_s": time.time() - t0,
           "note": ("ranks are virtual GPUs: disjoint green-context SM partitions of one B200 "
                    "computing concurrently, occupancy emulated inside each partition; HBM/L2 "
                    "shared, no NVLink hop"),
           "context": PAPER_CONTEXT}
    return out


# --------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOADS))
    ap.add_argument("--occupancy", default="half50")
    ap.add_argument("--transport", default="ipc", choices=["ipc", "nccl"],
                    help="N > 1 exchange transport (IPC: fused one-sided P2P, the default)")
    ap.add_argument("--mode", default="headline",
                    choices=["headline", "ablation", "fig8", "fig9", "alphabeta", "replan",
                             "cfgsplit"],
                    help="method-level measurements on virtual GPUs (one device)")
    ap.add_argument("--vgpu-sms", type=int, default=0, help="SMs per virtual GPU (mult. of 8)")
    ap.add_argument("--m-base", type=int, default=0, help="override the workload's M_base")
    ap.add_argument("--no-method", action="store_true",
                    help="skip the default run's 2-virtual-GPU STADI vs uniform-PP leg")
    ap.add_argument("--no-uniform", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-occ-sweep", action="store_true")
    ap.add_argument("--ncu", action="store_true",
                    help="profiling pass under ncu: 1 untimed request after profiling, no "
                         "uniform / e2e / cpu legs (its numbers are never bench values)")
    args = ap.parse_args()
    if args.ncu:
        args.warmup, args.steps = 0, 1
        args.no_uniform = args.no_e2e = args.no_cpu_baseline = True
    args.metric = "per-image latency ms & images/s at 1/2/4/8 B200 vs uniform patch-par"
    assert args.warmup >= 3 or args.impl == "reference" or args.ncu, "W >= 3 warm-up steps"

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    wl = WORKLOADS[args.workload]
    cfg = configs.model(wl["model"])

    if args.impl == "reference":
        run_reference(args, cfg, wl, rank, world)
        return
    if args.mode != "headline":
        assert world == 1, "method modes run on virtual GPUs of one device"
        print(json.dumps(run_method(args, cfg, wl)), flush=True)
        return

    # stdout carries exactly one JSON line: everything else written to fd 1 (NCCL's
    # "NCCL version" banner at communicator init, library / CUDA messages) goes to
    # stderr; the result is written to the saved stdout at the end
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)

    import torch
    import torch.distributed as dist
    from paper_2509_04719_b200 import stadi as S

    assert torch.cuda.is_available(), "bench.py needs a CUDA device"
    # one rank per GPU; more ranks than GPUs (a functional check of the N > 1 path on a
    # smaller box) share devices round-robin -- never a performance configuration
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        # control plane only (barriers, the ncclUniqueId broadcast, max-over-ranks):
        # gloo on the host, because ProcessGroupNCCL's barrier synchronises the whole
        # device, which never returns while an occupancy-emulator kernel is resident.
        # The data path is the library's own NCCL communicator over NVLink.
        dist.init_process_group("gloo")
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- context.  N > 1: the IPC transport by default (one-sided: the QKV epilogue
    # stores K/V straight into the peers' slots over NVLink, flags by stream memory
    # ops), or the library's NCCL communicator (--transport nccl); the 128-byte
    # session / unique id goes through torch.distributed
    nid = None
    transport = S.TRANSPORT_IPC if args.transport == "ipc" else S.TRANSPORT_NCCL
    if world > 1:
        obj = [(S.ipc_session_id() if transport == S.TRANSPORT_IPC else S.nccl_unique_id())
               if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    desc = S.model_desc(wl["model"], S.DTYPE_BF16)
    ctx = S.Context(desc, rank=rank, world=world, device=local, nccl_id=nid, transport=transport)
    W = gen.weights(cfg)
    ctx.load_weights([W[n] for n, _, _ in configs.manifest(cfg)])
    del W
    x = gen.noise(cfg)
    c = gen.cond(cfg)
    p = configs.rows_per_unit(cfg)          # R6: latent rows per planner unit
    p_total = cfg["latent_h"] // p

    # ---- a9 occupancy emulation, a1 profiling, a2/a3 plans
    occ = occupancy_list(args.occupancy, world)
    # one untimed probe before the emulator starts: every kernel of the path is
    # then loaded (CUDA lazy loading of a kernel first launched while the
    # emulator's resident kernel runs can need a context sync -> deadlock; the
    # library force-loads the SM-count-dependent tcgen05 variants itself)
    ctx.profile_warmup(1, world)
    # host-side buffers of the e2e leg, pinned now: nothing that may synchronise the
    # device (allocator / stream-pool first use) runs while the emulator is resident
    noise_h = torch.from_numpy(x).pin_memory()
    out_h = torch.empty_like(noise_h).pin_memory()
    cond_h = dict(c)
    if "text" in c:
        cond_h = {k: (torch.from_numpy(v).pin_memory() if k != "time_ids" else v)
                  for k, v in c.items()}
    noise_dev = torch.from_numpy(x).cuda()
    cond = dict(c)
    if "text" in c:  # conditioning resident in HBM for the device-timed legs
        cond = {k: (torch.from_numpy(v).cuda() if k != "time_ids" else v) for k, v in c.items()}
    out_dev = torch.empty_like(noise_dev)
    stream = torch.cuda.current_stream()
    e_pre = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e_pre[0].record(stream)
    e_pre[1].record(stream)
    stream.synchronize()

    if occ[rank]:
        ctx.emulator_start(occ[rank])
    barrier()
    ms_prof, speed = ctx.profile_warmup(3, world)
    plan = S.plan(speed, wl["m_base"], wl["m_warmup"], p_total, p)
    uplan = S.plan(speed, wl["m_base"], wl["m_warmup"], p_total, p, flags=S.NO_TA | S.NO_SA)

    # NOTE: stream synchronisation, not torch.cuda.synchronize(): on the ranks with
    # emulated occupancy a persistent spin kernel stays resident on the device for
    # the whole run, so a device-wide sync would never return.  Every kernel of a
    # request runs on `stream` (and the library's comm stream, which joins it).
    def sync():
        stream.synchronize()

    def timed(pl, noise, out, cnd, k, w, ktime=False):
        for _ in range(w):
            ctx.run(pl, noise, cnd, out, stream=stream)
        sync()
        l0 = S.launch_count()
        if ktime:
            ctx.kernel_timing(True)
        barrier()
        sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            ctx.run(pl, noise, cnd, out, stream=stream)
        e1.record(stream)
        sync()
        barrier()
        ms = e0.elapsed_time(e1)
        launches = S.launch_count() - l0
        return max_over_ranks(ms), launches

    # ---- STADI, device-resident inputs: `value` from a clean timed region, then
    # the same K requests again with CUDA events around every launch of the timed
    # kernel classes (their per-launch record overhead would inflate `value` on
    # the launch-heavy workloads, so the two are separate timed regions)
    with ClockSampler(local) as clk:
        ms, launches = timed(plan, noise_dev, out_dev, cond, args.steps, args.warmup)
    ms_img = ms / args.steps
    value = 1e3 / ms_img
    ms_kt, _ = timed(plan, noise_dev, out_dev, cond, args.steps, 0, ktime=True)
    kst = {k: ctx.kernel_stats(k) for k in S.KCLASS}
    ctx.kernel_timing(False)

    # ---- uniform patch parallelism, same kernels (NO_TA | NO_SA)
    uni = None
    if not args.no_uniform:
        ums, _ = timed(uplan, noise_dev, out_dev, cond, args.steps, args.warmup)
        u_img = ums / args.steps
        uni = {"value": 1e3 / u_img, "ms_per_image": u_img, "plan": _plan_json(uplan),
               "stadi_latency_reduction": 1.0 - ms_img / u_img}

    # ---- e2e: through the C ABI with pinned HOST buffers (H2D + D2H inside)
    e2e = None
    if not args.no_e2e:
        ems, _ = timed(plan, noise_h, out_h, cond_h, args.steps, 1)
        h2d = x.nbytes + sum(v.nbytes for v in c.values())
        e2e = {"value": 1e3 / (ems / args.steps), "unit": "images/s",
               "ms_per_image": ems / args.steps, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(x.nbytes)}

    if occ[rank]:
        ctx.emulator_stop()

    # ---- occupancy sweep (N = 1): the single GPU's probe step time under 0/20/40/60%
    # emulated occupancy (a9 + a1), and the plan the planner makes from those measured
    # speeds for a 4-GPU job with one GPU at each level.  The per-image latencies of
    # that job are a PROJECTION (measured per-step ms x rows_i / H x M_i, no exchange
    # cost), labelled as such -- gpurun provides one GPU.
    occ_sweep = None
    if world == 1 and not args.ncu and not args.no_occ_sweep:
        pcts = [0, 20, 40, 60]
        pms = []
        for pct in pcts:
            if pct:
                ctx.emulator_start(pct)
            m_, _ = ctx.profile_warmup(3, 1)
            if pct:
                ctx.emulator_stop()
            pms.append(m_[0])
        sq = [int(round((1 << 20) * min(pms) / v)) for v in pms]
        p4 = S.plan(sq, wl["m_base"], wl["m_warmup"], p_total, p).to_dict()
        u4 = S.plan(sq, wl["m_base"], wl["m_warmup"], p_total, p, flags=S.NO_TA | S.NO_SA).to_dict()
        H = cfg["latent_h"]

        def proj(pd):
            return max(pd["steps"][i] * pms[i] * pd["rows"][i] / H
                       for i in range(4) if pd["tier"][i])
        ts, tu = proj(p4), proj(u4)
        occ_sweep = {"occupancy_pct": pcts, "probe_ms_per_step": pms, "speed_q20": sq,
                     "plan_4gpu": {k: p4[k] for k in ("tier", "steps", "units", "rows")},
                     "projected_4gpu_ms": {"stadi": ts, "uniform_pp": tu,
                                           "stadi_latency_reduction": 1.0 - ts / tu},
                     "note": "probe times measured on this GPU under the emulator; the 4-GPU "
                             "latencies are a compute-only projection, not a measurement"}

    # ---- roofline of the dominant kernel class (largest share of kernel time)
    peaks = load_peaks()
    names = {"attn": "tc_attn_kernel (own Q x full stale K/V, tcgen05/TMEM, TMA)",
             "gemm": "tc_gemm_kernel (tcgen05/TMEM + TMA; linear layers and im2col convs)",
             "xattn": "tc_attn_kernel (cross-attention to the text tokens)"}
    step_kernel_ms = sum(v[1] for v in kst.values())
    dom = max(("attn", "gemm", "xattn"), key=lambda k: kst[k][1])
    n_k, ms_k, fl_k, _ = kst[dom]
    roof = None
    if n_k:
        avg_ms = ms_k / n_k
        ach = fl_k / n_k / (avg_ms * 1e-3) / 1e12
        roof = {"kernel": names[dom], "class": dom, "bound": "tensor", "achieved": ach,
                "peak": peaks["tflops"], "unit": "TFLOP/s", "frac": ach / peaks["tflops"],
                "traffic": _traffic(dom),
                "peak_src": peaks["src"] + ", bf16 dense sustained",
                "flops_per_launch": fl_k / n_k, "avg_launch_ms": avg_ms, "launches": n_k,
                "share_of_kernel_time": ms_k / max(step_kernel_ms, 1e-9),
                "measured_in": "second timed region of the same K requests with per-launch "
                               "CUDA events (stadi_kernel_timing); its wall time: "
                               f"{ms_kt / args.steps:.1f} ms per image"}
    kernels = {k: {"launches": v[0], "ms": v[1],
                   "tflops": (v[2] / (v[1] * 1e-3) / 1e12) if v[1] and v[2] else None,
                   "gbs": (v[3] / (v[1] * 1e-3) / 1e9) if v[1] and v[3] else None}
               for k, v in kst.items()}

    # ---- whole-path roofline: SURVEY §8(d) lower bound of the plan vs measured latency
    path_roof = path_lower_bound(cfg, plan.to_dict(), occ, peaks["tflops"])
    path_roof["frac"] = path_roof["lb_ms"] / ms_img
    if uni is not None:
        ulb = path_lower_bound(cfg, uplan.to_dict(), occ, peaks["tflops"])
        uni["path_roofline"] = dict(ulb, frac=ulb["lb_ms"] / uni["ms_per_image"])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, wl)

    # ---- the method on one device: 2 virtual GPUs (SM partitions), the second at 50%
    # emulated occupancy (C5's "half50" pattern), STADI vs same-kernel uniform PP
    method = None
    if world == 1 and not args.no_method and not args.ncu:
        try:
            method = run_method(args, cfg, wl, mode="fig8", pairs=[[0, 50]], steps=2)
        except Exception as e:  # reported, never silently dropped
            method = {"error": str(e)}

    if rank == 0:
        res = {
            "metric": args.metric, "value": value, "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_img,
            "latency_ms": ms_img, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded noise / T5-shaped text, random-init weights)",
            "config": {"workload": wl["name"], "n_gpus": world, "occupancy_pct": occ,
                       "speed_q20": [int(s) for s in speed], "profile_ms": ms_prof,
                       "plan": _plan_json(plan),
                       "l2": "inputs larger than L2: the K/V slots + bf16 weights streamed per "
                             "image exceed the 126 MB L2 (C5: 8.5 GB + 1.3 GB)",
                       "parallelism": f"stadi-patch{world}",
                       "transport": args.transport if world > 1 else "none"},
            "uniform_pp": uni, "e2e": e2e, "roofline": roof, "path_roofline": path_roof,
            "kernels": kernels,
            "cpu_baseline": cpu, "clocks": clk.summary(), "gpu_launches": int(launches),
            "occupancy_sweep": occ_sweep, "method_vgpu": method,
            "context": PAPER_CONTEXT,
        }
        sys.stdout.flush()
        os.write(json_fd, (json.dumps(res) + "\n").encode())
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def _plan_json(p):
    d = p.to_dict()
    return {k: d[k] for k in ("tier", "steps", "units", "rows", "n_exchange_rounds")}


def _traffic(kernel):
    """DRAM bytes per launch from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


if __name__ == "__main__":
    main()
