import sys, os, numpy as np, time, faulthandler
sys.path.insert(0, os.getcwd())
faulthandler.dump_traceback_later(50, exit=True)
from paper_2509_04719_b200 import stadi as S
from paper_2509_04719_b200.vgpu import VirtualGpus
from synth import configs, gen
cfg = configs.model("dit_xl2", depth=2); W, x, c = gen.weights(cfg), gen.noise(cfg), gen.cond(cfg)
speed = [65536, 39322, 60000, 30000]
p = S.plan(speed, 50, 4, 16, 2, flags=S.CFG_SPLIT)
vg = VirtualGpus(S.model_desc("dit_xl2", 0, depth=2), 4, 24, [W[k] for k, _, _ in configs.manifest(cfg)])
print("created", flush=True)
vo = [np.zeros_like(x) for _ in range(4)]
st = vg.call("run", p, x, c, per_rank=lambda r: {"out": vo[r]})
print("ran", [s.ms_total for s in st], flush=True)
vg.close()
