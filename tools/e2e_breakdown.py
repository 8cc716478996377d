"""Where the e2e (host latents in / host latents + traces out) time goes for
one C3 generate of 4 videos versus the device-resident run: the step loop,
the latent read-back and the trace construction, timed separately."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench
from paper_2503_06545_b200.engine import EngineOptions, QuantCacheEngine
from paper_2503_06545_b200.model import DiTConfig
from paper_2503_06545_b200.sampler import linear_beta_schedule
from paper_2503_06545_b200.schedule import ThresholdConfig, Toggles

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
T = 100
cfg = DiTConfig(seed=0, **bench.C3)
S, d = cfg.seq_len, cfg.model_dim
model = bench.fast_model(torch, cfg)
absmax = {l: {s: np.abs(getattr(b, s)).max(axis=1).astype(np.float64)
              for s in ("sta_q", "sta_k", "sta_v", "sta_o", "ca_q", "ca_k", "ca_v", "ca_o",
                        "ffn1", "ffn2")} for l, b in enumerate(model.blocks)}
sched = linear_beta_schedule(T)
th = ThresholdConfig(delta1=1.17e10, delta2=2.54e10, v_low=9.9e6, v_high=1.9e7)
eng = QuantCacheEngine(model, sched.alpha_bar, Toggles(True, True, True, True), th,
                       {l: 6 for l in range(28)}, absmax, max_videos=B,
                       options=EngineOptions(attention="fast", noise="device"))
x0h = torch.randn((B, S, d), generator=torch.Generator().manual_seed(11)).pin_memory()
ch = torch.randn((B, cfg.cond_dim), generator=torch.Generator().manual_seed(12)).pin_memory()
x0d, cd = x0h.cuda(), ch.cuda()
seeds = lambda k: [k * 10 + i for i in range(B)]
for w in range(2):
    eng.generate(seeds(w), device_noise_seed=w, x0_dev=x0h, cond_dev=ch)
torch.cuda.synchronize()

for rep in range(3):
    t0 = time.perf_counter()
    eng.generate(seeds(5 + rep), device_noise_seed=5, x0_dev=x0d, cond_dev=cd,
                 return_device=True)
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t0

    t0 = time.perf_counter()
    out, vids = eng.generate(seeds(9 + rep), device_noise_seed=9, x0_dev=x0h, cond_dev=ch,
                             return_device=True)
    torch.cuda.synchronize()
    t_loop = time.perf_counter() - t0
    t1 = time.perf_counter()
    host = out.cpu().numpy()
    t_d2h = time.perf_counter() - t1
    t1 = time.perf_counter()
    tr = eng._collect_traces(vids)
    t_tr = time.perf_counter() - t1

    t0 = time.perf_counter()
    eng.generate(seeds(20 + rep), device_noise_seed=20, x0_dev=x0h, cond_dev=ch)
    torch.cuda.synchronize()
    t_e2e = time.perf_counter() - t0
    print(f"rep {rep}: device-input loop {t_dev*1e3:.1f} ms | host-input loop {t_loop*1e3:.1f} ms"
          f" + d2h {t_d2h*1e3:.1f} ms + traces {t_tr*1e3:.1f} ms | full e2e {t_e2e*1e3:.1f} ms"
          f" | records {sum(len(x) for x in tr)}", flush=True)
