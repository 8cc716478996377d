"""GPU timeline of one C3 generation (2 videos, T = 100) via torch.profiler
(CUPTI): busy vs idle time on the device, and the largest idle gaps with the
kernels on either side.  Thresholds: a bench-style calibration pass."""
import collections
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench
from paper_2503_06545_b200.engine import EngineOptions, QuantCacheEngine
from paper_2503_06545_b200.model import DiTConfig
from paper_2503_06545_b200.sampler import linear_beta_schedule
from paper_2503_06545_b200.schedule import ThresholdConfig, Toggles

T, B = 100, 2
cfg = DiTConfig(seed=0, **bench.C3)
model = bench.fast_model(torch, cfg)
absmax = {l: {s: np.abs(getattr(b, s)).max(axis=1).astype(np.float64)
              for s in ("sta_q", "sta_k", "sta_v", "sta_o", "ca_q", "ca_k", "ca_v", "ca_o",
                        "ffn1", "ffn2")} for l, b in enumerate(model.blocks)}
sched = linear_beta_schedule(T)
wb = {l: 6 for l in range(28)}
opts = EngineOptions(attention="fast", noise="device")
cal = QuantCacheEngine(model, sched.alpha_bar, Toggles(True, True, True, False),
                       ThresholdConfig(0.0, 0.0), wb, absmax, max_videos=B, options=opts)
_, tr = cal.generate([1000], device_noise_seed=1000)
ds = [r.d for r in tr[0] if r.d is not None]
vs = [r.v for r in tr[0] if r.layer == 0 and r.v is not None and r.v > 0]
th = ThresholdConfig(delta1=float(np.percentile(ds, 33)), delta2=float(np.percentile(ds, 66)),
                     v_low=float(np.percentile(vs, 25)), v_high=float(np.percentile(vs, 75)))
del cal
eng = QuantCacheEngine(model, sched.alpha_bar, Toggles(True, True, True, True), th, wb, absmax,
                       max_videos=B, options=opts)
x0 = torch.randn((B, cfg.seq_len, cfg.model_dim), device="cuda")
cond = torch.randn((B, cfg.cond_dim), device="cuda")
for k in range(2):
    eng.generate([0, 1], device_noise_seed=k, x0_dev=x0, cond_dev=cond, return_device=True)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    eng.generate([0, 1], device_noise_seed=5, x0_dev=x0, cond_dev=cond, return_device=True)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
span = ev[-1].time_range.end - ev[0].time_range.start
busy = 0
last_end = ev[0].time_range.start
gaps = []
for a, b in zip(ev, ev[1:]):
    pass
# merge intervals (streams may overlap)
cur_s, cur_e = ev[0].time_range.start, ev[0].time_range.end
prev = ev[0]
for e in ev[1:]:
    s, t = e.time_range.start, e.time_range.end
    if s > cur_e:
        busy += cur_e - cur_s
        gaps.append((s - cur_e, prev.name[:50], e.name[:50]))
        cur_s, cur_e = s, t
    else:
        cur_e = max(cur_e, t)
    if t >= cur_e:
        prev = e
busy += cur_e - cur_s
print(f"span_ms {span / 1e3:.2f} busy_ms {busy / 1e3:.2f} idle_ms {(span - busy) / 1e3:.2f} "
      f"kernels {len(ev)}")
agg = collections.defaultdict(lambda: [0, 0.0])
for g, a, b in gaps:
    k = (a, b)
    agg[k][0] += 1
    agg[k][1] += g
print("top idle transitions (count, total ms, avg us):")
for (a, b), (n, tot) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {n:5d} {tot / 1e3:8.2f} {tot / n:8.1f}  {a} -> {b}")
kt = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    kt[e.name[:60]][0] += 1
    kt[e.name[:60]][1] += e.time_range.end - e.time_range.start
print("top kernels by time (count, ms):")
for k, (n, tot) in sorted(kt.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"  {n:6d} {tot / 1e3:8.2f}  {k}")
