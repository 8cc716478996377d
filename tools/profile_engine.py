"""Per-phase device/host timing of one C3 QuantCache generation (profiling aid).

Uses bench.py's C3 model and synthetic calibration with fixed thresholds taken
from a bench calibration pass, so the run is short enough for an ncu launch list."""
import argparse
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench
from paper_2503_06545_b200 import device as Dv
from paper_2503_06545_b200.engine import EngineOptions, QuantCacheEngine
from paper_2503_06545_b200.model import DiTConfig
from paper_2503_06545_b200.sampler import linear_beta_schedule
from paper_2503_06545_b200.schedule import ThresholdConfig, Toggles

ap = argparse.ArgumentParser()
ap.add_argument("--timesteps", type=int, default=20)
ap.add_argument("--videos", type=int, default=1)
ap.add_argument("--recompute-all", action="store_true")
args = ap.parse_args()
cfg = DiTConfig(seed=0, **bench.C3)
model = bench.fast_model(torch, cfg)
absmax = {l: {s: np.abs(getattr(b, s)).max(axis=1).astype(np.float64)
              for s in ("sta_q", "sta_k", "sta_v", "sta_o", "ca_q", "ca_k", "ca_v", "ca_o",
                        "ffn1", "ffn2")} for l, b in enumerate(model.blocks)}
sched = linear_beta_schedule(args.timesteps)
if args.recompute_all:
    th = ThresholdConfig(delta1=0.0, delta2=0.0)
    tog = Toggles(hlc=True, aigq_weights=True, aigq_acts=True, srap=False)
else:
    th = ThresholdConfig(delta1=1.17e10, delta2=2.54e10, v_low=6.8e6, v_high=1.3e7)
    tog = Toggles(True, True, True, True)
eng = QuantCacheEngine(model, sched.alpha_bar, tog, th, {l: 6 for l in range(28)}, absmax,
                       max_videos=args.videos,
                       options=EngineOptions(attention="fast", noise="device"))
seeds = list(range(args.videos))
eng.generate(seeds, device_noise_seed=0, return_device=True)   # warm-up
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
l0 = Dv.LAUNCHES[0]
t0 = time.perf_counter()
e0.record()
_, vids = eng.generate(seeds, device_noise_seed=1, return_device=True)
e1.record()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
tr = eng.traces_of(vids)
rec = sum(r.action == "recompute" for t in tr for r in t if r.layer != "head")
print(json.dumps({"timesteps": args.timesteps, "videos": args.videos,
                  "device_ms": e0.elapsed_time(e1), "wall_ms": wall * 1e3,
                  "launches": Dv.LAUNCHES[0] - l0, "recomputed_blocks": rec,
                  "blocks": args.timesteps * 28 * args.videos}))
