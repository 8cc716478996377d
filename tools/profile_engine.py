"""Host-side profile of one C3 QuantCache generation (4 videos, T = 100):
cProfile of generate() plus the device time, to find the Python work on the
critical path between a step's decision sync and its first launch."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2503_06545_b200.engine import EngineOptions, QuantCacheEngine  # noqa: E402
from paper_2503_06545_b200.model import DiTConfig  # noqa: E402
from paper_2503_06545_b200.sampler import linear_beta_schedule  # noqa: E402
from paper_2503_06545_b200.schedule import ThresholdConfig, Toggles  # noqa: E402

cfg = DiTConfig(seed=0, **bench.model_dims("c3"))
model = bench.fast_model(cfg)
absmax = bench.synthetic_absmax(model)
sched = linear_beta_schedule(100)
th = ThresholdConfig(delta1=11740291439.2, delta2=25524842316.4, v_low=9995031.5,
                     v_high=18937808.3)
eng = QuantCacheEngine(model, sched.alpha_bar, Toggles(True, True, True, True), th,
                       {l: 6 for l in range(28)}, absmax, max_videos=4,
                       options=EngineOptions(attention="fast", noise="device"))
g = torch.Generator(device="cuda").manual_seed(1)
x0 = torch.randn((4, cfg.seq_len, cfg.model_dim), device="cuda", generator=g)
cond = torch.randn((4, cfg.cond_dim), device="cuda", generator=g)
eng.generate([1, 2, 3, 4], x0_dev=x0, cond_dev=cond, return_device=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
eng.generate([5, 6, 7, 8], x0_dev=x0, cond_dev=cond, return_device=True)
torch.cuda.synchronize()
print("wall ms", (time.perf_counter() - t0) * 1e3)
pr = cProfile.Profile()
pr.enable()
eng.generate([9, 10, 11, 12], x0_dev=x0, cond_dev=cond, return_device=True)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
