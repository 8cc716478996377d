"""Microbench: one video's DDPM update at the C3 latent size (4096 x 1152 f32),
device-noise mode, CUDA-event timing of back-to-back calls."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_06545_b200 import device as D

n = 4096 * 1152
x = torch.randn(n, device="cuda")
e = torch.randn(n, device="cuda")
outs = [torch.empty(n, device="cuda") for _ in range(8)]
for o in outs:
    D.ddpm(x, e, 0.01, 0.999, None, 0.1, out=o, noise_gen=(5, 0))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for k in range(40):
    D.ddpm(x, e, 0.01, 0.999, None, 0.1, out=outs[k % 8], noise_gen=(5, k * n))
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 40 * 1e3
print("ddpm_us %.2f  alg_GBs %.0f" % (us, 12 * n / us / 1e3))
