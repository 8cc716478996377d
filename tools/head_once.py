"""One noise-head call at the bench shape (M = 2 x 4096, K = N = 1152), for an
ncu launch list; with --time, CUDA-event timing of back-to-back calls."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_06545_b200 import device as D

torch.manual_seed(0)
a = torch.randn(int(__import__("os").environ.get("HEAD_M", "8192")), 1152, device="cuda")
w = torch.randn(1152, 1152, device="cuda") / 1152 ** 0.5
hw = D.HeadWeights(w)
out = torch.empty(a.shape[0], 1152, device="cuda")
D.head_gemm(a, hw, out=out)
torch.cuda.synchronize()
if "--time" in sys.argv:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        D.head_gemm(a, hw, out=out)
    e1.record()
    torch.cuda.synchronize()
    print("head_us", e0.elapsed_time(e1) / 20 * 1e3)
if "--count" in sys.argv:
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    D.head_gemm(a, hw, out=out, fallback_count=cnt)
    torch.cuda.synchronize()
    print("fallback", int(cnt.item()), "of", a.shape[0] * w.shape[1],
          "frac", int(cnt.item()) / (a.shape[0] * w.shape[1]))
