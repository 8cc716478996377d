"""Microbench: the f64-accumulating GEMM (reference `mm`) at the noise-head
shape, M = videos x 4096 tokens, K = N = 1152."""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_06545_b200 import device as D

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=8192)
ap.add_argument("--K", type=int, default=1152)
ap.add_argument("--N", type=int, default=1152)
ap.add_argument("--iters", type=int, default=10)
args = ap.parse_args()
torch.manual_seed(0)
a = torch.randn(args.M, args.K, device="cuda")
w = torch.randn(args.K, args.N, device="cuda") / args.K ** 0.5
out = torch.empty(args.M, args.N, device="cuda")
for _ in range(2):
    D.gemm_f64(a, w, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.iters):
    D.gemm_f64(a, w, out=out)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / args.iters * 1e3
ref = (a[:256].double() @ w.double()).float()
print(json.dumps({"M": args.M, "K": args.K, "N": args.N, "us": us,
                  "dfma_tflops": 2 * args.M * args.K * args.N / us / 1e6,
                  "max_abs_diff_vs_torch_f64_256rows": (out[:256] - ref).abs().max().item()}))

# certified int8 head at the same shape (+ bias), vs the f64 kernel, bit-compared
from paper_2503_06545_b200 import _native as Nat
bias = torch.randn(args.N, device="cuda") * 0.1
hw = D.HeadWeights(w)
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
out2 = torch.empty_like(out)
for _ in range(2):
    D.head_gemm(a, hw, out=out2, bias=bias)
torch.cuda.synchronize()
e0.record()
for _ in range(args.iters):
    D.head_gemm(a, hw, out=out2, bias=bias)
e1.record()
torch.cuda.synchronize()
us2 = e0.elapsed_time(e1) / args.iters * 1e3
D.head_gemm(a, hw, out=out2, bias=bias, fallback_count=cnt)
ref = D.gemm_f64(a, w, epilogue=Nat.EPI_BIAS, bias=bias)
same = bool(torch.equal(out2.view(torch.int32), ref.view(torch.int32)))
print(json.dumps({"head_int8_us": us2, "f64_us": us, "speedup": us / us2,
                  "fallback_elements": int(cnt.item()), "elements": args.M * args.N,
                  "bit_identical": same}))
