"""Microbench: the exact in-place GELU at the FFN hidden shape (M x 4608)."""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_06545_b200 import device as D

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=8192)
ap.add_argument("--iters", type=int, default=10)
args = ap.parse_args()
torch.manual_seed(0)
x0 = torch.randn(args.M, 4608, device="cuda") * 1.5
x = x0.clone()
D.gelu_inplace(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
tot = 0.0
for _ in range(args.iters):
    x.copy_(x0)
    e0.record()
    D.gelu_inplace(x)
    e1.record()
    torch.cuda.synchronize()
    tot += e0.elapsed_time(e1)
us = tot / args.iters * 1e3
print(json.dumps({"M": args.M, "N": 4608, "us": us, "gelem_s": args.M * 4608 / us / 1e3,
                  "alg_gbs": args.M * 4608 * 8 / us / 1e3}))
