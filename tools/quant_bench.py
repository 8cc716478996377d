"""Microbench: the AIGQ activation quantizer alone at the STDiT block's call
shapes (M = videos x 4096 tokens): the LN-prologue triple output (q/k/v), the
LN single output (ca_q, ffn1), plain K=1152 (sta_o, ca_o) and K=4608 (ffn2).
Prints one JSON line per case with the algorithmic HBM rate (f32 read once,
u8 codes written once per output)."""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_06545_b200 import device as D

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=16384)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--cases", default="")
args = ap.parse_args()
torch.manual_seed(0)
M = args.M
cases = [("qkv_ln", 1152, 3, True), ("ln1", 1152, 1, True), ("plain1152", 1152, 1, False),
         ("plain4608", 4608, 1, False), ("gelu4608", 4608, 1, "gelu")]
for name, K, nout, ln in cases:
    gelu = ln == "gelu"
    ln = ln is True
    if args.cases and name not in args.cases.split(","):
        continue
    x = torch.randn(M, K, device="cuda")
    trs = []
    for o in range(nout):
        c = torch.rand(K, dtype=torch.float64, device="cuda") + 0.5
        sg = torch.as_tensor(D.sign_vector(o, D.pow2_floor(K))).cuda()
        trs.append((c, sg))
    lnp = (torch.rand(K, device="cuda") + 0.5, torch.randn(K, device="cuda") * 0.1) if ln else None
    outs = D.act_quant(x, 8, trs, ln=lnp, mod=(1.1, 0.05), gelu=gelu)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.iters):
        D.act_quant(x, 8, trs, ln=lnp, mod=(1.1, 0.05), out=outs, gelu=gelu)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / args.iters * 1e3
    alg = M * K * 4 + nout * M * K
    print(json.dumps({"case": name, "M": M, "K": K, "n_out": nout, "us": us,
                      "alg_gbs": alg / us / 1e3}), flush=True)
