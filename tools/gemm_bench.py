"""C2 microbench: AIGQ quantizer + tcgen05 u8 GEMM at STDiT-XL/2 shapes,
M = 16384 tokens (one 16-frame 512x512 video), back-to-back launches so the
GPU (not the host) is the bottleneck.  Prints one JSON line per shape."""
import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2503_06545_b200 import _native as N
from paper_2503_06545_b200 import device as D

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=16384)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--shapes", default="1152x1152,1152x4608,4608x1152")
ap.add_argument("--epi", default="store")
ap.add_argument("--bn", type=int, default=0)
args = ap.parse_args()
epi = {"store": N.EPI_STORE, "gelu": N.EPI_GELU, "gate": N.EPI_GATE_RESID, "acc": N.EPI_ACC}[args.epi]
torch.manual_seed(0)
for shp in args.shapes.split(","):
    K, Nn = map(int, shp.split("x"))
    M = args.M
    x = torch.randn(M, K, device="cuda")
    w = torch.randn(K, Nn, device="cuda") / K ** 0.5
    c = torch.ones(K, dtype=torch.float64, device="cuda")
    sg = torch.as_tensor(D.sign_vector(0, D.pow2_floor(K))).cuda()
    pw = D.weight_prep(w, 8, c, sg)
    (a,) = D.act_quant(x, 8, [(c, sg)])
    out = torch.empty(M, Nn, device="cuda")
    resid = torch.randn(M, Nn, device="cuda")
    for _ in range(3):
        D.gemm_u8(a, pw, out=out, epilogue=epi, resid=resid, block_n=args.bn)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.iters):
        D.gemm_u8(a, pw, out=out, epilogue=epi, resid=resid, block_n=args.bn)
    e1.record()
    torch.cuda.synchronize()
    tg = e0.elapsed_time(e1) / args.iters / 1e3
    e0.record()
    for _ in range(args.iters):
        D.act_quant(x, 8, [(c, sg)], out=[a])
    e1.record()
    torch.cuda.synchronize()
    tq = e0.elapsed_time(e1) / args.iters / 1e3
    ops = 2.0 * M * Nn * K
    qbytes = M * K * 4 + M * K  # algorithmic: read f32 once, write u8 once
    print(json.dumps({"shape": f"{M}x{K}x{Nn}", "epi": args.epi, "gemm_us": tg * 1e6,
                      "gemm_tops": ops / tg / 1e12, "quant_us": tq * 1e6,
                      "quant_alg_gbs": qbytes / tq / 1e9,
                      "block_n": args.bn or "auto"}), flush=True)
