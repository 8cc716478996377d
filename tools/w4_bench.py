"""u8 vs nibble-packed W4 weight operand: tcgen05 GEMM time at M = 16384."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_06545_b200 import device as D

M = 16384
for K, Nn in ((1152, 1152), (1152, 4608), (4608, 1152)):
    x = torch.randn(M, K, device="cuda")
    w = torch.randn(K, Nn, device="cuda") / K ** 0.5
    c = torch.ones(K, dtype=torch.float64, device="cuda")
    sg = torch.as_tensor(D.sign_vector(0, D.pow2_floor(K))).cuda()
    (a,) = D.act_quant(x, 8, [(c, sg)])
    out = torch.empty(M, Nn, device="cuda")
    for pack in (False, True):
        pw = D.weight_prep(w, 4, c, sg, pack4=pack)
        for _ in range(3):
            D.gemm_u8(a, pw, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            D.gemm_u8(a, pw, out=out)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        print(json.dumps({"K": K, "N": Nn, "packed_w4": pack, "us": round(us, 2),
                          "tops": round(2 * M * K * Nn / us / 1e6, 1)}), flush=True)
