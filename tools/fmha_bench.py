"""qcb_attention_bf16 vs cuDNN SDPA at the STDiT target shape (videos x 16
heads x S=16384, dh=72), CUDA events, plus the MUFU exp2 bound."""
import json
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
from paper_2503_06545_b200 import device as D  # noqa: E402

import os
H, dh, S = 16, int(os.environ.get("DH", "72")), int(os.environ.get("S", "16384"))
for B in (1, 4):
    d = H * dh
    q, k, v = (torch.randn((B * S, d), device="cuda").to(torch.bfloat16) for _ in range(3))
    out = torch.empty_like(q)
    qq, kk, vv = (t.view(B, S, H, dh).permute(0, 2, 1, 3) for t in (q, k, v))

    def ours():
        D.attention_bf16(q, k, v, H, S, nseg=B, out=out)

    def lib():
        F.scaled_dot_product_attention(qq, kk, vv)

    for name, fn in (("ours", ours), ("sdpa", lib)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(json.dumps({"impl": name, "videos": B, "ms": round(ms, 3),
                          "dh": dh, "tflops": round(4.0 * B * H * S * S * dh / ms / 1e9, 1),
                          "exp2_per_s": round(B * H * S * S / ms / 1e9, 1)}), flush=True)
