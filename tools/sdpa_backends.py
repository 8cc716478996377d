"""Time the available attention kernels at the STDiT-XL/2 self-attention shape
(B = 2 videos, H = 16, S = 4096, d = 72, bf16)."""
import json
import sys

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

B, H, S, D = 2, 16, 4096, 72
torch.manual_seed(0)
# the engine's layout: [B, S, H, D] rows viewed as [B, H, S, D]
q, k, v = (torch.randn(B, S, H, D, device="cuda", dtype=torch.bfloat16).permute(0, 2, 1, 3)
           for _ in range(3))
flops = 4.0 * B * H * S * S * D


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


ref = F.scaled_dot_product_attention(q, k, v)
for name, be in [("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                 ("efficient", SDPBackend.EFFICIENT_ATTENTION)]:
    try:
        with sdpa_kernel([be]):
            us = timeit(lambda: F.scaled_dot_product_attention(q, k, v))
            err = float((F.scaled_dot_product_attention(q, k, v) - ref).abs().max())
        print(json.dumps({"backend": name, "us": us, "tflops": flops / us / 1e6, "maxdiff": err}))
    except Exception as ex:   # noqa: BLE001
        print(json.dumps({"backend": name, "error": str(ex)[:120]}))
try:
    import flashinfer
    qf, kf, vf = (t.permute(0, 2, 1, 3).reshape(B * S, H, D).contiguous() for t in (q, k, v))
    def fi():
        outs = []
        for b in range(B):
            sl = slice(b * S, (b + 1) * S)
            outs.append(flashinfer.single_prefill_with_kv_cache(qf[sl], kf[sl], vf[sl]))
        return outs
    us = timeit(fi)
    print(json.dumps({"backend": "flashinfer", "us": us, "tflops": flops / us / 1e6}))
except Exception as ex:   # noqa: BLE001
    print(json.dumps({"backend": "flashinfer", "error": str(ex)[:160]}))
