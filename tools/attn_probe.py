"""Attention at the target shape (4 videos x 16 heads x S=16384) by head dim
for cuDNN SDPA (and the other torch SDPA backends where they run), to read
what the library does with dh=72 (padding) before writing our own kernel."""
import json
import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

H, S, B = 16, 16384, 4
for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
    for dh in (64, 72, 80, 96, 128):
        q = torch.randn(B, S, H, dh, device="cuda", dtype=torch.bfloat16).permute(0, 2, 1, 3)
        k = torch.randn_like(q)
        v = torch.randn_like(q)
        try:
            with sdpa_kernel([be]):
                for _ in range(2):
                    F.scaled_dot_product_attention(q, k, v)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(5):
                    F.scaled_dot_product_attention(q, k, v)
                e1.record()
                torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            print(json.dumps({"backend": str(be), "dh": dh, "ms": round(ms, 3),
                              "tflops_at_dh": round(4.0 * B * H * S * S * dh / ms / 1e9, 1)}),
                  flush=True)
        except Exception as ex:   # backend not available for this shape
            print(json.dumps({"backend": str(be), "dh": dh, "error": str(ex)[:120]}), flush=True)
