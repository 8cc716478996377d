"""Host-blocking and device time of torch SDPA backends at the C3 attention shape
(2 videos x 16 heads x 4096 tokens x dh 72, bf16)."""
import json
import time

import torch
from torch.nn.attention import SDPBackend, sdpa_kernel

B, H, S, D = 2, 16, 4096, 72
q, k, v = (torch.randn(B, S, H, D, device="cuda").permute(0, 2, 1, 3).to(torch.bfloat16)
           for _ in range(3))
busy = torch.randn(8192, 8192, device="cuda")
for name, be in [("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                 ("efficient", SDPBackend.EFFICIENT_ATTENTION), ("default", None)]:
    try:
        ctx = sdpa_kernel([be]) if be is not None else torch.autograd.grad_mode.no_grad()
        with ctx:
            for _ in range(3):
                torch.nn.functional.scaled_dot_product_attention(q, k, v)
            torch.cuda.synchronize()
            # host time with a busy GPU queue ahead (does the call block the host?)
            for _ in range(4):
                busy @ busy
            t0 = time.perf_counter()
            torch.nn.functional.scaled_dot_product_attention(q, k, v)
            host = time.perf_counter() - t0
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                torch.nn.functional.scaled_dot_product_attention(q, k, v)
            e1.record()
            torch.cuda.synchronize()
            print(json.dumps({"backend": name, "host_ms": host * 1e3,
                              "device_us": e0.elapsed_time(e1) / 10 * 1e3}))
    except Exception as exc:
        print(json.dumps({"backend": name, "error": str(exc)[:200]}))
