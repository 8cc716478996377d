"""Reproduce the engine's attention call pattern and time host blocking."""
import json
import time

import torch

S, Sp, H, D = 4096, 4096, 16, 72
big = [torch.randn(2 * Sp, H * D, device="cuda") for _ in range(3)]
out = torch.empty(2 * Sp, H * D, device="cuda")
busy = torch.randn(8192, 8192, device="cuda")
side = torch.cuda.Stream()


def attn(nseg):
    qq, kk, vv = (t[:nseg * Sp].view(nseg, Sp, H, D)[:, :S].permute(0, 2, 1, 3) for t in big)
    o = torch.nn.functional.scaled_dot_product_attention(
        qq.to(torch.bfloat16), kk.to(torch.bfloat16), vv.to(torch.bfloat16))
    out[:nseg * Sp].view(nseg, Sp, H, D)[:, :S].copy_(o.permute(0, 2, 1, 3))


for nseg in (1, 2, 1, 2):
    attn(nseg)
torch.cuda.synchronize()
for pattern in ([2, 2, 2, 2], [1, 2, 1, 2]):
    hs = []
    for nseg in pattern:
        for _ in range(3):
            busy @ busy
        with torch.cuda.stream(side):
            busy @ busy
        t0 = time.perf_counter()
        attn(nseg)
        hs.append((time.perf_counter() - t0) * 1e3)
    torch.cuda.synchronize()
    print(json.dumps({"pattern": pattern, "host_ms": [round(h, 3) for h in hs]}))
