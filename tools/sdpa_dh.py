"""cuDNN SDPA at the target shape (videos x 16 heads x S=16384) for the STDiT
head dim 72 and zero-padded 80 (explicit 1/sqrt(72) scale), with the output
slice copy the engine needs for the padded case."""
import json
import math
import torch
import torch.nn.functional as F

H, S = 16, 16384
for B in (1, 4):
    for dh, scale, sl in ((72, None, False), (80, None, False), (80, 1 / math.sqrt(72), False),
                          (80, 1 / math.sqrt(72), True)):
        q = torch.randn(B, S, H, dh, device="cuda", dtype=torch.bfloat16).permute(0, 2, 1, 3)
        k = torch.randn_like(q)
        v = torch.randn_like(q)

        def run():
            o = F.scaled_dot_product_attention(q, k, v, scale=scale)
            if sl:
                o = o.permute(0, 2, 1, 3)[..., :72].contiguous()
            return o
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(json.dumps({"B": B, "dh": dh, "scale": scale is not None, "slice_copy": sl,
                          "ms": round(ms, 3),
                          "useful_tflops": round(4.0 * B * H * S * S * 72 / ms / 1e9, 1)}),
              flush=True)
