"""qcb_gelu_inplace at the target's ffn1 output (4 videos x 16384 rows x 4608,
f32, N(0,1)-like values), CUDA events; elements/s and GB/s (read + write)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_06545_b200 import device as D  # noqa: E402

rows, cols = 4 * 16384, 4608
g = torch.Generator(device="cuda")
g.manual_seed(0)
base = torch.randn((rows, cols), device="cuda", generator=g)
x = base.clone()
for _ in range(2):
    x.copy_(base)
    D.gelu_inplace(x)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    x.copy_(base)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    D.gelu_inplace(x)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[2]
n = rows * cols
print(json.dumps({"ms": round(ms, 3), "gelem_s": round(n / ms / 1e6, 1),
                  "gbs": round(8 * n / ms / 1e6, 1)}))
