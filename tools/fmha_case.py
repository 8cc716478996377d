"""Run one qcb_attention_bf16 case (debugging): S heads dh nseg stride."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_06545_b200 import device as D  # noqa: E402

S, H, dh, nseg, stride = (int(x) for x in sys.argv[1:6])
g = torch.Generator(device="cuda").manual_seed(1)
q, k, v = (torch.randn((nseg * stride, H * dh), generator=g, device="cuda").to(torch.bfloat16)
           for _ in range(3))
out = D.attention_bf16(q, k, v, H, S, nseg=nseg, seg_stride=stride)
torch.cuda.synchronize()
qq, kk, vv = (t.view(nseg, stride, H, dh)[:, :S].permute(0, 2, 1, 3).float() for t in (q, k, v))
ref = torch.softmax(qq @ kk.transpose(-1, -2) / math.sqrt(dh), -1) @ vv
got = out.view(nseg, stride, H, dh)[:, :S].permute(0, 2, 1, 3).float()
print(S, H, dh, nseg, stride, "max err", (got - ref).abs().max().item(), flush=True)
