"""Exhaustive check of the certified GELU fast paths (qcb_gelu_inplace) against
the exact cephes replica (the f64 GEMM's GELU epilogue on a K=1 identity
product, itself pinned to SciPy by tests/test_gpu_kernels.py) over EVERY f32
value in [lo, hi].  usage: python tools/gelu_exhaustive.py [lo hi]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2503_06545_b200 import _native as N
from paper_2503_06545_b200 import device as D

lo = float(sys.argv[1]) if len(sys.argv) > 1 else -14.0
hi = float(sys.argv[2]) if len(sys.argv) > 2 else 6.0
one = torch.ones((1, 1), dtype=torch.float32, device="cuda")
CH = 1 << 22
COLS = 1 << 12


def bits_range(a, b):
    """f32 bit patterns of all values in [a, b] as int64 ranges (sign-split)."""
    out = []
    if a < 0:
        na = np.float32(min(-0.0, b)).view(np.uint32).item()
        nb = np.float32(a).view(np.uint32).item()
        out.append((int(na), int(nb)))           # negative: increasing bits = decreasing value
    if b >= 0:
        pa = np.float32(max(0.0, a)).view(np.uint32).item()
        pb = np.float32(b).view(np.uint32).item()
        out.append((int(pa), int(pb)))
    return out


t0 = time.time()
total = bad = 0
examples = []
for a, b in bits_range(lo, hi):
    for s in range(a, b + 1, CH):
        e = min(b + 1, s + CH)
        u = torch.arange(s, e, dtype=torch.int64, device="cuda").to(torch.int32)
        x = u.view(torch.float32)
        n = x.numel()
        pad = (-n) % COLS
        xx = torch.cat([x, torch.zeros(pad, device="cuda")]).view(-1, COLS)
        fast = xx.clone()
        D.gelu_inplace(fast)
        exact = D.gemm_f64(xx.reshape(-1, 1), one, epilogue=N.EPI_GELU).view(-1, COLS)
        diff = (fast.view(torch.int32) != exact.view(torch.int32)).view(-1)[:n]
        k = int(diff.sum().item())
        total += n
        bad += k
        if k and len(examples) < 5:
            idx = torch.nonzero(diff)[:3].view(-1)
            examples += [(float(x[i]), float(fast.view(-1)[i]), float(exact.view(-1)[i]))
                         for i in idx.tolist()]
print(json.dumps({"range": [lo, hi], "values": total, "mismatches": bad, "examples": examples,
                  "seconds": round(time.time() - t0, 1)}))
