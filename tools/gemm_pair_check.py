"""Run with QCB_GEMM_PAIR=1: CTA-pair (tcgen05 cta_group::2) u8 GEMMs must equal
the oracle's exact integer GEMM for every epilogue mode (prints one JSON line)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import qc_oracle as O
from paper_2503_06545_b200 import _native as N
from paper_2503_06545_b200 import device as D

rng = np.random.default_rng(5)
bad = {}
for M, K, Nn in [(512, 256, 384), (640, 1152, 192), (1024, 128, 512)]:
    x = rng.standard_normal((M, K)).astype(np.float32)
    w = (rng.standard_normal((K, Nn)) / np.sqrt(K)).astype(np.float32)
    pw = D.weight_prep(torch.from_numpy(w).cuda(), 8)
    (a,) = D.act_quant(torch.from_numpy(x).cuda(), 8, [None])
    acc = D.gemm_u8(a, pw, epilogue=N.EPI_ACC).cpu().numpy()
    ca = a.codes[:M, :K].cpu().numpy().astype(np.int64) - int(a.zero[0])
    cw = pw.codes[:Nn, :K].cpu().numpy().astype(np.int64) - pw.zero.cpu().numpy()[:, None]
    want = (ca @ cw.T).astype(np.int32)
    bad[f"{M}x{K}x{Nn}"] = int(np.count_nonzero(acc.view(np.int32) != want))
print(json.dumps({"mismatches": bad}))
