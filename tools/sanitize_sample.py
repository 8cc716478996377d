"""Small multi-tile invocations of every kernel family for compute-sanitizer
(one tool per run: memcheck / racecheck / synccheck):

  compute-sanitizer --tool memcheck python tools/sanitize_sample.py

The quantizer (LN + 3 outputs over several row groups per CTA, GELU K=4608,
plain), the u8 GEMM (multi-tile, every epilogue, packed W4, small-M), the
certified head, GELU in place, the reductions, DDPM, the policy kernels and
CFG, via a short full-stack run of the reference's small config."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_06545_b200 import _native as N
from paper_2503_06545_b200 import device as D
from paper_2503_06545_b200 import harness
from paper_2503_06545_b200.engine import EngineOptions


def main():
    torch.manual_seed(0)
    dev = "cuda"
    # quantizer: LN + 3 outputs (several row groups per CTA), GELU K=4608, plain
    x = torch.randn(1024, 1152, device=dev)
    g, b = torch.rand(1152, device=dev) + 0.5, torch.randn(1152, device=dev) * 0.1
    sg = torch.as_tensor(D.sign_vector(0, 1024)).to(dev)
    trs = [(torch.rand(1152, dtype=torch.float64, device=dev) + 0.5, sg) for _ in range(3)]
    qs = D.act_quant(x, 8, trs, nseg=2, ln=(g, b), mod=(1.1, 0.1))
    h = torch.randn(512, 4608, device=dev)
    sg4 = torch.as_tensor(D.sign_vector(0, 4096)).to(dev)
    D.act_quant(h, 6, [(torch.rand(4608, dtype=torch.float64, device=dev) + 0.5, sg4)],
                gelu=True)
    # u8 GEMM: every epilogue, W4 packed, small M
    w = torch.randn(1152, 1152, device=dev) / 34
    pw = D.weight_prep(w, 6, trs[0][0], sg)
    resid = torch.randn(1024, 1152, device=dev)
    for epi in (N.EPI_STORE, N.EPI_GATE_RESID, N.EPI_RESID, N.EPI_ACC, N.EPI_STORE_BF16):
        D.gemm_u8(qs[0], pw, epilogue=epi, resid=resid, gate=0.5, seg_rows=512, seg_valid=500)
    pw4 = D.weight_prep(w, 4, trs[0][0], sg, pack4=True)
    D.gemm_u8(qs[0], pw4)
    (a1,) = D.act_quant(torch.randn(3, 1152, device=dev), 8, [(trs[0][0], sg)], nseg=3)
    D.gemm_u8(a1, pw, seg_rows=1, seg_valid=1)
    # head, GELU in place
    hw = D.HeadWeights(torch.randn(1152, 1152, device=dev) / 34)
    D.head_gemm(x, hw, bias=torch.randn(1152, device=dev) * 0.01, nseg=2)
    D.gelu_inplace(h)
    # full stack (reductions, DDPM, policy kernels), exact and CFG
    golden = os.path.join(ROOT, "tests", "golden")
    cfg = harness.parse_config({
        "seed": 3, "model": {"num_blocks": 3, "model_dim": 16, "num_heads": 2,
                             "tokens_per_frame": 4, "frames": 2, "cond_dim": 8},
        "schedule": {"steps": 10}, "calibration": os.path.join(golden, "calib_small.json"),
        "toggles": {"hlc": True, "aigq_weights": True, "aigq_acts": True, "srap": True}})
    calib = harness.load_calibration(cfg.calibration)
    harness.run_single(cfg, cfg.toggles_obj(), calib)
    eng, _ = harness.build_engine(cfg, cfg.toggles_obj(), calib, max_videos=4,
                                  options=EngineOptions(noise="device", cfg_scale=2.0,
                                                        attention="fast"))
    eng.generate([1, 2])
    torch.cuda.synchronize()
    print("sanitize sample done")


if __name__ == "__main__":
    main()
