"""Classifier-free guidance (a labelled EXTENSION: the reference has no CFG,
SPEC.md:468).  Each video runs a cond and an uncond (zero cond) branch as two
engine slots with their own QuantCache decisions; one DDPM update per video
from eps_u + scale * (eps_c - eps_u).  No oracle exists, so the checks are the
kernel's formula and two exact reductions to the reference-parity path:

  * qcb_cfg_combine == f32(fma(scale, f32(c - u), u)) elementwise;
  * scale = 0: the guided eps IS the uncond eps, so the video's latent and its
    uncond branch's trace equal a plain (non-CFG) run whose cond is zero.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SMALL = {"seed": 3, "model": {"num_blocks": 3, "model_dim": 16, "num_heads": 2,
                              "tokens_per_frame": 4, "frames": 2, "cond_dim": 8},
         "schedule": {"steps": 10},
         "toggles": dict(hlc=True, aigq_weights=True, aigq_acts=True, srap=True)}


def test_cfg_combine_kernel(cuda_dev):
    from paper_2503_06545_b200 import device as D
    rng = np.random.default_rng(0)
    for n in (1, 7, 4096, 100003):
        c = rng.standard_normal(n).astype(np.float32)
        u = rng.standard_normal(n).astype(np.float32)
        for s in (0.0, 1.0, 4.5, -0.75):
            got = D.cfg_combine(torch.as_tensor(c).cuda(), torch.as_tensor(u).cuda(), s)
            dlt = (c - u).astype(np.float32)                     # f32 subtraction
            want = (np.float64(np.float32(s)) * dlt.astype(np.float64) +
                    u.astype(np.float64)).astype(np.float32)     # one rounding (exact in f64)
            assert np.array_equal(got.cpu().numpy(), want), (n, s)


@pytest.mark.parametrize("noise", ["numpy", "device"])
def test_scale_zero_is_the_uncond_run(golden_dir, cuda_dev, noise):
    from paper_2503_06545_b200 import harness
    from paper_2503_06545_b200.engine import EngineOptions
    cfg = harness.parse_config(dict(SMALL, calibration=os.path.join(golden_dir,
                                                                    "calib_small.json")))
    calib = harness.load_calibration(cfg.calibration)
    tog = cfg.toggles_obj()
    rng = np.random.default_rng(5)
    S, d, c = 8, 16, 8
    x0 = torch.as_tensor(rng.standard_normal((2, S, d)).astype(np.float32)).cuda()
    cond = torch.as_tensor(rng.standard_normal((2, c)).astype(np.float32)).cuda()
    seeds = [21, 22]
    eng, _ = harness.build_engine(cfg, tog, calib, max_videos=4,
                                  options=EngineOptions(noise=noise, cfg_scale=0.0))
    got, tr = eng.generate(seeds, x0_dev=x0, cond_dev=cond)
    plain, _ = harness.build_engine(cfg, tog, calib, max_videos=2,
                                    options=EngineOptions(noise=noise))
    want, trp = plain.generate(seeds, x0_dev=x0, cond_dev=torch.zeros_like(cond))
    assert got.shape == want.shape == (2, 2, 4, 16)
    assert np.array_equal(got, want)
    for i in range(2):
        assert [r.to_json_obj() for r in tr[2 * i + 1]] == [r.to_json_obj() for r in trp[i]]
    # the cond branch decides on its own (different cond): its trace exists and is full
    assert len(tr[0]) == len(trp[0])
