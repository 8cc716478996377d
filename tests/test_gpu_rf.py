"""Rectified-flow sampling (C5, a labelled EXTENSION: the reference has no flow
sampler).  The engine's sampler="rf" mode runs the same blocks,
head and QuantCache policies, treats the head output as a velocity and takes
one Euler step x - v / T per timestep.  No reference oracle exists for the
loop; the check is against oracle.sample(sampler="rf"), which drives the
reference-restated blocks and policies through the same loop.  Bars as for
DDPM: decisions identical, D / S / V within 1e-9, latents bit-identical."""

import os
from dataclasses import fields

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SMALL = {"seed": 3, "model": {"num_blocks": 3, "model_dim": 16, "num_heads": 2,
                              "tokens_per_frame": 4, "frames": 2, "cond_dim": 8},
         "schedule": {"steps": 10}, "device": {"sampler": "rf"}}


@pytest.mark.parametrize("toggles", [
    dict(hlc=True, aigq_weights=True, aigq_acts=True, srap=True), dict(hlc=True), {}])
def test_rf_engine_matches_oracle_loop(golden_dir, cuda_dev, toggles):
    from oracle import qc_oracle as O
    from paper_2503_06545_b200 import harness
    cfg = harness.parse_config(dict(SMALL, toggles=toggles,
                                    calibration=os.path.join(golden_dir, "calib_small.json")))
    calib = harness.load_calibration(cfg.calibration)
    tog = cfg.toggles_obj()
    res = harness.run_single(cfg, tog, calib)
    got = [r.to_json_obj() for r in res.scheduler.trace]
    thr = harness.resolve_thresholds(cfg, calib, tog)
    th = O.Thresholds(**{f.name: getattr(thr, f.name) for f in fields(O.Thresholds)})
    want, st = O.sample(O.ModelDims(3, 16, 2, 4, 2, 8, cfg.seeds["model"]), 10, th,
                        (tog.hlc, tog.aigq_weights, tog.aigq_acts, tog.srap),
                        seed=cfg.seeds["sampling"], prune_seed=cfg.seeds["prune"],
                        weight_bits=harness.resolve_weight_bits(cfg, calib),
                        act_absmax=calib.act_absmax, sign_seed=cfg.seeds["model"], sampler="rf")
    assert len(st.trace) == len(got)
    for a, b in zip(st.trace, got):
        for k in ("t", "layer", "action", "bits", "wbits", "macs"):
            assert a[k] == b[k], (k, a, b)
        for k in ("D", "S", "V"):
            if a[k] is not None and b[k] is not None:
                assert b[k] == pytest.approx(a[k], rel=1e-9, abs=1e-12), (k, a, b)
    assert np.array_equal(res.output, want)


def test_rf_draws_no_noise(golden_dir, cuda_dev):
    """The flow sampler consumes no noise: numpy- and device-noise modes agree."""
    from paper_2503_06545_b200 import harness
    from paper_2503_06545_b200.engine import EngineOptions
    cfg = harness.parse_config(dict(SMALL, toggles=dict(hlc=True, srap=True),
                                    calibration=os.path.join(golden_dir, "calib_small.json")))
    calib = harness.load_calibration(cfg.calibration)
    outs = []
    for noise in ("numpy", "device"):
        eng, _ = harness.build_engine(cfg, cfg.toggles_obj(), calib, max_videos=2,
                                      options=EngineOptions(noise=noise, sampler="rf"))
        outs.append(eng.generate([4, 9])[0])
    assert np.array_equal(outs[0], outs[1])


def test_rf_with_cfg_scale_zero_is_the_uncond_run(golden_dir, cuda_dev):
    """The two extensions together: rectified flow with guidance 0 equals the
    plain flow run whose cond is zero (latents and the uncond branch's trace)."""
    from paper_2503_06545_b200 import harness
    from paper_2503_06545_b200.engine import EngineOptions
    cfg = harness.parse_config(dict(SMALL, toggles=dict(hlc=True, aigq_weights=True,
                                                        aigq_acts=True, srap=True),
                                    calibration=os.path.join(golden_dir, "calib_small.json")))
    calib = harness.load_calibration(cfg.calibration)
    tog = cfg.toggles_obj()
    rng = np.random.default_rng(9)
    x0 = torch.as_tensor(rng.standard_normal((2, 8, 16)).astype(np.float32)).cuda()
    cond = torch.as_tensor(rng.standard_normal((2, 8)).astype(np.float32)).cuda()
    eng, _ = harness.build_engine(cfg, tog, calib, max_videos=4,
                                  options=EngineOptions(sampler="rf", cfg_scale=0.0))
    got, tr = eng.generate([31, 32], x0_dev=x0, cond_dev=cond)
    plain, _ = harness.build_engine(cfg, tog, calib, max_videos=2,
                                    options=EngineOptions(sampler="rf"))
    want, trp = plain.generate([31, 32], x0_dev=x0, cond_dev=torch.zeros_like(cond))
    assert np.array_equal(got, want)
    for i in range(2):
        assert [r.to_json_obj() for r in tr[2 * i + 1]] == [r.to_json_obj() for r in trp[i]]
