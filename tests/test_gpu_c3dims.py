"""End-to-end parity at the production widths:
STDiT-XL/2 block dimensions (d = 1152, 16 heads of 72, FFN 4608) with a short
sequence (2 frames x 64 tokens) and schedule, every QuantCache toggle on, the
reference-parity modes (attention="precise", noise="numpy"), against the
oracle's `sample` restatement of the reference sampler.  At d = 1152 the
engine runs the production kernels the benchmark times (the 1024-wide
rotation quantizer with the numpy-order LN prologue, the u8 GEMM at N = 1152
and 4608, the int8 head) rather than the narrow generic paths of the small
reference configs.

Bars: every (step, layer) decision identical (action, activation / weight
bits, billed MACs); D / S / V within 1e-9 relative; final latent bit-identical."""

from dataclasses import fields

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

MODEL = {"num_blocks": 2, "model_dim": 1152, "num_heads": 16, "tokens_per_frame": 64,
         "frames": 2, "cond_dim": 64}


@pytest.mark.parametrize("tname,toggles", [
    ("full", dict(hlc=True, aigq_weights=True, aigq_acts=True, srap=True)),
    ("aigq", dict(aigq_weights=True, aigq_acts=True))])
def test_c3_width_engine_matches_oracle(cuda_dev, tmp_path, tname, toggles):
    from oracle import qc_oracle as O
    from paper_2503_06545_b200 import harness
    base = {"seed": 11, "model": MODEL, "schedule": {"steps": 6}}
    path = str(tmp_path / "calib.json")
    harness.calibrate(harness.parse_config(base), out_path=path)   # device calibration
    cfg = harness.parse_config(dict(base, calibration=path, toggles=toggles))
    calib = harness.load_calibration(path)
    tog = cfg.toggles_obj()
    res = harness.run_single(cfg, tog, calib)
    got = [r.to_json_obj() for r in res.scheduler.trace]
    thr = harness.resolve_thresholds(cfg, calib, tog)
    th = O.Thresholds(**{f.name: getattr(thr, f.name) for f in fields(O.Thresholds)})
    dims = O.ModelDims(**MODEL, seed=cfg.seeds["model"])
    want, st = O.sample(dims, 6, th, (tog.hlc, tog.aigq_weights, tog.aigq_acts, tog.srap),
                        seed=cfg.seeds["sampling"], prune_seed=cfg.seeds["prune"],
                        weight_bits=harness.resolve_weight_bits(cfg, calib),
                        act_absmax=calib.act_absmax, sign_seed=cfg.seeds["model"])
    assert len(st.trace) == len(got)
    for a, b in zip(st.trace, got):
        for k in ("t", "layer", "action", "bits", "wbits", "macs"):
            assert a[k] == b[k], (k, a, b)
        for k in ("D", "S", "V"):
            if a[k] is not None and b[k] is not None:
                assert b[k] == pytest.approx(a[k], rel=1e-9, abs=1e-12), (k, a, b)
    if tname == "full":   # the toggles do skip work at this width
        assert any(r["action"] != "recompute" for r in st.trace if r["layer"] != "head")
    assert np.array_equal(res.output, want)
