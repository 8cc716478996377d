"""End-to-end parity of the device engine with the REFERENCE on its own
configs: every ablation toggle set of the small config (seed 3) and the
default benchmark config (seed 7), with the reference's calibration.

Bars: decisions (actions, activation bits, weight bits, billed MACs) identical
at every (step, layer); D / S / V within 1e-9 relative (f64 sums in another
order); final latents bit-identical (asserted) -- the stated tolerance if a
future change breaks exactness would be rtol 1e-5 / atol 1e-5."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CASES = [(c, t) for c in ("small", "default")
         for t in ("none", "hlc", "hlc_aigq", "full", "aigq")]
TOGGLES = {"none": {}, "hlc": dict(hlc=True),
           "hlc_aigq": dict(hlc=True, aigq_weights=True, aigq_acts=True),
           "full": dict(hlc=True, aigq_weights=True, aigq_acts=True, srap=True),
           "aigq": dict(aigq_weights=True, aigq_acts=True)}
SMALL = {"seed": 3, "model": {"num_blocks": 3, "model_dim": 16, "num_heads": 2,
                              "tokens_per_frame": 4, "frames": 2, "cond_dim": 8},
         "schedule": {"steps": 10}}


def _cfg(golden_dir, cname, tname):
    from paper_2503_06545_b200 import harness
    base = dict(SMALL) if cname == "small" else {"seed": 7}
    base = dict(base, calibration=os.path.join(golden_dir, f"calib_{cname}.json"),
                toggles=TOGGLES[tname])
    return harness.parse_config(base)


@pytest.fixture(scope="module")
def runs(golden_dir, cuda_dev):
    return np.load(os.path.join(golden_dir, "runs.npz"))


@pytest.mark.parametrize("cname,tname", CASES)
def test_run_matches_reference(golden_dir, runs, cname, tname):
    from paper_2503_06545_b200 import harness
    cfg = _cfg(golden_dir, cname, tname)
    calib = harness.load_calibration(cfg.calibration)
    res = harness.run_single(cfg, cfg.toggles_obj(), calib)
    ref_trace = [json.loads(l) for l in
                 open(os.path.join(golden_dir, f"trace_{cname}_{tname}.jsonl"))]
    got = [r.to_json_obj() for r in res.scheduler.trace]
    assert len(got) == len(ref_trace)
    for a, b in zip(ref_trace, got):
        for k in ("t", "layer", "action", "bits", "wbits", "macs"):
            assert a[k] == b[k], (k, a, b)
        for k in ("D", "S", "V"):
            if a[k] is None:
                assert b[k] is None or (k == "V" and a["layer"] == "head"), (k, a, b)
            else:
                assert b[k] == pytest.approx(a[k], rel=1e-9, abs=1e-12), (k, a, b)
    meta = json.load(open(os.path.join(golden_dir, "runs_meta.json")))[f"{cname}_{tname}"]
    assert res.scheduler.executed_macs() == meta["executed"]
    assert res.scheduler.baseline_macs() == meta["baseline"]
    want = runs[f"{cname}_{tname}"]
    assert res.output.shape == want.shape
    assert np.array_equal(res.output, want), float(np.abs(res.output - want).max())


def test_reference_metrics_reproduced(golden_dir, runs):
    """reference_metrics.json: full-stack MSE / PSNR / bit-weighted MAC speedup."""
    from paper_2503_06545_b200 import harness
    cfg = _cfg(golden_dir, "default", "full")
    calib = harness.load_calibration(cfg.calibration)
    metrics, trace, base, conf = harness.run_benchmark(cfg, calib=calib)
    assert metrics.speedup_mac == 47.54406614227479
    assert metrics.mse_vs_baseline == pytest.approx(32.10987246021118, rel=1e-12)
    assert metrics.psnr_vs_baseline == pytest.approx(12.832895012303487, rel=1e-12)
    # golden_default (sha256 recorded in runs_meta.json) is the disabled path
    import hashlib
    meta = json.load(open(os.path.join(golden_dir, "runs_meta.json")))
    assert hashlib.sha256(base.astype("<f4").tobytes()).hexdigest() == \
        meta["golden_default_sha256"]


def test_batched_videos_match_single(golden_dir):
    """Per-video decisions in one batched engine call equal separate runs."""
    from paper_2503_06545_b200 import harness
    cfg = _cfg(golden_dir, "small", "full")
    calib = harness.load_calibration(cfg.calibration)
    eng, _ = harness.build_engine(cfg, cfg.toggles_obj(), calib, max_videos=3)
    outs, traces = eng.generate([3, 11, 12])
    for i, seed in enumerate([3, 11, 12]):
        e1, _ = harness.build_engine(cfg, cfg.toggles_obj(), calib, max_videos=1)
        o1, t1 = e1.generate([seed])
        assert np.array_equal(outs[i], o1[0])
        assert [r.to_json_obj() for r in traces[i]] == [r.to_json_obj() for r in t1[0]]


def test_repeat_runs_byte_identical(golden_dir):
    """Criterion 9 (test_acceptance.py:256-286) on the device path."""
    from paper_2503_06545_b200 import harness
    cfg = harness.parse_config(dict(SMALL, toggles={"hlc": True, "aigq_acts": True,
                                                     "srap": True},
                                    thresholds={"delta1": 100.0, "delta2": 300.0,
                                                "v_low": 50.0, "v_high": 150.0}))
    a = harness.run_single(cfg, cfg.toggles_obj())
    b = harness.run_single(cfg, cfg.toggles_obj())
    assert a.output.tobytes() == b.output.tobytes()
    assert [r.to_json_obj() for r in a.scheduler.trace] == \
        [r.to_json_obj() for r in b.scheduler.trace]


def _sync_cfg(golden_dir, tname="full"):
    from paper_2503_06545_b200 import harness
    base = dict(SMALL, calibration=os.path.join(golden_dir, "calib_small.json"),
                toggles=TOGGLES[tname], device={"decisions": "synchronized"})
    return harness.parse_config(base)


def test_sync_single_video_equals_per_video(golden_dir, runs):
    """With one video the synchronised mode is the reference run."""
    from paper_2503_06545_b200 import harness
    cfg = _sync_cfg(golden_dir)
    calib = harness.load_calibration(cfg.calibration)
    res = harness.run_single(cfg, cfg.toggles_obj(), calib)
    assert np.array_equal(res.output, runs["small_full"])
    ref_trace = [json.loads(l) for l in
                 open(os.path.join(golden_dir, "trace_small_full.jsonl"))]
    got = [r.to_json_obj() for r in res.scheduler.trace]
    for a, b in zip(ref_trace, got):
        for k in ("t", "layer", "action", "bits", "wbits", "macs"):
            assert a[k] == b[k], (k, a, b)


@pytest.mark.parametrize("tname", ["full", "hlc_aigq"])
def test_sync_mode_matches_concatenated_batch_oracle(golden_dir, tname):
    """Synchronised decisions (north_star: one all-reduce of the decision sums
    per step, every rank on one path) == oracle.sample_sync: the reference
    formulas on the concatenated batch.  Bars: one shared trace, decisions
    identical at every (step, layer), D / S / V within 1e-9 relative, latents
    bit-identical."""
    from dataclasses import fields
    from paper_2503_06545_b200 import harness
    from oracle import qc_oracle as O
    cfg = _sync_cfg(golden_dir, tname)
    calib = harness.load_calibration(cfg.calibration)
    tog = cfg.toggles_obj()
    seeds = [3, 11, 12]
    eng, _ = harness.build_engine(cfg, tog, calib, max_videos=len(seeds))
    outs, traces = eng.generate(seeds)
    thr = harness.resolve_thresholds(cfg, calib, tog)
    th = O.Thresholds(**{f.name: getattr(thr, f.name) for f in fields(O.Thresholds)})
    wbits = harness.resolve_weight_bits(cfg, calib) if tog.aigq_weights else {}
    want, st = O.sample_sync(O.ModelDims(3, 16, 2, 4, 2, 8, cfg.seeds["model"]), 10, th,
                             (tog.hlc, tog.aigq_weights, tog.aigq_acts, tog.srap), seeds,
                             prune_seed=cfg.seeds["prune"], weight_bits=wbits,
                             act_absmax=calib.act_absmax if tog.aigq_weights else None,
                             sign_seed=cfg.seeds["model"])
    for v in range(len(seeds)):
        got = [r.to_json_obj() for r in traces[v]]
        assert got == [r.to_json_obj() for r in traces[0]]      # one path for all
        assert len(got) == len(st.trace)
        for a, b in zip(st.trace, got):
            for k in ("t", "layer", "action", "bits", "wbits", "macs"):
                assert a[k] == b[k], (k, a, b)
            for k in ("D", "S", "V"):
                if a[k] is not None and b[k] is not None:
                    assert b[k] == pytest.approx(a[k], rel=1e-9, abs=1e-12), (k, a, b)
                elif k != "V":
                    assert a[k] is None and b[k] is None, (k, a, b)
        assert np.array_equal(outs[v], want[v]), float(np.abs(outs[v] - want[v]).max())


@pytest.mark.parametrize("cname", ["small", "default"])
def test_device_calibration_matches_reference(golden_dir, cname):
    """harness.calibrate on the device == the reference's calibrate
    (harness.py:298-351, fixtures calib_{small,default}.json): activation
    channel max |x| per (layer, site) exact, delta / variation percentiles and
    per-layer sensitivities within 1e-9 relative (f64 sums in another order)."""
    from paper_2503_06545_b200 import harness
    base = dict(SMALL) if cname == "small" else {"seed": 7}
    cfg = harness.parse_config(base)
    got = harness.calibrate(cfg)
    ref = harness.load_calibration(os.path.join(golden_dir, f"calib_{cname}.json"))
    assert sorted(got.act_absmax) == sorted(ref.act_absmax)
    for l, sites in ref.act_absmax.items():
        assert sorted(got.act_absmax[l]) == sorted(sites)
        for site, arr in sites.items():
            assert np.array_equal(got.act_absmax[l][site], arr), (l, site)
    for a, b in ((got.delta_p33, ref.delta_p33), (got.delta_p66, ref.delta_p66),
                 (got.v_p25, ref.v_p25), (got.v_p75, ref.v_p75)):
        assert a == pytest.approx(b, rel=1e-9)
    assert sorted(got.sensitivities) == sorted(ref.sensitivities)
    for l, v in ref.sensitivities.items():
        assert got.sensitivities[l] == pytest.approx(v, rel=1e-9), l
    assert got.meta == ref.meta


def test_hooked_generate_and_predict_noise(golden_dir, runs):
    """generate(..., collect_features / extra_hooks) and predict_noise run the
    per-block device path (forward.py): bit-identical to the reference's
    full-precision run, hooks see every block and every GEMM site."""
    from paper_2503_06545_b200 import LayerHooks, generate, harness, predict_noise
    from paper_2503_06545_b200.errors import DimensionError
    from paper_2503_06545_b200.forward import _mm
    from paper_2503_06545_b200.model import init_model
    cfg = harness.parse_config(dict(SMALL))
    model, sched = init_model(cfg.model_config()), cfg.noise_schedule()
    seed = cfg.seeds["sampling"]
    feats = []
    out = generate(model, sched, seed=seed, collect_features=feats).cpu().numpy()
    assert np.array_equal(out, runs["small_none"])
    L = model.cfg.num_blocks
    assert [f[0] for f in feats] == list(range(sched.steps - 1, -1, -1))
    assert all(len(f[2]) == L for f in feats)
    calls, seen = [], []
    hooks = LayerHooks(after_block=lambda l, o: seen.append(l),
                       gemm=lambda l, s, a, w: (calls.append((l, s)), _mm(a, w))[1])
    out2 = generate(model, sched, seed=seed, extra_hooks=hooks).cpu().numpy()
    assert np.array_equal(out2, runs["small_none"])
    assert len(calls) == sched.steps * L * 10 and len(seen) == sched.steps * L
    x = feats[0][1]
    with pytest.raises(ValueError):
        predict_noise(x, sched.steps, np.zeros(model.cfg.cond_dim, np.float32), model,
                      total_steps=sched.steps)
    with pytest.raises(DimensionError):
        predict_noise(np.zeros((1, 2, 3), np.float32), 0,
                      np.zeros(model.cfg.cond_dim, np.float32), model)
