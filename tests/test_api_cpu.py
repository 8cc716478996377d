"""Host-side API of the drop-in, mirroring the reference's own unit tests
(pkg/tests/test_harness.py, test_quant.py, test_schedule.py, test_model.py).
No GPU needed: configs, policies, bit allocation, traces, MAC accounting."""

import itertools
import json
import os

import numpy as np
import pytest

from paper_2503_06545_b200 import harness, model as M, schedule as Sch
from paper_2503_06545_b200.errors import BudgetError, ConfigurationError, TraceFormatError
from paper_2503_06545_b200.quant import (BIT_LEVELS, WeightBitPlan, _round_scale_up,
                                          allocate_weight_bits, bit_penalty, round_half_away)


def make_cfg(**kw):
    base = dict(delta1=1.0, delta2=2.0, v_low=10.0, v_high=20.0)
    base.update(kw)
    return Sch.ThresholdConfig(**base)


class TestConfig:  # test_harness.py:45-116
    def test_defaults_and_seed_shorthand(self):
        cfg = harness.parse_config({"seed": 7})
        assert cfg.seeds == {"model": 7, "sampling": 7, "prune": 7}
        assert cfg.model["num_blocks"] == 8 and cfg.schedule["steps"] == 50
        assert cfg.device == {"attention": "precise", "noise": "numpy", "decisions": "per_video",
                              "sampler": "ddpm"}

    @pytest.mark.parametrize("obj", [{"bogus": 1}, {"model": {"bogus": 1}},
                                     {"thresholds": {"nope": 1}}, {"device": {"x": 1}}])
    def test_unknown_keys_rejected(self, obj):
        with pytest.raises(ConfigurationError):
            harness.parse_config(obj)

    @pytest.mark.parametrize("obj", [
        {"model": {"model_dim": 10, "num_heads": 3}}, {"schedule": {"steps": 1}},
        {"schedule": {"beta_start": 0.5, "beta_end": 0.1}},
        {"thresholds": {"delta1": 3.0, "delta2": 1.0}}, {"toggles": {"hlc": 1}},
        {"weight_bits": {"0": 5}}, {"weight_bits": {"0": 8}}, {"bit_budget": 3},
        {"toggles": {"aigq_weights": True}}, {"device": {"attention": "magic"}},
        {"device": {"decisions": "global"}}])
    def test_validation(self, obj):
        with pytest.raises(ConfigurationError):
            harness.parse_config(obj)

    def test_round_trip(self, tmp_path):
        cfg = harness.parse_config({"seed": 3, "weight_bits": {str(i): 6 for i in range(8)}})
        p = tmp_path / "c.json"
        harness.save_config(cfg, p)
        again = harness.load_config(p)
        assert again.to_json_obj() == cfg.to_json_obj()

    def test_bad_json(self, tmp_path):
        p = tmp_path / "bad.json"
        p.write_text("{nope")
        with pytest.raises(ConfigurationError):
            harness.load_config(p)

    def test_thresholds_from_calibration(self, golden_dir):
        cfg = harness.parse_config({"seed": 7})
        cal = harness.load_calibration(os.path.join(golden_dir, "calib_default.json"))
        th = harness.resolve_thresholds(cfg, cal, Sch.Toggles(hlc=True, srap=True))
        assert (th.delta1, th.delta2) == (cal.delta_p33, cal.delta_p66)
        assert (th.v_low, th.v_high) == (cal.v_p25, cal.v_p75)
        with pytest.raises(ConfigurationError):
            harness.resolve_thresholds(cfg, None, Sch.Toggles(hlc=True))

    def test_auto_weight_bits_match_reference(self, golden_dir):
        meta = json.load(open(os.path.join(golden_dir, "runs_meta.json")))
        for cname in ("small", "default"):
            cal = harness.load_calibration(os.path.join(golden_dir, f"calib_{cname}.json"))
            nb = 3 if cname == "small" else 8
            cfg = harness.parse_config({"model": {"num_blocks": nb}})
            got = harness.resolve_weight_bits(cfg, cal)
            want = {int(k): v for k, v in meta[f"{cname}_full"]["weight_bits"].items()}
            assert got == want

    def test_calibration_json_round_trip(self, golden_dir, tmp_path):
        cal = harness.load_calibration(os.path.join(golden_dir, "calib_small.json"))
        p = tmp_path / "cal.json"
        harness.save_calibration(cal, p)
        assert open(p).read() == open(os.path.join(golden_dir, "calib_small.json")).read()


class TestQuantHost:  # test_quant.py:25-42, 182-232
    def test_half_away(self):
        x = np.array([0.5, -0.5, 1.5, -1.5, 2.5, 2.4, -2.6])
        assert np.array_equal(round_half_away(x), [1, -1, 2, -2, 3, 2, -3])

    def test_scale_up(self):
        s = np.random.default_rng(0).uniform(1e-6, 1e3, size=1000)
        r = _round_scale_up(s)
        assert np.all(r >= s) and np.all((r - s) / s < 2.0 ** -15)

    def test_penalties_and_plan(self):
        assert [bit_penalty(b) for b in (4, 6, 8)] == [1.0, 1 / 16, 1 / 256]
        with pytest.raises(BudgetError):
            WeightBitPlan({0: 8, 1: 8}, 15)
        with pytest.raises(BudgetError):
            allocate_weight_bits({0: 1.0, 1: 1.0}, 7)
        assert allocate_weight_bits({0: 1.0, 1: 1.0, 2: 1.0}, 14).bits_per_layer == \
            {0: 6, 1: 4, 2: 4}

    def test_greedy_matches_exhaustive(self):  # criterion 4
        rng = np.random.default_rng(404)
        for _ in range(60):
            sens = {l: float(rng.uniform(0.01, 5.0)) for l in range(4)}
            budget = int(rng.integers(16, 33))
            plan = allocate_weight_bits(sens, budget)
            got = sum(sens[l] * bit_penalty(b) for l, b in plan.bits_per_layer.items())
            best = min(sum(sens[l] * bit_penalty(b) for l, b in enumerate(c))
                       for c in itertools.product(BIT_LEVELS, repeat=4) if sum(c) <= budget)
            assert got == pytest.approx(best, rel=1e-12)


class TestPolicies:  # test_schedule.py / criterion 3 transcriptions
    @pytest.mark.parametrize("kw,name", [
        (dict(delta1=3.0, delta2=2.0), "delta1/delta2"), (dict(theta1=0.9, theta2=0.4), "theta1"),
        (dict(tau_low=0.99, tau_high=0.5), "tau_low"), (dict(v_low=30.0, v_high=20.0), "v_low"),
        (dict(tau_min=5, tau_mid=3), "tau_min"), (dict(bit_min=8, bit_mid=6), "bit_min"),
        (dict(p_base=1.5), "p_base"), (dict(prune_adjust=0.5), "prune_adjust"),
        (dict(history_k=0), "history_k")])
    def test_invariants(self, kw, name):
        with pytest.raises(ConfigurationError, match=name):
            make_cfg(**kw).validate()

    def test_transcriptions(self):
        rng = np.random.default_rng(303)
        cfg = make_cfg()
        for d in np.concatenate([rng.uniform(0, 3, 500), [1.0, 2.0]]):
            want = 6 if d < 1.0 else (3 if d < 2.0 else 1)
            assert Sch.refresh_interval(float(d), cfg) == want
        for s in np.concatenate([rng.uniform(-1, 1, 500), [0.5, 0.98]]):
            want = 1.0 if s > 0.98 else (0.3 if s >= 0.5 else 0.0)
            assert Sch.prune_probability(float(s), cfg) == want
        assert Sch.adapt_prune_rate(5.0, cfg) == pytest.approx(0.6)
        assert Sch.adapt_prune_rate(25.0, cfg) == pytest.approx(0.15)
        assert Sch.activation_bits(0.4, cfg) == 6 and Sch.activation_bits(0.8, cfg) == 4
        assert Sch.redundancy_metric([1.0, 3.0]) == pytest.approx(1 / 3)

    def test_prune_draw_keyed(self, golden_dir):
        f = np.load(os.path.join(golden_dir, "policy.npz"))
        got = np.array([[Sch.prune_draw(s, t, l) for l in range(6)]
                        for s in (0, 3) for t in range(12)])
        assert np.array_equal(got, f["draws"])
        assert np.array_equal(Sch.prune_draw_table(3, 12, 6), f["draws"][12:])

    def test_billing(self):
        cost = M.BlockCost(quantizable=100, fp_always=7)
        assert Sch.billed_macs(cost, 32, 32) == 107 * 1024
        assert Sch.billed_macs(cost, 4, 8) == 100 * 32 + 7 * 1024


class TestModelHost:  # test_model.py
    def test_checksums_match_reference(self, golden_dir):
        meta = json.load(open(os.path.join(golden_dir, "model_meta.json")))
        for name, m in meta.items():
            cfg = M.DiTConfig(**m["cfg"])
            assert M.weight_checksum(M.init_model(cfg)) == m["checksum"], name

    def test_mac_closed_form(self):  # criterion 7 closed form
        cfg = M.DiTConfig()
        s, d, c = cfg.seq_len, cfg.model_dim, cfg.cond_dim
        cost = M.block_mac_cost(cfg)
        assert cost.quantizable == 4 * s * d * d + 2 * s * d * d + 2 * c * d + 8 * s * d * d
        assert cost.fp_always == 2 * s * s * d + 2 * s * d + 6 * d
        assert M.head_mac_cost(cfg) == s * d * d

    def test_snapshot_round_trip(self, tmp_path):
        m = M.init_model(M.DiTConfig(num_blocks=2, model_dim=8, num_heads=2,
                                     tokens_per_frame=2, frames=2, cond_dim=4, seed=5))
        p = tmp_path / "w.bin"
        M.save_weights(m, p)
        assert M.weight_checksum(M.load_weights(p)) == M.weight_checksum(m)
        raw = p.read_bytes()
        p.write_bytes(raw[:-4])
        with pytest.raises(ValueError):
            M.load_weights(p)

    def test_config_validation(self):
        with pytest.raises(ConfigurationError):
            M.DiTConfig(model_dim=10, num_heads=3)
        with pytest.raises(ConfigurationError):
            M.DiTConfig(num_blocks=0)


class TestTraceIO:  # test_harness.py:249-312
    def _trace(self, golden_dir):
        return harness.import_trace(os.path.join(golden_dir, "trace_small_full.jsonl"))

    def test_round_trip_and_replay(self, golden_dir, tmp_path):
        tr = self._trace(golden_dir)
        p = tmp_path / "t.jsonl"
        harness.export_trace(tr, p)
        assert p.read_text() == open(os.path.join(golden_dir, "trace_small_full.jsonl")).read()
        cfg = harness.parse_config({"seed": 3, "model": {
            "num_blocks": 3, "model_dim": 16, "num_heads": 2, "tokens_per_frame": 4,
            "frames": 2, "cond_dim": 8}, "schedule": {"steps": 10}})
        rep = harness.replay_check(tr, cfg)
        assert rep["records"] == len(tr)
        tr[0].macs += 1
        with pytest.raises(TraceFormatError, match="MAC count"):
            harness.replay_check(tr, cfg)

    @pytest.mark.parametrize("line,msg", [
        ("{bad", "invalid JSON"), ('{"t": 1}', "missing fields"),
        ('{"t":1,"layer":0,"action":"skip","D":null,"S":null,"bits":8,"wbits":8,"macs":0}',
         "unknown action"),
        ('{"t":1,"layer":0,"action":"reuse","D":null,"S":null,"bits":8,"wbits":8,"macs":-1}',
         "nonnegative")])
    def test_rejections(self, tmp_path, line, msg):
        p = tmp_path / "t.jsonl"
        p.write_text(line + "\n")
        with pytest.raises(TraceFormatError, match=msg):
            harness.import_trace(p)

    def test_compare_outputs(self):
        a = np.ones((2, 2), np.float32)
        assert harness.compare_outputs(a, a) == (0.0, 99.0)
        mse, psnr = harness.compare_outputs(a, a * 2)
        assert mse == 1.0 and psnr == pytest.approx(0.0)


class TestPolicyStatsErrors:   # schedule.py:67-82, 108-116 error conventions
    def test_shape_and_k_checks(self):
        from paper_2503_06545_b200 import (cumulative_variation, divergence_score,
                                           layer_similarity)
        from paper_2503_06545_b200.errors import DimensionError
        with pytest.raises(DimensionError):
            divergence_score(np.zeros(3), np.zeros(4), 1, np.zeros(2), np.zeros(2))
        with pytest.raises(ValueError):
            divergence_score(np.zeros(3), np.zeros(3), 0, np.zeros(2), np.zeros(2))
        with pytest.raises(DimensionError):
            layer_similarity(np.zeros((2, 3)), np.zeros((3, 2)))
        assert cumulative_variation([], np.zeros(5)) == 0.0
