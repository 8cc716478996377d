"""Pin the CPU oracle (oracle/qc_oracle.py) to the reference's own outputs.

Every fixture under tests/golden/ was produced by importing the reference
package (tests/golden/make_golden.py); the known-answer values below are the
reference's unit-test constants (pkg/tests/*.py, cited per test)."""

import json
import os

import numpy as np
import pytest

from oracle import qc_oracle as O


def load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name))


class TestKnownAnswers:
    def test_half_away_ties(self):  # test_quant.py:25-28
        x = np.array([0.5, -0.5, 1.5, -1.5, 2.5, 2.4, -2.6])
        assert np.array_equal(O.rha(x), [1.0, -1.0, 2.0, -2.0, 3.0, 2.0, -3.0])

    def test_hand_params(self):  # test_quant.py:46-59
        s, z = O.act_params(np.array([0.0, 2.0]), 2)
        assert s >= 2.0 / 3.0 and s == pytest.approx(2.0 / 3.0, rel=2e-5) and z == 0
        s, z = O.act_params(np.array([-1.0, 1.0]), 8)
        assert 120 <= z <= 135
        assert O.act_params(np.full(5, 3.0), 8) == (1.0, 0)
        with pytest.raises(ValueError):
            O.act_params(np.zeros((0,)), 8)

    def test_divergence_hand_value(self):  # test_schedule.py:54-59
        d = O.divergence5(np.array([1.0, 2.0, 3.0]), np.array([0.0, 1.0, 2.0]), 2,
                          np.array([0.5, 0.0]), np.array([0.0, 0.0]))
        assert d == pytest.approx(0.75)
        with pytest.raises(ValueError):
            O.divergence5(np.ones(3), np.ones(3), 0, np.ones(3), np.ones(3))

    def test_similarity_and_variation(self):  # test_schedule.py:153-182
        assert O.similarity([1.0, 2.0], [2.0, 4.0]) == pytest.approx(1.0)
        assert O.similarity([1.0, 0.0], [-3.0, 0.0]) == pytest.approx(-1.0)
        assert O.similarity(np.zeros(3), np.ones(3)) == 0.0
        assert O.variation([np.zeros(4), np.ones(4)], np.full(4, 2.0)) == pytest.approx(12.0)
        assert O.variation([], np.ones(3)) == 0.0

    def test_overflow_guard(self):  # test_tensor.py:120-127
        assert not O.overflow_guard(4, 8, 8, 16)
        assert O.overflow_guard(4, 8, 8, 20)


class TestQuantizerFixtures:
    def test_act_params_and_codes(self, golden_dir):
        f = load(golden_dir, "quantizer.npz")
        cases = json.load(open(os.path.join(golden_dir, "quantizer_cases.json")))
        for c in cases:
            i = c["i"]
            x = f["ties_x"] if i == "ties" else f[f"x{i}"]
            s, z = O.act_params(x, c["bits"])
            assert (s, z) == (c["s"], c["z"])
            codes = O.codes_of(x, s, z, c["bits"])
            want = f["ties_codes"] if i == "ties" else f[f"codes{i}"]
            assert np.array_equal(codes, want)
            if i != "ties":
                assert np.array_equal(O.dequant(codes, s, z), f[f"deq{i}"])

    def test_channel_params(self, golden_dir):
        f = load(golden_dir, "quantizer.npz")
        for j, bits in enumerate((8, 6, 4)):
            s, z = O.chan_params(f[f"w{j}"], bits)
            assert np.array_equal(s, f[f"ws{j}"]) and np.array_equal(z, f[f"wz{j}"])
            assert np.array_equal(O.codes_of(f[f"w{j}"], s[None], z[None], bits),
                                  f[f"wcodes{j}"])

    def test_scale_round_up(self, golden_dir):
        f = load(golden_dir, "quantizer.npz")
        assert np.array_equal(O.scale_up16(f["scale_in"]), f["scale_out"])


class TestRotationFixtures:
    def test_dense_and_fwht_match_reference(self, golden_dir):
        f = load(golden_dir, "rotation.npz")
        i = 0
        while f"x{i}" in f:
            x, w, st, seed = f[f"x{i}"], f[f"w{i}"], f[f"stats{i}"], int(f[f"seed{i}"])
            c = O.balance_scales(w, st)
            assert np.array_equal(c, f[f"c{i}"])
            want = f[f"xe{i}"]
            if x.shape[1] <= 1152:
                assert np.array_equal(O.rotate_act(x, c, seed), want)
                assert np.array_equal(O.rotate_weight(w, c, seed), f[f"we{i}"])
            # the device formulation (FWHT) on the same inputs
            assert np.array_equal(O.rotate_act_fwht(x, c, seed), want), i
            i += 1


class TestMatmulFixtures:
    def test_criterion5_cases(self, golden_dir):
        f = load(golden_dir, "matmul_int.npz")
        for n in range(int(f["count"])):
            args = (f[f"ca{n}"], f[f"sa{n}"], f[f"za{n}"], f[f"cw{n}"], f[f"sw{n}"],
                    f[f"zw{n}"])
            want = f[f"out{n}"]
            assert np.array_equal(O.matmul_int_seq(*args), want)
            assert np.array_equal(O.matmul_int_single_rounding(*args), want)

    @pytest.mark.parametrize("name", ["qkv", "fc1", "fc2", "w4a6"])
    def test_c2_slices(self, golden_dir, name):
        f = load(golden_dir, "matmul_int.npz")
        args = tuple(f[f"{name}_{k}"] for k in ("ca", "sa", "za", "cw", "sw", "zw"))
        assert np.array_equal(O.matmul_int_single_rounding(*args), f[f"{name}_out"])


class TestPolicyFixtures:
    def test_reductions(self, golden_dir):
        f = load(golden_dir, "policy.npz")
        for i in range(6):
            a, b, c, k = f[f"a{i}"], f[f"b{i}"], f[f"c{i}"], int(f[f"k{i}"])
            assert O.divergence(a, b, k, c) == pytest.approx(float(f[f"D{i}"]), rel=1e-12)
            assert O.similarity(a, b) == pytest.approx(float(f[f"S{i}"]), rel=1e-12)
            hist = [b, c][: int(f[f"nh{i}"])]
            assert O.variation(hist, a) == pytest.approx(float(f[f"V{i}"]), rel=1e-12)

    def test_draws(self, golden_dir):
        f = load(golden_dir, "policy.npz")
        got = np.array([[O.draw(s, t, l) for l in range(6)] for s in (0, 3) for t in range(12)])
        assert np.array_equal(got, f["draws"])


class TestModelFixtures:
    CFGS = dict(tiny=O.ModelDims(2, 8, 2, 2, 2, 4, 5),
                small=O.ModelDims(3, 16, 2, 4, 2, 8, 3),
                default=O.ModelDims(8, 64, 4, 16, 4, 32, 7))

    @pytest.mark.parametrize("name", ["tiny", "small", "default"])
    def test_block_and_generate(self, golden_dir, name):
        import hashlib
        f = load(golden_dir, "model.npz")
        meta = json.load(open(os.path.join(golden_dir, "model_meta.json")))
        dims = self.CFGS[name]
        blocks, hw, hb = O.init_weights(dims)
        dig = hashlib.sha256()
        for b in blocks:
            for k in O.BLOCK_FIELDS:
                dig.update(b[k].astype("<f4").tobytes())
        dig.update(hw.astype("<f4").tobytes())
        dig.update(hb.astype("<f4").tobytes())
        assert dig.hexdigest() == meta[name]["checksum"]
        assert np.array_equal(O.modulation(7, blocks[0]["mod"]), f[f"{name}_mod7"])
        out = O.block(f[f"{name}_x"], f[f"{name}_cond"], 7, blocks[0], 0, dims.num_heads)
        assert np.array_equal(out, f[f"{name}_out"])
        gen, _ = O.sample(dims, 4, seed=2)
        assert np.array_equal(gen, f[f"{name}_gen4"])


def _oracle_run_args(golden_dir, tog):
    """The run_single wiring (harness.py:416-437) resolved on the host for the
    small config with the reference's calibration, as oracle.sample arguments."""
    from paper_2503_06545_b200 import harness
    from dataclasses import fields
    cfg = harness.parse_config({
        "seed": 3, "model": {"num_blocks": 3, "model_dim": 16, "num_heads": 2,
                             "tokens_per_frame": 4, "frames": 2, "cond_dim": 8},
        "schedule": {"steps": 10}, "toggles": tog,
        "calibration": os.path.join(golden_dir, "calib_small.json")})
    calib = harness.load_calibration(cfg.calibration)
    toggles = cfg.toggles_obj()
    thr = harness.resolve_thresholds(cfg, calib, toggles)
    th = O.Thresholds(**{f.name: getattr(thr, f.name) for f in fields(O.Thresholds)})
    wbits = harness.resolve_weight_bits(cfg, calib) if toggles.aigq_weights else {}
    dims = O.ModelDims(3, 16, 2, 4, 2, 8, cfg.seeds["model"])
    kw = dict(th=th, toggles=(toggles.hlc, toggles.aigq_weights, toggles.aigq_acts,
                              toggles.srap),
              prune_seed=cfg.seeds["prune"], weight_bits=wbits,
              act_absmax=calib.act_absmax if toggles.aigq_weights else None,
              sign_seed=cfg.seeds["model"])
    return dims, cfg.seeds["sampling"], kw


class TestSampler:
    FULL = dict(hlc=True, aigq_weights=True, aigq_acts=True, srap=True)

    def test_full_stack_sample_matches_reference(self, golden_dir):
        """oracle.sample with every toggle reproduces the reference's run_single
        output bit for bit and its trace decision for decision."""
        dims, seed, kw = _oracle_run_args(golden_dir, self.FULL)
        out, st = O.sample(dims, 10, seed=seed, **kw)
        assert np.array_equal(out, load(golden_dir, "runs.npz")["small_full"])
        ref = [json.loads(l) for l in open(os.path.join(golden_dir, "trace_small_full.jsonl"))]
        ref = [r for r in ref if r["layer"] != "head"]
        got = [r for r in st.trace if r["layer"] != "head"]
        assert len(got) == len(ref)
        for a, b in zip(ref, got):
            for k in ("t", "layer", "action", "bits", "wbits", "macs"):
                assert a[k] == b[k], (k, a, b)

    def test_sync_mode_single_video_is_sample(self, golden_dir):
        dims, seed, kw = _oracle_run_args(golden_dir, self.FULL)
        out, _ = O.sample_sync(dims, 10, seeds=[seed], **kw)
        assert np.array_equal(out[0], load(golden_dir, "runs.npz")["small_full"])

    def test_sync_mode_shares_one_path(self, golden_dir):
        """Two videos under one concatenated-batch policy: one trace, and the
        statistics are the reference formulas on the stacked features."""
        dims, seed, kw = _oracle_run_args(golden_dir, self.FULL)
        out, st = O.sample_sync(dims, 10, seeds=[seed, seed + 8], **kw)
        assert out.shape == (2, 2, 4, 16)
        assert len(st.trace) == 10 * (dims.num_blocks + 1)
        solo, _ = O.sample(dims, 10, seed=seed + 8, **kw)
        assert not np.array_equal(out[1], out[0])
        assert np.isfinite(out).all() and np.isfinite(solo).all()


def test_matmul_int_seq_shortcut_equals_the_loop():
    """matmul_int_seq's exact-partial-sum shortcut returns what the explicit
    ascending-k f64 loop of tensor.py:100-112 returns (random codes, zero
    points, 16-bit-significand scales, K up to 2000)."""
    import numpy as np
    from oracle import qc_oracle as O
    rng = np.random.default_rng(7)

    def loop(a_, sa, za, w_, sw, zw):
        a = np.asarray(a_, np.int64) - za
        w = np.asarray(w_, np.int64) - np.asarray(zw, np.int64)
        joint = float(sa) * np.atleast_1d(np.asarray(sw, np.float64))
        acc = np.zeros((a.shape[0], w.shape[1]))
        for k in range(a.shape[1]):
            acc += joint[None, :] * (a[:, k:k + 1] * w[k:k + 1, :])
        return acc.astype(np.float32)
    for _ in range(40):
        M, K, N = rng.integers(1, 24), rng.integers(1, 2000), rng.integers(1, 24)
        ab, wb = int(rng.choice([6, 8])), int(rng.choice([4, 6, 8]))
        a = rng.integers(0, 2 ** ab, (M, K))
        w = rng.integers(0, 2 ** wb, (K, N))
        za, zw = int(rng.integers(0, 2 ** ab)), rng.integers(0, 2 ** wb, N)
        sa, sw = O.scale_up16(rng.uniform(1e-3, 1)), O.scale_up16(rng.uniform(1e-3, 1, N))
        assert np.array_equal(O.matmul_int_seq(a, sa, za, w, sw, zw), loop(a, sa, za, w, sw, zw))


def test_seq_mm_shortcut_equals_the_loop():
    """seq_mm's exact-partial-sum shortcut returns what the ascending-k f64
    loop of tensor.py:43-60 returns: random f32 operands (mostly the loop),
    rotation matrices (the shortcut) and coarse dyadic values (exact sums)."""
    import numpy as np
    from oracle import qc_oracle as O
    rng = np.random.default_rng(3)

    def loop(a, b):
        a64, b64 = np.asarray(a, np.float64), np.asarray(b, np.float64)
        acc = np.zeros((a64.shape[0], b64.shape[1]))
        for k in range(a64.shape[1]):
            acc += a64[:, k:k + 1] * b64[k:k + 1, :]
        return acc.astype(np.float32)
    for t in range(30):
        M, K, N = rng.integers(1, 24), rng.integers(1, 1200), rng.integers(1, 24)
        if t % 3 == 0:
            a = rng.standard_normal((M, K)).astype(np.float32)
            b = rng.standard_normal((K, N)).astype(np.float32)
        elif t % 3 == 1:
            K2 = 1 << int(np.log2(max(K, 2)))
            a = (rng.standard_normal((M, K2)) * np.exp(rng.standard_normal(K2))).astype(np.float32)
            b = O.rotation_dense(K2, t).astype(np.float32)
        else:
            a = (rng.integers(-8, 8, (M, K)) * 2.0 ** -3).astype(np.float32)
            b = (rng.integers(-8, 8, (K, N)) * 2.0 ** -4).astype(np.float32)
        assert np.array_equal(O.seq_mm(a, b), loop(a, b))
