"""The Python drop-in API on the device, restating the reference's own tests.

  * matmul_int / compute_minmax_params / quantize / dequantize
    (tensor.py:68-112, quant.py:83-134): pkg/tests/test_tensor.py:94-127,
    test_quant.py:25-99 and acceptance criterion 5 (test_acceptance.py:181-198),
    plus equality with the CPU oracle;
  * QuantRuntime.gemm_fn in its three modes -- integer W+A, weight-only FP,
    activation-only fake quantization (runtime.py:63-81) -- against the
    oracle's QuantSites hook, and its ndarray-in / ndarray-out boundary
    (LayerHooks.gemm, model.py:89-90);
  * the Scheduler's plan_step / observe_block / finalize_step protocol driven
    model-free (test_schedule.py:226-361's drive()) against the oracle's
    PolicyState on identical inputs: identical actions, bits and billed MACs.
"""

import json
import os

import numpy as np
import pytest

from oracle import qc_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def api(cuda_dev):
    import paper_2503_06545_b200 as P
    return P


def host(t):
    d = getattr(t, "data", t)
    return d.cpu().numpy() if isinstance(d, torch.Tensor) else np.asarray(d)


def random_quantized(P, rng, shape, bits, per_channel=False):
    """pkg/tests/test_tensor.py:31-37"""
    x = P.Tensor(rng.uniform(-4.0, 4.0, size=shape).astype(np.float32))
    if per_channel:
        params = P.compute_minmax_params(x, bits, granularity="per-channel", axis=1)
    else:
        params = P.compute_minmax_params(x, bits)
    return P.quantize(x, params)


class TestMatmulInt:
    def test_equals_dequantized_float_path(self, api):
        P = api
        rng = np.random.default_rng(4)
        for _ in range(20):
            m, k, n = (int(v) for v in rng.integers(1, 16, size=3))
            aq = random_quantized(P, rng, (m, k), int(rng.choice([4, 6, 8])))
            wq = random_quantized(P, rng, (k, n), int(rng.choice([4, 6, 8])),
                                  per_channel=bool(rng.integers(2)))
            got = host(P.matmul_int(aq, wq))
            want = host(P.matmul_fp(P.Tensor(P.dequantize(aq)), P.Tensor(P.dequantize(wq))))
            assert np.array_equal(got, want)
            # and the oracle's ascending-k integer GEMM on the same codes
            sw = np.broadcast_to(np.atleast_1d(wq.params.scale), (n,))
            zw = np.broadcast_to(np.atleast_1d(wq.params.zero_point), (n,))
            ref = O.matmul_int_seq(host(aq.codes).astype(np.int64), float(aq.params.scale),
                                   int(aq.params.zero_point), host(wq.codes).astype(np.int64),
                                   sw, zw)
            assert np.array_equal(got, ref)

    def test_criterion_5_integer_kernel_exact(self, api):
        """test_acceptance.py:181-198, same generator and seed."""
        P = api
        rng = np.random.default_rng(505)
        for _ in range(100):
            m, k, n = (int(v) for v in rng.integers(1, 33, size=3))
            abits = int(rng.choice([4, 6, 8]))
            wbits = int(rng.choice([4, 6, 8]))
            a = P.Tensor((rng.standard_normal((m, k)) * rng.uniform(0.1, 10)).astype(np.float32))
            w = P.Tensor((rng.standard_normal((k, n)) * rng.uniform(0.1, 10)).astype(np.float32))
            aq = P.quantize(a, P.compute_minmax_params(a, abits))
            if rng.integers(2):
                wp = P.compute_minmax_params(w, wbits, granularity="per-channel", axis=1)
            else:
                wp = P.compute_minmax_params(w, wbits)
            wq = P.quantize(w, wp)
            got = host(P.matmul_int(aq, wq))
            want = host(P.matmul_fp(P.Tensor(P.dequantize(aq)), P.Tensor(P.dequantize(wq))))
            assert np.array_equal(got, want)

    def test_rejections(self, api):
        """test_tensor.py:105-127: per-channel activations, row-axis weights,
        the accumulator guard, operand types."""
        P = api
        from paper_2503_06545_b200.errors import ConfigurationError
        rng = np.random.default_rng(5)
        aq = random_quantized(P, rng, (3, 4), 8, per_channel=True)
        wq = random_quantized(P, rng, (4, 2), 8)
        with pytest.raises(ConfigurationError):
            P.matmul_int(aq, wq)
        aq = random_quantized(P, rng, (3, 4), 8)
        x = P.Tensor(rng.standard_normal((4, 2)).astype(np.float32))
        params = P.compute_minmax_params(x, 8, granularity="per-channel", axis=0)
        with pytest.raises(ConfigurationError):
            P.matmul_int(aq, P.quantize(x, params))
        a2 = random_quantized(P, rng, (2, 4), 8)
        w2 = random_quantized(P, rng, (4, 2), 8)
        with pytest.raises(ConfigurationError):   # 4 * 255 * 255 needs 19 bits
            P.matmul_int(a2, w2, acc_bits=16)
        P.matmul_int(a2, w2, acc_bits=20)
        with pytest.raises(TypeError):
            P.matmul_int(a2.codes, w2)


class TestQuantizer:
    def test_rounding_helpers(self, api):
        P = api
        from paper_2503_06545_b200.quant import _round_scale_up, round_half_away
        x = np.array([0.5, -0.5, 1.5, -1.5, 2.5, 2.4, -2.6])
        assert np.array_equal(round_half_away(x), [1.0, -1.0, 2.0, -2.0, 3.0, 2.0, -3.0])
        s = np.random.default_rng(0).uniform(1e-6, 1e3, size=1000)
        r = _round_scale_up(s)
        assert np.all(r >= s) and np.all((r - s) / s < 2.0 ** -15)

    def test_hand_params(self, api):
        """test_quant.py:46-59"""
        P = api
        p = P.compute_minmax_params(P.Tensor(np.array([0.0, 2.0])), 2)
        assert float(p.scale) >= 2.0 / 3.0 and float(p.scale) == pytest.approx(2.0 / 3.0, rel=2e-5)
        assert int(p.zero_point) == 0
        p = P.compute_minmax_params(P.Tensor(np.array([-1.0, 1.0])), 8)
        assert 120 <= int(p.zero_point) <= 135
        p = P.compute_minmax_params(P.Tensor(np.full(5, 3.0)), 8)
        assert float(p.scale) == 1.0 and int(p.zero_point) == 0
        with pytest.raises(ValueError):
            P.compute_minmax_params(P.Tensor(np.zeros((0,))), 8)
        p = P.compute_minmax_params(P.Tensor(np.random.default_rng(2).standard_normal((6, 4))
                                             .astype(np.float32)), 8, "per-channel", axis=1)
        assert p.scale.shape == (4,) and p.zero_point.shape == (4,)

    @pytest.mark.parametrize("bits", [2, 4, 6, 8])
    def test_round_trip_and_oracle(self, api, bits):
        """test_quant.py:75-99 plus bit-equality with the oracle's params/codes."""
        P = api
        rng = np.random.default_rng(bits)
        x = rng.uniform(-3.0, 5.0, size=(40, 50)).astype(np.float32)
        params = P.compute_minmax_params(P.Tensor(x), bits)
        q = P.quantize(P.Tensor(x), params)
        s, z = O.act_params(x, bits)
        assert float(params.scale) == s and int(params.zero_point) == z
        assert np.array_equal(host(q.codes).astype(np.int64), O.codes_of(x, s, z, bits))
        deq = host(P.dequantize(q))
        assert np.abs(deq - x).max() <= s / 2 + 1e-6
        assert np.array_equal(deq.astype(np.float64),
                              s * (host(q.codes).astype(np.float64) - z))

    def test_per_channel_round_trip(self, api):
        P = api
        rng = np.random.default_rng(3)
        x = (rng.standard_normal((64, 8)) *
             np.array([0.01, 0.1, 1, 10, 0.5, 2, 5, 0.02])).astype(np.float32)
        params = P.compute_minmax_params(P.Tensor(x), 6, granularity="per-channel", axis=1)
        s, z = O.chan_params(x, 6)
        assert np.array_equal(params.scale, s) and np.array_equal(params.zero_point, z)
        err = np.abs(host(P.dequantize(P.quantize(P.Tensor(x), params))) - x)
        assert np.all(err.max(axis=0) <= params.scale / 2 + 1e-6)


def _small():
    """The reference's small_config (pkg/tests/conftest.py:48-59) and calibration."""
    from paper_2503_06545_b200 import harness
    golden = os.path.join(os.path.dirname(__file__), "golden")
    calib = harness.load_calibration(os.path.join(golden, "calib_small.json"))
    return calib


class TestQuantRuntime:
    @pytest.mark.parametrize("mode", ["w+a", "w", "a"])
    def test_gemm_fn_modes_vs_oracle(self, api, mode):
        P = api
        from paper_2503_06545_b200.model import DiTConfig, init_model
        calib = _small()
        cfg = DiTConfig(num_blocks=3, model_dim=16, num_heads=2, tokens_per_frame=4, frames=2,
                        cond_dim=8, seed=3)
        model = init_model(cfg)
        aw, aa = mode in ("w+a", "w"), mode in ("w+a", "a")
        tog = P.Toggles(aigq_weights=aw, aigq_acts=aa)
        wbits = {l: 6 for l in range(3)}
        rt = P.QuantRuntime(model, tog, wbits, calib.act_absmax, sign_seed=3)
        blocks, _, _ = O.init_weights(O.ModelDims(3, 16, 2, 4, 2, 8, 3))
        qs = O.QuantSites(blocks, aw, aa, wbits, calib.act_absmax, sign_seed=3)
        rng = np.random.default_rng(11)
        for abits in (8, 6, 4):
            hook, ref = rt.gemm_fn(abits), qs.hook(abits)
            for l in range(3):
                for site in ("sta_q", "ca_o", "ffn1", "ffn2", "ca_k"):
                    wt = getattr(model.blocks[l], site)
                    x = rng.standard_normal((8 if site != "ca_k" else 1, wt.shape[0])) \
                        .astype(np.float32)
                    got = hook(l, site, x, wt)
                    assert isinstance(got, np.ndarray) and got.dtype == np.float32
                    assert np.array_equal(got, ref(l, site, x, wt)), (mode, abits, l, site)
                    dev = hook(l, site, torch.as_tensor(x).cuda(), wt)
                    assert isinstance(dev, torch.Tensor) and dev.is_cuda
                    assert np.array_equal(dev.cpu().numpy(), got)

    def test_disabled_returns_none(self, api):
        P = api
        from paper_2503_06545_b200.model import DiTConfig, init_model
        model = init_model(DiTConfig(num_blocks=1, model_dim=16, num_heads=2,
                                     tokens_per_frame=4, frames=2, cond_dim=8, seed=3))
        assert P.QuantRuntime(model, P.Toggles(), {0: 6}).gemm_fn(8) is None


def drive_both(P, sch, ps, steps, layers, rng, shape=(4, 3)):
    """test_schedule.py:226-235's drive(), fed identically to the device
    Scheduler and the oracle PolicyState."""
    for t in range(steps - 1, -1, -1):
        x = rng.standard_normal(shape).astype(np.float32)
        dec = sch.plan_step(t, P.Tensor(x))
        dref = ps.plan(t, x)
        assert dec.actions == dref.actions and dec.abits == dref.abits, t
        for l in range(layers):
            out = rng.standard_normal(shape).astype(np.float32)
            sch.observe_block(t, l, P.Tensor(out), dec)
            ps.observe(t, l, out, dref)
        sch.finalize_step(t, P.Tensor(x), dec)
        ps.finalize(t, x, dref)


class TestSchedulerProtocol:
    CASES = [
        (dict(hlc=True), dict(delta1=0.5, delta2=1.0)),
        (dict(hlc=True), dict(delta1=1e9, delta2=2e9)),
        (dict(hlc=True), dict(delta1=0.0, delta2=0.0)),
        (dict(srap=True), dict(delta1=0.5, delta2=1.0, tau_high=0.1, tau_low=-1.0, p_base=0.5)),
        (dict(srap=True), dict(delta1=0.5, delta2=1.0, tau_high=-1.0, tau_low=-1.0)),
        (dict(aigq_acts=True), dict(delta1=0.5, delta2=1.0, theta1=0.0, theta2=0.0)),
        (dict(hlc=True, aigq_weights=True, aigq_acts=True, srap=True),
         dict(delta1=2.0, delta2=8.0, tau_high=0.2, tau_low=-0.5, p_base=0.4, v_low=20.0,
              v_high=60.0)),
    ]

    @pytest.mark.parametrize("case", range(len(CASES)))
    def test_trace_equals_oracle(self, api, case):
        P = api
        from paper_2503_06545_b200.model import BlockCost
        tog_kw, th_kw = self.CASES[case]
        steps, layers = 10, 4
        th = P.ThresholdConfig(**th_kw)
        wb = {l: (4 if l % 2 else 8) for l in range(layers)}
        sch = P.Scheduler(layers, steps, th, P.Toggles(**tog_kw),
                          BlockCost(quantizable=50, fp_always=5), 10, prune_seed=6,
                          weight_bits=wb)
        ps = O.PolicyState(layers, steps, O.Thresholds(**th_kw), hlc=tog_kw.get("hlc", False),
                           aigq_w=tog_kw.get("aigq_weights", False),
                           aigq_a=tog_kw.get("aigq_acts", False), srap=tog_kw.get("srap", False),
                           quantizable=50, fp_always=5, head_macs=10, prune_seed=6,
                           weight_bits=wb)
        drive_both(P, sch, ps, steps, layers, np.random.default_rng(case))
        got = [(r.t, r.layer, r.action, r.bits, r.wbits, r.macs) for r in sch.trace]
        want = [(r["t"], r["layer"], r["action"], r["bits"], r["wbits"], r["macs"])
                for r in ps.trace]
        assert got == want
        for r, q in zip(sch.trace, ps.trace):
            for a, b in ((r.d, q["D"]), (r.s, q["S"]), (r.v, q["V"])):
                assert (a is None) == (b is None)
                if a is not None:
                    assert a == pytest.approx(b, rel=1e-9, abs=1e-12)
        assert sch.executed_macs() == sum(r["macs"] for r in ps.trace)
        assert sch.baseline_macs() == steps * (layers * 55 * 1024 + 10 * 1024)
