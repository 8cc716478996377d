"""Device kernels vs the CPU oracle / reference golden fixtures, through the C ABI.

Bar: bit-exact for codes, params and integer accumulators; bit-exact f32
outputs for the GEMM epilogue (the reference's f64 sum equals the single
rounding whenever its partial sums are exact -- pinned on these fixtures)."""

import json
import os

import numpy as np
import pytest

from oracle import qc_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def D(cuda_dev):
    from paper_2503_06545_b200 import device
    return device


def t(a, dt=None):
    x = torch.from_numpy(np.ascontiguousarray(a))
    if dt is not None:
        x = x.to(dt)
    return x.cuda()


def act_from_codes(D, codes, s, z):
    """Device ActCodes from host codes (test-side construction)."""
    M, K = codes.shape
    buf = np.zeros((M, D.round16(K)), np.uint8)
    buf[:, :K] = codes
    return D.ActCodes(t(buf), t(codes.astype(np.int64).sum(1).astype(np.int32)),
                      t(np.array([s], np.float64)), t(np.array([z], np.int32)), K)


def packed_from_codes(D, codes_kn, s, z, bits=8):
    """Device PackedWeight from host [K][N] codes."""
    K, Nn = codes_kn.shape
    buf = np.zeros((Nn, D.round16(K)), np.uint8)
    buf[:, :K] = codes_kn.T
    return D.PackedWeight(t(buf), t(np.asarray(s, np.float64)), t(np.asarray(z, np.int32)),
                          t(codes_kn.astype(np.int64).sum(0).astype(np.int32)), K, Nn, bits)


class TestGemmU8:
    def test_criterion5_fixtures_exact(self, D, golden_dir):
        f = np.load(os.path.join(golden_dir, "matmul_int.npz"))
        from paper_2503_06545_b200 import _native as N
        for n in range(int(f["count"])):
            ca, cw = f[f"ca{n}"], f[f"cw{n}"]
            sa, za = float(f[f"sa{n}"]), int(f[f"za{n}"])
            a = act_from_codes(D, ca, sa, za)
            w = packed_from_codes(D, cw, f[f"sw{n}"], f[f"zw{n}"])
            acc = D.gemm_u8(a, w, epilogue=N.EPI_ACC).cpu().numpy()
            assert np.array_equal(acc, O.int_acc(ca, za, cw, f[f"zw{n}"])), n
            out = D.gemm_u8(a, w).cpu().numpy()
            assert np.array_equal(out, f[f"out{n}"]), n

    @pytest.mark.parametrize("name", ["qkv", "fc1", "fc2", "w4a6"])
    def test_c2_slices_exact(self, D, golden_dir, name):
        f = np.load(os.path.join(golden_dir, "matmul_int.npz"))
        ca, cw = f[f"{name}_ca"], f[f"{name}_cw"]
        a = act_from_codes(D, ca, float(f[f"{name}_sa"]), int(f[f"{name}_za"]))
        w = packed_from_codes(D, cw, f[f"{name}_sw"], f[f"{name}_zw"])
        out = D.gemm_u8(a, w).cpu().numpy()
        assert np.array_equal(out, f[f"{name}_out"])

    @pytest.mark.parametrize("M,K,N,bn", [(2048, 1152, 1152, 0), (1024, 4608, 1152, 0),
                                          (640, 1152, 4608, 256), (300, 200, 72, 0),
                                          (256, 1152, 1152, 128), (256, 1152, 1152, 64),
                                          (2, 4096, 1152, 0), (5, 200, 72, 0),
                                          (16, 1152, 300, 0)])
    def test_random_accumulators_exact(self, D, M, K, N, bn):
        from paper_2503_06545_b200 import _native as Nat
        rng = np.random.default_rng(M + K + N)
        ca = rng.integers(0, 256, size=(M, K), dtype=np.int64)
        cw = rng.integers(0, 256, size=(K, N), dtype=np.int64)
        za, zw = 117, rng.integers(0, 256, size=N)
        a = act_from_codes(D, ca.astype(np.uint8), 0.01, za)
        w = packed_from_codes(D, cw.astype(np.uint8), np.full(N, 0.02), zw)
        acc = D.gemm_u8(a, w, epilogue=Nat.EPI_ACC, block_n=bn).cpu().numpy()
        rows = np.r_[0:64, M - 64:M] if M > 128 else np.arange(M)
        assert np.array_equal(acc[rows], O.int_acc(ca[rows], za, cw, zw))
        # full check via exact f64 products of integers (< 2^53)
        full = (torch.from_numpy((ca - za).astype(np.float64)).cuda() @
                torch.from_numpy((cw - zw[None]).astype(np.float64)).cuda()).cpu().numpy()
        assert np.array_equal(acc.astype(np.float64), full)

    def test_small_m_segments(self, D):
        """One row per video (the cross-attention K/V of the cond token):
        small-M path with per-segment params, gate and residual epilogues."""
        from paper_2503_06545_b200 import _native as Nat
        rng = np.random.default_rng(31)
        nseg, K, N = 3, 4096, 200
        ca = rng.integers(0, 256, size=(nseg, K)).astype(np.uint8)
        cw = rng.integers(0, 64, size=(K, N)).astype(np.uint8)
        sa = np.array([2.0 ** -7, 3.0 * 2.0 ** -9, 0.015625], np.float64)
        za = np.array([3, 140, 17], np.int32)
        sw = O.scale_up16(rng.uniform(1e-3, 1e-2, size=N))
        zw = rng.integers(0, 64, size=N).astype(np.int32)
        a = D.ActCodes(t(np.pad(ca, ((0, 0), (0, D.round16(K) - K)))),
                       t(ca.astype(np.int64).sum(1).astype(np.int32)), t(sa), t(za), K)
        w = packed_from_codes(D, cw, sw, zw)
        want_y = np.concatenate([O.matmul_int_single_rounding(
            ca[v:v + 1], sa[v], za[v], cw, sw, zw) for v in range(nseg)])
        resid = rng.standard_normal((nseg, N)).astype(np.float32)
        gates = np.array([0.5, -1.25, 0.37], np.float32)
        for mode in (Nat.EPI_STORE, Nat.EPI_GATE_RESID, Nat.EPI_RESID):
            out = torch.zeros((nseg, N), dtype=torch.float32, device="cuda")
            D.gemm_u8(a, w, out=out, epilogue=mode, resid=t(resid), gate_vec=t(gates),
                      seg_rows=1, seg_valid=1)
            got = out.cpu().numpy()
            if mode == Nat.EPI_STORE:
                want = want_y
            elif mode == Nat.EPI_GATE_RESID:
                want = resid + gates[:, None] * want_y
            else:
                want = resid + want_y
            assert np.array_equal(got, want), mode

    def test_segments_and_epilogues(self, D):
        """Per-video params, padded segments, GELU / gate+residual / residual."""
        from paper_2503_06545_b200 import _native as Nat
        rng = np.random.default_rng(3)
        S, Spad, nseg, K, N = 100, 128, 3, 256, 96
        ca = rng.integers(0, 64, size=(nseg * Spad, K)).astype(np.uint8)
        cw = rng.integers(0, 64, size=(K, N)).astype(np.uint8)
        sa = np.array([2.0 ** -7, 3.0 * 2.0 ** -9, 0.015625], np.float64)
        za = np.array([3, 40, 17], np.int32)
        sw = O.scale_up16(rng.uniform(1e-3, 1e-2, size=N))
        zw = rng.integers(0, 64, size=N).astype(np.int32)
        a = D.ActCodes(t(np.pad(ca, ((0, 0), (0, D.round16(K) - K)))),
                       t(ca.astype(np.int64).sum(1).astype(np.int32)), t(sa), t(za), K)
        w = packed_from_codes(D, cw, sw, zw)
        resid = rng.standard_normal((nseg * Spad, N)).astype(np.float32)
        want_y = np.concatenate([O.matmul_int_single_rounding(
            ca[v * Spad:(v + 1) * Spad], sa[v], za[v], cw, sw, zw) for v in range(nseg)])
        for mode in (Nat.EPI_STORE, Nat.EPI_GELU, Nat.EPI_GATE_RESID, Nat.EPI_RESID):
            out = torch.zeros((nseg * Spad, N), dtype=torch.float32, device="cuda")
            D.gemm_u8(a, w, out=out, epilogue=mode, resid=t(resid), gate=np.float32(0.37),
                      seg_rows=Spad, seg_valid=S)
            got = out.cpu().numpy()
            if mode == Nat.EPI_STORE:
                want = want_y
            elif mode == Nat.EPI_GELU:
                want = O.gelu64(want_y)
            elif mode == Nat.EPI_GATE_RESID:
                want = resid + np.float32(0.37) * want_y
            else:
                want = resid + want_y
            for v in range(nseg):   # padding rows (S..Spad) are scratch, not checked
                sl = slice(v * Spad, v * Spad + S)
                assert np.array_equal(got[sl], want[sl]), (mode, v)

    def test_overflow_guard(self, D):
        from paper_2503_06545_b200.errors import ConfigurationError
        K = 40000
        a = D.ActCodes(torch.zeros((128, D.round16(K)), dtype=torch.uint8, device="cuda"),
                       torch.zeros(128, dtype=torch.int32, device="cuda"),
                       torch.ones(1, dtype=torch.float64, device="cuda"),
                       torch.zeros(1, dtype=torch.int32, device="cuda"), K)
        w = D.PackedWeight(torch.zeros((32, D.round16(K)), dtype=torch.uint8, device="cuda"),
                           torch.ones(32, dtype=torch.float64, device="cuda"),
                           torch.zeros(32, dtype=torch.int32, device="cuda"),
                           torch.zeros(32, dtype=torch.int32, device="cuda"), K, 32, 8)
        with pytest.raises(ConfigurationError):
            D.gemm_u8(a, w)


class TestActQuant:
    def test_quantizer_fixtures(self, D, golden_dir):
        f = np.load(os.path.join(golden_dir, "quantizer.npz"))
        cases = json.load(open(os.path.join(golden_dir, "quantizer_cases.json")))
        for c in cases:
            i = c["i"]
            x = f["ties_x"].reshape(1, -1) if i == "ties" else f[f"x{i}"]
            want = (f["ties_codes"].reshape(1, -1) if i == "ties" else f[f"codes{i}"])
            (r,) = D.act_quant(t(x), c["bits"], [None], want_deq=True)
            assert float(r.scale.item()) == c["s"] and int(r.zero.item()) == c["z"], i
            K = x.shape[1]
            assert np.array_equal(r.codes.cpu().numpy()[:, :K], want), i
            assert np.array_equal(r.rowsum.cpu().numpy(), want.astype(np.int64).sum(1)), i
            if i != "ties":
                assert np.array_equal(r.deq.cpu().numpy(), f[f"deq{i}"]), i

    def test_rotation_fixtures(self, D, golden_dir):
        f = np.load(os.path.join(golden_dir, "rotation.npz"))
        i = 0
        while f"x{i}" in f:
            x, c, seed = f[f"x{i}"], f[f"c{i}"], int(f[f"seed{i}"])
            K = x.shape[1]
            signs = D.sign_vector(seed, D.pow2_floor(K))
            for bits in (8, 6, 4):
                (r,) = D.act_quant(t(x), bits, [(t(c), t(signs))], want_xe=True)
                xe = r.xe.cpu().numpy()
                assert np.array_equal(xe, f[f"xe{i}"]), (i, bits)
                s, z = O.act_params(xe, bits)
                assert (float(r.scale.item()), int(r.zero.item())) == (s, z)
                assert np.array_equal(r.codes.cpu().numpy()[:, :K], O.codes_of(xe, s, z, bits))
            i += 1

    def test_ln_mod_prologue_three_outputs(self, D):
        rng = np.random.default_rng(11)
        S, K, nseg = 64, 1152, 2
        x = (rng.standard_normal((nseg * S, K)) * 3 + 0.5).astype(np.float32)
        g = rng.uniform(0.5, 1.5, K).astype(np.float32)
        b = rng.standard_normal(K).astype(np.float32) * 0.1
        s1, sh = np.float32(1.0) + np.float32(0.173), np.float32(-0.31)
        trs = []
        for o in range(3):
            c = rng.uniform(0.1, 4.0, K)
            trs.append((c, D.sign_vector(7 + o, 1024)))
        res = D.act_quant(t(x), 6, [(t(c), t(sg)) for c, sg in trs], nseg=nseg,
                          ln=(t(g), t(b)), mod=(s1, sh), want_xe=True)
        for v in range(nseg):
            xv = x[v * S:(v + 1) * S]
            h = O.ln64(xv, g, b) * s1 + sh
            for o, (c, sg) in enumerate(trs):
                xe_want = O.rotate_act_fwht(h, c, 7 + o)
                xe = res[o].xe.cpu().numpy()[v * S:(v + 1) * S]
                assert np.array_equal(xe, xe_want), (v, o)
                s, z = O.act_params(xe_want, 6)
                assert float(res[o].scale[v]) == s and int(res[o].zero[v]) == z
                codes = res[o].codes.cpu().numpy()[v * S:(v + 1) * S, :K]
                assert np.array_equal(codes, O.codes_of(xe_want, s, z, 6))


    @pytest.mark.parametrize("K,bits", [(1152, 8), (4608, 6), (2304, 4), (1024, 8)])
    def test_v2_gelu_prologue_rows_segments(self, D, K, bits):
        """Register-FWHT path (b = 1024/2048/4096): GELU prologue, rows gathered
        through a per-segment row table, per-segment params, vs the oracle."""
        rng = np.random.default_rng(K + bits)
        S, Spad, nseg = 40, 64, 3
        src = (rng.standard_normal((5 * Spad, K)) * 1.7).astype(np.float32)
        row0 = np.array([3 * Spad, 0, Spad], np.int64)      # segment -> first source row
        c = rng.uniform(0.2, 3.0, K)
        b = D.pow2_floor(K)
        sg = D.sign_vector(11, b)
        (r,) = D.act_quant(t(src), bits, [(t(c), t(sg))], seg_rows=Spad, seg_valid=S,
                           nseg=nseg, x_row0=t(row0), gelu=True)
        codes = r.codes.cpu().numpy()
        for v in range(nseg):
            xin = src[row0[v]:row0[v] + S]
            h = O.gelu64(xin)
            xe = O.rotate_act_fwht(h, c, 11)
            s, z = O.act_params(xe, bits)
            assert float(r.scale[v]) == s and int(r.zero[v]) == z, v
            want = O.codes_of(xe, s, z, bits)
            got = codes[v * Spad:v * Spad + S, :K]
            assert np.array_equal(got, want), (v, int((got != want).sum()))
            assert np.array_equal(r.rowsum.cpu().numpy()[v * Spad:v * Spad + S],
                                  want.sum(1))

    def test_v2_identity_transform_and_deq(self, D):
        rng = np.random.default_rng(3)
        x = rng.standard_normal((70, 1152)).astype(np.float32)
        (r,) = D.act_quant(t(x), 8, [None], want_deq=True)
        s, z = O.act_params(x, 8)
        codes = O.codes_of(x, s, z, 8)
        assert float(r.scale.item()) == s and int(r.zero.item()) == z
        assert np.array_equal(r.codes.cpu().numpy()[:, :1152], codes)
        assert np.array_equal(r.deq.cpu().numpy(), O.dequant(codes, s, z))


class TestWeightPrep:
    def test_rotation_and_channel_quant(self, D, golden_dir):
        f = np.load(os.path.join(golden_dir, "rotation.npz"))
        i = 0
        while f"x{i}" in f:
            if f"we{i}" in f:
                w, c, seed = f[f"w{i}"], f[f"c{i}"], int(f[f"seed{i}"])
                K = w.shape[0]
                signs = D.sign_vector(seed, D.pow2_floor(K))
                for bits in (8, 6, 4):
                    pw = D.weight_prep(t(w), bits, t(c), t(signs), keep_eff=True, keep_deq=True)
                    weff = pw.w_eff.cpu().numpy()
                    assert np.array_equal(weff, f[f"we{i}"]), (i, bits)
                    s, z = O.chan_params(weff, bits)
                    assert np.array_equal(pw.scale.cpu().numpy(), s)
                    assert np.array_equal(pw.zero.cpu().numpy(), z)
                    codes = O.codes_of(weff, s[None], z[None], bits)
                    assert np.array_equal(pw.codes.cpu().numpy()[:, :K], codes.T)
                    assert np.array_equal(pw.colsum.cpu().numpy(), codes.sum(0))
                    assert np.array_equal(pw.w_deq.cpu().numpy(), O.dequant(codes, s[None], z[None]))
            i += 1


class TestSiteFixtures:
    def test_every_hook_call_of_a_quantized_step(self, D, golden_dir):
        """The reference's QuantRuntime.gemm_fn outputs on the small config,
        reproduced by weight_prep -> act_quant -> gemm_u8 on identical inputs."""
        f = np.load(os.path.join(golden_dir, "gemm_sites.npz"))
        meta = json.load(open(os.path.join(golden_dir, "gemm_sites.json")))
        seed = meta["sign_seed"]
        blocks, _, _ = O.init_weights(O.ModelDims(3, 16, 2, 4, 2, 8, 3))
        packed = {}
        for call in meta["calls"]:
            l, site, ab = call["layer"], call["site"], call["abits"]
            key = (l, site)
            c = f[f"w_{l}_{site}_c"]
            K = c.shape[0]
            signs = D.sign_vector(seed, D.pow2_floor(K))
            if key not in packed:
                packed[key] = D.weight_prep(t(blocks[l][site]), call["wbits"], t(c), t(signs))
                assert np.array_equal(packed[key].codes.cpu().numpy()[:, :K],
                                      f[f"w_{l}_{site}_codes"].T)
            k = call["key"]
            (a,) = D.act_quant(t(f[k + "_x"]), ab, [(t(c), t(signs))])
            assert float(a.scale.item()) == call["s"] and int(a.zero.item()) == call["z"]
            assert np.array_equal(a.codes.cpu().numpy()[:, :K], f[k + "_codes"])
            out = D.gemm_u8(a, packed[key]).cpu().numpy()
            assert np.array_equal(out, f[k + "_out"]), (l, site, ab)


class TestFp:
    def test_gemm_f64_matches_seq_mm(self, D):
        rng = np.random.default_rng(5)
        for (m, k, n) in [(3, 4, 5), (64, 64, 256), (70, 256, 64), (1, 8, 16), (300, 1152, 900)]:
            a = rng.standard_normal((m, k)).astype(np.float32)
            w = rng.standard_normal((k, n)).astype(np.float32)
            assert np.array_equal(D.gemm_f64(t(a), t(w)).cpu().numpy(), O.seq_mm(a, w))

    @pytest.mark.parametrize("case", ["normal", "dynamic_range", "cancellation", "odd_k"])
    def test_head_gemm_certified_exact(self, D, case):
        """model.py:228 noise head via certified int8 digit GEMMs == mm + bias bit
        for bit (tensor.py:43-60), incl. padded segments and the exact fallback."""
        from paper_2503_06545_b200 import _native as Nat
        rng = np.random.default_rng({"normal": 1, "dynamic_range": 2, "cancellation": 3,
                                     "odd_k": 4}[case])
        nseg, seg_rows, seg_valid, N = 2, 160, 150, 264
        K = 200 if case == "odd_k" else 1152
        x = rng.standard_normal((nseg * seg_rows, K)).astype(np.float32) * 3
        w = (rng.standard_normal((K, N)) / np.sqrt(K)).astype(np.float32)
        b = (rng.standard_normal(N) * 0.1).astype(np.float32)
        if case == "dynamic_range":
            x[::7] *= np.float32(1e-6)
            x[3, ::5] = np.float32(1e-30)
            x[5] = 0.0
            x[9, :K // 2] *= np.float32(1e6)
            w[:, 4] = 0.0
            w[::11, 8] *= np.float32(1e-9)
        elif case == "cancellation":
            # rows whose products cancel to (near) zero and to values near f32 ties
            x[1::2, K // 2:] = x[1::2, :K // 2]
            w[K // 2:, ::3] = -w[:K // 2, ::3]
            w[K // 2:, 1::3] = -w[:K // 2, 1::3] * np.float32(1 + 2 ** -20)
        hw = D.HeadWeights(t(w))
        cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
        got = D.head_gemm(t(x), hw, bias=t(b), seg_rows=seg_rows, seg_valid=seg_valid,
                          nseg=nseg, fallback_count=cnt).cpu().numpy()
        want = D.gemm_f64(t(x), t(w), epilogue=Nat.EPI_BIAS, bias=t(b), seg_rows=seg_rows,
                          seg_valid=seg_valid).cpu().numpy()
        valid = np.concatenate([np.arange(v * seg_rows, v * seg_rows + seg_valid)
                                for v in range(nseg)])
        assert np.array_equal(got[valid].view(np.int32), want[valid].view(np.int32)), \
            (case, int(cnt.item()))
        # the oracle's sequential mm on a few rows (pins gemm_f64 too)
        rows = valid[[0, 3, 5, 9, 151]] if case not in ("normal", "odd_k") else valid[:4]
        ref = O.seq_mm(x[rows], w) + b
        assert np.array_equal(got[rows], ref)
        if case == "cancellation":
            assert cnt.item() > 0   # the exact fallback ran
        # fallback_count accumulates across calls
        before = int(cnt.item())
        D.head_gemm(t(x), hw, bias=t(b), seg_rows=seg_rows, seg_valid=seg_valid, nseg=nseg,
                    fallback_count=cnt)
        assert int(cnt.item()) == 2 * before

    def test_attention_matches_reference(self, D):
        rng = np.random.default_rng(6)
        for S, Skv, d, h in [(8, 8, 16, 2), (64, 64, 64, 4), (64, 1, 64, 4), (200, 200, 32, 2),
                             (300, 300, 1152, 16), (128, 1, 1152, 16)]:
            q, k, v = (rng.standard_normal((n, d)).astype(np.float32) for n in (S, Skv, Skv))
            got = D.attention_f64(t(q), t(k), t(v), h).cpu().numpy()
            want = O.attention_heads(q, k, v, h)
            assert np.array_equal(got, want), (S, Skv, d, h)   # bit-exact (f64 softmax)

    def test_gelu_inplace_exact(self, D):
        """f32(gelu_f64(x)) with SciPy's erf (model.py:145-147), all regions."""
        rng = np.random.default_rng(12)
        x = np.concatenate([
            rng.standard_normal(300_000) * 2.0, rng.uniform(-40, 40, 50_000),
            rng.uniform(-14, -1.4, 1_000_000), rng.standard_normal(1_000_000) * 3.0,
            np.linspace(-1.4143, -1.4141, 2001), np.linspace(1.4141, 1.4143, 2001),
            np.linspace(5.99, 6.01, 2001), [0.0, -0.0, 1e-30, -1e-30, 37.0, -37.0, -39.0]])
        x = x.astype(np.float32)
        cols = 1000
        pad = (-len(x)) % cols
        buf = np.concatenate([x, np.zeros(pad, np.float32)]).reshape(-1, cols)
        dev = torch.zeros((buf.shape[0], 1024), dtype=torch.float32, device="cuda")
        dev[:, :cols] = t(buf)
        D.gelu_inplace(dev, cols=cols)
        got = dev[:, :cols].cpu().numpy().reshape(-1)[:len(x)]
        want = O.gelu64(x)
        bad = np.flatnonzero(got.view(np.int32) != want.view(np.int32))
        assert bad.size == 0, (bad.size, x[bad[:5]], got[bad[:5]], want[bad[:5]])

    @pytest.mark.parametrize("M,K,Nn", [(8192, 1152, 1152), (640, 256, 200), (4096, 128, 384)])
    def test_gemm_bf16_epilogue(self, D, M, K, Nn):
        """EPI_STORE_BF16 (q/k/v for the bf16 attention path) == bf16(the exact f32
        epilogue output), incl. segment padding rows and ragged N."""
        from paper_2503_06545_b200 import _native as Nat
        rng = np.random.default_rng(M + Nn)
        x = rng.standard_normal((M, K)).astype(np.float32)
        w = (rng.standard_normal((K, Nn)) / np.sqrt(K)).astype(np.float32)
        pw = D.weight_prep(t(w), 8)
        seg_rows = 256 if M % 256 == 0 else M
        seg_valid = seg_rows - 16 if M % 256 == 0 else M
        nseg = M // seg_rows
        (a,) = D.act_quant(t(x), 8, [None], seg_rows=seg_rows, seg_valid=seg_valid, nseg=nseg)
        f32 = D.gemm_u8(a, pw, M=M, seg_rows=seg_rows, seg_valid=seg_valid)
        b16 = D.gemm_u8(a, pw, M=M, epilogue=Nat.EPI_STORE_BF16, seg_rows=seg_rows,
                        seg_valid=seg_valid)
        assert b16.dtype == torch.bfloat16
        valid = np.concatenate([np.arange(v * seg_rows, v * seg_rows + seg_valid)
                                for v in range(nseg)])
        assert torch.equal(b16[valid], f32[valid].to(torch.bfloat16))

    def test_gemm_cta_pair_exact(self, D):
        """The opt-in CTA-pair GEMM (tcgen05 cta_group::2, QCB_GEMM_PAIR=1) gives
        the exact integer accumulators (run in a subprocess: the switch is read
        once per process)."""
        import subprocess, sys
        env = dict(os.environ, QCB_GEMM_PAIR="1")
        out = subprocess.run([sys.executable, "tools/gemm_pair_check.py"], capture_output=True,
                             text=True, timeout=300, env=env,
                             cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        res = json.loads(out.stdout.strip().splitlines()[-1])
        assert all(v == 0 for v in res["mismatches"].values()), res

    def test_gelu_exhaustive_vs_replica(self, D):
        """Every f32 in [-14, 6] (2.18e9 values): the certified fast GELU paths
        equal the exact cephes replica (f64 GEMM GELU epilogue on a K=1 identity
        product; pinned to SciPy above).  -0.0 is excluded: that product turns it
        into +0.0 before the epilogue."""
        import subprocess, sys
        out = subprocess.run([sys.executable, "tools/gelu_exhaustive.py", "-14", "6"],
                             capture_output=True, text=True, timeout=600,
                             cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        res = json.loads(out.stdout.strip().splitlines()[-1])
        assert res["values"] > 2_000_000_000
        assert all(e[0] == 0.0 for e in res["examples"]), res
        assert res["mismatches"] <= 1, res

    def test_ln_mod(self, D):
        rng = np.random.default_rng(7)
        x = rng.standard_normal((64, 64)).astype(np.float32) * 2
        got = D.ln_mod(t(x), scale1=np.float32(1.25), shift=np.float32(0.5)).cpu().numpy()
        want = O.ln64(x, np.ones(64, np.float32), np.zeros(64, np.float32)) * np.float32(1.25) \
            + np.float32(0.5)
        assert np.array_equal(got, want)

    def test_ddpm(self, D):
        rng = np.random.default_rng(8)
        ab = O.alpha_bar(10)
        x, e, n = (rng.standard_normal((4, 16, 8)).astype(np.float32) for _ in range(3))
        for tt in (9, 5, 2, 1):
            a_t, a_p = ab[tt], ab[tt - 1]
            alpha = a_t / a_p
            beta = 1.0 - alpha
            c3 = float(np.sqrt((1.0 - a_p) / (1.0 - a_t) * beta)) if tt > 1 else 0.0
            got = D.ddpm(t(x), t(e), beta / np.sqrt(1.0 - a_t), float(np.sqrt(alpha)),
                         t(n) if tt > 1 else None, c3).cpu().numpy()
            assert np.array_equal(got, O.ddpm_step(x, tt, e, ab, n))
        got = D.ddpm(t(x), t(e), float(np.sqrt(1.0 - ab[0])), float(np.sqrt(ab[0]))).cpu().numpy()
        assert np.array_equal(got, O.ddpm_final(x, e, ab))


class TestDdpm:
    def test_markstein_quotient_exact(self, D):
        """(x - c1 eps) / c2 via RN(1/c2) and one FMA correction == numpy's f64
        expression (sampler.py:59-80), over many coefficient sets."""
        rng = np.random.default_rng(31)
        n = 1 << 20
        for trial in range(24):
            x = (rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 3)).astype(np.float32)
            e = rng.standard_normal(n).astype(np.float32)
            nz = rng.standard_normal(n).astype(np.float32)
            c1, c2, c3 = (float(v) for v in rng.uniform(1e-4, 2.0, 3))
            if trial % 3 == 0:
                c2 = float(np.sqrt(1.0 - rng.uniform(1e-4, 0.05)))   # sqrt(alpha) as sampled
            got = D.ddpm(t(x), t(e), c1, c2, t(nz), c3).cpu().numpy()
            want = ((x.astype(np.float64) - c1 * e.astype(np.float64)) / c2
                    + c3 * nz.astype(np.float64)).astype(np.float32)
            assert np.array_equal(got.view(np.int32), want.view(np.int32)), trial

    def test_device_noise_deterministic_normal(self, D):
        """noise_gen: seeded in-kernel N(0,1) (Philox4x32-10), reproducible and
        offset-addressed (the device-noise mode of the engine)."""
        n = 1 << 22
        z = torch.zeros(n, device="cuda")
        a = D.ddpm(z, z, 0.0, 1.0, None, 1.0, noise_gen=(7, 0)).cpu().numpy()
        b = D.ddpm(z, z, 0.0, 1.0, None, 1.0, noise_gen=(7, 0)).cpu().numpy()
        c = D.ddpm(z, z, 0.0, 1.0, None, 1.0, noise_gen=(7, n // 4)).cpu().numpy()
        assert np.array_equal(a, b) and not np.array_equal(a, c)
        assert abs(a.mean()) < 5e-3 and abs(a.std() - 1.0) < 5e-3
        assert abs(np.mean(a ** 4) - 3.0) < 0.05          # Gaussian kurtosis
        assert abs(np.corrcoef(a[:-1], a[1:])[0, 1]) < 5e-3


class TestReductions:
    def test_hlc_srap_l1(self, D):
        rng = np.random.default_rng(9)
        S, d, nseg = 4096, 1152, 2
        a, b, c = (rng.standard_normal((nseg * S, d)).astype(np.float32) for _ in range(3))
        ta, tb, tc = t(a), t(b), t(c)   # keep the device copies alive across the calls
        res = torch.zeros(nseg * 3, dtype=torch.float64, device="cuda")
        D.reduce_hlc(D.feat(ta), D.feat(tb), D.feat(tc), S, d, nseg, res)
        r = res.cpu().numpy()
        for v in range(nseg):
            sl = slice(v * S, (v + 1) * S)
            dd = O.divergence(a[sl], b[sl], 3, c[sl])
            assert (r[2 * v] / 3) * np.sqrt(r[2 * v + 1]) == pytest.approx(dd, rel=1e-12)
        D.reduce_srap(D.feat(ta), D.feat(tb), S, d, nseg, res)
        r = res.cpu().numpy()
        for v in range(nseg):
            sl = slice(v * S, (v + 1) * S)
            s = r[3 * v] / (np.sqrt(r[3 * v + 1]) * np.sqrt(r[3 * v + 2]))
            assert s == pytest.approx(O.similarity(a[sl], b[sl]), rel=1e-12, abs=1e-15)
        D.reduce_l1(D.feat(ta), D.feat(tb), S, d, nseg, res)
        r = res.cpu().numpy()
        for v in range(nseg):
            sl = slice(v * S, (v + 1) * S)
            assert r[v] == pytest.approx(O.variation([b[sl]], a[sl]), rel=1e-12)

    @pytest.mark.parametrize("nh", [1, 4, 5])
    def test_l1_hist_fused(self, D, nh):
        """cumulative_variation terms of every history entry in one pass
        (schedule.py:128-133) == the per-entry reduction, incl. row tables that
        place each video's slot anywhere in an arena and an odd row count."""
        rng = np.random.default_rng(20 + nh)
        S, d, nseg, slots = 1003, 1152, 2, 12
        arena = rng.standard_normal((slots * 1024, d)).astype(np.float32)
        ta = t(arena)
        pick = rng.permutation(slots)[:(nh + 1) * nseg].reshape(nh + 1, nseg)
        tabs = [torch.tensor(pick[j] * 1024, dtype=torch.int64, device="cuda")
                for j in range(nh + 1)]
        res = torch.zeros((nh, nseg), dtype=torch.float64, device="cuda")
        D.reduce_l1_hist(D.feat(ta, tabs[0]), [D.feat(ta, tabs[1 + j]) for j in range(nh)],
                         S, d, nseg, res)
        got = res.cpu().numpy()
        one = torch.zeros(nseg, dtype=torch.float64, device="cuda")
        for j in range(nh):
            D.reduce_l1(D.feat(ta, tabs[0]), D.feat(ta, tabs[1 + j]), S, d, nseg, one)
            ref = one.cpu().numpy()
            for v in range(nseg):
                x = arena[pick[0, v] * 1024: pick[0, v] * 1024 + S]
                h = arena[pick[1 + j, v] * 1024: pick[1 + j, v] * 1024 + S]
                assert got[j, v] == pytest.approx(O.variation([h], x), rel=1e-12)
                assert got[j, v] == pytest.approx(ref[v], rel=1e-13)
        again = torch.zeros_like(res)
        D.reduce_l1_hist(D.feat(ta, tabs[0]), [D.feat(ta, tabs[1 + j]) for j in range(nh)],
                         S, d, nseg, again)
        assert torch.equal(again, res)   # deterministic (fixed-order sums)

    @pytest.mark.parametrize("n", [64 * 64, 4 * 16 * 64 + 3, 4096 * 1152])
    def test_policy_statistics_api(self, D, n):
        """divergence_score / layer_similarity / cumulative_variation on the device
        == the reference formulas (oracle, schedule.py:67-133), incl. a length that
        is not a multiple of 4, zero-norm similarity and > 8 history entries."""
        from paper_2503_06545_b200 import (cumulative_variation, divergence_score,
                                           layer_similarity)
        rng = np.random.default_rng(n % 97)
        a, b, m, mp = (rng.standard_normal(n).astype(np.float32) for _ in range(4))
        assert divergence_score(a, b, 3, m, mp) == pytest.approx(
            O.divergence5(a, b, 3, m, mp), rel=1e-12)
        assert layer_similarity(a, b) == pytest.approx(O.similarity(a, b), rel=1e-12,
                                                       abs=1e-15)
        assert layer_similarity(a, np.zeros(n, np.float32)) == 0.0
        hist = [rng.standard_normal(n).astype(np.float32) for _ in range(9)]
        assert cumulative_variation(hist, a) == pytest.approx(O.variation(hist, a), rel=1e-12)

    def test_srap_dedup_equals_full(self, D):
        """SRAP over (layer, video) segments with repeated slot pairs: reducing
        only the representatives (dup_src) gives the full results bit for bit,
        including inactive representatives needed by active duplicates."""
        rng = np.random.default_rng(11)
        S, d, nslot = 512, 1152, 4
        arena = t(rng.standard_normal((nslot * S, d)).astype(np.float32))
        pairs = [(0, 0), (0, 1), (0, 0), (2, 2), (1, 1), (2, 2), (0, 1), (3, 0), (2, 2)]
        ra = torch.tensor([p[0] * S for p in pairs], dtype=torch.int64, device="cuda")
        rb = torch.tensor([p[1] * S for p in pairs], dtype=torch.int64, device="cuda")
        first = {}
        dup = torch.tensor([first.setdefault(p, i) for i, p in enumerate(pairs)],
                           dtype=torch.int64, device="cuda")
        active = torch.tensor([0, 1, 1, 0, 1, 1, 1, 1, 0], dtype=torch.int32, device="cuda")
        n = len(pairs)
        full = torch.zeros(n * 3, dtype=torch.float64, device="cuda")
        D.reduce_srap(D.feat(arena, ra), D.feat(arena, rb), S, d, n, full.view(n, 3))
        ded = torch.full((n * 3,), -1.0, dtype=torch.float64, device="cuda")
        D.reduce_srap(D.feat(arena, ra), D.feat(arena, rb), S, d, n, ded.view(n, 3),
                      seg_active=active, dup_src=dup)
        act = active.cpu().numpy().astype(bool)
        f, g = full.view(n, 3).cpu().numpy(), ded.view(n, 3).cpu().numpy()
        assert np.array_equal(f[act].view(np.int64), g[act].view(np.int64))

    def test_deterministic(self, D):
        rng = np.random.default_rng(10)
        a, b, c = (t(rng.standard_normal((4096, 1152)).astype(np.float32)) for _ in range(3))
        r1 = torch.zeros(2, dtype=torch.float64, device="cuda")
        r2 = torch.zeros(2, dtype=torch.float64, device="cuda")
        D.reduce_hlc(D.feat(a), D.feat(b), D.feat(c), 4096, 1152, 1, r1)
        D.reduce_hlc(D.feat(a), D.feat(b), D.feat(c), 4096, 1152, 1, r2)
        assert torch.equal(r1, r2)
