"""Parity of the production kernels at the BENCHMARKED shapes.

The bench runs the quantizer, the u8 GEMM and the noise head on 4 videos x
4,096 rows (C3) or 16,384-row videos (north_star target) per call: persistent
CTAs that loop over many row groups / tiles, flush min/max keys at segment
boundaries, flip TMEM accumulator and mbarrier phases.  These tests run exactly
those kernel variants at those sizes and compare EVERY output with the CPU
oracle (oracle/qc_oracle.py, pinned to the reference by tests/golden):

  * quantizer: codes, row sums and per-segment (scale, zero) bit-exact vs
    ln64 / gelu64 -> rotate_act_fwht -> act_params -> codes_of
    (model.py:137-147, quant.py:83-123, 163-165);
  * u8 GEMM: s32 accumulators bit-exact vs the exact integer contraction
    (computed as f64 products of integers < 2^53, i.e. exactly), f32 outputs
    bit-exact vs f32(f64(sa*sw[n]) * acc) for every epilogue, and that
    formulation equal to the reference's ascending-k matmul_int on sampled rows
    (tensor.py:68-112);
  * noise head: bit-exact vs the f64 FMA-chain kernel on all rows and vs
    seq_mm (the reference `mm`, tensor.py:43-60) on sampled rows.
"""

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


def residual_rows(rng, n, K, scale=1.0):
    """Residual-stream-like rows: N(0,1) with a per-row scale, a mean offset and
    a few large outlier channels (the dynamic range LN and the rotation see)."""
    x = rng.standard_normal((n, K)) * np.exp(0.3 * rng.standard_normal((n, 1))) * scale
    x += 0.2 * rng.standard_normal((n, 1))
    out = rng.choice(K, size=8, replace=False)
    x[:, out] *= 12.0
    return x.astype(np.float32)


def check_quant(res, want_xe, seg, rows, K, bits, o):
    """res: ActCodes of output o; want_xe: the oracle's rotated f32 rows of the
    segment; rows: the segment's row slice in the code buffer."""
    s, z = O.act_params(want_xe, bits)
    assert float(res.scale[seg]) == s and int(res.zero[seg]) == z, (seg, o)
    want = O.codes_of(want_xe, s, z, bits)
    got = res.codes[rows, :K].cpu().numpy()
    bad = int((got != want).sum())
    assert bad == 0, f"segment {seg} output {o}: {bad} code mismatches"
    assert np.array_equal(res.rowsum[rows].cpu().numpy(), want.sum(1)), (seg, o)


class TestQuantizerAtScale:
    """aq4_pass1 + aq2_pass2_hot with many row groups per CTA."""

    @pytest.mark.parametrize("nseg,S", [(4, 4096), (1, 16384)])
    def test_ln_mod_three_outputs(self, D, nseg, S):
        """sta_q/k/v: LN + modulation prologue, 3 outputs with their own balance
        scales and the shared rotation signs, rows gathered from arena slots
        through a row table (the engine's layout), K = 1152."""
        rng = np.random.default_rng(100 + nseg)
        K, bits = 1152, 8
        src = residual_rows(rng, (nseg + 1) * S, K)
        row0 = np.array([((v * 3) % (nseg + 1)) * S for v in range(nseg)], np.int64)
        g = rng.uniform(0.6, 1.4, K).astype(np.float32)
        b = (0.05 * rng.standard_normal(K)).astype(np.float32)
        s1, sh = np.float32(1.0) + np.float32(0.0731), np.float32(-0.0417)
        signs = D.sign_vector(0, 1024)
        cs = [np.exp(0.5 * rng.standard_normal(K)) for _ in range(3)]
        res = D.act_quant(t(src), bits, [(t(c), t(signs)) for c in cs], seg_rows=S,
                          seg_valid=S, nseg=nseg, x_row0=t(row0), ln=(t(g), t(b)),
                          mod=(s1, sh))
        for v in range(nseg):
            h = O.ln64(src[row0[v]:row0[v] + S], g, b) * s1 + sh
            for o, c in enumerate(cs):
                xe = O.rotate_act_fwht(h, c, 0)
                check_quant(res[o], xe, v, slice(v * S, (v + 1) * S), K, bits, o)

    def test_plain_k1152_padded_segments(self, D):
        """sta_o / ca_o: no prologue, one output, 4 videos of 4,000 valid rows in
        4,096-row segments (padding rows are not part of the tensor), 6 bits."""
        rng = np.random.default_rng(7)
        K, bits, nseg, Sp, S = 1152, 6, 4, 4096, 4000
        x = residual_rows(rng, nseg * Sp, K, scale=0.3)
        x[S:Sp] = 1e6   # padding rows of segment 0: must not enter the min/max
        c = np.exp(0.5 * rng.standard_normal(K))
        (r,) = D.act_quant(t(x), bits, [(t(c), t(D.sign_vector(0, 1024)))], seg_rows=Sp,
                           seg_valid=S, nseg=nseg)
        for v in range(nseg):
            xe = O.rotate_act_fwht(x[v * Sp:v * Sp + S], c, 0)
            check_quant(r, xe, v, slice(v * Sp, v * Sp + S), K, bits, 0)

    def test_gelu_prologue_k4608(self, D):
        """ffn2: GELU prologue on the ffn1 output, K = 4608 (b = 4096, tail 512)."""
        rng = np.random.default_rng(9)
        K, bits, nseg, S = 4608, 8, 4, 4096
        y = (1.5 * rng.standard_normal((nseg * S, K))).astype(np.float32)
        c = np.exp(0.5 * rng.standard_normal(K))
        (r,) = D.act_quant(t(y), bits, [(t(c), t(D.sign_vector(0, 4096)))], seg_rows=S,
                           seg_valid=S, nseg=nseg, gelu=True)
        for v in range(nseg):
            h = O.gelu64(y[v * S:(v + 1) * S])
            xe = O.rotate_act_fwht(h, c, 0)
            check_quant(r, xe, v, slice(v * S, (v + 1) * S), K, bits, 0)


def exact_acc(ca, za, cw, zw):
    """sum_k (a - za[seg])(w - zw[n]) exactly: f64 GEMM of integers (every
    product and partial sum is an integer < 2^53, so no rounding occurs)."""
    a = torch.from_numpy(ca.astype(np.float64)).cuda() - torch.from_numpy(
        np.asarray(za, np.float64)).cuda()[:, None]
    w = torch.from_numpy(cw.astype(np.float64)).cuda() - torch.from_numpy(
        np.asarray(zw, np.float64)).cuda()[None, :]
    return a @ w


class TestGemmAtScale:
    """gemm_u8_tcgen05 at M = 16,384: 86-344 tiles, >1 tile per CTA, both TMEM
    accumulators and every mbarrier phase flip."""

    @pytest.mark.parametrize("K,N,wb,ab", [(1152, 1152, 6, 8), (1152, 4608, 6, 8),
                                           (4608, 1152, 6, 8), (1152, 1152, 4, 6)])
    def test_every_epilogue(self, D, K, N, wb, ab):
        from paper_2503_06545_b200 import _native as Nat
        rng = np.random.default_rng(K + N + wb)
        nseg, S = 4, 4096
        M = nseg * S
        ca = rng.integers(0, 2 ** ab, size=(M, K)).astype(np.uint8)
        cw = rng.integers(0, 2 ** wb, size=(K, N)).astype(np.uint8)
        sa = O.scale_up16(rng.uniform(1e-3, 3e-2, size=nseg))
        za = rng.integers(0, 2 ** ab, size=nseg).astype(np.int32)
        sw = O.scale_up16(rng.uniform(1e-3, 1e-2, size=N))
        zw = rng.integers(0, 2 ** wb, size=N).astype(np.int32)
        a = D.ActCodes(t(np.pad(ca, ((0, 0), (0, D.round16(K) - K)))),
                       t(ca.astype(np.int64).sum(1).astype(np.int32)), t(sa), t(za), K)
        cwp = np.zeros((N, D.round16(K)), np.uint8)
        cwp[:, :K] = cw.T
        w = D.PackedWeight(t(cwp), t(sw), t(zw), t(cw.astype(np.int64).sum(0).astype(np.int32)),
                           K, N, wb)
        acc = exact_acc(ca, np.repeat(za, S), cw, zw)
        joint = torch.from_numpy(np.repeat(sa, S)).cuda()[:, None] * \
            torch.from_numpy(sw).cuda()[None, :]
        y = (joint * acc).to(torch.float32)
        got = D.gemm_u8(a, w, epilogue=Nat.EPI_ACC, seg_rows=S, seg_valid=S)
        assert torch.equal(got.to(torch.float64), acc)
        # the single-rounding formulation equals the reference's ascending-k
        # matmul_int on sampled rows of every segment
        for v in range(nseg):
            rows = np.r_[v * S:v * S + 8, (v + 1) * S - 8:(v + 1) * S]
            ref = O.matmul_int_seq(ca[rows], sa[v], za[v], cw, sw, zw)
            assert np.array_equal(ref, y[torch.from_numpy(rows).cuda()].cpu().numpy()), v
        resid = torch.randn((M, N), generator=torch.Generator().manual_seed(1)).cuda()
        gate = np.float32(-0.6171875)
        for mode in (Nat.EPI_STORE, Nat.EPI_GATE_RESID, Nat.EPI_RESID, Nat.EPI_STORE_BF16):
            out = D.gemm_u8(a, w, epilogue=mode, resid=resid, gate=gate, seg_rows=S,
                            seg_valid=S)
            if mode == Nat.EPI_STORE:
                want = y
            elif mode == Nat.EPI_GATE_RESID:   # xv + gate * y: two f32 roundings (numpy)
                want = resid + torch.tensor(gate).cuda() * y
            elif mode == Nat.EPI_RESID:
                want = resid + y
            else:
                want = y.to(torch.bfloat16)
            assert torch.equal(out, want), (mode, int((out != want).sum()))

    def test_row_tables_in_an_arena(self, D):
        """Output and residual rows addressed through per-segment row tables
        (the engine's slot layout), gate+residual in place (out == resid rows)."""
        from paper_2503_06545_b200 import _native as Nat
        rng = np.random.default_rng(5)
        K, N, nseg, S = 1152, 1152, 4, 4096
        M = nseg * S
        ca = rng.integers(0, 256, size=(M, K)).astype(np.uint8)
        cw = rng.integers(0, 64, size=(K, N)).astype(np.uint8)
        sa = O.scale_up16(rng.uniform(1e-3, 3e-2, size=nseg))
        za = rng.integers(0, 256, size=nseg).astype(np.int32)
        sw = O.scale_up16(rng.uniform(1e-3, 1e-2, size=N))
        zw = rng.integers(0, 64, size=N).astype(np.int32)
        a = D.ActCodes(t(ca), t(ca.astype(np.int64).sum(1).astype(np.int32)), t(sa), t(za), K)
        cwp = np.ascontiguousarray(cw.T)
        w = D.PackedWeight(t(cwp), t(sw), t(zw), t(cw.astype(np.int64).sum(0).astype(np.int32)),
                           K, N, 6)
        arena = torch.randn((8 * S, N), generator=torch.Generator().manual_seed(2)).cuda()
        before = arena.clone()
        slots = np.array([5, 1, 6, 3], np.int64) * S
        rt = t(slots)
        D.gemm_u8(a, w, out=arena, epilogue=Nat.EPI_GATE_RESID, resid=arena, gate=np.float32(0.25),
                  seg_rows=S, seg_valid=S, out_row0=rt, resid_row0=rt)
        acc = exact_acc(ca, np.repeat(za, S), cw, zw)
        y = ((torch.from_numpy(np.repeat(sa, S)).cuda()[:, None] *
              torch.from_numpy(sw).cuda()[None, :]) * acc).to(torch.float32)
        for v in range(nseg):
            sl = slice(int(slots[v]), int(slots[v]) + S)
            want = before[sl] + torch.tensor(np.float32(0.25)).cuda() * y[v * S:(v + 1) * S]
            assert torch.equal(arena[sl], want), v
        untouched = [s for s in range(8) if s * S not in set(slots.tolist())]
        for s in untouched:
            assert torch.equal(arena[s * S:(s + 1) * S], before[s * S:(s + 1) * S])


class TestHeadAtScale:
    def test_head_16384_rows(self, D):
        """The certified int8 digit-plane head at M = 16,384 (4 segments), bit-exact
        vs the f64 FMA-chain kernel on every element and vs seq_mm on sampled rows."""
        rng = np.random.default_rng(4)
        d, nseg, S = 1152, 4, 4096
        x = residual_rows(rng, nseg * S, d)
        w = (rng.standard_normal((d, d)) / np.sqrt(d)).astype(np.float32)
        bias = (rng.standard_normal(d) / np.sqrt(d)).astype(np.float32)
        from paper_2503_06545_b200 import _native as Nat
        hw = D.HeadWeights(t(w))
        fb = torch.zeros(1, dtype=torch.int32, device="cuda")
        got = D.head_gemm(t(x), hw, bias=t(bias), seg_rows=S, seg_valid=S, nseg=nseg,
                          fallback_count=fb)
        want = D.gemm_f64(t(x), t(w), epilogue=Nat.EPI_BIAS, bias=t(bias))
        assert torch.equal(got, want), int((got != want).sum())
        rows = np.r_[0:16, 8190:8200, nseg * S - 16:nseg * S]
        ref = O.seq_mm(x[rows], w) + bias
        assert np.array_equal(got.cpu().numpy()[rows], ref)
        assert 0 <= int(fb.item()) < nseg * S * d // 50


class TestLayerNormOrder:
    """LN mean / variance in numpy's pairwise order (model.py:137-142): rows
    whose f64 sums are NOT exact (a large offset plus small values, wide
    dynamic range), where any other summation order changes the last bits of
    the mean or variance and then, near f32 ties, the normalised values."""

    @staticmethod
    def rows(rng, n, K):
        x = 3.0e3 + rng.standard_normal((n, K)) * np.exp(2.0 * rng.standard_normal((n, 1)))
        x[:, ::7] *= 1e-3
        x[:, 5::11] = rng.standard_normal((n, len(range(5, K, 11)))) * 1e-9
        return x.astype(np.float32)

    @pytest.mark.parametrize("K", [1152, 64, 16, 200])
    def test_ln_mod_kernel(self, D, K):
        rng = np.random.default_rng(K)
        x = self.rows(rng, 4096 if K == 1152 else 512, K)
        g = rng.uniform(0.5, 1.5, K).astype(np.float32)
        b = (0.1 * rng.standard_normal(K)).astype(np.float32)
        s1, sh = np.float32(1.0) + np.float32(0.25), np.float32(-0.125)
        got = D.ln_mod(t(x), t(g), t(b), s1, sh).cpu().numpy()
        want = O.ln64(x, g, b) * s1 + sh
        assert np.array_equal(got, want), int((got != want).sum())

    def test_quantizer_ln_prologue_inexact_sums(self, D):
        """The v4 quantizer's LN (K = 1152, 3 outputs): rotated rows bit-exact."""
        rng = np.random.default_rng(77)
        K, S, nseg = 1152, 2048, 2
        x = self.rows(rng, nseg * S, K)
        g = rng.uniform(0.5, 1.5, K).astype(np.float32)
        b = (0.1 * rng.standard_normal(K)).astype(np.float32)
        cs = [np.exp(0.5 * rng.standard_normal(K)) for _ in range(3)]
        sg = D.sign_vector(0, 1024)
        res = D.act_quant(t(x), 8, [(t(c), t(sg)) for c in cs], nseg=nseg, ln=(t(g), t(b)),
                          mod=(np.float32(1.0), np.float32(0.0)))
        for v in range(nseg):
            h = O.ln64(x[v * S:(v + 1) * S], g, b)
            for o, c in enumerate(cs):
                check_quant(res[o], O.rotate_act_fwht(h, c, 0), v, slice(v * S, (v + 1) * S),
                            K, 8, o)


class TestPackedW4:
    """W4 weights stored nibble-packed ([N][K/2], quant.py:206 BIT_LEVELS 4) and
    unpacked to u8 in shared memory by the GEMM's producer warps (tcgen05 has no
    4-bit integer MMA): accumulators and outputs identical to the u8 operand."""

    @pytest.mark.parametrize("M,K,N,ab", [(16384, 1152, 1152, 8), (16384, 4608, 1152, 6),
                                          (4096, 1152, 4608, 8), (300, 200, 72, 8),
                                          (5, 200, 72, 8), (16, 1152, 300, 6)])
    def test_packed_equals_u8(self, D, M, K, N, ab):
        from paper_2503_06545_b200 import _native as Nat
        rng = np.random.default_rng(M + K + N)
        ca = rng.integers(0, 2 ** ab, size=(M, K)).astype(np.uint8)
        cw = rng.integers(0, 16, size=(K, N)).astype(np.uint8)
        sa = O.scale_up16(rng.uniform(1e-3, 3e-2, size=1))
        za = rng.integers(0, 2 ** ab, size=1).astype(np.int32)
        sw = O.scale_up16(rng.uniform(1e-3, 1e-2, size=N))
        zw = rng.integers(0, 16, size=N).astype(np.int32)
        a = D.ActCodes(t(np.pad(ca, ((0, 0), (0, D.round16(K) - K)))),
                       t(ca.astype(np.int64).sum(1).astype(np.int32)), t(sa), t(za), K)
        cwp = np.zeros((N, D.round16(K)), np.uint8)
        cwp[:, :K] = cw.T
        w8 = D.PackedWeight(t(cwp), t(sw), t(zw), t(cw.astype(np.int64).sum(0).astype(np.int32)),
                            K, N, 4)
        packed = D.pack_w4(w8.codes, K)
        # the packed bytes: low nibble = even k, high nibble = odd k, zero padding
        pk = packed.cpu().numpy()
        assert pk.shape[1] % 64 == 0
        un = np.zeros((N, 2 * pk.shape[1]), np.uint8)
        un[:, 0::2], un[:, 1::2] = pk & 15, pk >> 4
        assert np.array_equal(un[:, :K], cw.T) and not un[:, K:].any()
        w4 = D.PackedWeight(w8.codes, w8.scale, w8.zero, w8.colsum, K, N, 4, packed=packed)
        acc = exact_acc(ca, np.repeat(za, M), cw, zw)
        got = D.gemm_u8(a, w4, epilogue=Nat.EPI_ACC)
        assert torch.equal(got.to(torch.float64), acc)
        for mode in (Nat.EPI_STORE, Nat.EPI_GATE_RESID):
            resid = torch.randn((M, N), generator=torch.Generator().manual_seed(3)).cuda()
            o4 = D.gemm_u8(a, w4, epilogue=mode, resid=resid, gate=np.float32(0.5))
            o8 = D.gemm_u8(a, w8, epilogue=mode, resid=resid, gate=np.float32(0.5))
            assert torch.equal(o4, o8), mode

    def test_weight_prep_packs_w4(self, D):
        rng = np.random.default_rng(8)
        w = (rng.standard_normal((1152, 384)) / 34).astype(np.float32)
        c = np.exp(0.3 * rng.standard_normal(1152))
        pw = D.weight_prep(t(w), 4, t(c), t(D.sign_vector(0, 1024)), pack4=True)
        assert pw.packed is not None
        pk = pw.packed.cpu().numpy()
        un = np.zeros((384, 2 * pk.shape[1]), np.uint8)
        un[:, 0::2], un[:, 1::2] = pk & 15, pk >> 4
        assert np.array_equal(un[:, :1152], pw.codes.cpu().numpy()[:, :1152])
        assert D.weight_prep(t(w), 4).packed is None
        with pytest.raises(ValueError):
            D.weight_prep(t(w), 6, pack4=True)


class TestBf16Input:
    def test_bf16_rows_widened_exactly(self, D):
        """The sta_o quantizer reading the bf16 attention output directly
        (QCB_PRO_BF16, rows through a per-segment table) == the f32 path on the
        widened rows == the oracle."""
        rng = np.random.default_rng(12)
        K, S, Sp, nseg = 1152, 4000, 4096, 4
        xb = torch.as_tensor(residual_rows(rng, nseg * S, K)).cuda().to(torch.bfloat16)
        c = np.exp(0.5 * rng.standard_normal(K))
        tr = [(t(c), t(D.sign_vector(0, 1024)))]
        row0 = t(np.arange(nseg, dtype=np.int64) * S)
        (rb,) = D.act_quant(xb, 8, tr, seg_rows=Sp, seg_valid=S, nseg=nseg, x_row0=row0)
        xf = xb.float()
        (rf,) = D.act_quant(xf, 8, tr, seg_rows=Sp, seg_valid=S, nseg=nseg, x_row0=row0)
        xh = xf.cpu().numpy()
        for v in range(nseg):
            sl = slice(v * Sp, v * Sp + S)
            assert torch.equal(rb.codes[sl], rf.codes[sl]) and float(rb.scale[v]) == float(rf.scale[v])
            check_quant(rb, O.rotate_act_fwht(xh[v * S:(v + 1) * S], c, 0), v, sl, K, 8, 0)

    def test_engine_fast_attention_direct_equals_copy(self, D):
        """bench mode (bf16 SDPA): the bf16-direct sta_o input gives the same
        latents and decisions as the f32 copy of the attention output."""
        from paper_2503_06545_b200.engine import EngineOptions, QuantCacheEngine
        from paper_2503_06545_b200.model import DiTConfig, init_model
        from paper_2503_06545_b200.sampler import linear_beta_schedule
        from paper_2503_06545_b200.schedule import ThresholdConfig, Toggles
        cfg = DiTConfig(num_blocks=2, model_dim=1152, num_heads=16, tokens_per_frame=64,
                        frames=2, cond_dim=64, seed=1)
        model = init_model(cfg)
        absmax = {l: {s: np.abs(getattr(b, s)).max(axis=1).astype(np.float64) * 2.0
                      for s in ("sta_q", "sta_k", "sta_v", "sta_o", "ca_q", "ca_k", "ca_v",
                                "ca_o", "ffn1", "ffn2")} for l, b in enumerate(model.blocks)}
        sched = linear_beta_schedule(6)
        outs = []
        for direct in (True, False):
            eng = QuantCacheEngine(model, sched.alpha_bar,
                                   Toggles(hlc=True, aigq_weights=True, aigq_acts=True, srap=True),
                                   ThresholdConfig(delta1=1e3, delta2=1e6), {0: 6, 1: 6}, absmax,
                                   max_videos=2, options=EngineOptions(attention="fast",
                                                                       noise="device"))
            eng.attn_bf16_direct = direct
            lat, tr = eng.generate([5, 6])
            outs.append((lat, [[r.to_json_obj() for r in x] for x in tr]))
        assert np.array_equal(outs[0][0], outs[1][0])
        assert outs[0][1] == outs[1][1]
