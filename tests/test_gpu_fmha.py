"""qcb_attention_bf16: the tcgen05 attention of the bench-mode bf16 path
(model.py:150-156 `_mha` runs in f64 in the reference; this mode takes bf16
operands like the library SDPA it replaces).  Checked against an f32
reference computed from the same bf16 operands, with the tolerance written
here: relative Frobenius error <= 1e-2 and max error no worse than twice the
library SDPA's (bf16 P and bf16 output rounding are the only approximations).
Cases: ragged S (masked last key block, rows past S untouched), segments with a
stride, head dims 16..128 (zero-padded to a multiple of 16), growing logits
(lazy rescale), and the STDiT target shape (16 heads x dh 72, S = 16384)."""

import math

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _ref(q, k, v, heads, S, nseg, stride, scale):
    d = q.shape[1]
    dh = d // heads
    out = torch.zeros((nseg * stride, d), dtype=torch.float32, device=q.device)
    for s in range(nseg):
        r = slice(s * stride, s * stride + S)
        for h in range(heads):
            c = slice(h * dh, (h + 1) * dh)
            qs, ks, vs = q[r, c].float(), k[r, c].float(), v[r, c].float()
            for q0 in range(0, S, 4096):   # bounded score matrices
                sc = (qs[q0:q0 + 4096] @ ks.T) * scale
                out[s * stride + q0:s * stride + min(S, q0 + 4096), c] = torch.softmax(sc, -1) @ vs
    return out


def _sdpa(q, k, v, heads, S, nseg, stride):
    d = q.shape[1]
    dh = d // heads
    qq, kk, vv = (t[:nseg * stride].view(nseg, stride, heads, dh)[:, :S].permute(0, 2, 1, 3)
                  for t in (q, k, v))
    o = torch.nn.functional.scaled_dot_product_attention(qq, kk, vv)
    return o.permute(0, 2, 1, 3).reshape(nseg * S, d)


def _rows(t, S, nseg, stride):
    return torch.cat([t[s * stride:s * stride + S] for s in range(nseg)])


@pytest.mark.parametrize("S,heads,dh,nseg,stride", [
    (128, 2, 72, 1, 128), (300, 3, 72, 2, 384), (1000, 2, 64, 1, 1024), (256, 1, 128, 2, 256),
    (77, 2, 16, 1, 128), (513, 2, 40, 3, 640), (129, 4, 72, 2, 256), (200, 2, 96, 1, 256),
    (130, 1, 112, 1, 256), (384, 2, 24, 1, 384)])
def test_fmha_matches_f32_reference(cuda_dev, S, heads, dh, nseg, stride):
    from paper_2503_06545_b200 import device as D
    g = torch.Generator(device="cuda").manual_seed(S * 7 + dh)
    d = heads * dh
    q, k, v = (torch.randn((nseg * stride, d), generator=g, device="cuda").to(torch.bfloat16)
               for _ in range(3))
    out = torch.full((nseg * stride, d), 7.0, dtype=torch.bfloat16, device="cuda")
    D.attention_bf16(q, k, v, heads, S, nseg=nseg, seg_stride=stride, out=out)
    torch.cuda.synchronize()
    ref = _ref(q, k, v, heads, S, nseg, stride, 1.0 / math.sqrt(dh))
    got = _rows(out, S, nseg, stride).float()
    want = _rows(ref, S, nseg, stride)
    lib = _sdpa(q, k, v, heads, S, nseg, stride).float()
    err = (got - want).abs().max().item()
    lib_err = (lib - want).abs().max().item()
    rel = ((got - want).norm() / want.norm()).item()
    assert rel <= 1e-2, (rel, err, lib_err)
    assert err <= 2 * lib_err + 1e-3, (err, lib_err)
    for s in range(nseg):   # rows past S in each segment are not written
        assert bool((out[s * stride + S:(s + 1) * stride] == 7.0).all())


def test_fmha_growing_logits_rescale(cuda_dev):
    """Key magnitudes grow along the sequence, so the running max rises block
    after block by more than the lazy-rescale threshold."""
    from paper_2503_06545_b200 import device as D
    S, heads, dh = 1024, 2, 72
    g = torch.Generator(device="cuda").manual_seed(11)
    q = torch.randn((S, heads * dh), generator=g, device="cuda")
    k = torch.randn((S, heads * dh), generator=g, device="cuda")
    k *= torch.linspace(0.1, 6.0, S, device="cuda")[:, None]
    v = torch.randn((S, heads * dh), generator=g, device="cuda")
    q, k, v = (t.to(torch.bfloat16) for t in (q, k, v))
    out = D.attention_bf16(q, k, v, heads, S)
    ref = _ref(q, k, v, heads, S, 1, S, 1.0 / math.sqrt(dh))
    lib = _sdpa(q, k, v, heads, S, 1, S).float()
    err = (out.float() - ref).abs().max().item()
    lib_err = (lib - ref).abs().max().item()
    assert ((out.float() - ref).norm() / ref.norm()).item() <= 1e-2
    assert err <= 2 * lib_err + 1e-3, (err, lib_err)


def test_fmha_target_shape(cuda_dev):
    """STDiT target: 16 heads x dh 72, S = 16384 (one video), every row."""
    from paper_2503_06545_b200 import device as D
    S, heads, dh = 16384, 16, 72
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v = (torch.randn((S, heads * dh), generator=g, device="cuda").to(torch.bfloat16)
               for _ in range(3))
    out = D.attention_bf16(q, k, v, heads, S)
    ref = _ref(q, k, v, heads, S, 1, S, 1.0 / math.sqrt(dh))
    lib = _sdpa(q, k, v, heads, S, 1, S).float()
    err = (out.float() - ref).abs().max().item()
    lib_err = (lib - ref).abs().max().item()
    assert ((out.float() - ref).norm() / ref.norm()).item() <= 1e-2
    assert err <= 2 * lib_err + 1e-3, (err, lib_err)


def test_fmha_rejects_bad_shapes(cuda_dev):
    from paper_2503_06545_b200 import device as D
    from paper_2503_06545_b200.errors import DimensionError
    x = torch.zeros((128, 2 * 12), dtype=torch.bfloat16, device="cuda")   # dh = 12: not % 8
    with pytest.raises(DimensionError):
        D.attention_bf16(x, x, x, 2, 128)
    y = torch.zeros((128, 2 * 136), dtype=torch.bfloat16, device="cuda")  # dh = 136 > 128
    with pytest.raises(DimensionError):
        D.attention_bf16(y, y, y, 2, 128)


def test_engine_tcgen05_attention_mode(cuda_dev):
    """EngineOptions(attention="tcgen05") runs the STDiT block on this kernel
    (its bf16 output feeds the sta_o quantizer directly).  Its latents are as
    close to the f64-attention ("precise") run as the library-SDPA ("fast")
    run's are (AIGQ only, so every block recomputes and no decision can flip)."""
    import numpy as np
    from paper_2503_06545_b200.engine import EngineOptions, QuantCacheEngine
    from paper_2503_06545_b200.model import DiTConfig, init_model
    from paper_2503_06545_b200.sampler import linear_beta_schedule
    from paper_2503_06545_b200.schedule import ThresholdConfig, Toggles
    cfg = DiTConfig(num_blocks=2, model_dim=1152, num_heads=16, tokens_per_frame=96,
                    frames=2, cond_dim=64, seed=1)
    model = init_model(cfg)
    absmax = {l: {s: np.abs(getattr(b, s)).max(axis=1).astype(np.float64) * 2.0
                  for s in ("sta_q", "sta_k", "sta_v", "sta_o", "ca_q", "ca_k", "ca_v",
                            "ca_o", "ffn1", "ffn2")} for l, b in enumerate(model.blocks)}
    sched = linear_beta_schedule(4)
    lat = {}
    for mode in ("precise", "fast", "tcgen05"):
        eng = QuantCacheEngine(model, sched.alpha_bar,
                               Toggles(hlc=False, aigq_weights=True, aigq_acts=True, srap=False),
                               ThresholdConfig(delta1=1e3, delta2=1e6), {0: 8, 1: 8}, absmax,
                               max_videos=2, options=EngineOptions(attention=mode, noise="device"))
        lat[mode], _ = eng.generate([5, 6])
        assert np.isfinite(lat[mode]).all()

    def rel(a, b):
        return float(np.linalg.norm(a - b) / np.linalg.norm(b))
    e_fast = rel(lat["fast"], lat["precise"])
    e_ours = rel(lat["tcgen05"], lat["precise"])
    assert e_ours <= 2 * e_fast + 1e-6, (e_ours, e_fast)
