"""Localize engine vs oracle divergence on the default config (quantized path)."""
import json, sys
import numpy as np, torch
sys.path.insert(0, '.')
from oracle import qc_oracle as O
from paper_2503_06545_b200 import harness
cal = 'tests/golden/calib_default.json'
cfg = harness.parse_config({"seed": 7, "calibration": cal,
                            "toggles": dict(hlc=True, aigq_weights=True, aigq_acts=True)})
calib = harness.load_calibration(cal)
eng, sch = harness.build_engine(cfg, cfg.toggles_obj(), calib)
feats = []
eng.generate([7], collect_features=feats)
dims = O.ModelDims(8, 64, 4, 16, 4, 32, 7)
blocks, hw, hb = O.init_weights(dims)
wb = harness.resolve_weight_bits(cfg, calib)
qs = O.QuantSites(blocks, True, True, wb, calib.act_absmax, 7)
rng = np.random.default_rng(7)
x = rng.standard_normal((4, 16, 64)).astype(np.float32)
cond = rng.standard_normal(32).astype(np.float32)
t, xt, outs = feats[0]
print("x_T equal", np.array_equal(xt[0].reshape(4, 16, 64), x))
gemm = qs.hook(8)
h = x.reshape(64, 64)
for l in range(8):
    calls = {}
    def g(layer, site, a, w, calls=calls):
        y = gemm(layer, site, a, w); calls[site] = (a, y); return y
    h = O.block(h, cond, 49, blocks[l], l, 4, g)
    e = outs[l][0]
    print("layer", l, "equal", np.array_equal(h, e), "maxdiff", float(np.abs(h - e).max()))
    if not np.array_equal(h, e):
        break
# ---- step t=48
eps = (O.seq_mm(h, hw) + hb).reshape(4, 16, 64)
ab = O.alpha_bar(50)
noise = rng.standard_normal((4, 16, 64)).astype(np.float32)
x48 = O.ddpm_step(x, 49, eps, ab, noise)
t2, xt2, outs2 = feats[1]
print("t", t2, "x48 equal", np.array_equal(xt2[0].reshape(4, 16, 64), x48),
      float(np.abs(xt2[0].reshape(4,16,64) - x48).max()))
h = x48.reshape(64, 64)
for l in range(8):
    h = O.block(h, cond, 48, blocks[l], l, 4, gemm)
    e = outs2[l][0]
    print("t48 layer", l, "equal", np.array_equal(h, e), "maxdiff", float(np.abs(h - e).max()))
    if not np.array_equal(h, e):
        # per-site localisation
        hin = x48.reshape(64, 64) if l == 0 else outs2[l - 1][0]
        calls = {}
        def g(layer, site, a, w):
            y = gemm(layer, site, a, w); calls[site] = (a, y); return y
        O.block(hin, cond, 48, blocks[l], l, 4, g)
        for s, (a, y) in calls.items():
            print("  site", s, "in absmax", float(np.abs(a).max()))
        break
