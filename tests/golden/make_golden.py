"""Generate golden fixtures by running the REFERENCE package (`ditrt`).

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Outputs (committed, small): tests/golden/*.npz and *.json.  Nothing on the GPU
box reads /root/reference; the tests read these files instead.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

import ditrt
from ditrt import harness, model as rmodel, quant as rquant, runtime as rruntime
from ditrt import schedule as rsched, tensor as rtensor
from ditrt.tensor import Tensor

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrays):
    np.savez_compressed(os.path.join(OUT, name), **arrays)


def quantizer_fixtures():
    rng = np.random.default_rng(1234)
    arrays = {}
    cases = []
    for i, (shape, bits, scale) in enumerate([
        ((7, 5), 8, 1.0), ((33, 17), 6, 3.0), ((64, 64), 4, 0.2), ((5, 300), 8, 50.0),
        ((128, 1152), 8, 1.0), ((128, 1152), 6, 2.0), ((64, 4608), 4, 1.5),
        ((3, 3), 2, 1.0), ((16, 16), 8, 1e-3),
    ]):
        x = (rng.standard_normal(shape) * scale).astype(np.float32)
        p = rquant.compute_minmax_params(Tensor(x), bits)
        q = rquant.quantize(Tensor(x), p)
        arrays[f"x{i}"] = x
        arrays[f"codes{i}"] = q.codes.astype(np.uint8)
        arrays[f"deq{i}"] = rquant.dequantize(q).data
        cases.append(dict(i=i, bits=bits, s=float(p.scale), z=int(p.zero_point)))
    # ties: values exactly on half-code boundaries
    s = float(rquant._round_scale_up(np.float64(0.1)))
    ties = (np.arange(-40, 41, dtype=np.float64) + 0.5) * s
    ties = ties.astype(np.float32)
    p = rquant.compute_minmax_params(Tensor(ties), 8)
    arrays["ties_x"] = ties
    arrays["ties_codes"] = rquant.quantize(Tensor(ties), p).codes.astype(np.uint8)
    cases.append(dict(i="ties", bits=8, s=float(p.scale), z=int(p.zero_point)))
    # per-channel weights
    for j, (shape, bits) in enumerate([((16, 8), 8), ((1152, 64), 6), ((64, 256), 4)]):
        w = (rng.standard_normal(shape) / np.sqrt(shape[0])).astype(np.float32)
        p = rquant.compute_minmax_params(Tensor(w), bits, granularity="per-channel", axis=1)
        arrays[f"w{j}"] = w
        arrays[f"wcodes{j}"] = rquant.quantize(Tensor(w), p).codes.astype(np.uint8)
        arrays[f"ws{j}"] = p.scale
        arrays[f"wz{j}"] = p.zero_point
    svals = rng.uniform(1e-6, 1e3, size=2000)
    arrays["scale_in"] = svals
    arrays["scale_out"] = rquant._round_scale_up(svals)
    save("quantizer.npz", **arrays)
    with open(os.path.join(OUT, "quantizer_cases.json"), "w") as fh:
        json.dump(cases, fh, indent=1)


def rotation_fixtures():
    rng = np.random.default_rng(99)
    arrays = {}
    for i, (rows, k, seed) in enumerate([(4, 8, 5), (6, 16, 3), (5, 32, 7), (9, 64, 7),
                                         (3, 12, 1), (8, 256, 0), (16, 1152, 7),
                                         (4, 4608, 7)]):
        x = rng.standard_normal((rows, k)).astype(np.float32)
        w = rng.standard_normal((k, 8)).astype(np.float32)
        stats = rng.uniform(0.05, 20.0, size=k).astype(np.float32)
        _, tr = rquant.balance_channels(Tensor(w), Tensor(stats), sign_seed=seed)
        arrays[f"x{i}"] = x
        arrays[f"w{i}"] = w
        arrays[f"stats{i}"] = stats
        arrays[f"seed{i}"] = np.array(seed)
        arrays[f"c{i}"] = tr.channel_scales
        arrays[f"xe{i}"] = tr.apply_to_activation(x)
        if k <= 1152:
            arrays[f"we{i}"] = tr.apply_to_weight(w)
    save("rotation.npz", **arrays)


def matmul_fixtures():
    """Criterion-5 generator (test_acceptance.py:181-198) plus C2 row slices."""
    rng = np.random.default_rng(505)
    arrays = {}
    n = 0
    for _ in range(100):
        m, k, nn = (int(v) for v in rng.integers(1, 33, size=3))
        abits = int(rng.choice([4, 6, 8]))
        wbits = int(rng.choice([4, 6, 8]))
        a = Tensor((rng.standard_normal((m, k)) * rng.uniform(0.1, 10)).astype(np.float32))
        w = Tensor((rng.standard_normal((k, nn)) * rng.uniform(0.1, 10)).astype(np.float32))
        aq = rquant.quantize(a, rquant.compute_minmax_params(a, abits))
        if rng.integers(2):
            wp = rquant.compute_minmax_params(w, wbits, granularity="per-channel", axis=1)
        else:
            wp = rquant.compute_minmax_params(w, wbits)
        wq = rquant.quantize(w, wp)
        out = rtensor.matmul_int(aq, wq).data
        arrays[f"ca{n}"] = aq.codes.astype(np.uint8)
        arrays[f"sa{n}"] = np.array(float(aq.params.scale))
        arrays[f"za{n}"] = np.array(int(aq.params.zero_point))
        arrays[f"ab{n}"] = np.array(abits)
        arrays[f"cw{n}"] = wq.codes.astype(np.uint8)
        arrays[f"sw{n}"] = np.broadcast_to(np.atleast_1d(wp.scale), (nn,)).astype(np.float64)
        arrays[f"zw{n}"] = np.broadcast_to(np.atleast_1d(wp.zero_point), (nn,)).astype(np.int64)
        arrays[f"wb{n}"] = np.array(wbits)
        arrays[f"out{n}"] = out
        n += 1
    # row slices of the C2 shapes (M=16384 in the bench; 64 rows recorded here)
    rng = np.random.default_rng(7)
    for name, (rows, k, nn, wb, ab) in dict(
            qkv=(64, 1152, 384, 8, 8), fc1=(32, 1152, 512, 6, 8),
            fc2=(32, 4608, 256, 4, 8), w4a6=(64, 1152, 256, 4, 6)).items():
        a = Tensor(rng.standard_normal((rows, k)).astype(np.float32))
        w = Tensor((rng.standard_normal((k, nn)) / np.sqrt(k)).astype(np.float32))
        aq = rquant.quantize(a, rquant.compute_minmax_params(a, ab))
        wp = rquant.compute_minmax_params(w, wb, granularity="per-channel", axis=1)
        wq = rquant.quantize(w, wp)
        arrays[f"{name}_ca"] = aq.codes.astype(np.uint8)
        arrays[f"{name}_sa"] = np.array(float(aq.params.scale))
        arrays[f"{name}_za"] = np.array(int(aq.params.zero_point))
        arrays[f"{name}_cw"] = wq.codes.astype(np.uint8)
        arrays[f"{name}_sw"] = wp.scale
        arrays[f"{name}_zw"] = wp.zero_point
        arrays[f"{name}_out"] = rtensor.matmul_int(aq, wq).data
        arrays[f"{name}_bits"] = np.array([wb, ab])
    arrays["count"] = np.array(n)
    save("matmul_int.npz", **arrays)


def policy_fixtures():
    rng = np.random.default_rng(11)
    arrays = {}
    for i in range(6):
        shape = (int(rng.integers(1, 40)), int(rng.integers(1, 40)))
        a, b, c = (rng.standard_normal(shape).astype(np.float32) for _ in range(3))
        k = int(rng.integers(1, 6))
        arrays[f"a{i}"], arrays[f"b{i}"], arrays[f"c{i}"] = a, b, c
        arrays[f"k{i}"] = np.array(k)
        arrays[f"D{i}"] = np.array(rsched.divergence_score(Tensor(a), Tensor(b), k,
                                                           Tensor(a), Tensor(c)))
        arrays[f"S{i}"] = np.array(rsched.layer_similarity(Tensor(a), Tensor(b)))
        hist = [Tensor(b), Tensor(c)][: (i % 3)]
        arrays[f"V{i}"] = np.array(rsched.cumulative_variation(hist, Tensor(a)))
        arrays[f"nh{i}"] = np.array(i % 3)
    draws = np.array([[rsched.prune_draw(s, t, l) for l in range(6)]
                      for s in (0, 3) for t in range(12)])
    arrays["draws"] = draws
    save("policy.npz", **arrays)


def model_fixtures():
    """Weights checksum, mod scalars, one block forward, one plain generate."""
    arrays = {}
    meta = {}
    for name, cfg in dict(
            tiny=rmodel.DiTConfig(num_blocks=2, model_dim=8, num_heads=2,
                                  tokens_per_frame=2, frames=2, cond_dim=4, seed=5),
            small=harness.parse_config({"seed": 3, "model": {
                "num_blocks": 3, "model_dim": 16, "num_heads": 2,
                "tokens_per_frame": 4, "frames": 2, "cond_dim": 8}}).model_config(),
            default=harness.parse_config({"seed": 7}).model_config()).items():
        m = rmodel.init_model(cfg)
        meta[name] = dict(checksum=rmodel.weight_checksum(m), cfg=cfg.__dict__)
        rng = np.random.default_rng(42)
        x = rng.standard_normal((cfg.seq_len, cfg.model_dim)).astype(np.float32)
        cond = rng.standard_normal(cfg.cond_dim).astype(np.float32)
        temb = rmodel.timestep_embedding(7, cfg.model_dim)
        out = rmodel.block_forward(Tensor(x), Tensor(cond), Tensor(temb), m.blocks[0],
                                   0, None, cfg.num_heads).data
        arrays[f"{name}_x"], arrays[f"{name}_cond"], arrays[f"{name}_out"] = x, cond, out
        arrays[f"{name}_mod7"] = rtensor.mm(temb.reshape(1, -1), m.blocks[0].mod)[0]
        sched = ditrt.linear_beta_schedule(4)
        arrays[f"{name}_gen4"] = ditrt.generate(m, sched, seed=2).data
    save("model.npz", **arrays)
    with open(os.path.join(OUT, "model_meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


def run_fixtures():
    """End-to-end runs: calibration, then the four ablation toggle sets, on the
    reference's small_config (seed 3) and default config (seed 7)."""
    arrays = {}
    meta = {}
    small = {"seed": 3, "model": {"num_blocks": 3, "model_dim": 16, "num_heads": 2,
                                  "tokens_per_frame": 4, "frames": 2, "cond_dim": 8},
             "schedule": {"steps": 10}}
    for cname, obj in dict(small=small, default={"seed": 7}).items():
        cfg = harness.parse_config(obj)
        calib = harness.calibrate(cfg)
        harness.save_calibration(calib, os.path.join(OUT, f"calib_{cname}.json"))
        for tname, tog in dict(
                none={}, hlc=dict(hlc=True),
                hlc_aigq=dict(hlc=True, aigq_weights=True, aigq_acts=True),
                full=dict(hlc=True, aigq_weights=True, aigq_acts=True, srap=True),
                aigq=dict(aigq_weights=True, aigq_acts=True)).items():
            toggles = rsched.Toggles(**tog)
            res = harness.run_single(cfg, toggles, calib)
            key = f"{cname}_{tname}"
            arrays[key] = res.output.data
            tr = [r.to_json_obj() for r in res.scheduler.trace]
            with open(os.path.join(OUT, f"trace_{key}.jsonl"), "w") as fh:
                for r in tr:
                    fh.write(json.dumps(r) + "\n")
            meta[key] = dict(executed=res.scheduler.executed_macs(),
                             baseline=res.scheduler.baseline_macs(),
                             weight_bits=(harness.resolve_weight_bits(cfg, calib)
                                          if tog.get("aigq_weights") else {}))
        if cname == "default":
            gd = arrays["default_none"]
            meta["golden_default_sha256"] = hashlib.sha256(
                gd.astype("<f4").tobytes()).hexdigest()
    save("runs.npz", **arrays)
    with open(os.path.join(OUT, "runs_meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True, default=str)


def gemm_site_fixtures():
    """Every GEMM-hook call of one quantized step of the small config (full
    stack): the site input, the quantized codes/params and the output, plus the
    prepared weights. These drive the device parity tests on identical inputs."""
    cfg = harness.parse_config({"seed": 3, "model": {
        "num_blocks": 3, "model_dim": 16, "num_heads": 2, "tokens_per_frame": 4,
        "frames": 2, "cond_dim": 8}, "schedule": {"steps": 10}})
    calib = harness.load_calibration(os.path.join(OUT, "calib_small.json"))
    m = rmodel.init_model(cfg.model_config())
    wbits = harness.resolve_weight_bits(cfg, calib)
    rt = rruntime.QuantRuntime(m, rsched.Toggles(aigq_weights=True, aigq_acts=True),
                               wbits, calib.act_absmax, sign_seed=cfg.seeds["model"])
    arrays = {}
    for (l, site), (wq, wdeq, tr) in rt._prepared.items():
        arrays[f"w_{l}_{site}_codes"] = wq.codes.astype(np.uint8)
        arrays[f"w_{l}_{site}_s"] = wq.params.scale
        arrays[f"w_{l}_{site}_z"] = wq.params.zero_point
        arrays[f"w_{l}_{site}_c"] = tr.channel_scales
    calls = []
    rng = np.random.default_rng(5)
    for abits in (8, 6, 4):
        hook = rt.gemm_fn(abits)
        for l in range(cfg.model_config().num_blocks):
            for site in rmodel.QUANT_SITES:
                wt = getattr(m.blocks[l], site)
                rows = 1 if site in ("ca_k", "ca_v") else 8
                x = (rng.standard_normal((rows, wt.shape[0])) *
                     rng.uniform(0.2, 3.0)).astype(np.float32)
                out = hook(l, site, x, wt)
                _, _, tr = rt._prepared[(l, site)]
                xe = tr.apply_to_activation(x)
                ap = rquant.compute_minmax_params(Tensor(xe), abits)
                key = f"c{len(calls)}"
                arrays[key + "_x"], arrays[key + "_xe"], arrays[key + "_out"] = x, xe, out
                arrays[key + "_codes"] = rquant.quantize(Tensor(xe), ap).codes.astype(np.uint8)
                calls.append(dict(key=key, layer=l, site=site, abits=abits,
                                  wbits=wbits[l], s=float(ap.scale), z=int(ap.zero_point)))
    save("gemm_sites.npz", **arrays)
    with open(os.path.join(OUT, "gemm_sites.json"), "w") as fh:
        json.dump(dict(calls=calls, weight_bits={str(k): v for k, v in wbits.items()},
                       sign_seed=cfg.seeds["model"]), fh, indent=1)


if __name__ == "__main__":
    which = sys.argv[1:] or ["quant", "rot", "mm", "policy", "model", "runs", "sites"]
    if "quant" in which:
        quantizer_fixtures()
    if "rot" in which:
        rotation_fixtures()
    if "mm" in which:
        matmul_fixtures()
    if "policy" in which:
        policy_fixtures()
    if "model" in which:
        model_fixtures()
    if "runs" in which:
        run_fixtures()
    if "sites" in which:
        gemm_site_fixtures()
    print("golden fixtures written to", OUT)
