#!/usr/bin/env python
"""QuantCache B200 benchmark -- prints ONE JSON line (driver contract).

Headline workload (BASELINE.json north_star Target): STDiT-XL/2 dimensions in
the reference block (28 blocks, hidden 1152, 16 heads, FFN 4608, cond width
4096), 16 frames of 512x512 (S = 16 x 32 x 32 = 16,384 tokens: 8x spatial VAE,
2x2 patches), 100 DDPM steps with full QuantCache (HLC + AIGQ W6 with
mixed-bit activations + SRAP), random-init weights, synthetic latents.  A bench
"step" = one batch of videos sampled end to end (`--workload c3` selects
BASELINE configs[2], 16 frames 256x256, S = 4096, as the headline instead).

  value     videos/s of the whole job, device-timed (CUDA events, inputs in HBM)
  e2e       the same metric through the engine's public generate() with pinned
            host latents in and host latents out (H2D/D2H inside the timed region)
  roofline  the dominant kernel class of OUR kernels in a profiled step;
            all classes under roofline_kernels (attention = library bf16 SDPA)
  lines     secondary measurements at N = 1: the other workload (C3 or target),
            an all-recompute AIGQ-only run (every block recomputed every step:
            the quantized block path without HLC/SRAP skipping), the C2 GEMM /
            quantizer microbench (W8A8 / W6A8 / W4A8 / W4A6 at M = 16,384) and
            the C1 latency of the reference's tiny configs

Multi-GPU: one process per GPU.  `--gpus N` re-launches itself under
torch.distributed.run when WORLD_SIZE is unset.  Videos are sharded across
ranks with no collective in the sampling loop (per-video decisions, reference
semantics) -> "scaling": "weak"; barrier + max-over-ranks timing.

`--impl reference` times the reference's own CPU implementation (the
unmodified `ditrt` package installed in baseline/_ref; the oracle port when
absent) on all host cores: one recomputed block + head + DDPM update on row
slices, extrapolated to videos/s of the same workload (bench_cpu.py).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

STDIT = dict(num_blocks=28, model_dim=1152, num_heads=16, cond_dim=4096, frames=16)
WORKLOADS = {
    "target": dict(tokens_per_frame=1024, label="north_star Target: STDiT-XL/2 dims (28x1152, "
                   "16 heads, FFN 4608, cond 4096), 16 frames 512x512 (S=16384), DDPM T=100, "
                   "full QuantCache"),
    "c3": dict(tokens_per_frame=256, label="C3: STDiT-XL/2 dims (28x1152, 16 heads, FFN 4608, "
               "cond 4096), 16 frames 256x256 (S=4096), DDPM T=100, full QuantCache"),
}
# Recompute fraction of the full-QuantCache runs, measured by this bench on the
# B200 (recompute_fraction in BENCH lines); the reference's decisions equal ours
# (tests/test_gpu_engine.py), so the CPU arm extrapolates with the same fraction.
RECOMPUTE_FRACTION = {"target": 0.030, "c3": 0.030}
NOMINAL_INT8_TOPS = 4500.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="target", choices=sorted(WORKLOADS))
    ap.add_argument("--videos", type=int, default=4, help="videos per GPU per step")
    ap.add_argument("--timesteps", type=int, default=100)
    ap.add_argument("--wbits", type=int, default=6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the secondary lines")
    ap.add_argument("--decisions", default="per_video", choices=["per_video", "synchronized"],
                    help="per-video decisions (reference semantics, no collective) or one "
                         "policy for the whole batch (one NCCL all-reduce per step)")
    return ap.parse_args()


def model_dims(workload: str) -> dict:
    w = WORKLOADS[workload]
    return dict(STDIT, tokens_per_frame=w["tokens_per_frame"])


# ---------------------------------------------------------------------------
# CPU arm


def _ref_worker(args):
    """One core's sample (fork child: the BlockSample was built before fork)."""
    r1, r2, S, warm = args
    os.environ["OMP_NUM_THREADS"] = "1"
    import bench_cpu
    s = _SAMPLE[0]
    if warm:
        return s.block_seconds(r1), s.head_seconds(r1)
    fb = bench_cpu.fit_seconds(s.block_seconds, r1, r2, S)
    fh = bench_cpu.fit_seconds(s.head_seconds, r1, r2, S)
    return fb, fh


_SAMPLE = [None]
R1, R2 = 4, 16


def cpu_sample_line(workload: str, steps: int, warmup: int, cores: int, timesteps: int,
                    wbits: int) -> dict:
    """Reference CPU throughput (videos/s) on `cores` processes; each step times
    one recomputed block + the head + DDPM on R1 and R2 rows per process and
    extrapolates with the linear fit t(S) = a + b S."""
    import multiprocessing as mp
    import bench_cpu
    dims = model_dims(workload)
    S = dims["tokens_per_frame"] * dims["frames"]
    _SAMPLE[0] = bench_cpu.BlockSample(S, dims["model_dim"], dims["num_heads"],
                                       dims["cond_dim"], wbits=wbits, abits=8)
    frac = RECOMPUTE_FRACTION[workload]
    ctx = mp.get_context("fork")
    rates, step_s = [], []
    with ctx.Pool(cores) as pool:
        for _ in range(warmup):
            pool.map(_ref_worker, [(R1, R2, S, True)] * cores)
        for _ in range(steps):
            t0 = time.perf_counter()
            res = pool.map(_ref_worker, [(R1, R2, S, False)] * cores)
            step_s.append(time.perf_counter() - t0)
            # every process extrapolates its own per-video time; the job's rate
            # is the sum over the concurrently running processes
            rates.append(sum(bench_cpu.videos_per_s(fb["t_S"], fh["t_S"], timesteps,
                                                    dims["num_blocks"], frac)
                             for fb, fh in res))
            last = res
    fb, fh = last[0]
    kind = _SAMPLE[0].kind
    return {
        "value": statistics.median(rates), "unit": "videos/s", "cores": cores, "kind": kind,
        "ms_per_step": statistics.median(step_s) * 1e3,
        "sample": (f"{'ditrt (unmodified reference, baseline/_ref)' if kind == 'reference' else 'oracle port'}: "
                   f"one recomputed block (10 GEMM sites via QuantRuntime.gemm_fn, _ln, _mha over "
                   f"all {S} keys, _gelu) and head mm + reverse_step on {R1} and {R2} rows per "
                   f"process x {cores} processes; per-process fit t(S)=a+b*S "
                   f"(block a={fb['a']:.2f}s b={fb['b'] * 1e3:.1f}ms/row -> {fb['t_S']:.0f}s, head "
                   f"{fh['t_S']:.1f}s at S={S}); per video = {timesteps} x (head + {frac} "
                   f"recompute fraction x {dims['num_blocks']} blocks)"),
    }


def run_reference(args):
    """--impl reference: rank 0 only (other ranks exit without work)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    cores = os.cpu_count() or 1
    c = cpu_sample_line(args.workload, args.steps, args.warmup, cores, args.timesteps,
                        args.wbits)
    line = {
        "impl": "reference", "metric": "videos_per_s", "value": c["value"], "unit": "videos/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": c["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic latents, random-init weights",
        "config": {"workload": WORKLOADS[args.workload]["label"] + " (CPU reference sample)",
                   "timesteps": args.timesteps, "weight_bits": args.wbits},
        "cpu_baseline": {k: c[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": c["value"], "unit": "videos/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def _peaks() -> dict:
    """Roofline denominators from the driver-written MEASURED_PEAKS.json."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm": float(p["hbm_gbs"]), "bf16": float(p["bf16_tflops"]),
                "bf16_sustained": float(p.get("bf16_tflops_sustained", p["bf16_tflops"])),
                "source": "MEASURED_PEAKS.json"}
    except Exception:
        return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md; MEASURED_PEAKS.json absent)"}


def _ncu_traffic() -> dict:
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of
    each roofline kernel from the committed `ncu --set full` capture summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def measured_int8_peak(torch) -> dict:
    """Library int8 GEMM (cuBLASLt via torch._int_mm, s8 x s8 -> s32, 8192^3) as the
    measured tensor-pipe reference; MEASURED_PEAKS.json carries bf16 only."""
    try:
        n = 8192
        a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
        b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
        for _ in range(3):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        return {"tops": 2.0 * n ** 3 / best / 1e12, "source": "measured torch._int_mm "
                "(cuBLASLt) s8 8192^3 burst, best of 10"}
    except Exception as exc:  # pragma: no cover - library path absent
        return {"tops": None, "source": f"unavailable: {type(exc).__name__}"}


def fast_model(cfg):
    """Random-init weights of the STDiT-XL/2 block architecture (N(0, fan_in^-1/2),
    like init_model) drawn with NumPy's float32 normal generator for speed."""
    from paper_2503_06545_b200.model import BlockWeights, DiTModel, _shapes
    rng = np.random.default_rng(cfg.seed)
    blocks = []
    for _ in range(cfg.num_blocks):
        vals = {}
        for name, shape, fan in _shapes(cfg):
            if fan == "one":
                vals[name] = np.ones(shape, np.float32)
            elif fan == "zero":
                vals[name] = np.zeros(shape, np.float32)
            else:
                vals[name] = rng.standard_normal(shape, dtype=np.float32) * np.float32(fan ** -0.5)
        blocks.append(BlockWeights(**vals))
    d = cfg.model_dim
    return DiTModel(cfg, blocks,
                    rng.standard_normal((d, d), dtype=np.float32) * np.float32(d ** -0.5),
                    rng.standard_normal(d, dtype=np.float32) * np.float32(d ** -0.5))


# sites that read the same activation tensor share its calibration statistics
_INPUT_OF = {"sta_q": "h1", "sta_k": "h1", "sta_v": "h1", "sta_o": "att", "ca_q": "h2",
             "ca_k": "cond", "ca_v": "cond", "ca_o": "ca", "ffn1": "h3", "ffn2": "hid"}


def synthetic_absmax(model, seed: int = 0):
    """Per-(layer, site) channel |x| maxima standing in for harness.calibrate's
    (harness.py:305-311): one log-normal vector per block INPUT tensor, shared by
    the sites that read it, so every site gets its own balance scales
    c_j = sqrt(absmax_x / absmax_w) (quant.py:179-200) and the q/k/v quantizer
    emits three different rotations of h1, as with a real calibration."""
    rng = np.random.default_rng(seed)
    out = {}
    for l, b in enumerate(model.blocks):
        per_input = {}
        out[l] = {}
        for site, inp in _INPUT_OF.items():
            K = getattr(b, site).shape[0]
            if inp not in per_input:
                per_input[inp] = 4.0 * np.exp(0.5 * rng.standard_normal(K))
            out[l][site] = per_input[inp]
    return out


def _events(torch):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def _agg(prof):
    tot_work, tot_t, sites = 0, 0.0, {}
    for e_s, e_e, work, site in prof:
        dt = e_s.elapsed_time(e_e) / 1e3
        tot_work += work
        tot_t += dt
        a = sites.setdefault(site, [0, 0.0, 0])
        a[0] += work
        a[1] += dt
        a[2] += 1
    return tot_work, tot_t, sites


def profile_call(torch, eng, seeds, x0, cond, S, d, H, int8_peak, peaks, traffic):
    """One generate() with CUDA events around every quantizer call, every u8 GEMM
    and every other phase (attention, GELU, head, plan, HLC, sampler): per
    kernel-class time, achieved rate and roofline fraction."""
    eng.gemm_profile, eng.quant_profile, eng.phase_profile, eng.host_profile = [], [], [], []
    eng.head_fallbacks.zero_()
    eng.att_flops = 0.0
    p0, p1 = _events(torch)
    p0.record()
    eng.generate(seeds, x0_dev=x0, cond_dev=cond, return_device=True)
    p1.record()
    torch.cuda.synchronize()
    step = p0.elapsed_time(p1) / 1e3
    g_ops, g_time, per_site = _agg(eng.gemm_profile)
    q_bytes, q_time, q_sites = _agg(eng.quant_profile)
    phases = {"act_quant": q_time * 1e3, "gemm_u8": g_time * 1e3}
    for name, e_s, e_e in eng.phase_profile:
        phases[name] = phases.get(name, 0.0) + e_s.elapsed_time(e_e)
    phases["other_and_gaps"] = step * 1e3 - sum(phases.values())
    host_loop_ms = sum(h[0] for h in eng.host_profile) * 1e3
    nv = len(seeds)
    head_fb = int(eng.head_fallbacks.item()) / float(eng.T * nv * S * d)
    att_flops = eng.att_flops
    eng.att_flops = 0.0
    eng.gemm_profile = eng.quant_profile = eng.phase_profile = eng.host_profile = None
    peak_tops = int8_peak.get("tops") or NOMINAL_INT8_TOPS
    tops = g_ops / g_time / 1e12 if g_time > 0 else None
    qgbs = q_bytes / q_time / 1e9 if q_time > 0 else None
    kern = {
        "act_quant": {
            "bound": "hbm", "achieved": qgbs, "peak": peaks["hbm"], "unit": "GB/s",
            "frac": (qgbs / peaks["hbm"]) if qgbs else None,
            "traffic": traffic.get("act_quant"),
            "traffic_call": (traffic.get("notes") or {}).get("act_quant"),
            "kernel": "act_quant (aq4_pass1 + aq2_pass2_hot + init_keys)",
            "peak_source": peaks["source"] + " hbm_gbs (burst copy)",
            "share_of_step": q_time / step if step else None,
            "algorithmic": "4*M_valid*K (f32 read) + n_out*M_valid*K (u8 codes) bytes per call",
            "per_site": {s: {"gbs": a[0] / a[1] / 1e9, "launches": a[2], "ms_total": a[1] * 1e3}
                         for s, a in q_sites.items()}},
        "gemm_u8": {
            "bound": "tensor", "achieved": tops, "peak": peak_tops, "unit": "TOP/s",
            "frac": (tops / peak_tops) if tops else None,
            "traffic": traffic.get("gemm_u8_tcgen05"),
            "traffic_call": (traffic.get("notes") or {}).get("gemm_u8_tcgen05"),
            "kernel": "gemm_u8_tcgen05 (+ gemm_u8_small_m for the cond token)",
            "peak_source": int8_peak.get("source"), "nominal_int8_dense_tops": NOMINAL_INT8_TOPS,
            "share_of_step": g_time / step if step else None,
            "algorithmic": "2*M_valid*N*K ops per launch",
            "per_site": {s: {"tops": a[0] / a[1] / 1e12, "launches": a[2], "ms_total": a[1] * 1e3}
                         for s, a in per_site.items()}},
    }
    att_ms = phases.get("attention", 0.0)
    if att_ms > 0 and att_flops > 0:
        tf = att_flops / (att_ms / 1e3) / 1e12
        kern["attention"] = {
            "bound": "tensor", "achieved": tf, "peak": peaks["bf16"], "unit": "TFLOP/s",
            "frac": tf / peaks["bf16"], "library": "cuDNN SDPA via torch (bf16), not ours",
            "peak_source": peaks["source"] + " bf16_tflops (burst cuBLAS)",
            "share_of_step": att_ms / 1e3 / step,
            "algorithmic": "4*S^2*d flops per recomputed block per video (QK^T + PV)"}
    return step, {k: round(v, 3) for k, v in phases.items()}, kern, host_loop_ms, head_fb


def _rank_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _calibrated_thresholds(torch, model, sched, wbits, absmax, T, sampler="ddpm"):
    """Threshold calibration pass (harness.py:319-345 on the quantized path):
    every block recomputed (HLC with delta = 0), D/V recorded, delta = p33/p66 of
    D, v = p25/p75 of V.  The same calibration video on every rank."""
    from paper_2503_06545_b200.engine import EngineOptions, QuantCacheEngine
    from paper_2503_06545_b200.schedule import ThresholdConfig, Toggles
    tog_cal = Toggles(hlc=True, aigq_weights=True, aigq_acts=True, srap=False)
    eng = QuantCacheEngine(model, sched.alpha_bar, tog_cal,
                           ThresholdConfig(delta1=0.0, delta2=0.0), wbits, absmax,
                           sign_seed=0, prune_seed=0, max_videos=1,
                           options=EngineOptions(attention="fast", noise="device",
                                                 sampler=sampler))
    _, tr = eng.generate([1000])
    ds = [r.d for r in tr[0] if r.d is not None]
    vs = [r.v for r in tr[0] if r.layer == 0 and r.v is not None and r.v > 0]
    del eng
    torch.cuda.empty_cache()
    return ThresholdConfig(delta1=float(np.percentile(ds, 33)),
                           delta2=float(np.percentile(ds, 66)),
                           v_low=float(np.percentile(vs, 25)), v_high=float(np.percentile(vs, 75)))


def run_workload(torch, args, workload, model, absmax, *, world, rank, local, int8_peak,
                 peaks, traffic, headline):
    """Full-QuantCache videos/s of one workload (device-timed), its profiled
    step and (headline only) the e2e run through the public generate()."""
    import torch.distributed as dist
    from paper_2503_06545_b200 import device as Dv
    from paper_2503_06545_b200 import dist as qdist
    from paper_2503_06545_b200.engine import EngineOptions, QuantCacheEngine
    from paper_2503_06545_b200.sampler import linear_beta_schedule
    from paper_2503_06545_b200.schedule import Toggles
    cfg = model.cfg
    B, T = args.videos, args.timesteps
    S, d = cfg.seq_len, cfg.model_dim
    wbits = {l: args.wbits for l in range(cfg.num_blocks)}
    sched = linear_beta_schedule(T)
    th = _calibrated_thresholds(torch, model, sched, wbits, absmax, T)
    tog = Toggles(hlc=True, aigq_weights=True, aigq_acts=True, srap=True)
    opts = EngineOptions(attention="fast", noise="device",
                         decisions=args.decisions if headline else "per_video")
    eng = QuantCacheEngine(model, sched.alpha_bar, tog, th, wbits, absmax, sign_seed=0,
                           prune_seed=0, max_videos=B, options=opts)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7 + rank)
    x0 = torch.randn((B, S, d), device="cuda", generator=gen)
    cond = torch.randn((B, cfg.cond_dim), device="cuda", generator=gen)
    # video sharding: the global video ids of this rank for bench step k (weak
    # scaling: B videos per GPU per step); a video's seed follows its id
    seeds = lambda k: qdist.video_seeds(qdist.shard_videos(B * world, world, rank), 1_000 * k)
    n_steps, n_warm = (args.steps, args.warmup) if headline else (max(2, min(args.steps, 3)), 1)
    for k in range(n_warm):
        eng.generate(seeds(k), x0_dev=x0, cond_dev=cond, return_device=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local) if headline else None
    if clocks:
        clocks.start()
    launches0 = Dv.LAUNCHES[0]
    eng.head_calls = eng.head_skipped = 0
    e0, e1 = _events(torch)
    torch.cuda.synchronize()
    # QC_PROFILE_RANGE=1: open the CUDA profiler range around the timed steps only,
    # so `ncu --profile-from-start off` lists exactly the timed region's launches
    prof_range = headline and os.environ.get("QC_PROFILE_RANGE") == "1"
    if prof_range:
        torch.cuda.cudart().cudaProfilerStart()
    e0.record()
    vids_all = []
    for k in range(n_steps):
        _, vids = eng.generate(seeds(n_warm + k), x0_dev=x0, cond_dev=cond, return_device=True)
        vids_all.append(vids)
    e1.record()
    torch.cuda.synchronize()
    if prof_range:
        torch.cuda.cudart().cudaProfilerStop()
    elapsed = e0.elapsed_time(e1) / 1e3
    launches = Dv.LAUNCHES[0] - launches0
    clk = clocks.stop() if clocks else None
    if world > 1:
        dist.barrier()
    elapsed = qdist.max_over_ranks(elapsed, device="cuda")
    traces = [eng.traces_of(v) for v in vids_all]
    recs = [r for trs in traces for tv in trs for r in tv if r.layer != "head"]
    frac = sum(r.action == "recompute" for r in recs) / max(1, len(recs))
    prune_frac = sum(r.action == "prune" for r in recs) / max(1, len(recs))
    executed = sum(r.macs for trs in traces for tv in trs for r in tv)
    out = {
        "value": n_steps * B * world / elapsed, "unit": "videos/s",
        "ms_per_step": elapsed / n_steps * 1e3, "s_per_video": elapsed / (n_steps * B),
        "steps": n_steps, "warmup": n_warm, "videos_per_gpu_per_step": B,
        "recompute_fraction": frac, "prune_fraction": prune_frac,
        "head_reuse_fraction": eng.head_skipped / max(1, eng.head_calls),
        "executed_bit_macs_per_video": executed / (n_steps * B), "gpu_launches": launches,
        "thresholds": {"delta1": th.delta1, "delta2": th.delta2, "v_low": th.v_low,
                       "v_high": th.v_high},
        "arena_gib": round(eng.arena.numel() * 4 / 2 ** 30, 2),
    }
    if clk:
        out["clocks"] = clk
    step, phases, kern, host_ms, head_fb = profile_call(
        torch, eng, seeds(900), x0, cond, S, d, cfg.num_heads, int8_peak, peaks, traffic)
    out.update({"profiled_call_ms": round(step * 1e3, 3), "profiled_step_ms": phases,
                "roofline_kernels": kern, "host_block_loop_ms": round(host_ms, 3),
                "head_exact_fallback_fraction": head_fb})
    if headline:
        # e2e through the public API on every rank: the step's inputs live in
        # pinned host memory, generate() copies them in (H2D inside the timed
        # region) and returns the latents on the host (D2H); max over ranks
        g = torch.Generator().manual_seed(11 + rank)
        x0_host = torch.randn((B, S, d), generator=g).pin_memory()
        cond_host = torch.randn((B, cfg.cond_dim), generator=g).pin_memory()
        eng.generate(seeds(499), x0_dev=x0_host, cond_dev=cond_host)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for k in range(n_steps):
            eng.generate(seeds(500 + k), x0_dev=x0_host, cond_dev=cond_host)
        torch.cuda.synchronize()
        wall = qdist.max_over_ranks(time.perf_counter() - t0, device="cuda")
        out["e2e"] = {"value": n_steps * B * world / wall, "unit": "videos/s",
                      "h2d_bytes_per_step": B * (S * d + cfg.cond_dim) * 4,
                      "d2h_bytes_per_step": B * S * d * 4}
    del eng
    torch.cuda.empty_cache()
    return out


def all_recompute_line(torch, args, model, absmax, int8_peak, peaks, traffic):
    """AIGQ only (HLC/SRAP off): every block of every step recomputed through
    the quantizer + u8 GEMM path, 1 video, T steps (device-timed, + a profiled
    call for the per-kernel-class breakdown)."""
    from paper_2503_06545_b200.engine import EngineOptions, QuantCacheEngine
    from paper_2503_06545_b200.sampler import linear_beta_schedule
    from paper_2503_06545_b200.schedule import ThresholdConfig, Toggles
    cfg = model.cfg
    S, d, T = cfg.seq_len, cfg.model_dim, args.timesteps
    sched = linear_beta_schedule(T)
    wbits = {l: args.wbits for l in range(cfg.num_blocks)}
    eng = QuantCacheEngine(model, sched.alpha_bar,
                           Toggles(hlc=False, aigq_weights=True, aigq_acts=True, srap=False),
                           ThresholdConfig(delta1=1.0, delta2=2.0), wbits, absmax, sign_seed=0,
                           prune_seed=0,
                           max_videos=1, options=EngineOptions(attention="fast", noise="device"))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)
    x0 = torch.randn((1, S, d), device="cuda", generator=gen)
    cond = torch.randn((1, cfg.cond_dim), device="cuda", generator=gen)
    eng.generate([1], x0_dev=x0, cond_dev=cond, return_device=True)
    torch.cuda.synchronize()
    e0, e1 = _events(torch)
    e0.record()
    eng.generate([2], x0_dev=x0, cond_dev=cond, return_device=True)
    e1.record()
    torch.cuda.synchronize()
    el = e0.elapsed_time(e1) / 1e3
    step, phases, kern, host_ms, _ = profile_call(torch, eng, [3], x0, cond, S, d,
                                                  cfg.num_heads, int8_peak, peaks, traffic)
    del eng
    torch.cuda.empty_cache()
    blocks = cfg.num_blocks * T
    return {"workload": f"AIGQ only (W{args.wbits}A8, HLC/SRAP off: all {cfg.num_blocks} blocks "
                        f"recomputed at every one of {T} steps), S={S}, 1 video",
            "value": 1.0 / el, "unit": "videos/s", "s_per_video": el,
            "ms_per_block": el / blocks * 1e3, "profiled_call_ms": round(step * 1e3, 3),
            "profiled_step_ms": phases, "roofline_kernels": kern}


def c4_cfg_line(torch, args, model, absmax, th_target, S_target, cfg_scale=4.5):
    """BASELINE configs[3] (C4) on one GPU: STDiT-XL/2 dims, 64 frames 512x512
    (S = 65,536), classifier-free guidance (an EXTENSION: the reference has no
    CFG) as a cond and an uncond branch per video with their own QuantCache
    decisions, HLC + SRAP + mixed-bit AIGQ, T steps, 1 video.  Thresholds: the
    target's calibrated ones scaled by the D / V scaling laws (D = L1 x L2 over
    S x d elements ~ S^1.5, V = L1 ~ S) -- an all-recompute calibration pass at
    this size would take minutes."""
    from paper_2503_06545_b200.engine import EngineOptions, QuantCacheEngine
    from paper_2503_06545_b200.model import DiTConfig, DiTModel
    from paper_2503_06545_b200.sampler import linear_beta_schedule
    from paper_2503_06545_b200.schedule import ThresholdConfig, Toggles
    cfg = DiTConfig(seed=0, **dict(STDIT, frames=64, tokens_per_frame=1024))
    m4 = DiTModel(cfg, model.blocks, model.head_w, model.head_b)
    S, d, T = cfg.seq_len, cfg.model_dim, args.timesteps
    r = S / S_target
    th = ThresholdConfig(delta1=th_target["delta1"] * r ** 1.5,
                         delta2=th_target["delta2"] * r ** 1.5,
                         v_low=th_target["v_low"] * r, v_high=th_target["v_high"] * r)
    wbits = {l: args.wbits for l in range(cfg.num_blocks)}
    sched = linear_beta_schedule(T)
    eng = QuantCacheEngine(m4, sched.alpha_bar,
                           Toggles(hlc=True, aigq_weights=True, aigq_acts=True, srap=True),
                           th, wbits, absmax, sign_seed=0, prune_seed=0, max_videos=2,
                           options=EngineOptions(attention="fast", noise="device",
                                                 cfg_scale=cfg_scale))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(4)
    x0 = torch.randn((1, S, d), device="cuda", generator=gen)
    cond = torch.randn((1, cfg.cond_dim), device="cuda", generator=gen)
    eng.generate([40], x0_dev=x0, cond_dev=cond, return_device=True)
    torch.cuda.synchronize()
    e0, e1 = _events(torch)
    e0.record()
    _, vids = eng.generate([41], x0_dev=x0, cond_dev=cond, return_device=True)
    e1.record()
    torch.cuda.synchronize()
    el = e0.elapsed_time(e1) / 1e3
    recs = [r_ for tv in eng.traces_of(vids) for r_ in tv if r_.layer != "head"]
    frac = sum(r_.action == "recompute" for r_ in recs) / max(1, len(recs))
    out = {"workload": f"C4 (extension: CFG): STDiT-XL/2 dims, 64 frames 512x512 (S={S}), "
                       f"cond + uncond branches (guidance {cfg_scale}), DDPM T={T}, full "
                       f"QuantCache per branch, 1 video on 1 GPU",
           "value": 1.0 / el, "unit": "videos/s", "s_per_video": el,
           "recompute_fraction": frac, "arena_gib": round(eng.arena.numel() * 4 / 2 ** 30, 2),
           "thresholds": {"delta1": th.delta1, "delta2": th.delta2, "v_low": th.v_low,
                          "v_high": th.v_high, "note": "target thresholds x (S ratio)^1.5 "
                                                        "for delta, x S ratio for v"}}
    del eng
    torch.cuda.empty_cache()
    return out


def c5_rf_line(torch, args, model, absmax, batches=(1, 8, 32, 64), steps=30):
    """BASELINE configs[4] (C5, an EXTENSION: the reference has no flow sampler,
    SPEC.md:474): rectified-flow sampling (head output = velocity, 30 Euler
    steps) at STDiT-XL/2 dims, 16 frames 256x256 (S = 4096, the C3 size), full
    QuantCache with per-video decisions, batch sweep of videos per GPU.
    Thresholds from an all-recompute flow calibration pass at this size."""
    from paper_2503_06545_b200.engine import EngineOptions, QuantCacheEngine
    from paper_2503_06545_b200.model import DiTConfig, DiTModel
    from paper_2503_06545_b200.sampler import linear_beta_schedule
    from paper_2503_06545_b200.schedule import Toggles
    cfg = DiTConfig(seed=0, **model_dims("c3"))
    m5 = DiTModel(cfg, model.blocks, model.head_w, model.head_b)
    S, d = cfg.seq_len, cfg.model_dim
    wbits = {l: args.wbits for l in range(cfg.num_blocks)}
    sched = linear_beta_schedule(steps)
    th = _calibrated_thresholds(torch, m5, sched, wbits, absmax, steps, sampler="rf")
    res = {}
    for B in batches:
        eng = QuantCacheEngine(m5, sched.alpha_bar,
                               Toggles(hlc=True, aigq_weights=True, aigq_acts=True, srap=True),
                               th, wbits, absmax, sign_seed=0, prune_seed=0, max_videos=B,
                               options=EngineOptions(attention="fast", noise="device",
                                                     sampler="rf"))
        gen = torch.Generator(device="cuda")
        gen.manual_seed(5)
        x0 = torch.randn((B, S, d), device="cuda", generator=gen)
        cond = torch.randn((B, cfg.cond_dim), device="cuda", generator=gen)
        eng.generate(list(range(100, 100 + B)), x0_dev=x0, cond_dev=cond, return_device=True)
        torch.cuda.synchronize()
        e0, e1 = _events(torch)
        e0.record()
        _, vids = eng.generate(list(range(200, 200 + B)), x0_dev=x0, cond_dev=cond,
                               return_device=True)
        e1.record()
        torch.cuda.synchronize()
        el = e0.elapsed_time(e1) / 1e3
        recs = [r_ for tv in eng.traces_of(vids) for r_ in tv if r_.layer != "head"]
        frac = sum(r_.action == "recompute" for r_ in recs) / max(1, len(recs))
        res[str(B)] = {"videos_per_s": round(B / el, 3), "s_per_video": round(el / B, 4),
                       "recompute_fraction": round(frac, 4),
                       "arena_gib": round(eng.arena.numel() * 4 / 2 ** 30, 2)}
        del eng, x0, cond
        torch.cuda.empty_cache()
    return {"workload": f"C5 (extension: rectified flow, no reference sampler): STDiT-XL/2 "
                        f"dims, 16 frames 256x256 (S={S}), {steps} Euler steps, full "
                        f"QuantCache, per-video decisions, batch sweep on 1 GPU",
            "unit": "videos/s", "results": res,
            "thresholds": {"delta1": th.delta1, "delta2": th.delta2, "v_low": th.v_low,
                           "v_high": th.v_high}}


def c2_microbench(torch, int8_peak, peaks):
    """BASELINE configs[1] (C2): the AIGQ quantized linear at M = 16,384 tokens
    (one 16-frame 512^2 video), K,N in {1152, 4608}: quantizer (rotation +
    per-tensor params + codes, no prologue) GB/s and tcgen05 u8 GEMM TOP/s, for
    W8A8 / W6A8 / W4A8 / W4A6.  Each launch is timed alone with CUDA events on
    its stream after a 256 MiB write that flushes L2."""
    from paper_2503_06545_b200 import device as Dv
    M = 16384
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rng = torch.Generator(device="cuda")
    rng.manual_seed(0)
    res = {}
    reps = 5

    def timed(fn):
        ts = []
        for i in range(reps + 1):
            flush.fill_(i & 0xFF)
            e0, e1 = _events(torch)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            if i:
                ts.append(e0.elapsed_time(e1) / 1e3)
        return statistics.median(ts)

    peak_tops = int8_peak.get("tops") or NOMINAL_INT8_TOPS
    for K, Nn in ((1152, 1152), (1152, 4608), (4608, 1152)):
        x = torch.randn((M, K), device="cuda", generator=rng)
        w = torch.randn((K, Nn), device="cuda", generator=rng) / K ** 0.5
        c = torch.exp(0.5 * torch.randn(K, device="cuda", generator=rng, dtype=torch.float64))
        signs = torch.as_tensor(Dv.sign_vector(0, Dv.pow2_floor(K))).cuda()
        for wb, ab in ((8, 8), (6, 8), (4, 8), (4, 6)):
            pw = Dv.weight_prep(w, wb, c, signs)
            tr = [(pw.chan_scale, pw.signs, pw.chan_recip)]
            (a,) = Dv.act_quant(x, ab, tr)
            out = torch.empty((M, Nn), dtype=torch.float32, device="cuda")
            tq = timed(lambda: Dv.act_quant(x, ab, tr, out=[a]))
            tg = timed(lambda: Dv.gemm_u8(a, pw, out=out))
            tops = 2.0 * M * Nn * K / tg / 1e12
            gbs = (4 + 1) * M * K / tq / 1e9
            r = {"gemm_us": round(tg * 1e6, 2), "gemm_tops": round(tops, 1),
                 "gemm_frac_int8_peak": round(tops / peak_tops, 4),
                 "quant_us": round(tq * 1e6, 2), "quant_gbs": round(gbs, 1),
                 "quant_frac_hbm": round(gbs / peaks["hbm"], 4)}
            if wb <= 4:   # the nibble-packed weight operand (unpacked in shared memory)
                pw4 = Dv.weight_prep(w, wb, c, signs, pack4=True)
                t4 = timed(lambda: Dv.gemm_u8(a, pw4, out=out))
                r["packed_w4_gemm_us"] = round(t4 * 1e6, 2)
                r["packed_w4_gemm_tops"] = round(2.0 * M * Nn * K / t4 / 1e12, 1)
                del pw4
            res[f"K{K}_N{Nn}_W{wb}A{ab}"] = r
        del x, w
    del flush
    torch.cuda.empty_cache()
    return {"workload": "C2: quantized linear at M=16384, (K,N) in {(1152,1152),(1152,4608),"
                        "(4608,1152)}, weights per-channel, activations per-tensor with the "
                        "balance/rotation transform; L2 flushed before every timed launch",
            "int8_peak_tops": peak_tops, "int8_peak_source": int8_peak.get("source"),
            "hbm_peak_gbs": peaks["hbm"], "results": res}


def attention_microbench(torch, peaks):
    """The STDiT self-attention at the target shape (4 videos x 16 heads x
    S = 16384, dh = 72, bf16): our tcgen05 kernel (qcb_attention_bf16) against
    the library SDPA the headline uses, CUDA events, median of 5."""
    import torch.nn.functional as F
    from paper_2503_06545_b200 import device as Dv
    H, dh, S, B = 16, 72, 16384, 4
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    q, k, v = (torch.randn((B * S, H * dh), device="cuda", generator=g).to(torch.bfloat16)
               for _ in range(3))
    out = torch.empty_like(q)
    qq, kk, vv = (t.view(B, S, H, dh).permute(0, 2, 1, 3) for t in (q, k, v))
    res = {}
    for name, fn in (("tcgen05_ours", lambda: Dv.attention_bf16(q, k, v, H, S, nseg=B, out=out)),
                     ("sdpa_library", lambda: F.scaled_dot_product_attention(qq, kk, vv))):
        fn()
        ts = []
        for _ in range(5):
            e0, e1 = _events(torch)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        tf = 4.0 * B * H * S * S * dh / ms / 1e9
        res[name] = {"ms": round(ms, 3), "tflops_dh72": round(tf, 1),
                     "frac_bf16_peak": round(tf / peaks["bf16"], 4)}
    del q, k, v, out
    torch.cuda.empty_cache()
    return {"workload": "self-attention at the north_star target: 4 videos x 16 heads x "
                        "S=16384, dh=72, bf16 operands, f32 softmax/accumulation",
            "bf16_peak_tflops": peaks["bf16"], "results": res,
            "engine_default": "sdpa_library (faster); attention='tcgen05' selects ours"}


def c1_latency(torch):
    """BASELINE configs[0] (C1): the reference's tiny configs (small seed 3,
    default seed 7) with full QuantCache and the reference's calibration, exact
    mode (f64-softmax attention, NumPy noise): wall ms per sampling step through
    harness.run_single."""
    from paper_2503_06545_b200 import harness
    golden = os.path.join(ROOT, "tests", "golden")
    small = {"seed": 3, "model": {"num_blocks": 3, "model_dim": 16, "num_heads": 2,
                                  "tokens_per_frame": 4, "frames": 2, "cond_dim": 8},
             "schedule": {"steps": 10}, "calibration": os.path.join(golden, "calib_small.json")}
    default = {"seed": 7, "calibration": os.path.join(golden, "calib_default.json")}
    out = {}
    full = {"hlc": True, "aigq_weights": True, "aigq_acts": True, "srap": True}
    for name, obj in (("small", small), ("default", default)):
        cfg = harness.parse_config(dict(obj, toggles=full))
        calib = harness.load_calibration(cfg.calibration)
        harness.run_single(cfg, cfg.toggles_obj(), calib)
        walls = [harness.run_single(cfg, cfg.toggles_obj(), calib).wall_time_ms for _ in range(3)]
        T = cfg.noise_schedule().steps
        out[name] = {"ms_per_run": round(statistics.median(walls), 3),
                     "us_per_step": round(statistics.median(walls) / T * 1e3, 1), "steps": T}
    return {"workload": "C1: reference tiny configs, full QuantCache, exact mode "
                        "(bit-identical to the reference), wall time through run_single "
                        "(includes engine-internal host work; excludes engine construction)",
            "results": out}


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2503_06545_b200.model import DiTConfig, DiTModel

    world, rank, local = _rank_env()
    # QCB_BENCH_SHARED_GPU=1: a functional check of the multi-rank code path on
    # a one-GPU box (every rank on cuda:0, gloo); its numbers are not a
    # measurement.  Per-video ranks never wait on one another's kernels.
    shared = os.environ.get("QCB_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks = _peaks()
    traffic = _ncu_traffic()
    int8_peak = measured_int8_peak(torch) if rank == 0 else {"tops": None}
    cfg = DiTConfig(seed=0, **model_dims(args.workload))
    model = fast_model(cfg)
    absmax = synthetic_absmax(model)
    head = run_workload(torch, args, args.workload, model, absmax, world=world, rank=rank,
                        local=local, int8_peak=int8_peak, peaks=peaks, traffic=traffic,
                        headline=True)
    if rank == 0:
        print("headline:", json.dumps({k: head[k] for k in ("value", "s_per_video",
              "recompute_fraction", "head_reuse_fraction", "profiled_step_ms")}),
              file=sys.stderr, flush=True)
    extra = {}
    if rank == 0 and world == 1 and not args.no_extra:
        extra["all_recompute"] = all_recompute_line(torch, args, model, absmax, int8_peak,
                                                    peaks, traffic)
        other = "c3" if args.workload == "target" else "target"
        # the same block weights: only the token count S differs
        m2 = DiTModel(DiTConfig(seed=0, **model_dims(other)), model.blocks, model.head_w,
                      model.head_b)
        o = run_workload(torch, args, other, m2, absmax, world=1, rank=0, local=local,
                         int8_peak=int8_peak, peaks=peaks, traffic=traffic, headline=False)
        extra[other] = dict({"workload": WORKLOADS[other]["label"]}, **o)
        tgt = head if args.workload == "target" else o
        extra["c4_cfg"] = c4_cfg_line(torch, args, model, absmax, tgt["thresholds"],
                                      model_dims("target")["tokens_per_frame"] * 16)
        print("extra:", json.dumps(extra, default=str)[:3000], file=sys.stderr, flush=True)
        extra["c2_gemm"] = c2_microbench(torch, int8_peak, peaks)
        extra["c1_latency"] = c1_latency(torch)
        extra["attention"] = attention_microbench(torch, peaks)
        extra["c5_rf"] = c5_rf_line(torch, args, model, absmax)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        c = cpu_sample_line(args.workload, 1, 0, 1, args.timesteps, args.wbits)
        cpu = {k: c[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        kern = head["roofline_kernels"]
        ours = {k: v for k, v in kern.items() if k in ("act_quant", "gemm_u8")}
        dominant = max(ours.values(), key=lambda r: r.get("share_of_step") or 0.0)
        line = {
            "metric": "videos_per_s", "value": head["value"], "unit": "videos/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic latents, random-init weights",
            "config": {"workload": WORKLOADS[args.workload]["label"],
                       "videos_per_gpu_per_step": args.videos, "timesteps": args.timesteps,
                       "weight_bits": args.wbits,
                       "parallelism": f"video-sharded x{world}" + (
                           ", synchronised decisions (1 NCCL all-reduce of 1.1 KB per step)"
                           if args.decisions == "synchronized" else ", per-video decisions"),
                       "decisions": args.decisions, "attention": "bf16 SDPA (library)",
                       "noise": "device Philox keyed by each video's seed",
                       "calibration": "synthetic per-input channel absmax (log-normal), "
                                      "thresholds from a device calibration pass",
                       "l2": f"inputs > L2 (activation arena {head['arena_gib']} GiB per GPU)",
                       "thresholds": head["thresholds"]},
            "s_per_video": head["s_per_video"],
            "recompute_fraction": head["recompute_fraction"],
            "prune_fraction": head["prune_fraction"],
            "head_reuse_fraction": head["head_reuse_fraction"],
            "executed_bit_macs_per_video": head["executed_bit_macs_per_video"],
            "roofline": dominant,
            "roofline_kernels": kern,
            "profiled_step_ms": head["profiled_step_ms"],
            "profiled_call_ms": head["profiled_call_ms"],
            "head_exact_fallback_fraction": head["head_exact_fallback_fraction"],
            "host_block_loop_ms": head["host_block_loop_ms"],
            "cpu_baseline": cpu,
            "e2e": head["e2e"],
            "gpu_launches": head["gpu_launches"],
            "clocks": head.get("clocks"),
            "lines": extra,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def relaunch(args) -> int:
    """--gpus N without a torchrun environment: one process per GPU."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
