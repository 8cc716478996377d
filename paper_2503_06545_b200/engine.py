"""Device engine for QuantCache sampling: the reference's `generate` loop
(sampler.py:91-134) with `Scheduler` decisions (schedule.py:281-351) and the
`QuantRuntime` GEMM hook (runtime.py:63-81) executed by libqcb200 kernels.

Data layout in HBM
  * residual-stream ARENA  f32 [nvid * P * S_pad][d]: every block output, cache
    entry, previous-step feature and latent lives in a slot of S_pad rows.
    Cache reuse and layer pruning are zero-copy: the host refcounts slots per
    video exactly like the reference's Python references (a pruned layer's
    `prev` aliases its input, a reused layer's output *is* the cache entry;
    schedule.py:337-351, sampler.py:150-156).  No buffer is mutated while a
    cache entry or prev feature refers to it.
  * per-step scratch for the active videos: u8 codes [rows][roundup16(K)],
    f32 q/k/v/attention/hidden, row sums, per-video scale/zero.
  * device policy state QcbPolicyVideo[nvid] (cache steps/taus, last D, prev
    flags, the step's actions) + prune-draw table + reduction results.

Per step: V reductions -> plan_reuse -> SRAP reductions -> plan_finish on the
device, ONE device->host copy of the plan (actions, bits) so the host can
dispatch only recomputed blocks, then per layer the block kernels for the
recomputing videos, the HLC reduction and the device observe kernel.  Trace
values (D, S, V) stay on device until the end of the run.
"""

from __future__ import annotations

import contextlib
import gc
import time
import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import _native as N
from . import device as Dv
from .errors import ConfigurationError
from .model import QUANT_SITES, DiTModel, block_mac_cost, head_mac_cost, timestep_embedding
from .schedule import FP_BITS, ThresholdConfig, Toggles, TraceRecord, billed_macs, \
    prune_draw_table

ACTION_NAMES = ("recompute", "reuse", "prune")
_POLICY_DTYPE = None


def _policy_dtype() -> np.dtype:
    """numpy structured dtype of QcbPolicyVideo (same field offsets)."""
    global _POLICY_DTYPE
    if _POLICY_DTYPE is None:
        _POLICY_DTYPE = np.dtype(N.QcbPolicyVideo)
    return _POLICY_DTYPE


def balance_scales(w: np.ndarray, act_absmax: np.ndarray) -> np.ndarray:
    """c_j = clip(sqrt(absmax_x / absmax_w), 1e-3, 1e3), 1 for dead channels
    (reference quant.py:179-200); host-side offline prep of K scalars."""
    w64 = np.asarray(w, np.float64)
    st = np.asarray(act_absmax, np.float64)
    if st.shape != (w64.shape[0],):
        from .errors import ConfigurationError
        raise ConfigurationError(
            f"balance stats shape {st.shape} does not match weight rows {w64.shape}")
    wa = np.abs(w64).max(axis=1)
    ok = (st > 0) & (wa > 0)
    c = np.ones_like(st)
    c[ok] = np.clip(np.sqrt(st[ok] / wa[ok]), 1e-3, 1e3)
    return c


def noise_key(seed: int, salt: Optional[int] = None) -> int:
    """64-bit Philox key of a video's device noise stream: splitmix64 of its
    seed (and of the optional salt), so nearby seeds get unrelated streams."""
    def mix(z: int) -> int:
        z = (z + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return z ^ (z >> 31)
    k = mix(int(seed) & 0xFFFFFFFFFFFFFFFF)
    if salt is not None:
        k = mix(k ^ (int(salt) & 0xFFFFFFFFFFFFFFFF))
    return k


class DevRows:
    """An uploaded int64 row table: its device address (all the kernels need)
    and, on demand, the torch view of it."""
    __slots__ = ("ptr", "n", "_src", "_off")

    def __init__(self, ptr: int, n: int, src: torch.Tensor, off: int):
        self.ptr, self.n, self._src, self._off = ptr, n, src, off

    def data_ptr(self) -> int:
        return self.ptr

    def __len__(self) -> int:
        return self.n

    @property
    def t(self) -> torch.Tensor:
        return self._src[self._off:self._off + self.n]


class SlotPool:
    """Refcounted residual-stream slots of one video."""

    def __init__(self, first: int, count: int):
        self.free = list(range(first + count - 1, first - 1, -1))
        self.ref: Dict[int, int] = {}

    def alloc(self) -> int:
        if not self.free:
            raise RuntimeError("residual-stream arena exhausted")
        s = self.free.pop()
        self.ref[s] = 1
        return s

    def inc(self, s: int) -> int:
        self.ref[s] += 1
        return s

    def dec(self, s: Optional[int]):
        if s is None:
            return
        self.ref[s] -= 1
        if self.ref[s] == 0:
            del self.ref[s]
            self.free.append(s)


@dataclass
class VideoState:
    pool: SlotPool
    rng: np.random.Generator
    x: int = -1                         # slot of the current latent x_t
    cache: List[Optional[int]] = field(default_factory=list)
    prev: List[Optional[int]] = field(default_factory=list)
    hist: List[int] = field(default_factory=list)
    seen: int = 0
    head_src: Optional[int] = None      # slot whose noise head is in eps (held)
    trace: List[TraceRecord] = field(default_factory=list)


@dataclass
class EngineOptions:
    attention: str = "precise"     # "precise" (f64 softmax kernel) | "fast" (bf16 library
                                   # SDPA) | "tcgen05" (bf16, our qcb_attention_bf16)
    noise: str = "numpy"           # "numpy" (reference RNG stream) | "device" (Philox)
    head: str = "int8"             # "int8" (certified digit GEMMs) | "f64" (FMA chains);
                                   # both give the reference's mm bit for bit
    decisions: str = "per_video"   # "per_video" (reference semantics) | "synchronized"
                                   # (one policy for the whole batch, all ranks)
    pack_w4: bool = False               # W4 layers' weights nibble-packed (footprint option)
    cfg_scale: Optional[float] = None   # classifier-free guidance (EXTENSION, no reference:
                                        # SPEC.md:468): each video runs a cond and an
                                        # uncond (null cond) branch as two slots
    sampler: str = "ddpm"          # "ddpm" (reference) | "rf": rectified flow, EXTENSION
                                   # (C5; no reference sampler): the head
                                   # output is a velocity, x <- x - v / T, no noise
    record_features: bool = False


class _PhaseEvents:
    """Records (name, start event, end event) around a phase on the current stream."""

    def __init__(self, prof: list, name: str):
        self.prof, self.name = prof, name

    def __enter__(self):
        self.e0 = torch.cuda.Event(enable_timing=True)
        self.e1 = torch.cuda.Event(enable_timing=True)
        self.e0.record()
        return self

    def __exit__(self, *exc):
        self.e1.record()
        self.prof.append((self.name, self.e0, self.e1))
        return False


class QuantCacheEngine:
    """Batched, per-video-decision QuantCache sampler on one GPU."""

    def __init__(self, model: DiTModel, alpha_bar: np.ndarray, toggles: Toggles,
                 thresholds: ThresholdConfig, weight_bits: Optional[Dict[int, int]] = None,
                 act_absmax: Optional[Dict[int, Dict[str, np.ndarray]]] = None,
                 sign_seed: int = 0, prune_seed: int = 0, max_videos: int = 1,
                 options: Optional[EngineOptions] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("QuantCacheEngine needs a CUDA device (no CPU fallback)")
        N.lib()
        thresholds.validate()
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.stream = torch.cuda.current_stream()
        self.model, self.cfg = model, model.cfg
        self.opts = options or EngineOptions()
        self.tog, self.th = toggles, thresholds
        self.thc = Dv.thresholds_struct(thresholds, toggles)
        self.ab = np.asarray(alpha_bar, np.float64)
        if self.opts.sampler not in ("ddpm", "rf"):
            raise ConfigurationError("sampler must be 'ddpm' or 'rf'")
        self.T = len(self.ab)
        self.L = self.cfg.num_blocks
        if self.L > N.MAX_LAYERS:
            raise ValueError(f"at most {N.MAX_LAYERS} blocks")
        self.S = self.cfg.seq_len
        self.Sp = (self.S + 127) // 128 * 128
        self.d = self.cfg.model_dim
        self.H = self.cfg.num_heads
        self.c = self.cfg.cond_dim
        self.nv = max_videos
        self.weight_bits = dict(weight_bits or {})
        self.sign_seed, self.prune_seed = sign_seed, prune_seed
        self.block_cost = block_mac_cost(self.cfg)
        self.head_macs = head_mac_cost(self.cfg)
        self.gemm_profile: Optional[list] = None   # set to [] to time every u8 GEMM
        self.quant_profile: Optional[list] = None  # set to [] to time every act_quant
        self.phase_profile: Optional[list] = None  # set to [] to time the other phases
        self.att_flops = 0.0                       # self-attention flops while phase-profiled
        self.attn_bf16_direct = True               # sta_o quantizer reads the bf16 SDPA rows
        self.head_calls = 0                        # video-steps whose eps was needed
        self.head_skipped = 0                      # ... of which the held eps was exact
        self.host_profile: Optional[list] = None   # set to []: host s from plan sync to the
                                                   # end of the block loop, per step
        # set to {} to record, per (layer, site), the channel max |x| of every
        # full-precision GEMM input (calibration, harness.py:305-311)
        self.absmax_rec: Optional[Dict[tuple, torch.Tensor]] = None
        if self.opts.decisions not in ("per_video", "synchronized"):
            raise ValueError("decisions must be 'per_video' or 'synchronized'")
        self.sync = self.opts.decisions == "synchronized"
        self.cfg_scale = self.opts.cfg_scale
        if self.cfg_scale is not None and (self.sync or max_videos % 2):
            raise ValueError("CFG needs per-video decisions and an even slot count "
                             "(2 branches per video)")
        self.sync_group = None    # process group of the synchronised mode (None: default)
        self._upload_weights(act_absmax or {})
        self._alloc()

    # ------------------------------------------------------------------ setup
    def _t(self, a, dt=torch.float32):
        return torch.as_tensor(np.ascontiguousarray(a)).to(self.dev, dt)

    def _upload_weights(self, act_absmax):
        m, tog = self.model, self.tog
        self.fpw = []          # per layer: dict site -> f32 [K][N] (FP / act-only modes)
        self.packed = []       # per layer: dict site -> PackedWeight
        self.ln = []
        signs_by_b = {}
        need_fp = not tog.aigq_weights
        for l, blk in enumerate(m.blocks):
            self.ln.append(tuple(self._t(getattr(blk, n)) for n in
                                 ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "ln3_g", "ln3_b")))
            fp, pk = {}, {}
            for site in QUANT_SITES:
                w = getattr(blk, site)
                if need_fp:
                    fp[site] = self._t(w)
                if tog.aigq_weights:
                    stats = act_absmax.get(l, {}).get(site)
                    K = w.shape[0]
                    if stats is not None:
                        b = Dv.pow2_floor(K)
                        if b not in signs_by_b:
                            signs_by_b[b] = self._t(Dv.sign_vector(self.sign_seed, b))
                        tr = (self._t(balance_scales(w, stats), torch.float64), signs_by_b[b])
                    else:
                        tr = (None, None)
                    pk[site] = Dv.weight_prep(self._t(w), self.weight_bits[l], tr[0], tr[1],
                                              keep_deq=not tog.aigq_acts,
                                              pack4=self.opts.pack_w4 and self.weight_bits[l] <= 4)
            self.fpw.append(fp)
            self.packed.append(pk)
        self.head_w = self._t(m.head_w)
        self.head_prep = Dv.HeadWeights(self.head_w) if self.opts.head == "int8" else None
        # running count of head outputs recomputed by the exact f64 chain
        self.head_fallbacks = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.head_b = self._t(m.head_b)
        # modulation scalars for every (t, layer): t_emb @ mod on device (f64 acc)
        temb = self._t(np.stack([timestep_embedding(t, self.d) for t in range(self.T)]))
        mods = []
        for blk in m.blocks:
            mods.append(Dv.gemm_f64(temb, self._t(blk.mod)).cpu().numpy())
        self.mod = np.stack(mods)            # [L][T][6] f32
        self.draws = self._t(prune_draw_table(self.prune_seed, self.T, self.L), torch.float64)

    def _alloc(self):
        nv, Sp, d, L = self.nv, self.Sp, self.d, self.L
        self.P = 2 * L + self.th.history_k + 7   # (+1: the held head-input slot)
        dev = self.dev
        self.arena = torch.zeros((nv * self.P * Sp, d), dtype=torch.float32, device=dev)
        rows = nv * Sp
        K4 = 4 * d
        self.codes = [torch.zeros((rows, Dv.round16(K4)), dtype=torch.uint8, device=dev)
                      for _ in range(3)]
        self.q = torch.zeros((rows, d), dtype=torch.float32, device=dev)
        self.k = torch.zeros_like(self.q)
        self.v = torch.zeros_like(self.q)
        self.att = torch.zeros_like(self.q)
        self.xe = torch.zeros((rows, K4), dtype=torch.float32, device=dev)
        self.hid = torch.zeros((rows, K4), dtype=torch.float32, device=dev)
        self.eps = torch.zeros((rows, d), dtype=torch.float32, device=dev)
        # guided eps per video (CFG extension)
        self.eps_cfg = torch.zeros((nv // 2, self.S, d), dtype=torch.float32, device=dev) \
            if self.opts.cfg_scale is not None else None
        self.q2 = torch.zeros_like(self.q)
        # bf16 q/k/v written by the integer GEMMs' epilogue for the bf16 attention
        bf16_att = self.opts.attention in ("fast", "tcgen05")
        self.qkv16 = [torch.zeros((rows, d), dtype=torch.bfloat16, device=dev) for _ in range(3)] \
            if bf16_att else None
        # bf16 attention output of the tcgen05 kernel (read by the sta_o quantizer)
        self.att16 = torch.zeros((rows, d), dtype=torch.bfloat16, device=dev) \
            if self.opts.attention == "tcgen05" else None
        self.cond = torch.zeros((nv, self.c), dtype=torch.float32, device=dev)
        self.ac = [Dv.ActCodes(self.codes[o][:, :Dv.round16(d)],
                               torch.zeros(rows, dtype=torch.int32, device=dev),
                               torch.zeros(nv, dtype=torch.float64, device=dev),
                               torch.zeros(nv, dtype=torch.int32, device=dev), d)
                   for o in range(3)]
        self.noise_dev = torch.zeros((nv, self.S, d), dtype=torch.float32, device=dev)
        self.noise_host = torch.zeros((nv, self.S, d), dtype=torch.float32).pin_memory()
        self.pol_size = C.sizeof(N.QcbPolicyVideo)
        self._act_off = N.QcbPolicyVideo.action.offset // 4
        self._abits_off = N.QcbPolicyVideo.abits.offset // 4
        self.pol = torch.zeros(nv * self.pol_size, dtype=torch.uint8, device=dev)
        self.pol_host = torch.zeros(nv * self.pol_size, dtype=torch.uint8).pin_memory()
        # per-step policy records, copied D2H after each step's observe into pinned
        # host memory, where the host turns finished steps into TraceRecords while
        # it waits on the next decision sync
        self.pol_trace = torch.zeros((self.T, nv * self.pol_size), dtype=torch.uint8).pin_memory()
        self.srap = torch.zeros((L, nv, 3), dtype=torch.float64, device=dev)
        self.mask = torch.zeros((L, nv), dtype=torch.int32, device=dev)
        self.hist_l1 = torch.zeros((self.th.history_k + 1, nv), dtype=torch.float64, device=dev)
        self.hlc = torch.zeros((L, nv, 2), dtype=torch.float64, device=dev)
        # synchronised mode: the packed per-step decision sums, summed over the
        # local videos and then all-reduced over ranks:
        # [L][2] HLC (sum|out-ref|, sum (out-prev)^2) | [L][3] SRAP (<a,b>, |a|^2,
        # |b|^2) | [history_k + 1] V terms
        hk1 = self.th.history_k + 1
        self.stats = torch.zeros(5 * L + hk1, dtype=torch.float64, device=dev)
        self.hlc_g = self.stats[:2 * L].view(L, 1, 2)
        self.srap_g = self.stats[2 * L:5 * L].view(L, 1, 3)
        self.l1_g = self.stats[5 * L:].view(hk1, 1)
        self.sync_mask = torch.ones((L, nv), dtype=torch.int32, device=dev)
        self.sync_mask[0].zero_()
        # the next step's reuse plan + SRAP similarities run on a side stream
        # while this step's FP64 noise head runs (see _early_plan)
        self.side = torch.cuda.Stream(device=dev)
        # the side stream's reduction workspace is sized and zeroed HERE, on the
        # main stream, and the constructor synchronises below: its tickets must be
        # zero before the side stream's first SRAP launch (the kernels' last CTA
        # re-zeroes them after every use)
        self._srap_ws = Dv.Workspace()
        self._srap_ws.get(int(N.lib().qcb_reduce_workspace_bytes(L * nv)))
        n_idx = 2 * max(1 << 15, 16 * L * (nv + 4) + 64)
        self.idx_host = torch.zeros(n_idx, dtype=torch.int64).pin_memory()
        self.idx_dev = torch.zeros(n_idx, dtype=torch.int64, device=dev)
        self._idx_np = self.idx_host.numpy()
        self._idx_hptr = self.idx_host.data_ptr()
        self._idx_dptr = self.idx_dev.data_ptr()
        self._begin_step(0)
        torch.cuda.synchronize(dev)

    # ------------------------------------------------------------------ index tables
    def _begin_step(self, t: int):
        """Staging for index tables is double-buffered by step parity: every
        upload of step t gets a fresh region of half (t & 1), and the plan sync
        of step t-1 guarantees step t-2's copies (same half) have retired."""
        half = self.idx_host.numel() // 2
        self._idx_base = (t & 1) * half
        self._idx_end = self._idx_base + half
        self._idx_cur = self._idx_base

    def _upload_idx(self, arrays: Sequence[Sequence[int]], stream=None) -> List[DevRows]:
        """Pack small int64 row tables into a pinned region, one H2D copy (on
        `stream`, default the current one: the stream whose kernels read them)."""
        lo = off = self._idx_cur
        buf = self._idx_np
        out = []
        for a in arrays:
            n = len(a)
            if off + n > self._idx_end:
                raise RuntimeError("index table staging overflow")
            buf[off:off + n] = a
            out.append(DevRows(self._idx_dptr + 8 * off, n, self.idx_dev, off))
            off += n
        if off > lo:
            N.check(N.lib().qcb_copy_async(self._idx_dptr + 8 * lo, self._idx_hptr + 8 * lo,
                                           8 * (off - lo), N.stream_ptr(stream)), "copy_async")
        self._idx_cur = off
        return out

    def rows(self, slot: int) -> int:
        return slot * self.Sp

    def _ph(self, name: str):
        """CUDA-event bracket for a phase when phase profiling is on."""
        prof = self.phase_profile
        if prof is None:
            return contextlib.nullcontext()
        return _PhaseEvents(prof, name)

    def slot_view(self, slot: int) -> torch.Tensor:
        return self.arena[slot * self.Sp: slot * self.Sp + self.S]

    # ------------------------------------------------------------------ sites
    def _site(self, l, site, bits, x, nseg, *, x_row0=None, seg_rows=None, seg_valid=None,
              ln=None, mod=(1.0, 0.0), epi=N.EPI_STORE, out=None, out_row0=None,
              resid=None, resid_row0=None, gate=1.0, outs=None, sites=None,
              gelu_in=False):
        """One GEMM site (or a fused group sharing the same input) through the
        mode the reference's QuantRuntime.gemm_fn would pick (runtime.py:69-79)."""
        tog = self.tog
        sites = sites or (site,)
        seg_rows = seg_rows or self.Sp
        seg_valid = seg_valid or self.S
        M = nseg * seg_rows
        quant_acts = tog.aigq_acts and bits < FP_BITS
        if tog.aigq_weights and quant_acts:
            pws = [self.packed[l][s] for s in sites]
            trs = [(p.chan_scale, p.signs, p.chan_recip) if p.chan_scale is not None else None
                   for p in pws]
            acs = []
            for o, p in enumerate(pws):
                a = self.ac[o]
                acs.append(Dv.ActCodes(self.codes[o][:M, :Dv.round16(p.K)],
                                       a.rowsum[:M], a.scale[:nseg], a.zero[:nseg], p.K))
            qprof = self.quant_profile
            if qprof is not None:
                q0 = torch.cuda.Event(enable_timing=True)
                q1 = torch.cuda.Event(enable_timing=True)
                q0.record()
            Dv.act_quant(x, bits, trs, seg_rows=seg_rows, seg_valid=seg_valid, nseg=nseg,
                         x_row0=x_row0, ln=ln, mod=mod, out=acs, gelu=gelu_in)
            if qprof is not None:
                q1.record()
                # algorithmic bytes: f32 rows read once, u8 codes written once per output
                K = pws[0].K
                rows = nseg * seg_valid
                qprof.append((q0, q1, rows * K * 4 + len(pws) * rows * K, sites[0]))
            targets = outs or [out]
            prof = self.gemm_profile
            for o, p in enumerate(pws):
                if prof is not None:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                Dv.gemm_u8(acs[o], p, M=M, out=targets[o], epilogue=epi, resid=resid,
                           gate=gate, seg_rows=seg_rows, seg_valid=seg_valid,
                           out_row0=out_row0, resid_row0=resid_row0)
                if prof is not None:
                    e1.record()
                    # algorithmic work: 2*M_valid*N*K ops (padding rows excluded)
                    prof.append((e0, e1, 2 * nseg * seg_valid * p.N * p.K, sites[o]))
            return
        # full-precision GEMMs (weight-only, act-only or plain)
        for o, s in enumerate(sites):
            target = (outs or [out])[o]
            if tog.aigq_weights:
                p = self.packed[l][s]
                w = p.w_deq
                if p.chan_scale is not None:
                    (r,) = Dv.act_quant(x, 8, [(p.chan_scale, p.signs)], seg_rows=seg_rows,
                                        seg_valid=seg_valid, nseg=nseg, x_row0=x_row0, ln=ln,
                                        mod=mod, want_codes=False, want_xe=True)
                    a, a_row0 = r.xe, None
                else:
                    a, a_row0 = self._prologue(x, ln, mod, nseg, seg_rows, seg_valid, x_row0,
                                               p.K)
            elif quant_acts:   # activation-only fake quantization (runtime.py:78-79)
                w = self.fpw[l][s]
                (r,) = Dv.act_quant(x, bits, [None], seg_rows=seg_rows, seg_valid=seg_valid,
                                    nseg=nseg, x_row0=x_row0, ln=ln, mod=mod,
                                    want_codes=False, want_deq=True)
                a, a_row0 = r.deq, None
            else:
                w = self.fpw[l][s]
                a, a_row0 = self._prologue(x, ln, mod, nseg, seg_rows, seg_valid, x_row0,
                                           w.shape[0])
            if self.absmax_rec is not None:
                rec = self.absmax_rec.get((l, s))
                if rec is None:
                    rec = torch.zeros(w.shape[0], dtype=torch.float32, device=self.dev)
                    self.absmax_rec[(l, s)] = rec
                Dv.col_absmax(a, w.shape[0], rec, nseg=nseg, seg_rows=seg_rows,
                              seg_valid=seg_valid, x_row0=a_row0)
            Dv.gemm_f64(a, w, out=target, epilogue=epi, resid=resid, gate=gate,
                        seg_rows=seg_rows, seg_valid=seg_valid, a_row0=a_row0,
                        out_row0=out_row0, resid_row0=resid_row0, M=M)

    def _prologue(self, x, ln, mod, nseg, seg_rows, seg_valid, x_row0, K):
        if ln is None:
            return x, x_row0
        h = self.xe[:nseg * seg_rows, :K]
        Dv.ln_mod(x, ln[0], ln[1], mod[0], mod[1], out=h, seg_rows=seg_rows,
                  seg_valid=seg_valid, nseg=nseg, x_row0=x_row0)
        return h, None

    def _attention(self, q, k, v, out, nseg, Skv, kv_stride):
        """Returns None, or (bf16 rows [nseg * S][d], their per-segment first-row
        table) when the fast path's output can feed the next quantizer directly."""
        S, Sp, d, H = self.S, self.Sp, self.d, self.H
        if self.opts.attention == "tcgen05" and Skv > 1:
            bf = torch.bfloat16
            qq, kk, vv = (t if t.dtype == bf else t.to(bf) for t in (q, k, v))
            Dv.attention_bf16(qq, kk, vv, H, S, nseg=nseg, seg_stride=Sp, out=self.att16)
            if self.tog.aigq_weights and self.tog.aigq_acts:
                return self.att16, self._upload_idx([[v_ * Sp for v_ in range(nseg)]])[0]
            out[:nseg * Sp].copy_(self.att16[:nseg * Sp])
            return None
        if self.opts.attention == "fast" and Skv > 1:
            dh = d // H
            qq = q[:nseg * Sp].view(nseg, Sp, H, dh)[:, :S].permute(0, 2, 1, 3)
            kk = k[:nseg * Sp].view(nseg, Sp, H, dh)[:, :S].permute(0, 2, 1, 3)
            vv = v[:nseg * Sp].view(nseg, Sp, H, dh)[:, :S].permute(0, 2, 1, 3)
            bf = torch.bfloat16
            o = torch.nn.functional.scaled_dot_product_attention(
                qq if qq.dtype == bf else qq.to(bf), kk if kk.dtype == bf else kk.to(bf),
                vv if vv.dtype == bf else vv.to(bf))
            ob = o.permute(0, 2, 1, 3)
            if (self.attn_bf16_direct and self.tog.aigq_weights and self.tog.aigq_acts
                    and ob.is_contiguous() and d % 8 == 0 and ob.data_ptr() % 16 == 0):
                # the sta_o quantizer widens the bf16 rows itself (exact): no
                # bf16 -> f32 copy pass
                rows = ob.reshape(nseg * S, d)
                return rows, self._upload_idx([[v * S for v in range(nseg)]])[0]
            out[:nseg * Sp].view(nseg, Sp, H, dh)[:, :S].copy_(ob)
            return None
        a = N.QcbAttention(N.ptr(q), q.stride(0), N.ptr(k), k.stride(0), N.ptr(v), v.stride(0),
                           N.ptr(out), out.stride(0), S, Skv, H, d // H, nseg, Sp, kv_stride,
                           Sp, S)
        N.check(N.lib().qcb_attention_f64(C.byref(a), N.stream_ptr()), "attention")


    def _block(self, l, t, vids, bits, xin_row0, out_row0, cond_row0):
        """block_forward (model.py:159-199) for the videos `vids` at one bits."""
        n = len(vids)
        m = self.mod[l, t]
        one = np.float32(1.0)
        sh1, sc1, g1 = m[0], one + m[1], m[2]
        sh3, sc3, g3 = m[3], one + m[4], m[5]
        ln1g, ln1b, ln2g, ln2b, ln3g, ln3b = self.ln[l]
        A = self.arena
        # spatial-temporal self-attention; on the integer path with the bf16
        # attention kernel the q/k/v GEMMs write bf16 directly (no conversion pass)
        int_path = self.tog.aigq_weights and self.tog.aigq_acts and bits < FP_BITS
        qkv = self.qkv16 if (self.qkv16 is not None and int_path) else [self.q, self.k, self.v]
        self._site(l, None, bits, A, n, x_row0=xin_row0, ln=(ln1g, ln1b), mod=(sc1, sh1),
                   outs=qkv, sites=("sta_q", "sta_k", "sta_v"),
                   epi=N.EPI_STORE_BF16 if qkv is self.qkv16 else N.EPI_STORE)
        with self._ph("attention"):
            ob = self._attention(qkv[0], qkv[1], qkv[2], self.att, n, self.S, self.Sp)
        if self.phase_profile is not None:   # 4 S^2 d flops per video (QK^T and PV)
            self.att_flops += 4.0 * self.S * self.S * self.d * n
        if ob is not None and int_path:   # quantizer input: the bf16 attention rows
            self._site(l, "sta_o", bits, ob[0], n, x_row0=ob[1], epi=N.EPI_GATE_RESID, out=A,
                       out_row0=out_row0, resid=A, resid_row0=xin_row0, gate=g1)
        else:
            if ob is not None:
                self.att[:n * self.Sp].view(n, self.Sp, self.d)[:, :self.S].copy_(
                    ob[0].view(n, self.S, self.d))
            self._site(l, "sta_o", bits, self.att, n, epi=N.EPI_GATE_RESID, out=A,
                       out_row0=out_row0, resid=A, resid_row0=xin_row0, gate=g1)
        # cross-attention on the single cond token
        self._site(l, "ca_q", bits, A, n, x_row0=out_row0, ln=(ln2g, ln2b), out=self.q2)
        k2, v2 = self._cond_kv(l, bits, vids, cond_row0)
        with self._ph("attention_ca"):
            self._attention(self.q2, k2, v2, self.att, n, 1, 1)
        self._site(l, "ca_o", bits, self.att, n, epi=N.EPI_RESID, out=A, out_row0=out_row0,
                   resid=A, resid_row0=out_row0)
        # FFN.  On the integer path GELU (model.py:197) runs as its own in-place
        # kernel between ffn1 and the ffn2 quantizer: same f32(gelu_f64(y)) per
        # element, with divergent exact evaluations compacted per warp.  (As the
        # ffn2 quantizer's prologue it measured slower: the exact-erfc path
        # diverges per thread there and the variant runs at 2 CTAs per SM.)
        self._site(l, "ffn1", bits, A, n, x_row0=out_row0, ln=(ln3g, ln3b), mod=(sc3, sh3),
                   epi=N.EPI_STORE if int_path else N.EPI_GELU, out=self.hid)
        if int_path:
            with self._ph("gelu"):
                Dv.gelu_inplace(self.hid, rows=n * self.Sp)
        self._site(l, "ffn2", bits, self.hid, n, epi=N.EPI_GATE_RESID, out=A,
                   out_row0=out_row0, resid=A, resid_row0=out_row0, gate=g3)

    def _cond_kv(self, l, bits, vids, cond_row0):
        """Cross-attention K/V of the cond token (model.py:191-193).  They depend
        only on (layer, activation bits, the video's cond), all fixed for a
        generate() call, so they are computed once per (layer, bits) for every
        video of the call and reused by every later recompute: the same values
        the reference recomputes each time (per-video quantizer segments make a
        video's result independent of the others in the launch)."""
        key = (l, bits)
        kv = self._kv_cache.get(key)
        nv = self._nv_call
        if kv is None:
            kv = (torch.empty((nv, self.d), dtype=torch.float32, device=self.dev),
                  torch.empty((nv, self.d), dtype=torch.float32, device=self.dev))
            self._site(l, None, bits, self.cond, nv, x_row0=self._all_vids, seg_rows=1,
                       seg_valid=1, outs=list(kv), sites=("ca_k", "ca_v"))
            self._kv_cache[key] = kv
        if list(vids) == list(range(nv)):
            return kv
        return kv[0].index_select(0, cond_row0.t), kv[1].index_select(0, cond_row0.t)

    # ------------------------------------------------------------------ plan
    def _srap_tables(self, vids) -> List[List[int]]:
        """Row tables for one SRAP launch over every (layer, video) pair:
        prev[l-1] vs prev[l] (schedule.py:298-305)."""
        L = self.L
        ra = [self.rows(vs.prev[l - 1]) if l > 0 and vs.prev[l - 1] is not None else 0
              for l in range(L) for vs in vids]
        rb = [self.rows(vs.prev[l]) if vs.prev[l] is not None else 0
              for l in range(L) for vs in vids]
        # representative per distinct (a, b) pair: pruned chains alias one slot
        first: Dict[tuple, int] = {}
        dup = [first.setdefault((x, y), i) for i, (x, y) in enumerate(zip(ra, rb))]
        return [ra, rb, dup]

    def _plan_reuse_srap(self, t: int, nv: int, do_srap: bool, tabs, stream,
                         workspace=None):
        """plan_reuse (HLC liveness, schedule.py:285-291) + SRAP similarities of
        the layers it marks for recompute (schedule.py:296-306) on `stream`."""
        lib, pol, L, S, d = N.lib(), self.pol.data_ptr(), self.L, self.S, self.d
        sp = N.stream_ptr(stream)
        N.check(lib.qcb_policy_plan_reuse(pol, nv, L, t, self.thc, sp), "plan_reuse")
        Dv.count(1)
        if do_srap:
            N.check(lib.qcb_policy_sim_mask(pol, nv, L, self.thc, N.ptr(self.mask_v), sp),
                    "sim_mask")
            Dv.count(1)
            Dv.reduce_srap(Dv.feat(self.arena, tabs[0]), Dv.feat(self.arena, tabs[1]), S, d,
                           L * nv, self.srap_v.view(L * nv, 3), seg_active=self.mask_v.view(L * nv),
                           stream=stream, workspace=workspace, dup_src=tabs[2])

    def _early_plan(self, tn: int, vids, ready):
        """Launch step tn's plan_reuse + SRAP on the side stream once `ready` (an
        event recorded on the main stream after the observe kernel) has fired;
        returns (tn, completion event)."""
        do_srap = self.tog.srap and tn != 0   # seen >= 1 here: boundary iff tn == 0
        # the tables travel on the side stream itself: main is already running
        # the head, queued after `ready`
        tabs = self._upload_idx(self._srap_tables(vids), stream=self.side) if do_srap else []
        self.side.wait_event(ready)
        self._plan_reuse_srap(tn, len(vids), do_srap, tabs, self.side, self._srap_ws)
        done = torch.cuda.Event()
        done.record(self.side)
        return (tn, done)

    # ------------------------------------------------------------------ run
    def generate(self, seeds: Sequence[int], device_noise_seed: Optional[int] = None,
                 collect_features: Optional[list] = None, x0_dev: Optional[torch.Tensor] = None,
                 cond_dev: Optional[torch.Tensor] = None, return_device: bool = False):
        """Run the full reverse trajectory for len(seeds) videos (one per seed).

        The initial latent and cond are drawn from NumPy's stream per seed like
        the reference (sampler.py:108-111), unless x0_dev [nv,S,d] / cond_dev
        [nv,c] are given: device tensors (inputs already in HBM) or host tensors
        (pinned for an async copy), copied into the video's slots.
        collect_features (list, optional): appended per step with
        (t, x_t [nv,S,d], [block outputs [nv,S,d] per layer]) host copies, like
        the reference's generate(collect_features=...) (sampler.py:113-126).
        Returns (latents f32 [nv][F][T][d] on host, or a CUDA tensor with
        return_device, and traces per video).

        With EngineOptions.cfg_scale (classifier-free guidance, an extension)
        every video occupies two slots, its cond and its uncond (zero cond)
        branch, each with its own cache / prune / bit decisions; the returned
        traces are per slot (cond, uncond, cond, ...), the latents per video."""
        cfgm = self.cfg_scale is not None
        n_videos = len(seeds)
        nv = 2 * n_videos if cfgm else n_videos
        if nv > self.nv:
            raise ValueError(f"engine sized for {self.nv} slots")
        L, S, d, T = self.L, self.S, self.d, self.T
        F, Tk = self.cfg.frames, self.cfg.tokens_per_frame
        # every launch, copy, event and synchronize of this call goes to the
        # stream current at the call (the C ABI wrappers read it per launch)
        st = self.stream = torch.cuda.current_stream(self.dev)
        self.pol.zero_()
        vids = []
        for v in range(nv):
            i = v // 2 if cfgm else v          # video of slot v
            vs = VideoState(SlotPool(v * self.P, self.P), np.random.default_rng(seeds[i]),
                            cache=[None] * L, prev=[None] * L)
            vs.x = vs.pool.alloc()
            if cfgm and v % 2:                # uncond branch: the cond branch's x0, null cond
                self.slot_view(vs.x).copy_(self.slot_view(vids[v - 1].x))
                self.cond[v].zero_()
            elif x0_dev is not None:
                # async from pinned host memory (the first decision sync of the
                # loop orders it before generate() returns); device sources too
                self.slot_view(vs.x).copy_(x0_dev[i].reshape(S, d), non_blocking=True)
                self.cond[v].copy_(cond_dev[i], non_blocking=True)
            else:
                x0 = vs.rng.standard_normal((F, Tk, d)).astype(np.float32)
                cond = vs.rng.standard_normal(self.c).astype(np.float32)
                self.slot_view(vs.x).copy_(torch.from_numpy(x0.reshape(S, d)))
                self.cond[v].copy_(torch.from_numpy(cond))
            vids.append(vs)
        # device-noise mode: N(0,1) drawn inside the DDPM kernel, Philox4x32-10 keyed
        # by each video's OWN seed (mixed with the optional call-wide salt
        # device_noise_seed), one counter range per step: a video's noise does not
        # depend on its slot in the batch or on the rank that runs it
        gen = [noise_key(s, device_noise_seed) for s in seeds] \
            if self.opts.noise == "device" else None
        self._early = None
        # cross-attention K/V of the cond tokens, per (layer, bits), for this call
        self._kv_cache: Dict[tuple, tuple] = {}
        self._nv_call = nv
        self._all_vids = torch.arange(nv, dtype=torch.int64, device=self.dev)
        # reduction results laid out [.][nv][.] for the nv videos of this call
        # (the layout the policy kernels index with nvid = nv)
        hk1 = self.th.history_k + 1
        self.hlc_v = self.hlc.view(-1)[:L * nv * 2].view(L, nv, 2)
        self.srap_v = self.srap.view(-1)[:L * nv * 3].view(L, nv, 3)
        self.l1_v = self.hist_l1.view(-1)[:hk1 * nv].view(hk1, nv)
        self.mask_v = self.mask.view(-1)[:L * nv].view(L, nv)
        if self.sync:
            self.sync_mask_v = self.sync_mask.view(-1)[:L * nv].view(L, nv)
            self.sync_mask_v.fill_(1)
            self.sync_mask_v[0].zero_()
        traces = [[] for _ in range(nv)]
        t_built = T - 1   # the next step whose records are turned into TraceRecords
        for t in range(T - 1, -1, -1):
            self._begin_step(t)
            # ---------------- plan (device) ----------------
            if self.sync:
                if t == T - 1:
                    self._sync_plan(t, 0)    # later steps were planned by _sync_decide
            else:
                self._plan_step(t, vids)
            N.check(N.lib().qcb_copy_async(self.pol_host.data_ptr(), self.pol.data_ptr(),
                                           self.pol.numel(), N.stream_ptr()), "copy_async")
            # steps >= t + 2 had their records copied before the previous sync:
            # turn them into TraceRecords while the device runs this plan
            if t + 2 <= t_built:
                self._trace_steps(traces, range(t_built, t + 1, -1))
                t_built = t + 1
            st.synchronize()
            # the decisions straight from the pinned copy (QcbPolicyVideo.action /
            # .abits as int32 words; ctypes parsing costs ~10 us per video)
            npl = 1 if self.sync else nv
            r32 = self.pol_host.numpy()[:npl * self.pol_size].view(np.int32).reshape(npl, -1)
            act_tab = r32[:, self._act_off:self._act_off + L].tolist()
            abits_of = r32[:, self._abits_off].tolist()
            if self.sync:   # every video (and every rank) takes one path
                act_tab, abits_of = act_tab * nv, abits_of * nv
            for vs in vids:
                vs.seen += 1
            self._run_step(t, vids, act_tab, abits_of, collect_features, gen)
        outv = vids[::2] if cfgm else vids   # the latent of each video
        if return_device:
            out = torch.stack([self.slot_view(vs.x) for vs in outv]).reshape(len(outv), F, Tk, d)
            st.synchronize()
            self._trace_steps(traces, range(t_built, -1, -1))
            for vs, tr in zip(vids, traces):
                vs.trace = tr
            return out, vids
        # latents to the host: a pinned block from torch's caching host allocator
        # (a new array per call, reused only once the caller drops it) filled by
        # async per-video D2H copies on the engine stream (a pageable .cpu() of
        # the stacked latents ran at ~2 GB/s: 36 ms for 4 C3 videos)
        host = torch.empty((len(outv), S, d), dtype=torch.float32, pin_memory=True)
        for v, vs in enumerate(outv):
            host[v].copy_(self.slot_view(vs.x), non_blocking=True)
        st.synchronize()
        self._trace_steps(traces, range(t_built, -1, -1))
        for vs, tr in zip(vids, traces):
            vs.trace = tr
        return host.numpy().reshape(len(outv), F, Tk, d), traces

    def _plan_step(self, t: int, vids):
        """Per-video plan of step t: V reductions, plan_reuse + SRAP (unless the
        side stream already ran them during step t+1's head), plan_finish."""
        nv, L, S, d = len(vids), self.L, self.S, self.d
        st, lib, sp, pol = self.stream, N.lib(), N.stream_ptr(), self.pol.data_ptr()
        nh = len(vids[0].hist)
        pre = self._l1_tables(vids)
        early = self._early if (self._early is not None and self._early[0] == t) else None
        self._early = None
        if early is None:
            do_srap = self.tog.srap and not (vids[0].seen == 0 or t == 0)
            if do_srap:
                pre += self._srap_tables(vids)
        tabs = self._upload_idx(pre)
        with self._ph("plan"):
            self._reduce_l1(tabs, nh, nv)
            if early is None:
                self._plan_reuse_srap(t, nv, do_srap, tabs[-3:] if do_srap else [], st)
        with self._ph("plan_srap_wait"):
            if early is not None:
                st.wait_event(early[1])   # plan_reuse / SRAP of this step ran on the side stream
            N.check(lib.qcb_policy_plan_finish(pol, nv, L, t, self.thc, N.ptr(self.srap_v),
                                               N.ptr(self.l1_v), nh,
                                               N.ptr(self.draws[t]), 0, sp), "plan_finish")
            Dv.count(1)

    def _l1_tables(self, vids) -> List[List[int]]:
        """Row tables of x_t and its history entries (cumulative_variation)."""
        nh = len(vids[0].hist)
        if nh == 0:
            return []
        return [[self.rows(vs.x) for vs in vids]] + \
            [[self.rows(vs.hist[j]) for vs in vids] for j in range(nh)]

    def _reduce_l1(self, tabs, nh: int, nv: int):
        """V terms sum|x - h_j| of every history entry in one pass over x
        (schedule.py:128-133) into l1_v[j][video]."""
        if nh:
            Dv.reduce_l1_hist(Dv.feat(self.arena, tabs[0]),
                              [Dv.feat(self.arena, tabs[1 + j]) for j in range(nh)],
                              self.S, self.d, nv, self.l1_v)

    # ------------------------------------------------------------------ synchronised mode
    def _sync_plan(self, tn: int, nh: int):
        """plan_step of step tn for the ONE policy state of the synchronised
        mode, from the all-reduced sums in self.stats (schedule.py:281-328)."""
        lib, sp, pol, L = N.lib(), N.stream_ptr(), self.pol.data_ptr(), self.L
        N.check(lib.qcb_policy_plan_reuse(pol, 1, L, tn, self.thc, sp), "plan_reuse")
        N.check(lib.qcb_policy_plan_finish(pol, 1, L, tn, self.thc, N.ptr(self.srap_g),
                                           N.ptr(self.l1_g), nh, N.ptr(self.draws[tn]), 0, sp),
                "plan_finish")
        Dv.count(2)

    def _sync_decide(self, t: int, vids):
        """Synchronised mode, after reverse_step(t): every input of
        the next decisions is known -- D sums of step t's recomputes
        (schedule.py:342-350), S sums of the step-t features prev[l-1] vs prev[l]
        (:301-305, for every layer: which ones plan(t-1) keeps depends on D) and
        the V terms of x_{t-1} against the history (:293).  They are summed over
        the local videos, packed into one f64 vector and all-reduced over the
        ranks (ONE collective per step); then every rank runs the identical
        observe + plan kernels, so all videos of all ranks take the same path.
        Equals the reference formulas on the concatenated batch
        (oracle.sample_sync): L1 terms, squares, dots and norms are additive."""
        from . import dist as qdist
        nv, L, S, d = len(vids), self.L, self.S, self.d
        lib, sp, pol = N.lib(), N.stream_ptr(), self.pol.data_ptr()
        nh = len(vids[0].hist)             # history after finalize_step(t)
        do_plan = t > 0
        do_srap = self.tog.srap and t - 1 > 0   # plan(t-1) is a boundary iff t-1 == 0
        pre = self._l1_tables(vids) if do_plan else []
        n_l1 = len(pre)
        if do_srap:
            pre += self._srap_tables(vids)
        tabs = self._upload_idx(pre)
        with self._ph("plan"):
            if do_plan:
                self._reduce_l1(tabs, nh, nv)
            if do_srap:
                Dv.reduce_srap(Dv.feat(self.arena, tabs[n_l1]),
                               Dv.feat(self.arena, tabs[n_l1 + 1]), S, d, L * nv,
                               self.srap_v.view(L * nv, 3),
                               seg_active=self.sync_mask_v.view(L * nv),
                               workspace=self._srap_ws, dup_src=tabs[n_l1 + 2])
            # pack the local sums (fixed video order: deterministic), then ranks
            qdist.pack_decision_sums(self.stats, self.hlc_v, self.srap_v, self.l1_v)
            qdist.allreduce_sum(self.stats, group=self.sync_group)
            N.check(lib.qcb_policy_observe_all(pol, 1, L, t, self.thc, N.ptr(self.hlc_g), sp),
                    "observe_all")
            Dv.count(1)
            self.pol_trace[t, :self.pol_size].copy_(self.pol[:self.pol_size], non_blocking=True)
            if do_plan:
                self._sync_plan(t - 1, nh)

    # ------------------------------------------------------------------ one step
    def _run_step(self, t: int, vids, act_tab, abits_of, collect_features, gen):
        """Execute step t's plan: recomputed blocks with the HLC reductions,
        observe, the noise head and the DDPM update (sampler.py:114-133)."""
        nv, L, S, d = len(vids), self.L, self.S, self.d
        F, Tk = self.cfg.frames, self.cfg.tokens_per_frame
        st, lib, sp, pol = self.stream, N.lib(), N.stream_ptr(), self.pol.data_ptr()
        first_launch = None
        if self.host_profile is not None:
            t_sync = time.perf_counter()
        # ---------------- execute blocks ----------------
        fast = collect_features is None and not any(
            a == N.ACT_RECOMPUTE for row in act_tab for a in row)
        if fast:
            # nothing recomputes: the head reads each video's last reused cache
            # entry (or x_t); the prev bookkeeping runs after the head launch
            cur = []
            for v, vs in enumerate(vids):
                c = vs.x
                for l, a in enumerate(act_tab[v]):
                    if a == N.ACT_REUSE:
                        c = vs.cache[l]
                cur.append(vs.pool.inc(c))
            x_in = [vs.x for vs in vids]
        else:
            cur = [vs.pool.inc(vs.x) for vs in vids]     # block input slot per video
        feats = [] if collect_features is not None else None
        for l in range(0 if fast else L):
            acts = [act_tab[v][l] for v in range(nv)]
            outs = list(cur)
            rec = []
            for v in range(nv):
                a = acts[v]
                if a == N.ACT_REUSE:
                    outs[v] = vids[v].pool.inc(vids[v].cache[l])
                elif a == N.ACT_PRUNE:
                    outs[v] = vids[v].pool.inc(cur[v])
                else:
                    outs[v] = vids[v].pool.alloc()
                    rec.append(v)
            if rec:
                # group recomputing videos by activation bits
                groups: Dict[int, List[int]] = {}
                for v in rec:
                    groups.setdefault(abits_of[v], []).append(v)
                need_d = [acts[v] == N.ACT_RECOMPUTE and vids[v].prev[l] is not None
                          for v in range(nv)]
                tabl = []
                for bits, g in groups.items():
                    tabl += [[self.rows(cur[v]) for v in g], [self.rows(outs[v]) for v in g], g]
                if any(need_d):
                    tabl += [[self.rows(outs[v]) for v in range(nv)],
                             [self.rows(vids[v].cache[l] if vids[v].cache[l] is not None
                                        else (vids[v].prev[l] or 0)) for v in range(nv)],
                             [self.rows(vids[v].prev[l] or 0) for v in range(nv)],
                             [int(x) for x in need_d]]
                tl = self._upload_idx(tabl)
                if self.host_profile is not None and first_launch is None:
                    first_launch = time.perf_counter() - t_sync
                for gi, (bits, g) in enumerate(groups.items()):
                    self._block(l, t, g, bits, tl[3 * gi], tl[3 * gi + 1], tl[3 * gi + 2])
                if any(need_d):
                    base = 3 * len(groups)
                    act = tl[base + 3].t.to(torch.int32)
                    with self._ph("hlc"):
                        Dv.reduce_hlc(Dv.feat(self.arena, tl[base]),
                                      Dv.feat(self.arena, tl[base + 1]),
                                      Dv.feat(self.arena, tl[base + 2]), S, d, nv,
                                      self.hlc_v[l], seg_active=act)

            # host mirror of the cache / prev references (schedule.py:349-351)
            for v, vs in enumerate(vids):
                if acts[v] == N.ACT_RECOMPUTE and t > 0:
                    vs.pool.dec(vs.cache[l])
                    vs.cache[l] = vs.pool.inc(outs[v])
                vs.pool.dec(vs.prev[l])
                vs.prev[l] = vs.pool.inc(outs[v])
                vs.pool.dec(cur[v])
            cur = outs
            if feats is not None:
                feats.append(torch.stack([self.slot_view(s) for s in cur]).cpu().numpy())
        if self.host_profile is not None:
            now = time.perf_counter() - t_sync
            self.host_profile.append((now, first_launch if first_launch is not None else now))
        ready = None
        if not self.sync:
            # observe_block for every layer of the step (schedule.py:330-351)
            N.check(lib.qcb_policy_observe_all(pol, nv, L, t, self.thc, N.ptr(self.hlc_v), sp),
                    "observe_all")
            Dv.count(1)
            N.check(lib.qcb_copy_async(self.pol_trace.data_ptr() + t * self.pol.numel(), pol,
                                       self.pol.numel(), sp), "copy_async")
            if t > 0:
                ready = torch.cuda.Event()
                ready.record(st)
        if collect_features is not None:
            x_now = torch.stack([self.slot_view(vs.x) for vs in vids]).cpu().numpy()
            collect_features.append((t, x_now, feats))
        # ---------------- head + sampler update ----------------
        # A video whose head input is the very slot its eps was computed from at
        # an earlier step (an unchanged cache entry with every later layer
        # pruned or reused from it) gets bit-identical eps = mm(x, head_w) + b
        # (model.py:228): slots are never mutated while referenced, and the
        # video holds a reference to its head-input slot.  Only the others run.
        need = [v for v in range(nv) if vids[v].head_src != cur[v]]
        self.head_calls += nv
        self.head_skipped += nv - len(need)
        if need:
            tabh = self._upload_idx([[self.rows(cur[v]) for v in need],
                                     [v * self.Sp for v in need]])
            with self._ph("head"):
                if self.head_prep is not None:
                    Dv.head_gemm(self.arena, self.head_prep, out=self.eps, bias=self.head_b,
                                 seg_rows=self.Sp, seg_valid=S, nseg=len(need),
                                 a_row0=tabh[0], out_row0=tabh[1],
                                 fallback_count=self.head_fallbacks)
                else:
                    Dv.gemm_f64(self.arena, self.head_w, out=self.eps, epilogue=N.EPI_BIAS,
                                bias=self.head_b, seg_rows=self.Sp, seg_valid=S,
                                a_row0=tabh[0], out_row0=tabh[1], M=len(need) * self.Sp)
            for v in need:
                vs = vids[v]
                vs.pool.dec(vs.head_src)
                vs.head_src = vs.pool.inc(cur[v])
        with self._ph("sampler"):
            # CFG (extension): slots (2i, 2i+1) are video i's cond / uncond
            # branches; one DDPM update per video from the guided eps, its
            # result copied into the uncond branch's own slot
            step = 2 if self.cfg_scale is not None else 1
            rf = self.opts.sampler == "rf"
            if t > 0 and self.opts.noise == "numpy" and not rf:
                for i, v in enumerate(range(0, nv, step)):
                    self.noise_host[i].numpy()[:] = vids[v].rng.standard_normal(
                        (F, Tk, d)).astype(np.float32).reshape(S, d)
                self.noise_dev[:nv // step].copy_(self.noise_host[:nv // step], non_blocking=True)
            quads = (S * d + 3) // 4
            a_t = self.ab[t]
            for v, vs in enumerate(vids):
                if v % step:
                    continue   # an uncond branch: updated with its cond branch below
                i = v // step   # video index (noise stream, guided eps)
                new = vs.pool.alloc()
                eps_v = self.eps[v * self.Sp: v * self.Sp + S]
                if step == 2:
                    eps_v = Dv.cfg_combine(eps_v, self.eps[(v + 1) * self.Sp:(v + 1) * self.Sp + S],
                                           self.cfg_scale, out=self.eps_cfg[i])
                if rf:   # Euler step of the flow ODE: f32(x - (1/T) v) in f64
                    Dv.ddpm(self.slot_view(vs.x), eps_v, 1.0 / self.T, 1.0,
                            out=self.slot_view(new))
                elif t > 0:
                    a_p = self.ab[t - 1]
                    alpha = a_t / a_p
                    beta = 1.0 - alpha
                    c3 = float(np.sqrt((1.0 - a_p) / (1.0 - a_t) * beta)) if t > 1 else 0.0
                    dev_noise = gen is not None and t > 1
                    Dv.ddpm(self.slot_view(vs.x), eps_v, float(beta / np.sqrt(1.0 - a_t)),
                            float(np.sqrt(alpha)),
                            self.noise_dev[i] if (t > 1 and not dev_noise) else None, c3,
                            out=self.slot_view(new),
                            noise_gen=(gen[i], t * quads) if dev_noise else None)
                else:
                    Dv.ddpm(self.slot_view(vs.x), eps_v, float(np.sqrt(1.0 - self.ab[0])),
                            float(np.sqrt(self.ab[0])), out=self.slot_view(new))
                news = [(v, new)]
                if step == 2:
                    vu = vids[v + 1]
                    new_u = vu.pool.alloc()
                    N.check(N.lib().qcb_copy_async(N.ptr(self.slot_view(new_u)),
                                                   N.ptr(self.slot_view(new)), S * d * 4, sp),
                            "copy_async")
                    news.append((v + 1, new_u))
                for w, nw in news:
                    ws = vids[w]
                    ws.pool.dec(cur[w])
                    # finalize_step: latent history window (schedule.py:353-357)
                    ws.hist.append(ws.x)
                    if len(ws.hist) > self.th.history_k:
                        ws.pool.dec(ws.hist.pop(0))
                    ws.x = nw
        if fast:
            # prev references of the step (schedule.py:349-351): a reused layer's
            # output is its cache entry, a pruned layer passes its input through
            for v, vs in enumerate(vids):
                c = x_in[v]
                for l, a in enumerate(act_tab[v]):
                    if a == N.ACT_REUSE:
                        c = vs.cache[l]
                    vs.pool.dec(vs.prev[l])
                    vs.prev[l] = vs.pool.inc(c)
        if ready is not None:
            # the next step's reuse plan depends only on the cache state just
            # observed (schedule.py:286-309): it runs on the side stream while
            # the head (launched above) runs
            self._early = self._early_plan(t - 1, vids, ready)
        if self.sync:
            self._sync_decide(t, vids)

    def traces_of(self, vids) -> List[List[TraceRecord]]:
        return [vs.trace for vs in vids]

    def _collect_traces(self, vids) -> List[List[TraceRecord]]:
        """Per-video TraceRecords (schedule.py:187-210) of every step, from the
        per-step policy records in pinned host memory."""
        traces = [[] for _ in range(len(vids))]
        self._trace_steps(traces, range(self.T - 1, -1, -1))
        return traces

    def _trace_steps(self, traces, steps) -> None:
        """Append the records of `steps` (descending t) to traces[v]: one
        structured numpy view of those rows of the [T][videos] QcbPolicyVideo
        array, columns converted to Python lists once (per-record ctypes access
        cost ~40 ms per 4-video call)."""
        steps = list(steps)
        if not steps:
            return
        gc_was = gc.isenabled()
        gc.disable()   # ~12k new records would trigger collections (+45 ms when one hits gen 2)
        try:
            self._trace_steps_impl(traces, steps)
        finally:
            if gc_was:
                gc.enable()

    def _trace_steps_impl(self, traces, steps) -> None:
        nv, L = len(traces), self.L
        npv = 1 if self.sync else nv
        lo, hi = steps[-1], steps[0]
        raw = self.pol_trace[lo:hi + 1, :npv * self.pol_size].numpy()
        rec = np.ascontiguousarray(raw).view(_policy_dtype()).reshape(hi + 1 - lo, npv)
        A, DV, DN = rec["action"].tolist(), rec["d_valid"].tolist(), rec["d_now"].tolist()
        SV, SM = rec["sim_valid"].tolist(), rec["sim"].tolist()
        AB, VV = rec["abits"].tolist(), rec["v"].tolist()
        wbs = [self.weight_bits.get(l, FP_BITS) if self.tog.aigq_weights else FP_BITS
               for l in range(L)]
        macs_of: Dict[int, list] = {}   # abits -> billed MACs per layer when recomputed
        rc = N.ACT_RECOMPUTE
        head_macs = self.head_macs * FP_BITS * FP_BITS
        layers = range(L)
        for t in steps:
            k = t - lo
            for v in range(nv):
                pv = 0 if self.sync else v
                ab, vf = int(AB[k][pv]), float(VV[k][pv])
                mt = macs_of.get(ab)
                if mt is None:
                    mt = macs_of[ab] = [billed_macs(self.block_cost, wb, ab) for wb in wbs]
                out = traces[v]
                out.extend([TraceRecord(t, l, ACTION_NAMES[a], dn if dv else None,
                                        sm if sv else None, ab, wb, m if a == rc else 0, vf)
                            for l, a, dv, dn, sv, sm, wb, m in
                            zip(layers, A[k][pv], DV[k][pv], DN[k][pv], SV[k][pv], SM[k][pv],
                                wbs, mt)])
                out.append(TraceRecord(t, "head", "recompute", None, None, FP_BITS, FP_BITS,
                                       head_macs))
