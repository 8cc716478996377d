"""CPU arm of bench.py: the reference's own hot path timed on host cores.

TEST/BENCH INFRASTRUCTURE -- never imported by the product package.

The reference (`ditrt`, pure Python/NumPy) is installed unmodified into
`baseline/_ref` (pip --target), which travels to the
GPU box with the repo snapshot.  One recomputed block of the sampling path is
timed through the reference's OWN functions on a slice of r token rows:

  * the 10 GEMM sites through `QuantRuntime.gemm_fn(abits)` (runtime.py:63-81):
    `BalanceTransform.apply_to_activation` (the sequential f64 rotation,
    quant.py:163-165), `compute_minmax_params`, `quantize` (quant.py:83-123),
    `matmul_int` (tensor.py:68-112);
  * `_ln`, `_gelu`, residual/gate arithmetic of `block_forward` (model.py:159-199);
  * `_mha` (model.py:150-156) for the r query rows against all S keys/values;
  * the FP noise head `mm(x, head_w) + head_b` (model.py:228) and
    `reverse_step` (sampler.py:59-80) on the r rows.

Setup (random-init weights, the weight-side rotation, weight quantization,
the dense rotation matrix, K/V of all S tokens) is done once, outside the
timed region.  The weight-side rotation R^T (c (.) W) is computed by a fast
FWHT restatement for setup speed; the reference's own `compute_minmax_params`
and `quantize` then quantize it.  Each sample times r1 and r2 rows and fits
t(r) = a + b r (a: per-call costs such as the cond-token sites and the
Python k-loop overheads, b: per-row cost including attention over S keys),
then evaluates t(S).  Falls back to the oracle port (oracle/qc_oracle.py)
when the installed reference is absent.
"""

from __future__ import annotations

import os
import sys
import time
from typing import Dict, Optional

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
SITES = ("sta_q", "sta_k", "sta_v", "sta_o", "ca_q", "ca_k", "ca_v", "ca_o", "ffn1", "ffn2")


def load_reference():
    """The installed reference package `ditrt`, or None."""
    if os.path.isdir(os.path.join(REF_DIR, "ditrt")):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        try:
            import ditrt  # noqa: F401
            import ditrt.model, ditrt.runtime, ditrt.quant, ditrt.sampler, ditrt.tensor  # noqa
            return ditrt
        except Exception:
            return None
    return None


def _fwht_cols(v: np.ndarray) -> np.ndarray:
    """Unnormalised Walsh-Hadamard transform along axis 0 (f64)."""
    v = np.array(v, dtype=np.float64, copy=True)
    n = v.shape[0]
    h = 1
    while h < n:
        v = v.reshape(n // (2 * h), 2, h, -1)
        a = v[:, 0].copy()
        b = v[:, 1].copy()
        v[:, 0] = a + b
        v[:, 1] = a - b
        v = v.reshape(n, -1)
        h *= 2
    return v


def _weight_eff(w: np.ndarray, c: np.ndarray, seed: int) -> np.ndarray:
    """R^T (c (.) W) (quant.py:167-169) via an f64 FWHT (setup only)."""
    K = w.shape[0]
    b = 1 << (K.bit_length() - 1)
    sc = (c[:, None] * w.astype(np.float64)).astype(np.float32).astype(np.float64)
    signs = np.where(np.random.default_rng(seed).random(b) < 0.5, -1.0, 1.0)
    out = sc.copy()
    out[:b] = _fwht_cols(signs[:, None] * sc[:b]) * np.float64(np.float32(1.0 / np.sqrt(b)))
    return out.astype(np.float32)


class BlockSample:
    """One recomputed block + head + DDPM update of the reference path on r rows."""

    def __init__(self, S: int, d: int, heads: int, cond_dim: int, wbits: int = 6,
                 abits: int = 8, seed: int = 0):
        self.ref = load_reference()
        self.kind = "reference" if self.ref is not None else "port"
        self.S, self.d, self.H, self.c = S, d, heads, cond_dim
        self.abits = abits
        rng = np.random.default_rng(seed)
        f = 4 * d
        shapes = {"sta_q": (d, d), "sta_k": (d, d), "sta_v": (d, d), "sta_o": (d, d),
                  "ca_q": (d, d), "ca_k": (cond_dim, d), "ca_v": (cond_dim, d),
                  "ca_o": (d, d), "ffn1": (d, f), "ffn2": (f, d)}
        self.w = {s: rng.standard_normal(sh, dtype=np.float32) * np.float32(sh[0] ** -0.5)
                  for s, sh in shapes.items()}
        self.ln = [(np.ones(d, np.float32), np.zeros(d, np.float32)) for _ in range(3)]
        self.head_w = rng.standard_normal((d, d), dtype=np.float32) * np.float32(d ** -0.5)
        self.head_b = rng.standard_normal(d, dtype=np.float32) * np.float32(d ** -0.5)
        self.mod = (rng.standard_normal(6) * 0.1).astype(np.float32)
        self.cond = rng.standard_normal((1, cond_dim), dtype=np.float32)
        # K/V of all S tokens for the r query rows' attention (setup)
        self.kf = rng.standard_normal((S, d), dtype=np.float32)
        self.vf = rng.standard_normal((S, d), dtype=np.float32)
        self.x_all = rng.standard_normal((S, d), dtype=np.float32)
        self.noise = rng.standard_normal((S, d), dtype=np.float32)
        # balance statistics shared by the sites that read the same input
        absmax = {}
        for s, (K, _) in shapes.items():
            a = np.abs(self.w[s]).max(axis=1).astype(np.float64)
            absmax[s] = a * np.exp(rng.standard_normal(K) * 0.5)
        if self.ref is not None:
            self._prep_reference(absmax, wbits)
        else:
            self._prep_port(absmax, wbits)

    # -------------------------------------------------------------- setup
    def _prep_reference(self, absmax, wbits):
        R = self.ref
        from ditrt.quant import (BalanceTransform, compute_minmax_params, dequantize,
                                 quantize)
        from ditrt.runtime import QuantRuntime
        from ditrt.schedule import Toggles
        from ditrt.tensor import Tensor
        rt = object.__new__(QuantRuntime)
        rt.toggles = Toggles(hlc=False, aigq_weights=True, aigq_acts=True, srap=False)
        rt._prepared = {}
        for s, w in self.w.items():
            K = w.shape[0]
            wa = np.abs(w.astype(np.float64)).max(axis=1)
            c = np.clip(np.sqrt(absmax[s] / wa), 1e-3, 1e3)
            b = 1 << (K.bit_length() - 1)
            tr = BalanceTransform(c, b, 0)
            tr.rotation_matrix()     # built and cached here, not in the timed region
            w_eff = _weight_eff(w, c, 0)
            params = compute_minmax_params(Tensor(w_eff), wbits, granularity="per-channel",
                                           axis=1)
            wq = quantize(Tensor(w_eff), params)
            rt._prepared[(0, s)] = (wq, dequantize(wq).data, tr)
        self.gemm = rt.gemm_fn(self.abits)
        self._ln = R.model._ln
        self._gelu = R.model._gelu
        self._mha = R.model._mha
        self._mm = R.tensor.mm
        self._reverse = R.sampler.reverse_step
        self._sched = R.sampler.linear_beta_schedule(100)
        self._Tensor = R.tensor.Tensor

    def _prep_port(self, absmax, wbits):
        from oracle import qc_oracle as O
        prep = {}
        for s, w in self.w.items():
            K = w.shape[0]
            wa = np.abs(w.astype(np.float64)).max(axis=1)
            c = np.clip(np.sqrt(absmax[s] / wa), 1e-3, 1e3)
            w_eff = _weight_eff(w, c, 0)
            sw, zw = O.chan_params(w_eff, wbits)
            cw = O.codes_of(w_eff, sw[None], zw[None], wbits)
            prep[s] = (c, O.rotation_dense(K, 0).astype(np.float32), cw, sw, zw)
        ab = self.abits

        def gemm(_l, s, x, _w):
            c, rot, cw, sw, zw = prep[s]
            y = (x.astype(np.float64) / c[None, :]).astype(np.float32)
            xe = O.seq_mm(y, rot)
            sa, za = O.act_params(xe, ab)
            return O.matmul_int_seq(O.codes_of(xe, sa, za, ab), sa, za, cw, sw, zw)
        self.gemm = gemm
        self._ln = O.ln64
        self._gelu = O.gelu64
        self._mha = O.attention_heads
        self._mm = O.seq_mm
        ab_ = O.alpha_bar(100)
        self._reverse = lambda x, t, e, _s, n: O.ddpm_step(x, t, e, ab_, n)
        self._sched = None
        self._Tensor = lambda a, **k: a

    # -------------------------------------------------------------- timed
    def _wrap(self, a):
        return self._Tensor(a) if self.kind == "reference" else a

    def _data(self, a):
        return a.data if hasattr(a, "data") and not isinstance(a, np.ndarray) else a

    def block_seconds(self, r: int) -> float:
        """block_forward (model.py:159-199) for r token rows (attention over S keys)."""
        g = self.gemm
        m = self.mod
        one = np.float32(1.0)
        x = self.x_all[:r].copy()
        t0 = time.perf_counter()
        h1 = self._ln(x, *self.ln[0]) * (one + m[1]) + m[0]
        q = g(0, "sta_q", h1, self.w["sta_q"])
        g(0, "sta_k", h1, self.w["sta_k"])      # the rows' own k/v (attention uses all S)
        g(0, "sta_v", h1, self.w["sta_v"])
        att = self._mha(q, self.kf, self.vf, self.H)
        x = x + m[2] * g(0, "sta_o", att, self.w["sta_o"])
        h2 = self._ln(x, *self.ln[1])
        q2 = g(0, "ca_q", h2, self.w["ca_q"])
        k2 = g(0, "ca_k", self.cond, self.w["ca_k"])
        v2 = g(0, "ca_v", self.cond, self.w["ca_v"])
        ca = self._mha(q2, k2, v2, self.H)
        x = x + g(0, "ca_o", ca, self.w["ca_o"])
        h3 = self._ln(x, *self.ln[2]) * (one + m[4]) + m[3]
        hid = self._gelu(g(0, "ffn1", h3, self.w["ffn1"]))
        x = x + m[5] * g(0, "ffn2", hid, self.w["ffn2"])
        return time.perf_counter() - t0

    def head_seconds(self, r: int) -> float:
        """Noise head mm(x, head_w) + head_b (model.py:228) + reverse_step on r rows."""
        x = self.x_all[:r]
        t0 = time.perf_counter()
        eps = self._data(self._mm(x, self.head_w)) + self.head_b
        self._reverse(self._wrap(x), 50, self._wrap(eps), self._sched,
                      self._wrap(self.noise[:r]))
        return time.perf_counter() - t0


def fit_seconds(fn, r1: int, r2: int, S: int) -> Dict[str, float]:
    """Times fn at r1 and r2 rows, fits t = a + b r, returns t(S)."""
    t1 = fn(r1)
    t2 = fn(r2)
    b = max(0.0, (t2 - t1) / (r2 - r1))
    a = max(0.0, t1 - b * r1)
    return {"a": a, "b": b, "t_S": a + b * S, "sample_s": t1 + t2}


def videos_per_s(block_S: float, head_S: float, steps: int, layers: int,
                 recompute_frac: float) -> float:
    """Per video: T steps x (head + DDPM on S rows + frac x L recomputed blocks)."""
    return 1.0 / (steps * (head_S + recompute_frac * layers * block_S))
