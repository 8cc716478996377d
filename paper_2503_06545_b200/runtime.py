"""QuantRuntime (mirror of ditrt.runtime, runtime.py:31-81) on the device.

Holds the immutable prepared-weight snapshot of one run and exposes the
per-step GEMM hook `gemm_fn(abits)` with the reference's signature
`gemm(layer, site, x, w) -> y`, where x is a CUDA f32 [M, K] tensor.  The hook
routes exactly as the reference does: integer W+A GEMM (act_quant ->
tcgen05 u8 GEMM), weight-only (rotated activations x dequantized weights), or
activation-only fake quantization; all three are libqcb200 kernels."""

from __future__ import annotations

from typing import Dict, Optional

import numpy as np
import torch

from . import _native as N
from . import device as Dv
from .engine import balance_scales
from .model import QUANT_SITES, DiTModel
from .schedule import FP_BITS, Toggles


class QuantRuntime:
    def __init__(self, model: DiTModel, toggles: Toggles, weight_bits: Dict[int, int],
                 site_act_absmax: Optional[Dict[int, Dict[str, np.ndarray]]] = None,
                 sign_seed: int = 0):
        self.toggles = toggles
        self.weight_bits = dict(weight_bits)
        self.site_act_absmax = site_act_absmax
        self.sign_seed = sign_seed
        self._prepared: Dict[tuple, Dv.PackedWeight] = {}
        self._model = model
        if not toggles.aigq_weights:
            return
        signs = {}
        for l, blk in enumerate(model.blocks):
            stats = (site_act_absmax or {}).get(l, {})
            for site in QUANT_SITES:
                w = getattr(blk, site)
                wt = torch.as_tensor(w).cuda()
                if stats.get(site) is not None:
                    b = Dv.pow2_floor(w.shape[0])
                    if b not in signs:
                        signs[b] = torch.as_tensor(Dv.sign_vector(sign_seed, b)).cuda()
                    c = torch.as_tensor(balance_scales(w, stats[site])).cuda()
                    pw = Dv.weight_prep(wt, weight_bits[l], c, signs[b], keep_deq=True)
                else:
                    pw = Dv.weight_prep(wt, weight_bits[l], keep_deq=True)
                self._prepared[(l, site)] = pw

    def gemm_fn(self, abits: int):
        """GEMM hook for one step; abits >= 32 means full-precision activations."""
        tog = self.toggles
        if not (tog.aigq_weights or tog.aigq_acts):
            return None
        quant_acts = tog.aigq_acts and abits < FP_BITS

        def gemm(layer: int, site: str, x, w):
            # type-preserving at the LayerHooks boundary (model.py:89-90): an
            # ndarray in (the reference's block_forward) gives an ndarray out
            if not isinstance(x, torch.Tensor):
                y = gemm_dev(layer, site, torch.as_tensor(np.asarray(x, np.float32)), w)
                return y.cpu().numpy()
            return gemm_dev(layer, site, x, w)

        def gemm_dev(layer: int, site: str, x: torch.Tensor, w):
            xt = x.float().cuda().contiguous()
            if tog.aigq_weights:
                pw = self._prepared[(layer, site)]
                tr = [(pw.chan_scale, pw.signs)] if pw.chan_scale is not None else [None]
                if quant_acts:
                    (a,) = Dv.act_quant(xt, abits, tr)
                    return Dv.gemm_u8(a, pw)
                if tr[0] is not None:
                    (r,) = Dv.act_quant(xt, 8, tr, want_codes=False, want_xe=True)
                    xt = r.xe
                return Dv.gemm_f64(xt, pw.w_deq)
            wt = w if isinstance(w, torch.Tensor) else torch.as_tensor(np.asarray(w, np.float32))
            (r,) = Dv.act_quant(xt, abits, [None], want_codes=False, want_deq=True)
            return Dv.gemm_f64(r.deq, wt.float().cuda().contiguous())

        return gemm
