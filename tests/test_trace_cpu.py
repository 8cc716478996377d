"""Trace records from the per-step policy array (engine._collect_traces), checked
against a per-record ctypes reading of the same bytes (CPU, no kernels)."""
import ctypes as C
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from paper_2503_06545_b200 import _native as N
from paper_2503_06545_b200.engine import ACTION_NAMES, QuantCacheEngine
from paper_2503_06545_b200.schedule import FP_BITS, TraceRecord


def _fake_engine(T, nv, sync, seed):
    L = len(N.QcbPolicyVideo().action)
    size = C.sizeof(N.QcbPolicyVideo)
    npv = 1 if sync else nv
    rng = np.random.default_rng(seed)
    recs = (N.QcbPolicyVideo * (T * npv))()
    for r in recs:
        r.abits = int(rng.choice([4, 6, 8]))
        r.v = float(rng.standard_normal())
        for l in range(L):
            r.action[l] = int(rng.integers(0, len(ACTION_NAMES)))
            r.d_valid[l] = int(rng.integers(0, 2))
            r.d_now[l] = float(rng.standard_normal())
            r.sim_valid[l] = int(rng.integers(0, 2))
            r.sim[l] = float(rng.uniform(-1, 1))
    raw = np.frombuffer(bytes(recs), dtype=np.uint8).reshape(T, npv * size)
    full = np.zeros((T, nv * size), dtype=np.uint8)
    full[:, :npv * size] = raw
    eng = SimpleNamespace(
        L=L, T=T, sync=sync, pol_size=size, pol_trace=torch.from_numpy(full),
        weight_bits={l: 4 + (l % 3) for l in range(L)},
        tog=SimpleNamespace(aigq_weights=True), head_macs=1000,
        block_cost=None)
    for name in ("_trace_steps", "_trace_steps_impl"):
        setattr(eng, name, getattr(QuantCacheEngine, name).__get__(eng))
    return eng


def _macs(wb, ab):   # stand-in cost model (the block cost itself is tested elsewhere)
    return 7 * wb + int(ab)


def _reference(eng, nv):
    raw = eng.pol_trace.numpy()
    traces = [[] for _ in range(nv)]
    for t in range(eng.T - 1, -1, -1):
        for v in range(nv):
            pv = 0 if eng.sync else v
            p = N.QcbPolicyVideo.from_buffer_copy(
                raw[t, pv * eng.pol_size:(pv + 1) * eng.pol_size].tobytes())
            for l in range(eng.L):
                a = p.action[l]
                wb = eng.weight_bits[l]
                macs = _macs(wb, p.abits) if a == N.ACT_RECOMPUTE else 0
                traces[v].append(TraceRecord(
                    t, l, ACTION_NAMES[a], float(p.d_now[l]) if p.d_valid[l] else None,
                    float(p.sim[l]) if p.sim_valid[l] else None, int(p.abits), wb, macs,
                    float(p.v)))
            traces[v].append(TraceRecord(t, "head", "recompute", None, None, FP_BITS,
                                         FP_BITS, eng.head_macs * FP_BITS * FP_BITS))
    return traces


@pytest.mark.parametrize("sync", [False, True])
def test_collect_traces_matches_per_record_reading(monkeypatch, sync):
    import paper_2503_06545_b200.engine as E
    monkeypatch.setattr(E, "billed_macs", lambda cost, wb, ab: _macs(wb, ab))
    nv = 3
    eng = _fake_engine(T=5, nv=nv, sync=sync, seed=1)
    got = QuantCacheEngine._collect_traces(eng, [None] * nv)
    want = _reference(eng, nv)
    assert [[r.to_json_obj() for r in tv] for tv in got] == \
        [[r.to_json_obj() for r in tv] for tv in want]


@pytest.mark.parametrize("sync", [False, True])
def test_incremental_trace_build_matches_full_reading(monkeypatch, sync):
    """generate() builds finished steps while it waits on each decision sync
    (steps >= t + 2 at step t, the rest after the loop): same records, same order."""
    import paper_2503_06545_b200.engine as E
    monkeypatch.setattr(E, "billed_macs", lambda cost, wb, ab: _macs(wb, ab))
    nv, T = 2, 7
    eng = _fake_engine(T=T, nv=nv, sync=sync, seed=2)
    traces = [[] for _ in range(nv)]
    t_built = T - 1
    for t in range(T - 1, -1, -1):
        if t + 2 <= t_built:
            eng._trace_steps(traces, range(t_built, t + 1, -1))
            t_built = t + 1
    eng._trace_steps(traces, range(t_built, -1, -1))
    want = _reference(eng, nv)
    assert [[r.to_json_obj() for r in tv] for tv in traces] == \
        [[r.to_json_obj() for r in tv] for tv in want]
