"""The engine's synchronised-decision mode with TWO processes (world size 2,
gloo) sharing one GPU: every step all-reduces the packed decision sums of the
two ranks' videos (engine._sync_decide, dist.allreduce_sum), then both ranks
run the identical plan kernels.  Compared with oracle.sample_sync on the
concatenated batch: one shared trace, identical decisions at
every (step, layer), D / S / V within 1e-9, bit-identical latents per video.

The ranks' kernels never wait on one another (the only cross-rank dependency
is the host-side gloo all-reduce), so running both on one GPU is safe."""

import os
import pickle
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
SEEDS = {0: [3, 11], 1: [12]}
SMALL = {"seed": 3, "model": {"num_blocks": 3, "model_dim": 16, "num_heads": 2,
                              "tokens_per_frame": 4, "frames": 2, "cond_dim": 8},
         "schedule": {"steps": 10},
         "toggles": dict(hlc=True, aigq_weights=True, aigq_acts=True, srap=True),
         "device": {"decisions": "synchronized"}}


def _rank(rank, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    from paper_2503_06545_b200 import harness
    cfg = harness.parse_config(dict(SMALL, calibration=os.path.join(GOLDEN, "calib_small.json")))
    calib = harness.load_calibration(cfg.calibration)
    eng, _ = harness.build_engine(cfg, cfg.toggles_obj(), calib, max_videos=len(SEEDS[rank]))
    outs, traces = eng.generate(SEEDS[rank])
    with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as f:
        pickle.dump((np.asarray(outs), [[r.to_json_obj() for r in tr] for tr in traces]), f)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_synchronised_decisions_match_oracle(tmp_path, cuda_dev):
    import torch.multiprocessing as mp
    from dataclasses import fields
    from oracle import qc_oracle as O
    from paper_2503_06545_b200 import harness
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.start_processes(_rank, args=(port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    got = {r: pickle.load(open(tmp_path / f"rank{r}.pkl", "rb")) for r in (0, 1)}
    cfg = harness.parse_config(dict(SMALL, calibration=os.path.join(GOLDEN, "calib_small.json")))
    calib = harness.load_calibration(cfg.calibration)
    tog = cfg.toggles_obj()
    thr = harness.resolve_thresholds(cfg, calib, tog)
    th = O.Thresholds(**{f.name: getattr(thr, f.name) for f in fields(O.Thresholds)})
    seeds = SEEDS[0] + SEEDS[1]
    want, st = O.sample_sync(O.ModelDims(3, 16, 2, 4, 2, 8, cfg.seeds["model"]), 10, th,
                             (tog.hlc, tog.aigq_weights, tog.aigq_acts, tog.srap), seeds,
                             prune_seed=cfg.seeds["prune"],
                             weight_bits=harness.resolve_weight_bits(cfg, calib),
                             act_absmax=calib.act_absmax, sign_seed=cfg.seeds["model"])
    outs = list(got[0][0]) + list(got[1][0])
    traces = got[0][1] + got[1][1]
    assert len(st.trace) == len(traces[0])
    for tr in traces:
        assert tr == traces[0]                       # every video of both ranks: one path
    for a, b in zip(st.trace, traces[0]):
        for k in ("t", "layer", "action", "bits", "wbits", "macs"):
            assert a[k] == b[k], (k, a, b)
        for k in ("D", "S", "V"):
            if a[k] is not None and b[k] is not None:
                assert b[k] == pytest.approx(a[k], rel=1e-9, abs=1e-12), (k, a, b)
            elif k != "V":
                assert a[k] is None and b[k] is None, (k, a, b)
    assert any(r["action"] != "recompute" for r in st.trace)
    for v in range(len(seeds)):
        assert np.array_equal(outs[v], want[v]), v
