import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2503_06545_b200 import harness
SMALL = {"seed": 3, "model": {"num_blocks": 3, "model_dim": 16, "num_heads": 2,
         "tokens_per_frame": 4, "frames": 2, "cond_dim": 8}, "schedule": {"steps": 10}}
for tog in [{}, dict(hlc=True), dict(aigq_weights=True, aigq_acts=True), dict(hlc=True, aigq_weights=True, aigq_acts=True, srap=True)]:
    cfg = harness.parse_config(dict(SMALL, calibration='tests/golden/calib_small.json', toggles=tog))
    calib = harness.load_calibration(cfg.calibration)
    eng, _ = harness.build_engine(cfg, cfg.toggles_obj(), calib, max_videos=2)
    fb = []; ob, tb = eng.generate([3, 11], collect_features=fb)
    e1, _ = harness.build_engine(cfg, cfg.toggles_obj(), calib, max_videos=1)
    fs = []; o1, t1 = e1.generate([11], collect_features=fs)
    print(tog, "video1 equal", np.array_equal(ob[1], o1[0]))
    done = False
    for (t, xb, lb), (_, xs, ls) in zip(fb, fs):
        if not np.array_equal(xb[1], xs[0]):
            print("  x differs at t", t); break
        for l in range(3):
            if not np.array_equal(lb[l][1], ls[l][0]):
                print("  layer out differs t", t, "l", l, float(np.abs(lb[l][1]-ls[l][0]).max()),
                      [r.action for r in tb[1] if r.t == t], [r.action for r in t1[0] if r.t == t])
                done = True; break
        if done: break
