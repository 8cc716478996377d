"""Run bench.py's C5 rectified-flow batch-sweep line alone (for iteration)."""
import json
import sys
import types

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_06545_b200.model import DiTConfig  # noqa: E402

cfg = DiTConfig(seed=0, **bench.model_dims("target"))
model = bench.fast_model(cfg)
absmax = bench.synthetic_absmax(model)
args = types.SimpleNamespace(wbits=6, timesteps=100)
batches = tuple(int(b) for b in sys.argv[1:]) or (1, 8, 32, 64)
print(json.dumps(bench.c5_rf_line(torch, args, model, absmax, batches=batches)))
