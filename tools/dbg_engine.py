import json, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from oracle import qc_oracle as O
from paper_2503_06545_b200.model import DiTConfig, init_model
from paper_2503_06545_b200.schedule import ThresholdConfig, Toggles
from paper_2503_06545_b200.engine import QuantCacheEngine
f = np.load('tests/golden/runs.npz')
cal = json.load(open('tests/golden/calib_small.json'))
meta = json.load(open('tests/golden/runs_meta.json'))
cfg = DiTConfig(3, 16, 2, 4, 2, 8, 3)
m = init_model(cfg)
ab = O.alpha_bar(10)
absmax = {int(l): {s: np.asarray(v) for s, v in d.items()} for l, d in cal['act_absmax'].items()}
th = ThresholdConfig(delta1=cal['delta_percentiles']['p33'], delta2=cal['delta_percentiles']['p66'],
                     v_low=cal['variation_percentiles']['p25'], v_high=cal['variation_percentiles']['p75'])
for name, tog in [('none', Toggles()), ('hlc', Toggles(hlc=True)),
                  ('hlc_aigq', Toggles(True, True, True, False)), ('full', Toggles(True, True, True, True)),
                  ('aigq', Toggles(False, True, True, False))]:
    wb = {int(k): v for k, v in meta[f'small_{name}']['weight_bits'].items()}
    eng = QuantCacheEngine(m, ab, tog, th, wb, absmax, sign_seed=3, prune_seed=3)
    t0 = time.time()
    out, tr = eng.generate([3])
    want = f[f'small_{name}']
    ref_tr = [json.loads(l) for l in open(f'tests/golden/trace_small_{name}.jsonl')]
    acts_ok = [r['action'] for r in ref_tr] == [r.action for r in tr[0]]
    bits_ok = [r['bits'] for r in ref_tr] == [r.bits for r in tr[0]]
    print(name, 'exact', np.array_equal(out[0], want), 'maxdiff', float(np.abs(out[0]-want).max()),
          'actions', acts_ok, 'bits', bits_ok, 'time', round(time.time()-t0, 3))
    if not acts_ok:
        for a, b in zip(ref_tr, tr[0]):
            if a['action'] != b.action:
                print('  first diff', a, b); break
