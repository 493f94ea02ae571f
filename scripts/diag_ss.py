"""Diagnostic: PPO update gradient blocks (bf16 tcgen05) uncapped vs capped grids vs the reference."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import test_steady_state as T
import oracle as O
from _util import THREE_M
for env_id, cfg in [("SMAX_5m_vs_6m", THREE_M), ("MPE_simple_spread_v3", {})]:
    res = {}
    for cap in (0, 1, 2, 4):
        if cap:
            c = T._Cap(cap); c.__enter__()
        tr = T._trainer(env_id, cfg, 1024, 24, "bf16")
        tr.begin(O.key_from_seed(61)); tr.collect()
        buf = {k: t.cpu().numpy() for k, t in tr.rollout._views.items()}
        a, cc = tr.params(); R = tr.rollout.R
        idx = np.random.default_rng(9).choice(24 * R, size=50000, replace=False).astype(np.int32)
        g, st = tr.minibatch_grad(idx)
        if cap:
            c.__exit__()
        res[cap] = g
    gr, sr = O.ref_ff_minibatch(env_id, cfg, a, cc, buf, idx)
    for lo, hi in T._blocks(tr.spec):
        y = gr[lo:hi]
        print(env_id, lo, hi, "ref %.4g" % np.linalg.norm(y),
              " ".join("cap%d %.4g" % (k, np.linalg.norm(v[lo:hi])) for k, v in res.items()),
              "max|cap1-cap0| %.3g" % np.abs(res[1][lo:hi] - res[0][lo:hi]).max())
