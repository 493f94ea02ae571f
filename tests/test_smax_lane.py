"""The one-thread-per-env SMAX step (smax_lane.cu: 3m, 5m_vs_6m, 2s3z,
smacv2_5_units) against the lane-group kernel (smax.cu, forced with
MARL_SMAX_GROUP=1; the lane kernel forced with MARL_SMAX_LANE=1, since by
default it only takes batches of >= 24 576 envs) and against the oracle at the
bench shape.

Both kernels are separately parity-tested against the oracle at small sizes
(test_gpu_parity.py runs whichever kernel the roster selects); here they must
produce the same bytes for every output of every step, on the probe's random
stream and on caller actions, with the heuristic or controlled enemies, and
over enough steps that episodes end by wipe-out, by timeout and by draw."""
import numpy as np
import pytest

import oracle as O
from _util import STEP_FIELDS, THREE_M, gpu_outputs, probe_keys

pytestmark = pytest.mark.gpu

ROSTERS = [
    ("SMAX_5m_vs_6m", THREE_M),
    ("SMAX_5m_vs_6m", dict(THREE_M, enemy_controlled=True, max_steps=40)),
    ("SMAX_5m_vs_6m", {}),
    ("SMAX_2s3z", {}),
    ("SMAX_smacv2_5_units", {}),
]


def _run(env_id, cfg, n, T, group, monkeypatch, explicit=False):
    import paper_2311_10090_b200 as m
    if group:
        monkeypatch.setenv("MARL_SMAX_GROUP", "1")
        monkeypatch.delenv("MARL_SMAX_LANE", raising=False)
    else:  # the lane kernel at any size (by default it takes batches of >= 24 576 envs)
        monkeypatch.delenv("MARL_SMAX_GROUP", raising=False)
        monkeypatch.setenv("MARL_SMAX_LANE", "1")
    v = m.VectorEnv(m.make_env(env_id, cfg), n, device=0)
    n_info = 3
    key, ak = probe_keys(71, T)
    v.reset(key)
    rng = np.random.default_rng(5)
    outs = []
    for t in range(T):
        if explicit:
            legal = v.legal_actions().cpu().numpy()  # [N][A][n_act]
            u = rng.random(legal.shape[:2] + (1,))
            c = np.cumsum(legal, -1)
            k = (u * c[..., -1:]).astype(np.int64)
            a = (c <= k).sum(-1).astype(np.int32)
            v.step(None, a)
        else:
            v.step_random(ak[t])
        outs.append(gpu_outputs(v, n_info))
    return outs


@pytest.mark.parametrize("env_id,cfg", ROSTERS)
@pytest.mark.parametrize("explicit", [False, True])
def test_smax_lane_equals_group(env_id, cfg, explicit, monkeypatch):
    n, T = 1000 + 37, 110
    a = _run(env_id, cfg, n, T, False, monkeypatch, explicit)
    b = _run(env_id, cfg, n, T, True, monkeypatch, explicit)
    ends = 0
    for t, (x, y) in enumerate(zip(a, b)):
        for f in STEP_FIELDS:
            assert np.array_equal(x[f], y[f]), (env_id, t, f)
        fin = y["finished"].astype(bool)
        ends += int(fin.sum())
        assert np.array_equal(x["final_obs"][fin], y["final_obs"][fin]), (env_id, t)
    assert ends > 0


def test_smax3m_bench_shape_matches_oracle_on_shards():
    """configs[1] at its bench size (65 536 envs): the GPU steps the whole
    batch, the oracle replays sampled 64-env shards at their global offsets
    (keys derive from global indices), 60 steps, every field bit-exact."""
    import paper_2311_10090_b200 as m
    n, T = 65536, 60
    v = m.VectorEnv(m.make_env("SMAX_5m_vs_6m", THREE_M), n, device=0)
    key, ak = probe_keys(0, T)
    v.reset(key)
    shards = [0, 13 * 64, 511 * 64, n - 64]
    ports = []
    for off in shards:
        p = O.PortVenv("SMAX_5m_vs_6m", THREE_M, 64, global_offset=off, global_n=n)
        p.reset(key)
        ports.append(p)
    for t in range(T):
        v.step_random(ak[t])
        a = gpu_outputs(v, 3)
        for off, p in zip(shards, ports):
            b = p.step_random(ak[t])
            for f in STEP_FIELDS:
                if f == "state_hash":
                    continue
                x = a[f][off:off + 64]
                assert np.array_equal(x, b[f]), (t, off, f)
