"""The fused throughput_probe loop (marl_venv_probe_steps, vector_env.cpp:202-217).

MPE runs K probe steps in ONE launch with each env's state, carry key and
episode bookkeeping in registers across the steps (mpe_step_kernel's MULTI
instance, one-warp CTAs).  Every step still writes every output view, so after
the launch the views must hold exactly what K separate step_random launches
leave: every field, bit for bit, plus the state hash and the episode
statistics.  Chunkings that straddle the 25-step episode boundary, ragged
batches and the box-action (continuous) variant are covered, and the fused
path is compared with the oracle at the end of a 1000-step probe (configs[0]'s
protocol)."""
import numpy as np
import pytest

import oracle as O
from _util import STEP_FIELDS, gpu_outputs

pytestmark = pytest.mark.gpu

MPE = [("MPE_simple_spread_v3", {}), ("MPE_simple_tag_v3", {}), ("MPE_simple_speaker_listener_v4", {}),
       ("MPE_simple_spread_v3", {"continuous_actions": True})]


def _venv(env_id, cfg, n):
    import paper_2311_10090_b200 as m
    return m.VectorEnv(m.make_env(env_id, cfg), n, device=0)


@pytest.mark.parametrize("env_id,cfg", MPE)
@pytest.mark.parametrize("chunks", [(1, 1, 1), (7, 30, 3), (60,)])
def test_fused_probe_equals_single_steps(env_id, cfg, chunks):
    n = 1024 + 37
    key = O.key_from_seed(5)
    parent = O.fold_in(key, 2)
    a, b = _venv(env_id, cfg, n), _venv(env_id, cfg, n)
    a.reset(key)
    b.reset(key)
    a.episode_stats(clear=True)
    b.episode_stats(clear=True)
    ks = O.split(parent, sum(chunks) + 1)
    n_info = 0
    t = 0
    for K in chunks:
        a.probe_steps(parent, t, K)
        for k in range(K):
            b.step_random(ks[t + k])
        t += K
        x, y = gpu_outputs(a, n_info), gpu_outputs(b, n_info)
        for f in STEP_FIELDS + ["final_obs"]:
            if f == "final_obs":
                fin = y["finished"].astype(bool)
                assert np.array_equal(x[f][fin], y[f][fin]), (t, f)
            elif f == "actions" and cfg.get("continuous_actions"):
                continue
            else:
                assert np.array_equal(x[f], y[f]), (t, f)
        if cfg.get("continuous_actions"):
            assert np.array_equal(a.view("actions_f").cpu().numpy(), b.view("actions_f").cpu().numpy())
    assert a.episode_stats() == b.episode_stats()


def test_fused_probe_1000_steps_matches_oracle():
    """configs[0] end to end: reset, the probe's warm-up step (key T), then
    T = 1000 steps in one fused launch; the state against the oracle's after
    the same 1001 steps (keys / lengths / dones exact, obs within MPE's bar)."""
    env_id, n, T = "MPE_simple_spread_v3", 1024, 1000
    key = O.key_from_seed(0)
    parent = O.fold_in(key, 2)
    ks = O.split(parent, T + 1)
    v = _venv(env_id, {}, n)
    o = O.PortVenv(env_id, {}, n)
    v.reset(key)
    o.reset(key)
    v.step_random(ks[T])
    o.step_random(ks[T])
    v.probe_steps(parent, 0, T)
    for t in range(T):
        b = o.step_random(ks[t])
    a = gpu_outputs(v, 0)
    for f in ("actions", "dones", "finished", "final_lengths", "episode_lengths"):
        assert np.array_equal(a[f], b[f]), f
    assert np.array_equal(a["keys"], o.batch_state()["keys"])
    for f in ("obs", "rewards", "episode_returns"):
        x, y = a[f].astype(np.float64), b[f].astype(np.float64)
        assert np.all(np.abs(x - y) <= 1e-6 + 1e-5 * np.abs(y)), (f, np.abs(x - y).max())


def test_throughput_probe_uses_fused_path():
    import paper_2311_10090_b200 as m
    from paper_2311_10090_b200 import _native
    L = _native.lib()
    c0 = L.marl_launch_count()
    res = m.throughput_probe("MPE_simple_spread_v3", 1024, 500, O.key_from_seed(1))
    # reset + warm-up step + ONE launch for the 500 timed steps
    assert L.marl_launch_count() - c0 < 10
    assert res.sps > 0


def test_probe_steps_other_families_equal_single_steps():
    """SMAX / Overcooked: probe_steps is the same device launches as the
    step_random loop (one per step)."""
    from _util import THREE_M
    for env_id, cfg in (("SMAX_5m_vs_6m", THREE_M), ("overcooked_cramped_room_v0", {"max_steps": 9})):
        key = O.key_from_seed(8)
        parent = O.fold_in(key, 2)
        a, b = _venv(env_id, cfg, 300), _venv(env_id, cfg, 300)
        a.reset(key)
        b.reset(key)
        ks = O.split(parent, 21)
        a.probe_steps(parent, 0, 20)
        for k in range(20):
            b.step_random(ks[k])
        x, y = gpu_outputs(a, 3), gpu_outputs(b, 3)
        for f in STEP_FIELDS:
            assert np.array_equal(x[f], y[f]), (env_id, f)
