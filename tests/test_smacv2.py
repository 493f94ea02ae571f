"""SMAX smacv2 scenarios: per-episode random unit
types (randint1(fold_in(key, 10+i | 500+i), 0, 6), smax.cpp:169-175) and the
smacv2 spawns (reflected uniform, or centre + ring, smax.cpp:456-479) drawn in
the reset / auto-reset path of the step kernel, vs the compiled reference.

Bars: actions, rewards, dones, finished, episode lengths, carry keys exact;
observations and world_state within 1e-6 (the ring spawn's cos / sin are
CUDA's, not glibc's: positions may differ in the last bit, far below the
float32 observation grid).  Everything else in SMAX (types, health, heuristic,
damage) is exact arithmetic downstream of the same decisions.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O


def _need_ref():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")


def test_smacv2_env_describes_like_the_reference():
    _need_ref()
    import paper_2311_10090_b200 as m
    for units in (5, 10, 20):
        env_id = f"SMAX_smacv2_{units}_units"
        e = m.make_env(env_id, {})
        r = O.RefVenv(env_id, {}, 1)
        assert e.num_agents() == r.n_agents == units and e.obs_dim == r.obs_dim


@pytest.mark.gpu
@pytest.mark.parametrize("units,cfg", [(5, {}), (10, {"max_steps": 40}), (20, {"enemy_controlled": True}),
                                       (5, {"spawn_jitter": 0.0, "map_size": 20.0})])
def test_smacv2_random_stream_matches_reference(units, cfg):
    _need_ref()
    import torch
    import paper_2311_10090_b200 as m
    env_id = f"SMAX_smacv2_{units}_units"
    n, T = 96, 60
    v = m.VectorEnv(env_id, n, config=cfg)
    r = O.RefVenv(env_id, cfg, n)
    key = O.key_from_seed(21)
    v.reset(key)
    r.reset(key)
    ws0 = r.world_state()
    assert np.allclose(v.world_state().cpu().numpy(), ws0, atol=1e-6)
    for k in range(T):
        sk = O.fold_in(O.key_from_seed(22), k)
        v.step_random(sk)
        want = r.step_random(sk)
        got = v.download(("obs", "rewards", "dones", "finished", "final_returns", "final_lengths", "infos",
                          "actions"))
        got["keys"] = v.view("keys").cpu().numpy().view(np.uint32)
        torch.cuda.synchronize()
        for f in ("actions", "rewards", "dones", "finished", "final_lengths", "final_returns", "keys"):
            assert np.array_equal(got[f], want[f]), (k, f)
        assert np.array_equal(got["infos"][:, :, : r.n_info], want["infos"]), k
        assert np.allclose(got["obs"], want["obs"], atol=1e-6), (k, np.abs(got["obs"] - want["obs"]).max())
        assert np.allclose(v.world_state().cpu().numpy(), r.world_state(), atol=1e-6), k


@pytest.mark.gpu
def test_smacv2_types_vary_per_episode():
    """The roster is drawn per episode: world_state's type one-hots differ across envs."""
    import paper_2311_10090_b200 as m
    v = m.VectorEnv("SMAX_smacv2_10_units", 512)
    v.reset(O.key_from_seed(3))
    ws = v.world_state().cpu().numpy()[:, :-1].reshape(512, 20, 18)
    types = ws[:, :, 6:12].argmax(-1)
    assert len({tuple(t) for t in types}) > 400
    assert set(np.unique(types)) == set(range(6))
