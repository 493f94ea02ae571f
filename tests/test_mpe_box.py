"""Continuous-action MPE (box action spaces, mpe.cpp:91-99, 144-166;
SURVEY.md §8(f) rank 2) against the compiled reference.

Box actions: agent a's vector is its first action_space(a).flat_size() floats
(movement 5, speaker dim_c) of a [N][A][5] f32 row, each in [0, 1]
(SpaceDescriptor::contains, spaces.cpp:36-46).  The probe's box draw is
space.sample(fold_in(env_key, j)) (vector_env.cpp:179-181).

Bars: drawn actions, dones, finished, keys and episode lengths exact; obs,
rewards and returns within the MPE 1e-5 relative bar (CUDA vs glibc
exp/log1p in the contact term, as for discrete MPE).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O

SCEN = ["MPE_simple_spread_v3", "MPE_simple_speaker_listener_v4", "MPE_simple_tag_v3"]
CFG = {"continuous_actions": True}


def _need_ref():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")


def test_box_env_describes_like_the_reference():
    """Host-only: the config is accepted and the spec matches (no device needed)."""
    _need_ref()
    import paper_2311_10090_b200 as m
    for env_id in SCEN:
        e = m.make_env(env_id, CFG)
        r = O.RefVenv(env_id, CFG, 1)
        assert e.num_agents() == r.n_agents and e.obs_dim == r.obs_dim


def _cmp(got, ref, k, what):
    for f in ("dones", "finished", "final_lengths", "keys", "episode_lengths"):
        assert np.array_equal(got[f], ref[f]), (what, k, f)
    for f in ("obs", "rewards", "final_returns", "episode_returns"):
        assert np.allclose(got[f], ref[f], rtol=1e-5, atol=1e-6), (what, k, f, np.abs(got[f] - ref[f]).max())


def _gpu(v):
    import torch
    out = v.download(("obs", "rewards", "dones", "finished", "final_returns", "final_lengths"))
    out["keys"] = v.view("keys").cpu().numpy().view(np.uint32).copy()
    out["episode_returns"] = v.view("episode_returns").cpu().numpy().copy()
    out["episode_lengths"] = v.view("episode_lengths").cpu().numpy().copy()
    torch.cuda.synchronize()
    return out


def _ref(o, r):
    o = dict(o)
    o["keys"] = r.keys.copy()
    return o


@pytest.mark.gpu
@pytest.mark.parametrize("env_id", SCEN)
def test_box_random_stream_matches_reference(env_id):
    _need_ref()
    import paper_2311_10090_b200 as m
    n, T = 257, 60
    v = m.VectorEnv(env_id, n, config=CFG)
    r = O.RefVenv(env_id, CFG, n)
    key = O.key_from_seed(4)
    v.reset(key)
    r.reset(key)
    assert v.action_dim == 5
    for k in range(T):
        sk = O.fold_in(O.key_from_seed(5), k)
        v.step_random(sk)
        a = r.random_actions_box(sk)
        assert np.array_equal(v.view("actions_f").cpu().numpy(), a), k
        _cmp(_gpu(v), _ref(r.step(a), r), k, "random")


@pytest.mark.gpu
@pytest.mark.parametrize("env_id", SCEN)
@pytest.mark.parametrize("path", ["device", "host"])
def test_box_explicit_actions_match_reference(env_id, path):
    """Caller actions incl. the bounds 0 and 1 and garbage in the padding of
    short (speaker) rows, through the device and the host C-ABI entry points."""
    _need_ref()
    import torch
    import paper_2311_10090_b200 as m
    n, T = 100, 30
    v = m.VectorEnv(env_id, n, config=CFG)
    r = O.RefVenv(env_id, CFG, n)
    v.reset(O.key_from_seed(8))
    r.reset(O.key_from_seed(8))
    rng = np.random.default_rng(1)
    for k in range(T):
        a = rng.random((n, r.n_agents, 5), dtype=np.float32)
        a[rng.random(a.shape) < 0.05] = 0.0
        a[rng.random(a.shape) < 0.05] = 1.0
        ref_a = a.copy()
        if env_id == "MPE_simple_speaker_listener_v4":
            a[:, 0, 3:] = 7.0  # padding of the speaker's 3-float row: ignored
            ref_a[:, 0, 3:] = 0.0
        if path == "device":
            v.step(None, torch.as_tensor(a, device="cuda"))
        else:
            v.step(None, a)
        _cmp(_gpu(v), _ref(r.step(ref_a), r), k, path)


@pytest.mark.gpu
@pytest.mark.parametrize("bad", [np.nan, 1.5, -0.25, np.inf])
def test_box_invalid_actions_raise_and_leave_state(bad):
    import torch
    import paper_2311_10090_b200 as m
    v = m.VectorEnv("MPE_simple_spread_v3", 16, config=CFG)
    v.reset(O.key_from_seed(2))
    h0 = v.state_hash().cpu().numpy().copy()
    a = np.full((16, 3, 5), 0.5, np.float32)
    a[5, 1, 2] = bad
    with pytest.raises(m.ContractError, match="agent_1"):
        v.step(None, a)
    with pytest.raises(m.ContractError, match="agent_1"):
        v.step(None, torch.as_tensor(a, device="cuda"))
    assert np.array_equal(v.state_hash().cpu().numpy(), h0)
    with pytest.raises(m.ContractError):
        v.step(None, np.zeros((16, 3), np.int32))  # wrong shape for a box space
    v.step(None, np.full((16, 3, 5), 0.5, np.float32))  # the handle recovers


@pytest.mark.gpu
def test_box_env_refuses_categorical_rollout():
    import paper_2311_10090_b200 as m
    from paper_2311_10090_b200.rollout import IppoRollout
    v = m.VectorEnv("MPE_simple_spread_v3", 8, config=CFG)
    with pytest.raises(m.SchemaError):
        IppoRollout(v, 4)
