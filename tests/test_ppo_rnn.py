"""Recurrent (GRU) PPO: RnnBranch actor / critic
(actor_critic.hpp:74-200, gru_step / gru_backward nn.hpp:200-318), the
recurrent Collector (hidden states carried, reset at episode boundaries,
ppo.cpp:194-250) and rnn_minibatch (BPTT over whole row sequences,
ppo.cpp:444-509), against the reference's own train_ippo / train_mappo with
recurrent=true.

Bars as for the feed-forward trainer (tests/test_ppo.py): ppo_init_nets
bit-exact; step / update / n_episodes / lr exact; losses and final parameters
within 1e-3 relative (float reassociation in the gradient sums, CUDA vs glibc
expf / tanhf by an ulp).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from _util import THREE_M


def _need_ref():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")


@pytest.mark.parametrize("env_id,cfg", [("MPE_simple_spread_v3", {}), ("SMAX_5m_vs_6m", THREE_M),
                                        ("overcooked_cramped_room_v0", {})])
def test_init_rnn_bit_exact(env_id, cfg):
    _need_ref()
    from paper_2311_10090_b200.ppo import init_rnn
    sp = O.ref_ppo_spec(env_id, cfg)
    for seed, F, H in ((0, 64, 128), (3, 32, 48)):
        key = O.key_from_seed(seed)
        ra, rc = O.ref_ppo_init_rnn(env_id, cfg, key, F, H)
        a, c = init_rnn(sp["in_dim"], sp["critic_in"], sp["n_actions"], key, F, H)
        assert a.tobytes() == ra.tobytes() and c.tobytes() == rc.tobytes()


def _close(x, y, rel=1e-3, absf=1e-4):
    return np.all(np.abs(x - y) <= rel * np.abs(y) + absf * max(np.abs(y).max(), 1e-30))


def _compare(env_id, cfg, ppo_cfg, key, centralized=False):
    from paper_2311_10090_b200 import make_env
    from paper_2311_10090_b200.ppo import train_ippo, train_mappo
    ref = O.ref_train(env_id, cfg, ppo_cfg, key, centralized)
    got = (train_mappo if centralized else train_ippo)(make_env(env_id, cfg), ppo_cfg, key)
    m, rm = got.metrics.as_array(), ref["metrics"]
    assert m.shape == rm.shape and got.diverged == ref["diverged"] and got.steps_done == ref["steps_done"]
    for col in (0, 1, 3, 11):
        assert np.array_equal(m[:, col], rm[:, col]), O.PPO_COLUMNS[col]
    assert np.allclose(m[:, 2], rm[:, 2], rtol=1e-5, atol=1e-5)
    for col in range(4, 11):
        assert np.allclose(m[:, col], rm[:, col], rtol=1e-3, atol=1e-5), (O.PPO_COLUMNS[col], m[:, col], rm[:, col])
    assert _close(got.actor, ref["actor"]) and _close(got.critic, ref["critic"])


@pytest.mark.gpu
@pytest.mark.parametrize("env_id,cfg,n_envs,T", [("MPE_simple_spread_v3", {}, 8, 16),
                                                 ("SMAX_5m_vs_6m", THREE_M, 8, 24)])
def test_recurrent_train_ippo_matches_reference(env_id, cfg, n_envs, T):
    _need_ref()
    ppo_cfg = {"total_timesteps": 2 * n_envs * T, "n_envs": n_envs, "n_rollout_steps": T, "recurrent": True,
               "hidden_width": 32, "fc_width": 32, "update_epochs": 2}
    _compare(env_id, cfg, ppo_cfg, O.key_from_seed(7))


@pytest.mark.gpu
def test_recurrent_train_mappo_relu_matches_reference():
    _need_ref()
    ppo_cfg = {"total_timesteps": 2 * 8 * 16, "n_envs": 8, "n_rollout_steps": 16, "recurrent": True,
               "hidden_width": 24, "fc_width": 16, "activation": "relu", "n_minibatches": 4, "update_epochs": 2}
    _compare("MPE_simple_spread_v3", {}, ppo_cfg, O.key_from_seed(9), centralized=True)


@pytest.mark.gpu
def test_recurrent_default_widths_run():
    """PpoConfig defaults (fc 64, GRU 128): a sane run at a modest size."""
    from paper_2311_10090_b200 import make_env
    from paper_2311_10090_b200.ppo import train_ippo
    r = train_ippo(make_env("MPE_simple_spread_v3", {}),
                   {"total_timesteps": 3 * 32 * 32, "n_envs": 32, "n_rollout_steps": 32, "recurrent": True},
                   O.key_from_seed(1))
    m = r.metrics.as_array()
    assert m.shape == (3, 12) and np.isfinite(m).all() and not r.diverged


@pytest.mark.gpu
def test_recurrent_schema_errors():
    import paper_2311_10090_b200 as m
    from paper_2311_10090_b200.errors import SchemaError
    from paper_2311_10090_b200.ppo import PpoTrainer
    v = m.VectorEnv(m.make_env("MPE_simple_spread_v3", {}), 5, device=0)
    with pytest.raises(SchemaError, match="divisible"):  # R = 15 rows, 2 minibatches (ppo.cpp:548-552)
        PpoTrainer(v, {"n_envs": 5, "recurrent": True})
    with pytest.raises(SchemaError, match="fp32"):
        PpoTrainer(v, {"n_envs": 5, "recurrent": True, "n_minibatches": 3}, precision="bf16")


@pytest.mark.gpu
def test_recurrent_chunked_bptt_matches_reference(monkeypatch):
    """Minibatches processed in row chunks whose BPTT caches fit a budget
    (here a zero budget: one row per chunk) give the same training as the reference."""
    _need_ref()
    monkeypatch.setenv("MARL_RNN_CACHE_MB", "0")
    ppo_cfg = {"total_timesteps": 2 * 8 * 16, "n_envs": 8, "n_rollout_steps": 16, "recurrent": True,
               "hidden_width": 32, "fc_width": 32, "update_epochs": 2}
    _compare("MPE_simple_spread_v3", {}, ppo_cfg, O.key_from_seed(7))


@pytest.mark.gpu
@pytest.mark.parametrize("env_id,cfg", [("MPE_simple_spread_v3", {}), ("SMAX_5m_vs_6m", THREE_M)])
def test_recurrent_gemm_collector_matches_reference(monkeypatch, env_id, cfg):
    """The GEMM-structured acting step (used for large row counts) forced on a
    small batch: the same training as the reference."""
    _need_ref()
    monkeypatch.setenv("MARL_RNN_COLLECT", "gemm")
    ppo_cfg = {"total_timesteps": 2 * 8 * 16, "n_envs": 8, "n_rollout_steps": 16, "recurrent": True,
               "hidden_width": 32, "fc_width": 32, "update_epochs": 2}
    _compare(env_id, cfg, ppo_cfg, O.key_from_seed(7))
