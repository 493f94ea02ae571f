"""IPPO rollout collection (config 5).

Oracle: the reference's own Collector pieces (VectorEnv, TeamLayout,
ppo_init_nets, ff_forward, sample_masked, compute_gae) compiled from
/root/reference, with the private collect loop restated line for line
(oracle/ref_rollout.cpp, ppo.cpp:189-323).

Parity bars (fp32 policy path vs the reference):
* actions, resets, dones, legal masks, active flags: exact;
* SMAX: observation rows and rewards exact;
* MPE: observation rows / rewards within the env's 1e-5 bar (CUDA vs glibc
  exp/log1p in the contact term);
* logp / value / adv / vtarg: within 2e-5 relative + 2e-6 absolute (CUDA
  tanhf vs glibc tanhf differ by an ulp; every dot product is accumulated in
  the reference's order, nn.hpp:42-54).
bf16 tensor-core path vs fp32 path on identical inputs: logits-derived
log-probs / values within bf16 tolerance, action agreement >= 97%.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from _util import THREE_M

ENVS = [("MPE_simple_spread_v3", {}, 48, 24, 2, 0.0),
        ("SMAX_5m_vs_6m", THREE_M, 24, 20, 2, 0.0),
        ("overcooked_cramped_room_v0", {"max_steps": 30}, 8, 20, 2, 0.5)]


def _need_ref():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")


def test_reference_collector_invariants():
    _need_ref()
    key = O.key_from_seed(3)
    a, c = O.ref_ppo_init("MPE_simple_spread_v3", {}, key)
    out = O.ref_collect("MPE_simple_spread_v3", {}, 12, 30, key, a, c, n_windows=1)
    assert np.array_equal(out["vtarg"], out["adv"] + out["value"])   # compute_gae: vtarg = adv + v
    assert out["resets"][0].all()                                      # every row starts an episode
    assert (out["legal"] == 1).all() and (out["active"] == 1).all()    # MPE: all legal, all active
    assert np.array_equal(out["dones"][24], np.ones(36, np.uint8))     # 25-step episodes
    assert np.array_equal(out["resets"][25], out["dones"][24])
    oh = out["obs"][:, :, 18:]
    assert np.array_equal(oh, np.tile(np.eye(3, dtype=np.float32), (30, 12, 1)))  # TeamLayout one-hot


def test_policy_spec_matches_reference():
    _need_ref()
    import paper_2311_10090_b200 as m
    for env_id, cfg, *_ in ENVS:
        env = m.make_env(env_id, cfg)
        ref = O.ref_ppo_spec(env_id, cfg)
        A = env.num_agents()
        in_dim = env.obs_dim + (A if A > 1 else 0)
        n_act = env.n_actions_max
        W = 64
        assert (in_dim, n_act) == (ref["in_dim"], ref["n_actions"])
        assert W * in_dim + W + W * W + W + n_act * W + n_act == ref["n_actor"]
        assert W * in_dim + W + W * W + W + W + 1 == ref["n_critic"]


def _gpu_collect(env_id, cfg, n, T, windows, shaping, precision, key, a, c, centralized=False):
    import paper_2311_10090_b200 as m
    from paper_2311_10090_b200.rollout import IppoRollout
    v = m.VectorEnv(m.make_env(env_id, cfg), n, device=0)
    ro = IppoRollout(v, T, precision=precision, centralized=centralized)
    ro.set_params(a, c)
    ro.begin(key)
    for w in range(windows):
        views = ro.collect(seq_base=w * T, shaping=shaping)
    return {k: t.cpu().numpy().copy() for k, t in views.items()}


@pytest.mark.gpu
@pytest.mark.parametrize("env_id,cfg,n,T,windows,shaping", ENVS)
def test_fp32_rollout_matches_reference_collector(env_id, cfg, n, T, windows, shaping):
    _need_ref()
    key = O.key_from_seed(11)
    a, c = O.ref_ppo_init(env_id, cfg, O.fold_in(key, 10))
    ref = O.ref_collect(env_id, cfg, n, T, key, a, c, n_windows=windows, shaping=shaping)
    got = _gpu_collect(env_id, cfg, n, T, windows, shaping, "fp32", key, a, c)
    for f in ("actions", "resets", "dones", "legal", "active"):
        assert np.array_equal(got[f], ref[f]), f
    exact_env = not env_id.startswith("MPE")
    for f in ("obs", "rewards"):
        if exact_env:
            assert np.array_equal(got[f], ref[f]), f
        else:
            assert np.allclose(got[f], ref[f], rtol=1e-5, atol=1e-6), (f, np.abs(got[f] - ref[f]).max())
    for f in ("logp", "value", "adv", "vtarg"):
        err = np.abs(got[f].astype(np.float64) - ref[f])
        assert np.all(err <= 2e-6 + 2e-5 * np.abs(ref[f])), (f, err.max())


# input widths 18 / 95 / 163 / 180: the kernel's staging modes (two staged tiles + staged
# buffer rows, two tiles, one tile or none) and layer-1 K of 32 .. 192
@pytest.mark.gpu
@pytest.mark.parametrize("env_id,cfg,n", [("MPE_simple_spread_v3", {}, 512), ("SMAX_5m_vs_6m", THREE_M, 300),
                                          ("SMAX_2s3z", {}, 131), ("SMAX_5m_vs_6m", {}, 77),
                                          # wide rows (K-chunked layer 1): Overcooked's 520 + 2 columns
                                          ("overcooked_cramped_room_v0", {"max_steps": 20}, 300),
                                          ("overcooked_coordination_ring_v0", {"max_steps": 20}, 97),
                                          # 989 columns, 35 actions (head N = 48)
                                          ("SMAX_27m_vs_30m", {"max_steps": 20}, 40)])
def test_bf16_tensor_core_rollout_agrees_with_fp32(env_id, cfg, n):
    from paper_2311_10090_b200._native import lib
    _need_ref()
    key = O.key_from_seed(5)
    a, c = O.ref_ppo_init(env_id, cfg, O.fold_in(key, 10))
    T = 8
    f32 = _gpu_collect(env_id, cfg, n, T, 1, 0.0, "fp32", key, a, c)
    launches0 = lib().marl_launch_count()
    b16 = _gpu_collect(env_id, cfg, n, T, 1, 0.0, "bf16", key, a, c)
    assert lib().marl_launch_count() > launches0
    # step 0 sees identical inputs: compare the nets directly there
    assert np.array_equal(f32["obs"][0], b16["obs"][0])
    assert np.allclose(b16["value"][0], f32["value"][0], rtol=0.05, atol=0.03)
    assert np.allclose(b16["logp"][0], f32["logp"][0], rtol=0.02, atol=0.02)
    agree = (b16["actions"][0] == f32["actions"][0]).mean()
    assert agree >= 0.97, agree
    # the whole window is a valid rollout: legal actions, GAE identity
    act = b16["actions"]
    assert (act >= 0).all() and (act < b16["legal"].shape[-1]).all()
    assert np.take_along_axis(b16["legal"], act[..., None].astype(np.int64), -1).all()
    assert np.array_equal(b16["vtarg"], b16["adv"] + b16["value"])


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("n", [1, 5, 43])
def test_rollout_ragged_rows(precision, n):
    """Row counts that leave partial 128-row tensor-core tiles and unaligned
    bulk-copy tails: the fp32 path still equals the reference collector, the
    bf16 path stays a valid rollout that agrees on the first step."""
    _need_ref()
    env_id, cfg, T = "MPE_simple_spread_v3", {}, 6
    key = O.key_from_seed(40 + n)
    a, c = O.ref_ppo_init(env_id, cfg, O.fold_in(key, 10))
    ref = O.ref_collect(env_id, cfg, n, T, key, a, c)
    got = _gpu_collect(env_id, cfg, n, T, 1, 0.0, precision, key, a, c)
    assert np.array_equal(got["resets"], ref["resets"]) and np.array_equal(got["legal"], ref["legal"])
    assert np.array_equal(got["obs"][0], ref["obs"][0])
    if precision == "fp32":
        assert np.array_equal(got["actions"], ref["actions"])
        assert np.allclose(got["value"], ref["value"], rtol=2e-5, atol=2e-6)
    else:
        assert np.allclose(got["value"][0], ref["value"][0], rtol=0.05, atol=0.03)
        assert np.array_equal(got["vtarg"], got["adv"] + got["value"])


@pytest.mark.gpu
@pytest.mark.parametrize("env_id,cfg,n,T", [("MPE_simple_spread_v3", {}, 24, 30), ("SMAX_5m_vs_6m", THREE_M, 16, 24),
                                            ("overcooked_cramped_room_v0", {"max_steps": 20}, 4, 24)])
def test_mappo_rollout_matches_reference_collector(env_id, cfg, n, T):
    """train_mappo's collector (centralized=true): the critic reads
    Env::world_state (ppo.cpp:341-346); critic rows, values and GAE vs the
    reference."""
    _need_ref()
    import paper_2311_10090_b200 as m
    from paper_2311_10090_b200.rollout import IppoRollout
    key = O.key_from_seed(17)
    a, c = O.ref_ppo_init(env_id, cfg, O.fold_in(key, 10), centralized=True)
    ref = O.ref_collect(env_id, cfg, n, T, key, a, c, centralized=True)
    v = m.VectorEnv(m.make_env(env_id, cfg), n, device=0)
    ro = IppoRollout(v, T, precision="fp32", centralized=True)
    ro.set_params(a, c)
    ro.begin(key)
    got = {k: t.cpu().numpy() for k, t in ro.collect().items()}
    for f in ("actions", "resets", "dones", "legal", "active"):
        assert np.array_equal(got[f], ref[f]), f
    if env_id.startswith("MPE"):
        assert np.allclose(got["critic_in"], ref["critic_in"], rtol=1e-5, atol=1e-6)
    else:
        assert np.array_equal(got["critic_in"], ref["critic_in"])
    for f in ("value", "adv", "vtarg"):
        err = np.abs(got[f].astype(np.float64) - ref[f])
        assert np.all(err <= 2e-6 + 2e-5 * np.abs(ref[f])), (f, err.max())


# MAPPO on the tensor cores: the critic's layer 1 reads world_state rows of
# widths 54 (MPE spread), 109 (SMAX 3m) and 181 (2s3z) from its own X tile
@pytest.mark.gpu
@pytest.mark.parametrize("env_id,cfg,n", [("MPE_simple_spread_v3", {}, 700), ("SMAX_5m_vs_6m", THREE_M, 300),
                                          ("SMAX_2s3z", {}, 131)])
def test_bf16_mappo_rollout_agrees_with_fp32(env_id, cfg, n):
    """centralized=True with precision bf16: the critic_in rows equal the
    fp32 path's (and the reference's) exactly, values / log-probs within the
    bf16 tolerances, >= 97% identical actions at step 0, a valid rollout."""
    _need_ref()
    key = O.key_from_seed(23)
    a, c = O.ref_ppo_init(env_id, cfg, O.fold_in(key, 10), centralized=True)
    T = 6
    f32 = _gpu_collect(env_id, cfg, n, T, 1, 0.0, "fp32", key, a, c, centralized=True)
    b16 = _gpu_collect(env_id, cfg, n, T, 1, 0.0, "bf16", key, a, c, centralized=True)
    assert np.array_equal(f32["obs"][0], b16["obs"][0])
    assert np.array_equal(f32["critic_in"][0], b16["critic_in"][0])
    assert np.allclose(b16["value"][0], f32["value"][0], rtol=0.05, atol=0.03)
    assert np.allclose(b16["logp"][0], f32["logp"][0], rtol=0.02, atol=0.02)
    assert (b16["actions"][0] == f32["actions"][0]).mean() >= 0.97
    act = b16["actions"]
    assert np.take_along_axis(b16["legal"], act[..., None].astype(np.int64), -1).all()
    assert np.array_equal(b16["vtarg"], b16["adv"] + b16["value"])
    ref = O.ref_collect(env_id, cfg, n, 1, key, a, c, centralized=True)
    if env_id.startswith("MPE"):
        assert np.allclose(b16["critic_in"][0], ref["critic_in"][0], rtol=1e-5, atol=1e-6)
    else:
        assert np.array_equal(b16["critic_in"][0], ref["critic_in"][0])


@pytest.mark.gpu
def test_bf16_mappo_training_runs():
    """train_mappo with the bf16 tcgen05 collector (the update stays on the
    fp32 kernels for centralized critics): finite losses, counts as fp32."""
    _need_ref()
    import paper_2311_10090_b200 as m
    from paper_2311_10090_b200.ppo import train_mappo
    cfg = {"total_timesteps": 256 * 8 * 2, "n_envs": 256, "n_rollout_steps": 8}
    key = O.key_from_seed(3)
    r16 = train_mappo(m.make_env("MPE_simple_spread_v3", {}), cfg, key, precision="bf16").metrics.as_array()
    r32 = train_mappo(m.make_env("MPE_simple_spread_v3", {}), cfg, key, precision="fp32").metrics.as_array()
    assert np.isfinite(r16).all()
    assert np.array_equal(r16[:, [0, 1, 3]], r32[:, [0, 1, 3]])
