"""GPU parity: the CUDA engine vs the CPU oracle and the reference goldens.

Bars (BASELINE.json north_star):
* SMAX and Overcooked: bit-exact on every field of every step (obs, rewards,
  dones, infos, finished, final_*, carry keys, episode bookkeeping and the
  reference's own state_hash).
* MPE: keys, dones, finished, episode lengths, actions bit-exact; obs /
  rewards / returns within 1e-5 relative + 1e-6 absolute per step (the
  reference's own oracle bar is 1e-4 absolute, test_mpe.cpp:281).  The only
  non-identical arithmetic is CUDA's exp/log1p vs glibc's in the soft-contact
  term (mpe.cpp:39-41).
"""
import numpy as np
import pytest

import oracle as O
from _util import STEP_FIELDS, THREE_M, digest, golden_manifest, gpu_outputs, probe_keys

pytestmark = pytest.mark.gpu

MPE_RTOL, MPE_ATOL = 1e-5, 1e-6
EXACT_MPE = ["actions", "dones", "finished", "final_lengths", "keys", "episode_lengths"]


def _venv(env_id, cfg, n, **kw):
    import paper_2311_10090_b200 as m
    return m.VectorEnv(m.make_env(env_id, cfg), n, **kw)


def _compare(env_id, a, b, t, skip=()):
    fam = env_id.split("_")[0]
    if fam != "MPE":
        for f in STEP_FIELDS:
            if f in skip:
                continue
            assert np.array_equal(a[f], b[f]), f"{env_id} step {t}: {f} differs"
        fin = b["finished"].astype(bool)
        assert np.array_equal(a["final_obs"][fin], b["final_obs"][fin]), f"{env_id} step {t}: final_obs"
        return 0.0
    for f in EXACT_MPE:
        if f in skip:
            continue
        assert np.array_equal(a[f], b[f]), f"{env_id} step {t}: {f} differs"
    worst = 0.0
    for f in ("obs", "rewards", "final_returns", "episode_returns"):
        x, y = a[f].astype(np.float64), b[f].astype(np.float64)
        err = np.abs(x - y)
        assert np.all(err <= MPE_ATOL + MPE_RTOL * np.abs(y)), f"{env_id} step {t}: {f} max err {err.max()}"
        worst = max(worst, float(err.max(initial=0.0)))
    return worst


CASES = [
    ("MPE_simple_spread_v3", {}, 300, 80),
    ("MPE_simple_speaker_listener_v4", {}, 100, 60),
    ("MPE_simple_tag_v3", {}, 100, 60),
    ("MPE_simple_tag_v3", {"cooperative_prey_reward": True}, 64, 40),
    ("SMAX_5m_vs_6m", THREE_M, 1000, 120),
    ("SMAX_2s3z", {}, 300, 120),
    ("SMAX_5m_vs_6m", {}, 100, 60),
    ("SMAX_3s_vs_5z", {"enemy_controlled": True, "max_steps": 30}, 100, 60),
    ("SMAX_3s5z_vs_3s6z", {"max_steps": 40}, 50, 50),
    ("SMAX_27m_vs_30m", {"max_steps": 15}, 8, 25),
    ("SMAX_10m_vs_11m", {"unit_stats": {"marine": {"range": 3.0}}, "max_steps": 30}, 30, 40),
    ("overcooked_cramped_room_v0", {"max_steps": 60}, 512, 150),
    ("overcooked_asymmetric_advantages_v0", {"max_steps": 50}, 64, 60),
    ("overcooked_coordination_ring_v0", {"max_steps": 50}, 64, 60),
    ("overcooked_forced_coordination_v0", {"max_steps": 50}, 64, 60),
    ("overcooked_counter_circuit_v0", {"max_steps": 50, "cook_time": 4}, 64, 110),
    ("overcooked_cramped_room_v0", {"max_steps": 30, "random_conflict_resolution": True}, 128, 70),
]


@pytest.mark.parametrize("env_id,cfg,n,T", CASES)
def test_step_random_matches_oracle(env_id, cfg, n, T):
    v = _venv(env_id, cfg, n)
    o = O.PortVenv(env_id, cfg, n)
    key, ak = probe_keys(11, T)
    obs, _ = v.reset(key)
    ref0 = o.reset(key)
    if env_id.startswith("MPE"):
        assert np.allclose(obs.cpu().numpy(), ref0, rtol=MPE_RTOL, atol=MPE_ATOL)
    else:
        assert np.array_equal(obs.cpu().numpy(), ref0)
    finished = 0
    for t in range(T):
        v.step_random(ak[t])
        a = gpu_outputs(v, o.n_info)
        b = o.step_random(ak[t])
        _compare(env_id, a, b, t)
        finished += int(b["finished"].sum())
    assert finished > 0, "the sweep should cross episode boundaries"


@pytest.mark.parametrize("name", sorted(golden_manifest()))
def test_matches_reference_goldens(name):
    """Against trajectories dumped from the unmodified reference (no oracle in between)."""
    rec = golden_manifest()[name]
    v = _venv(rec["env_id"], rec["config"], rec["n_envs"])
    key, ak = probe_keys(rec["seed"], rec["steps"])
    obs, _ = v.reset(key)
    n_info = O.N_INFO[{"MPE": O.MPE, "SMAX": O.SMAX}.get(rec["env_id"].split("_")[0], O.OVERCOOKED)]
    if rec["env_id"].startswith("MPE"):
        import os
        from _util import GOLDEN
        g = np.load(os.path.join(GOLDEN, name + ".npz"))
        assert np.allclose(obs.cpu().numpy(), g["reset_obs"], rtol=MPE_RTOL, atol=MPE_ATOL)
        for t in range(rec["steps"]):
            v.step_random(ak[t])
            a = gpu_outputs(v, n_info)
            for f in ("actions", "keys", "finished", "dones", "episode_lengths"):
                assert np.array_equal(a[f], g[f][t]), (name, t, f)
            for f in ("obs", "rewards", "final_returns"):
                assert np.allclose(a[f], g[f][t], rtol=MPE_RTOL, atol=MPE_ATOL), (name, t, f)
        return
    assert digest(obs.cpu().numpy()) == rec["reset_obs"]
    for t, want in enumerate(rec["digests"]):
        v.step_random(ak[t])
        a = gpu_outputs(v, n_info)
        for f in STEP_FIELDS:
            assert digest(a[f]) == want[f], (name, t, f)
        fin = a["finished"].astype(bool)
        assert digest(a["final_obs"][fin]) == want["final_obs"], (name, t, "final_obs")


@pytest.mark.parametrize("env_id,cfg,n,T", [
    ("SMAX_5m_vs_6m", THREE_M, 256, 60),
    ("SMAX_2s3z", {"enemy_controlled": True}, 64, 50),
    ("overcooked_cramped_room_v0", {"max_steps": 40}, 256, 90),
    ("MPE_simple_spread_v3", {}, 128, 60),
])
def test_explicit_actions_device_and_host_paths(env_id, cfg, n, T):
    """VectorEnv::step with caller actions: device tensor path and host path
    both equal the oracle given the same (legal) random actions."""
    import torch
    vd, vh = _venv(env_id, cfg, n), _venv(env_id, cfg, n)
    o = O.PortVenv(env_id, cfg, n)
    key, ak = probe_keys(3, T)
    _, sd = vd.reset(key)
    _, sh = vh.reset(key)
    o.reset(key)
    for t in range(T):
        acts = o.random_actions(ak[t])
        rd = vd.step(sd, torch.from_numpy(acts).cuda())
        sd = rd.next
        rh = vh.step(sh, acts)
        sh = rh.next
        b = o.step(acts)
        # views.actions holds the actions of step_random / the host path's copy
        _compare(env_id, gpu_outputs(vd, o.n_info), b, t, skip=("actions",))
        gh = gpu_outputs(vh, o.n_info)
        assert np.array_equal(gh["actions"], acts)
        _compare(env_id, gh, b, t, skip=("actions",))


@pytest.mark.parametrize("env_id,cfg", [("SMAX_5m_vs_6m", THREE_M), ("SMAX_2s3z", {"enemy_controlled": True}),
                                        ("SMAX_27m_vs_30m", {})])
def test_legal_masks_match_oracle(env_id, cfg):
    n, T = 64 if "27m" not in env_id else 4, 30
    v = _venv(env_id, cfg, n)
    o = O.PortVenv(env_id, cfg, n)
    key, ak = probe_keys(8, T)
    v.reset(key)
    o.reset(key)
    for t in range(T):
        assert np.array_equal(v.legal_actions().cpu().numpy(), o.legal()), t
        v.step_random(ak[t])
        o.step_random(ak[t])


@pytest.mark.gpu
@pytest.mark.parametrize("env_id,cfg,n,T", [
    ("SMAX_5m_vs_6m", THREE_M, 64, 40), ("SMAX_2s3z", {}, 32, 40), ("MPE_simple_spread_v3", {}, 64, 30),
    ("MPE_simple_speaker_listener_v4", {}, 32, 30), ("overcooked_cramped_room_v0", {"max_steps": 25}, 32, 30)])
def test_world_state_matches_reference(env_id, cfg, n, T):
    """Env::world_state (MAPPO critic input) of the live batch vs the reference
    after the same random-legal steps: exact for SMAX/Overcooked, MPE within
    the env's bar."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    v = _venv(env_id, cfg, n, device=0)
    r = O.RefVenv(env_id, cfg, n)
    key, ak = probe_keys(21, T)
    v.reset(key)
    r.reset(key)
    for t in range(T):
        v.step_random(ak[t])
        r.step_random(ak[t])
        if t % 7 == 6 or t == T - 1:
            a, b = v.world_state().cpu().numpy(), r.world_state()
            assert a.shape == b.shape, (a.shape, b.shape)
            if env_id.startswith("MPE"):
                assert np.allclose(a, b, rtol=MPE_RTOL, atol=MPE_ATOL), (t, np.abs(a - b).max())
            else:
                assert np.array_equal(a, b), (env_id, t)


RAGGED = [(env_id, cfg, n) for env_id, cfg in
          [("MPE_simple_spread_v3", {}), ("SMAX_5m_vs_6m", THREE_M), ("SMAX_2s3z", {}),
           ("overcooked_cramped_room_v0", {"max_steps": 12})]
          for n in (1, 7, 41, 257)]


@pytest.mark.gpu
@pytest.mark.parametrize("env_id,cfg,n", RAGGED)
def test_ragged_batch_sizes_match_oracle(env_id, cfg, n):
    """Batch sizes that leave partial warps / blocks / bulk-store tiles (one
    env, odd counts, one past a block): every field still equals the oracle."""
    v = _venv(env_id, cfg, n, device=0)
    o = O.PortVenv(env_id, cfg, n)
    key, ak = probe_keys(31 + n, 30)
    v.reset(key)
    o.reset(key)
    for t in range(30):
        v.step_random(ak[t])
        a = gpu_outputs(v, o.n_info)
        b = o.step_random(ak[t])
        _compare(env_id, a, b, t)



@pytest.mark.gpu
@pytest.mark.parametrize("env_id,cfg", [("SMAX_5m_vs_6m", THREE_M), ("SMAX_5m_vs_6m", {}),
                                        ("SMAX_5m_vs_6m", {"enemy_controlled": True}), ("SMAX_2s3z", {})])
def test_smax_folded_instances_equal_generic(env_id, cfg, monkeypatch):
    """All-marine rosters run a step kernel with the unit type folded to a
    compile-time constant, and rosters that fill their lane group (3m: 6 of 6,
    2s3z: 10 of 10) one with the unit count folded; MARL_SMAX_GENERIC=1 forces
    the general kernel. Both must produce the same bytes (obs, rewards, dones,
    state) every step."""
    import paper_2311_10090_b200 as m
    n, T = 300, 40
    runs = []
    for generic in (False, True):
        if generic:
            monkeypatch.setenv("MARL_SMAX_GENERIC", "1")
        v = m.VectorEnv(env_id, n, config=cfg)
        v.reset(O.key_from_seed(17))
        out = []
        for k in range(T):
            v.step_random(O.fold_in(O.key_from_seed(18), k))
            d = v.download(("obs", "rewards", "dones", "finished"))
            d["hash"] = v.state_hash().cpu().numpy().copy()
            out.append(d)
        runs.append(out)
    for k, (a, b) in enumerate(zip(*runs)):
        for f in a:
            assert np.array_equal(a[f], b[f]), (k, f)
