"""Overcooked's reward-bearing transitions: soup delivery (reward 20), soup
pickup (shaping 5), plate and onion shaping (3).

Two action streams from the reference's own tests:
* the scripted soup of test_overcooked.cpp:227-317 (fill the pot with three
  onions, fetch a plate while it cooks, collect the soup, deliver it) played by
  agent 0 of every cramped_room env, started after a per-env delay so the
  batch is spread over every phase of the script, with agent 1 either idle (the
  reference's script) or on the interact-heavy random mix;
* the interact-heavy random rollouts of test_overcooked.cpp:466-527 (action
  weights {2,2,2,2,1,6}) on all five layouts: the reference's protocol
  (40 episodes x 120 steps, max_steps 120) and a wider one at the default
  400-step horizon, where deliveries happen.

CPU tests pin the oracle to the compiled reference on these streams; the GPU
tests compare every field of every step of the CUDA engine (device-action and
host-buffer paths; oc_step_kernel's grid capped so its grid-stride loop runs
several iterations) with the oracle, and require deliveries and soup pickups
to actually occur in the compared steps.
"""
import numpy as np
import pytest

import oracle as O
from _util import STEP_FIELDS, gpu_outputs

kUp, kDown, kLeft, kRight, kStay, kInteract = range(6)  # overcooked.cpp:16
LAYOUTS = ["cramped_room", "asymmetric_advantages", "coordination_ring", "forced_coordination", "counter_circuit"]
INTERACT_HEAVY = np.array([2, 2, 2, 2, 1, 6], np.float64) / 15.0  # test_overcooked.cpp:475
I_DELIV, I_SHAPED = 0, 1  # infos in std::map key order: deliveries, shaped_reward

# test_overcooked.cpp:245-311, agent 0's actions; 20 waits cover the rest of
# the cook (the reference loops until pot_ready, 16 steps)
SCRIPT = ([kUp, kLeft, kInteract, kRight, kUp, kInteract]
          + [kLeft, kLeft, kInteract, kRight, kUp, kInteract] * 2
          + [kDown, kLeft, kDown, kInteract] + [kStay] * 20
          + [kUp, kRight, kUp, kInteract]
          + [kDown, kRight, kDown, kInteract])
PICKUP_AT = len(SCRIPT) - 5   # the kInteract that lifts the soup (shaping 5)
DELIVER_AT = len(SCRIPT) - 1  # the kInteract at the serving window (reward 20)


def scripted_actions(n, T, seed=3):
    """[T, n, 2]: env i plays SCRIPT after i % 7 idle steps; odd envs give agent 1
    the interact-heavy random mix, even envs keep it idle as the reference does."""
    rng = np.random.default_rng(seed)
    a = np.full((T, n, 2), kStay, np.int32)
    for i in range(n):
        d = i % 7
        a[d:d + len(SCRIPT), i, 0] = SCRIPT[: max(0, min(len(SCRIPT), T - d))]
        if i % 2:
            a[:, i, 1] = rng.choice(6, size=T, p=INTERACT_HEAVY)
    return a


def interact_heavy(n, T, seed):
    rng = np.random.default_rng(seed)
    return rng.choice(6, size=(T, n, 2), p=INTERACT_HEAVY).astype(np.int32)


def _exact(a, b, tag):
    for f in STEP_FIELDS:
        if f == "actions" or f not in a or f not in b:
            continue
        assert np.array_equal(a[f], b[f]), f"{tag}: {f} differs"
    fin = b["finished"].astype(bool)
    assert np.array_equal(a["final_obs"][fin], b["final_obs"][fin]), f"{tag}: final_obs"


# ------------------------------------------------------------ oracle pinning
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="compiled reference (oracle/_ref) not built")


@needs_ref
def test_oracle_scripted_soup_matches_reference():
    env_id, n = "overcooked_cramped_room_v0", 14
    T = len(SCRIPT) + 8
    acts = scripted_actions(n, T)
    o, r = O.PortVenv(env_id, {}, n), O.RefVenv(env_id, {}, n)
    key = O.key_from_seed(5)
    assert np.array_equal(o.reset(key), r.reset(key))
    deliveries = pickups = 0
    for t in range(T):
        a, b = o.step(acts[t]), r.step(acts[t])
        _exact(a, b, f"step {t}")
        for i in range(n):
            if i % 2 == 0 and t == i % 7 + DELIVER_AT:  # the reference's own script: agent 1 idle
                assert b["rewards"][i, 0] == 20.0 and b["rewards"][i, 1] == 20.0
                assert b["infos"][i, 0, I_DELIV] == 1.0 and b["infos"][i, 0, I_SHAPED] == 0.0
            if i % 2 == 0 and t == i % 7 + PICKUP_AT:
                assert b["infos"][i, 0, I_SHAPED] == 5.0
        deliveries += int((b["rewards"][:, 0] > 0).sum())
        pickups += int((b["infos"][:, :, I_SHAPED] == 5.0).sum())
    assert deliveries >= n // 2 and pickups >= n // 2


@needs_ref
@pytest.mark.parametrize("layout", LAYOUTS)
def test_oracle_interact_heavy_matches_reference(layout):
    """test_overcooked.cpp:466-527's protocol (40 episodes x 120 steps) plus one
    crossing of the default 400-step horizon."""
    env_id = f"overcooked_{layout}_v0"
    for n, T, cfg in [(40, 121, {"max_steps": 120}), (64, 401, {})]:
        acts = interact_heavy(n, T, seed=LAYOUTS.index(layout))
        o, r = O.PortVenv(env_id, cfg, n), O.RefVenv(env_id, cfg, n)
        key = O.fold_in(O.key_from_seed(42), 1)
        assert np.array_equal(o.reset(key), r.reset(key))
        for t in range(T):
            _exact(o.step(acts[t]), r.step(acts[t]), f"{layout} n={n} step {t}")


# ------------------------------------------------------------------- GPU
def _venv(env_id, cfg, n):
    import paper_2311_10090_b200 as m
    return m.VectorEnv(m.make_env(env_id, cfg), n)


@pytest.fixture
def grid_cap():
    """Cap persistent grids at one CTA: oc_step_kernel's grid-stride loop then
    walks every env chunk of the batch in sequence."""
    from paper_2311_10090_b200 import _native
    L = _native.lib()
    old = L.marl_set_grid_cap(1)
    yield
    L.marl_set_grid_cap(old)


def _run(env_id, cfg, acts, key, path, tag):
    import torch
    T, n, _ = acts.shape
    v, o = _venv(env_id, cfg, n), O.PortVenv(env_id, cfg, n)
    obs, state = v.reset(key)
    assert np.array_equal(obs.cpu().numpy(), o.reset(key))
    deliveries = pickups = 0
    host = None
    if path == "host":
        A, D = v.env().num_agents(), v.env().obs_dim
        host = {"obs": np.zeros((n, A, D), np.float32), "rewards": np.zeros((n, A), np.float64),
                "dones": np.zeros((n, A + 1), np.uint8), "finished": np.zeros(n, np.uint8),
                "final_obs": np.zeros((n, A, D), np.float32), "final_returns": np.zeros(n, np.float64),
                "final_lengths": np.zeros(n, np.int32), "infos": np.zeros((n, A, 2), np.float64)}
    for t in range(T):
        if path == "device":
            v.step(None, torch.from_numpy(acts[t]).cuda())
        else:
            v.host_step(acts[t], host)
        a = gpu_outputs(v, o.n_info)
        b = o.step(acts[t])
        _exact(a, b, f"{tag} step {t}")
        if host is not None:  # the host-buffer copies are the same bytes as the device views
            for f in host:
                assert np.array_equal(host[f], a[f]), f"{tag} step {t}: host {f}"
        deliveries += int((b["rewards"][:, 0] > 0).sum())
        pickups += int((b["infos"][:, :, I_SHAPED] == 5.0).sum())
    return deliveries, pickups


@pytest.mark.gpu
@pytest.mark.parametrize("path", ["device", "host"])
def test_gpu_scripted_soup(path, grid_cap):
    """The scripted soup on every env of a 600-env batch (three grid-stride
    iterations at one CTA): bit-exact on every field, and every idle-partner
    env delivers."""
    n = 600
    acts = scripted_actions(n, len(SCRIPT) + 8)
    d, p = _run("overcooked_cramped_room_v0", {}, acts, O.key_from_seed(5), path, f"scripted/{path}")
    assert d >= n // 2 and p >= n // 2, (d, p)


@pytest.mark.gpu
@pytest.mark.parametrize("layout", LAYOUTS)
def test_gpu_interact_heavy(layout, grid_cap):
    """The reference's interact-heavy protocol (40 episodes x 120 steps at
    max_steps 120), then 1024 envs across the default 400-step horizon."""
    env_id = f"overcooked_{layout}_v0"
    key = O.fold_in(O.key_from_seed(42), 1)
    _run(env_id, {"max_steps": 120}, interact_heavy(40, 121, seed=1), key, "device", f"{layout}/120")
    d, p = _run(env_id, {}, interact_heavy(1024, 401, seed=2), key, "device", f"{layout}/400")
    assert p > 0 or layout == "counter_circuit", (layout, d, p)
    if layout in ("cramped_room", "asymmetric_advantages"):
        assert d > 0, (layout, d, p)
