"""GPU: the VectorEnv contract (vector_env.cpp, test_vector_env.cpp) on the
CUDA engine -- error behaviour, purity/determinism, shard invariance (the
analogue of the 1/4/16-thread invariance test, test_vector_env.cpp:117-154),
episode bookkeeping, and size-independent properties at full bench sizes."""
import numpy as np
import pytest

import oracle as O
from _util import THREE_M, gpu_outputs, probe_keys

pytestmark = pytest.mark.gpu


def _m():
    import paper_2311_10090_b200 as m
    return m


def test_invalid_actions_raise_and_leave_state_untouched():
    import torch
    m = _m()
    v = m.VectorEnv("SMAX_5m_vs_6m", 32, config=THREE_M)
    _, st = v.reset(O.key_from_seed(1))
    h0 = v.state_hash().cpu().numpy().copy()
    bad = torch.full((32, 3), 4, dtype=torch.int32, device="cuda")
    bad[7, 2] = 99
    with pytest.raises(m.ContractError, match="ally_2"):
        v.step(st, bad)
    assert np.array_equal(v.state_hash().cpu().numpy(), h0)
    with pytest.raises(m.ContractError):
        v.step(st, np.full((32, 3), -1, np.int32))
    with pytest.raises(m.ContractError):
        v.step(st, np.zeros((31, 3), np.int32))
    assert np.array_equal(v.state_hash().cpu().numpy(), h0)
    # the handle recovers: a valid step works and matches the oracle
    o = O.PortVenv("SMAX_5m_vs_6m", THREE_M, 32)
    o.reset(O.key_from_seed(1))
    good = np.full((32, 3), 4, np.int32)
    r = v.step(st, good)
    b = o.step(good)
    assert np.array_equal(gpu_outputs(v, 3)["obs"], b["obs"])
    with pytest.raises(m.ContractError, match="stale"):
        v.step(st, good)
    v.step(r.next, good)


def test_step_before_reset_is_contract_error():
    m = _m()
    v = m.VectorEnv("MPE_simple_spread_v3", 4)
    with pytest.raises(m.ContractError):
        v.step(None, np.zeros((4, 3), np.int32))


@pytest.mark.parametrize("env_id,cfg", [("SMAX_5m_vs_6m", THREE_M), ("overcooked_cramped_room_v0", {"max_steps": 20}),
                                        ("MPE_simple_spread_v3", {})])
def test_shard_invariance(env_id, cfg):
    """Splitting the batch across handles (as across GPUs) is bit-identical."""
    m = _m()
    N, T = 200, 45
    full = m.VectorEnv(env_id, N, config=cfg)
    parts = [m.VectorEnv(env_id, 70, config=cfg, global_offset=0, global_n=N),
             m.VectorEnv(env_id, 130, config=cfg, global_offset=70, global_n=N)]
    key, ak = probe_keys(21, T)
    full.reset(key)
    for p in parts:
        p.reset(key)
    for t in range(T):
        full.step_random(ak[t])
        for p in parts:
            p.step_random(ak[t])
        a = gpu_outputs(full, full.env().n_info)
        bs = [gpu_outputs(p, p.env().n_info) for p in parts]
        for f in a:
            assert np.array_equal(a[f], np.concatenate([b[f] for b in bs])), (t, f)
    assert full.episode_stats_raw() == [x + y for x, y in zip(parts[0].episode_stats_raw(),
                                                              parts[1].episode_stats_raw())]


def test_determinism_and_bookkeeping_identity():
    """Re-running is bit-identical; no transition lost across boundaries
    (test_vector_env.cpp:92-115): sum of finished lengths + in-flight == steps."""
    m = _m()
    N, T = 4096, 150
    runs = []
    for _ in range(2):
        v = m.VectorEnv("SMAX_5m_vs_6m", N, config=THREE_M)
        key, ak = probe_keys(5, T)
        v.reset(key)
        done_len = 0
        for t in range(T):
            r = v.step_random(ak[t])
            fin = r.finished.bool()
            done_len += int(r.final_lengths[fin].sum())
        in_flight = int(v.view("episode_lengths").sum())
        assert done_len + in_flight == N * T
        eps, lens, rets = v.episode_stats()
        assert lens == done_len and eps > 0
        runs.append((v.state_hash().cpu().numpy().copy(), v.keys_numpy().copy(), eps, lens, rets))
    assert np.array_equal(runs[0][0], runs[1][0]) and np.array_equal(runs[0][1], runs[1][1])
    assert runs[0][2:] == runs[1][2:]


def test_full_size_overcooked_properties():
    """C3 at full size (262144 envs): one-hot plane invariants every step and
    the synchronised horizon (all episodes end at t = max_steps)."""
    import torch
    m = _m()
    N, T, H = 262144, 40, 25
    v = m.VectorEnv("overcooked_cramped_room_v0", N, config={"max_steps": H})
    key, ak = probe_keys(2, T)
    v.reset(key)
    cells = 20
    for t in range(T):
        r = v.step_random(ak[t])
        obs = r.obs.view(N, 2, 541)
        planes = obs[:, :, :540].view(N, 2, 27, cells)
        assert torch.all(planes[:, :, 0].sum(-1) == 1)          # self position one-hot
        assert torch.all(planes[:, :, 2:6].sum((-1, -2)) == 1)  # exactly one facing plane set
        assert torch.all(planes[:, :, 10:15].sum(-2).max(-1).values <= 1)
        expect_done = (t + 1) % H == 0
        assert bool(torch.all(r.finished == int(expect_done)))
        clock = ((t + 1) % H) / H
        assert torch.allclose(obs[:, :, 540], torch.full_like(obs[:, :, 540], clock))
    torch.cuda.synchronize()


def test_full_size_smax_properties():
    """C2 at full size (65536 envs): rewards identical across allies, reward
    ledger bounded, health never increases, obs entries in [-1, 1]."""
    import torch
    m = _m()
    N, T = 65536, 60
    v = m.VectorEnv("SMAX_5m_vs_6m", N, config=THREE_M)
    key, ak = probe_keys(4, T)
    v.reset(key)
    for t in range(T):
        r = v.step_random(ak[t])
        rew = r.rewards
        assert torch.all(rew[:, 0] == rew[:, 1]) and torch.all(rew[:, 1] == rew[:, 2])
        assert torch.all(rew <= 1.0 + 1e-12) and torch.all(rew >= 0.0)
        assert torch.all(r.obs.abs() <= 1.0)
        assert torch.all(r.dones[:, 3] == r.finished)
    eps, lens, rets = v.episode_stats()
    assert eps > N // 2 and 5 < lens / eps < 60


def test_throughput_probe_runs():
    m = _m()
    res = m.throughput_probe("MPE_simple_spread_v3", 1024, 50, O.key_from_seed(1))
    assert res.sps > 0 and np.isfinite(res.sps) and res.cold_seconds > 0
    assert res.csv_row().startswith("MPE_simple_spread_v3,1024,50,")
    assert m.ThroughputResult.csv_header() == "env_id,n_envs,steps,seconds,sps"


@pytest.mark.parametrize("env_id,cfg,n", [("SMAX_5m_vs_6m", THREE_M, 40_003), ("MPE_simple_spread_v3", {}, 70_001),
                                          ("overcooked_cramped_room_v0", {"max_steps": 3}, 33_001)])
def test_host_buffer_step_matches_device_views(env_id, cfg, n):
    """The host-buffer step (C-ABI marl_venv_step_random_host / _step_host, run
    as env chunks whose outputs stream back while later chunks compute) equals
    the one-launch device step of a twin VectorEnv, every field, exactly."""
    m = _m()
    a = m.VectorEnv(env_id, n, config=cfg)
    b = m.VectorEnv(env_id, n, config=cfg)
    a.reset(O.key_from_seed(3))
    b.reset(O.key_from_seed(3))
    fields = ("obs", "rewards", "dones", "finished", "final_obs", "final_returns", "final_lengths", "infos",
              "actions")
    if not a.info_names:
        fields = tuple(f for f in fields if f != "infos")
    for k in range(4):
        key = O.fold_in(O.key_from_seed(9), k)
        a.step_random(key)
        want = a.download(fields)
        got = {f: np.zeros_like(want[f]) for f in fields}
        if k % 2 == 0:
            b.host_step_random(key, got)
        else:
            b.host_step(want["actions"], got)
        for f in fields:
            assert np.array_equal(got[f], want[f]), (k, f)
    assert np.array_equal(a.state_hash().cpu().numpy(), b.state_hash().cpu().numpy())


def test_generic_rollout_matches_oracle_loop():
    """rollout(venv, policy, T, key) (vector_env.cpp:131-165) with an
    observation-dependent policy vs the same loop on the plain-C oracle."""
    import torch
    m = _m()
    n, T = 50, 30
    env_id, cfg = "SMAX_5m_vs_6m", THREE_M
    v = m.VectorEnv(env_id, n, config=cfg)

    def policy(obs):  # stop (always legal) + observation-derived log-probs / values
        acts = torch.full(obs.shape[:2], 4, dtype=torch.int32, device=obs.device)
        return acts, obs[:, :, 0].double() - obs[:, :, 1].double(), obs[:, :, 2].double()

    tr = m.rollout(v, policy, T, O.key_from_seed(11))
    assert tr.n_steps == T and tr.n_envs == n and tuple(tr.obs.shape[:2]) == (T, n)
    o = O.PortVenv(env_id, cfg, n)
    ob = o.reset(O.key_from_seed(11))
    for t in range(T):
        assert np.array_equal(tr.obs[t].cpu().numpy(), ob), t
        r = o.step(np.full((n, 3), 4, np.int32))
        assert np.array_equal(tr.rewards[t].cpu().numpy(), r["rewards"]), t
        assert np.array_equal(tr.dones[t].cpu().numpy(), r["dones"]), t
        ob = r["obs"]
    assert np.array_equal(tr.final_obs.cpu().numpy(), ob)
    assert np.allclose(tr.log_probs.cpu().numpy(), tr.obs[..., 0].double().cpu().numpy() -
                       tr.obs[..., 1].double().cpu().numpy())
    with pytest.raises(m.ContractError):
        m.rollout(v, policy, 0, O.key_from_seed(1))


@pytest.mark.parametrize("env_id,cfg,n", [("SMAX_5m_vs_6m", THREE_M, 40_003),
                                          ("overcooked_cramped_room_v0", {"max_steps": 3}, 33_001)])
def test_host_final_obs_mapped_buffer_gets_finished_rows_only(env_id, cfg, n):
    """final_obs is valid where finished (vector_env.hpp:31): into a mapped
    pinned host buffer the device writes exactly the finished rows (equal to
    the device view) and leaves every other row as the caller left it."""
    import torch
    m = _m()
    a = m.VectorEnv(env_id, n, config=cfg)
    b = m.VectorEnv(env_id, n, config=cfg)
    a.reset(O.key_from_seed(5))
    b.reset(O.key_from_seed(5))
    shape = (n, a.env().num_agents(), a.env().obs_dim)
    fo = torch.full(shape, -7.0, dtype=torch.float32, pin_memory=True).numpy()
    fin = torch.zeros((n,), dtype=torch.uint8, pin_memory=True).numpy()
    seen = 0
    for k in range(25):
        key = O.fold_in(O.key_from_seed(11), k)
        a.step_random(key)
        want = a.download(("final_obs", "finished"))
        fo[:] = -7.0
        b.host_step_random(key, {"final_obs": fo, "finished": fin})
        f = want["finished"].astype(bool)
        assert np.array_equal(fin, want["finished"])
        assert np.array_equal(fo[f], want["final_obs"][f]), k
        assert np.all(fo[~f] == -7.0), k
        seen += int(f.sum())
    assert seen > 0
