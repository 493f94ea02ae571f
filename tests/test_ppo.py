"""PPO update on the device (ff_minibatch, ppo_row_loss,
clip_global_norm, adam_update, train_ippo / train_mappo).

Oracle: the reference compiled from /root/reference (oracle/_ref):
prng::permutation, ppo_init_nets, the private ff_minibatch restated over the
reference's public nn pieces (oracle/ref_rollout.cpp), and the reference's own
public train_ippo / train_mappo.

Parity bars:
* permutation (Fisher-Yates, prng.cpp:151-159): exact, every n;
* ppo_init_nets (host C++ restatement): bit-exact;
* one minibatch gradient vs ff_minibatch on identical buffers: within float
  accumulation tolerance (the reference sums rows sequentially in float, the
  device reassociates): |g - g_ref| <= 2e-3 |g_ref| + 1e-4 max|g_ref|; loss
  statistics within 1e-5 relative;
* a short train_ippo / train_mappo run vs the reference's: step / update /
  n_episodes exact, every loss column and the final parameters within 1e-3
  relative (Adam normalises the gradient, so parameter errors stay at the
  gradient's relative error times lr).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from _util import THREE_M


def _need_ref():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")


ENVS = [("MPE_simple_spread_v3", {}), ("SMAX_5m_vs_6m", THREE_M), ("overcooked_cramped_room_v0", {}),
        ("SMAX_27m_vs_30m", {"max_steps": 20})]


# ------------------------------------------------------------------ CPU tests
def _parallel_fisher_yates(key, n):
    """The device algorithm (ppo.cu perm_*_kernel) restated in numpy."""
    j = np.array([0] + [O.bits(key, i) % (i + 1) for i in range(1, n)], np.int64)
    ks, vs = j[1:], np.arange(1, n)
    order = np.argsort(ks, kind="stable")
    ks, vs = ks[order], vs[order]
    nxt = -np.ones(n, np.int64)
    fst = -np.ones(n, np.int64)
    for p in range(n - 1):
        q, k = ks[p], vs[p]
        nx = vs[p + 1] if p + 1 < n - 1 and ks[p + 1] == q else -1
        nxt[k] = nx
        if p == 0 or ks[p - 1] != q:
            fst[q] = k if k != q else nx
    out = np.zeros(n, np.int64)
    for i in range(n):
        v = 0 if i == 0 else nxt[i]
        if i > 0 and v < 0:
            out[i] = j[i]
            continue
        while fst[v] >= 0:
            v = fst[v]
        out[i] = v
    return out


@pytest.mark.parametrize("n", [1, 2, 3, 5, 17, 256, 1001])
def test_parallel_fisher_yates_formulation_matches_reference(n):
    _need_ref()
    for s in range(3):
        k = O.key_from_seed(100 + s)
        assert np.array_equal(_parallel_fisher_yates(k, n), O.ref_permutation(k, n))


@pytest.mark.parametrize("env_id,cfg", ENVS)
@pytest.mark.parametrize("centralized", [False, True])
def test_init_nets_bit_exact(env_id, cfg, centralized):
    """ppo_init_nets (ppo.cpp:109-124: Box-Muller normals, modified Gram-Schmidt)
    restated in the host library equals the reference bit for bit."""
    _need_ref()
    from paper_2311_10090_b200.ppo import init_nets
    sp = O.ref_ppo_spec(env_id, cfg, centralized)
    for seed in (0, 9):
        key = O.key_from_seed(seed)
        ra, rc = O.ref_ppo_init(env_id, cfg, key, centralized)
        a, c = init_nets(sp["in_dim"], sp["critic_in"], sp["n_actions"], key)
        assert a.tobytes() == ra.tobytes() and c.tobytes() == rc.tobytes()


def test_reference_train_invariants():
    """The oracle trainer itself: one row per update, annealed lr, steps column."""
    _need_ref()
    cfg = {"total_timesteps": 3 * 4 * 8, "n_envs": 4, "n_rollout_steps": 8}
    r = O.ref_train("MPE_simple_spread_v3", {}, cfg, O.key_from_seed(1))
    m = r["metrics"]
    assert m.shape == (3, 12) and not r["diverged"] and r["steps_done"] == 96
    assert np.array_equal(m[:, 0], [32, 64, 96]) and np.array_equal(m[:, 1], [0, 1, 2])
    assert np.allclose(m[:, 11], 5e-4 * (1 - np.arange(3) / 3))


# ------------------------------------------------------------------ GPU tests
@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 3, 10, 1000, 65537, 1 << 20])
def test_device_permutation_matches_reference(n):
    _need_ref()
    from paper_2311_10090_b200.ppo import permutation
    for s in range(2):
        k = O.key_from_seed(7 + s)
        got = permutation(k, n).cpu().numpy()
        assert np.array_equal(got, O.ref_permutation(k, n)), (n, s)


def _trainer(env_id, cfg, n_envs, T, centralized=False, precision="fp32", **ppo):
    import paper_2311_10090_b200 as m
    from paper_2311_10090_b200.ppo import PpoTrainer
    v = m.VectorEnv(m.make_env(env_id, cfg), n_envs, device=0)
    pc = {"n_envs": n_envs, "n_rollout_steps": T, "total_timesteps": 4 * n_envs * T}
    pc.update(ppo)
    return PpoTrainer(v, pc, centralized, precision)


def _close(got, ref, rel=2e-3, absf=1e-4):
    tol = rel * np.abs(ref) + absf * max(np.abs(ref).max(), 1e-30)
    return np.all(np.abs(got - ref) <= tol), np.abs(got - ref).max()


@pytest.mark.gpu
@pytest.mark.parametrize("env_id,cfg", ENVS)
@pytest.mark.parametrize("centralized", [False, True])
def test_minibatch_gradient_matches_ff_minibatch(env_id, cfg, centralized):
    _need_ref()
    if centralized and env_id == "SMAX_27m_vs_30m":
        pytest.skip("27m_vs_30m's world_state is wider than the collector's 1024-column critic input")
    n_envs, T = (16, 24) if env_id.startswith(("MPE", "SMAX_5m")) else (4, 24)
    tr = _trainer(env_id, cfg, n_envs, T, centralized)
    key = O.key_from_seed(21)
    tr.begin(key)
    tr.collect()
    buf = {k: t.cpu().numpy() for k, t in tr.rollout._views.items()}
    a, c = tr.params()
    R = tr.rollout.R
    rng = np.random.default_rng(3)
    for M in (T * R // 2, 1, 37):  # largest first: a smaller minibatch must not read its stale loss rows
        idx = rng.choice(T * R, size=M, replace=False).astype(np.int32)
        g, st = tr.minibatch_grad(idx)
        gr, sr = O.ref_ff_minibatch(env_id, cfg, a, c, buf, idx, centralized=centralized)
        ok, err = _close(g, gr)
        assert ok, (M, err)
        # the per-row kernels evaluate the forward in the reference's order (stats within 1e-5); wide
        # inputs run it as 3xTF32 GEMMs (fp32-accurate, another summation order), so a row whose value
        # sits near its target moves the value loss by more: the gradient's 2e-3 bar there
        rtol = 2e-3 if max(tr.spec.in_dim, tr.spec.critic_in) >= 256 else 1e-5
        assert np.allclose(st, sr, rtol=rtol, atol=1e-7), (M, st, sr)


@pytest.mark.gpu
def test_minibatch_all_inactive_rows_give_zero():
    """A fully masked minibatch: zero loss, zero gradient (actor_critic.hpp:353-354)."""
    _need_ref()
    tr = _trainer("SMAX_5m_vs_6m", THREE_M, 8, 40)
    tr.begin(O.key_from_seed(2))
    tr.collect()
    act = tr.rollout._views["active"].cpu().numpy().ravel()
    dead = np.nonzero(act == 0)[0].astype(np.int32)
    if dead.size == 0:
        pytest.skip("no inactive rows in this window")
    g, st = tr.minibatch_grad(dead[:64])
    assert not g.any() and not st.any()


def _compare_train(env_id, cfg, ppo_cfg, key, centralized=False):
    from paper_2311_10090_b200 import make_env
    from paper_2311_10090_b200.ppo import train_ippo, train_mappo
    ref = O.ref_train(env_id, cfg, ppo_cfg, key, centralized)
    fn = train_mappo if centralized else train_ippo
    got = fn(make_env(env_id, cfg), ppo_cfg, key)
    m, rm = got.metrics.as_array(), ref["metrics"]
    assert m.shape == rm.shape and got.diverged == ref["diverged"] and got.steps_done == ref["steps_done"]
    for col in (0, 1, 3, 11):  # step, update, n_episodes, lr
        assert np.array_equal(m[:, col], rm[:, col]), O.PPO_COLUMNS[col]
    assert np.allclose(m[:, 2], rm[:, 2], rtol=1e-5, atol=1e-5)  # mean_return (2^-24 fixed-point sums)
    for col in range(4, 11):
        assert np.allclose(m[:, col], rm[:, col], rtol=1e-3, atol=1e-5), (O.PPO_COLUMNS[col], m[:, col], rm[:, col])
    for x, rx in ((got.actor, ref["actor"]), (got.critic, ref["critic"])):
        ok, err = _close(x, rx, rel=1e-3, absf=1e-4)
        assert ok, err
    return got, ref


@pytest.mark.gpu
@pytest.mark.parametrize("env_id,cfg,n_envs,T", [("MPE_simple_spread_v3", {}, 8, 16),
                                                 ("SMAX_5m_vs_6m", THREE_M, 8, 32),
                                                 ("overcooked_cramped_room_v0", {"max_steps": 40}, 2, 40)])
def test_train_ippo_matches_reference(env_id, cfg, n_envs, T):
    _need_ref()
    ppo_cfg = {"total_timesteps": 2 * n_envs * T, "n_envs": n_envs, "n_rollout_steps": T}
    _compare_train(env_id, cfg, ppo_cfg, O.key_from_seed(5))


@pytest.mark.gpu
def test_train_mappo_matches_reference():
    _need_ref()
    ppo_cfg = {"total_timesteps": 2 * 8 * 16, "n_envs": 8, "n_rollout_steps": 16, "update_epochs": 2,
               "n_minibatches": 4, "anneal_lr": False, "activation": "relu"}
    _compare_train("MPE_simple_spread_v3", {}, ppo_cfg, O.key_from_seed(6), centralized=True)


@pytest.mark.gpu
def test_ppo_config_schema_errors():
    import paper_2311_10090_b200 as m
    from paper_2311_10090_b200.errors import ContractError, SchemaError
    from paper_2311_10090_b200.ppo import PpoTrainer
    v = m.VectorEnv(m.make_env("MPE_simple_spread_v3", {}), 4, device=0)
    for bad in ({"n_envs": 4, "bogus": 1}, {"n_envs": 4, "clip_eps": 1.5}, {"n_envs": 4, "activation": "gelu"},
                {"n_envs": 4, "n_rollout_steps": 5, "n_minibatches": 7},
                {"n_envs": 4, "recurrent": True, "n_minibatches": 5}):  # 12 rows % 5 (ppo.cpp:548-552)
        with pytest.raises(SchemaError):
            PpoTrainer(v, bad)
    with pytest.raises(ContractError):
        PpoTrainer(v, {"n_envs": 8})


# ------------------------------------------------ tcgen05 (bf16) minibatch step
def _cos(a, b):
    return float(np.dot(a, b) / (np.linalg.norm(a) * np.linalg.norm(b) + 1e-30))


def _blocks(sp):
    W, I, NA = sp.width, sp.in_dim, sp.n_actions
    out, off = [], 0
    for n in (W * I, W, W * W, W, NA * W, NA, W * I, W, W * W, W, W, 1):
        out.append((off, off + n))
        off += n
    return out


def _assert_blocks_close(g, gr, blocks, what):
    for lo, hi in blocks:
        x, y = g[lo:hi], gr[lo:hi]
        if np.linalg.norm(y) < 1e-12:
            continue
        assert _cos(x, y) >= 0.995, (what, lo, hi, _cos(x, y))
        assert abs(np.linalg.norm(x) / np.linalg.norm(y) - 1) < 0.03, (what, lo, hi)


# input widths: 18 (Kx 32), 95 (Kx 96, two X buffers), 163 (Kx 176, one X buffer), 180 (Kx 192, the widest)
TC_SHAPES = [("MPE_simple_spread_v3", {}), ("SMAX_5m_vs_6m", THREE_M), ("SMAX_2s3z", {}), ("SMAX_5m_vs_6m", {})]


@pytest.mark.gpu
@pytest.mark.parametrize("env_id,cfg", TC_SHAPES)
def test_tc_minibatch_gradient_matches_reference(env_id, cfg):
    """The bf16 tensor-core step (ppo_tc.cu) vs ff_minibatch on the same buffers:
    every parameter block's gradient has cosine >= 0.995 and norm within 3 %;
    loss statistics within 2 %."""
    _need_ref()
    tr = _trainer(env_id, cfg, 64, 32, precision="bf16")
    assert tr.tensor_core_update
    tr.begin(O.key_from_seed(31))
    tr.collect()
    buf = {k: t.cpu().numpy() for k, t in tr.rollout._views.items()}
    a, c = tr.params()
    R = tr.rollout.R
    rng = np.random.default_rng(5)
    for M in (200, 3000):
        idx = rng.choice(32 * R, size=M, replace=False).astype(np.int32)
        g, st = tr.minibatch_grad(idx)
        gr, sr = O.ref_ff_minibatch(env_id, cfg, a, c, buf, idx)
        _assert_blocks_close(g, gr, _blocks(tr.spec), M)
        assert np.allclose(st, sr, rtol=2e-2, atol=1e-4), (st, sr)


@pytest.mark.gpu
@pytest.mark.parametrize("activation", ["relu", "tanh"])
@pytest.mark.parametrize("env_id,cfg", TC_SHAPES[:2])
def test_tc_minibatch_gradient_matches_fp32_path(activation, env_id, cfg):
    """bf16 tcgen05 step vs the fp32 step (itself pinned to the reference above)
    on identical buffers copied between two trainers; relu covers the other
    activation the reference supports."""
    tc = _trainer(env_id, cfg, 64, 32, precision="bf16", activation=activation)
    f32 = _trainer(env_id, cfg, 64, 32, precision="fp32", activation=activation)
    key = O.key_from_seed(41)
    tc.begin(key)
    f32.begin(key)
    tc.collect()
    for k, v in tc.rollout._views.items():
        f32.rollout._views[k].copy_(v)
    a, c = tc.params()
    f32.set_params(a, c)
    R = tc.rollout.R
    idx = np.random.default_rng(6).choice(32 * R, size=3000, replace=False).astype(np.int32)
    g, st = tc.minibatch_grad(idx)
    gr, sr = f32.minibatch_grad(idx)
    _assert_blocks_close(g, gr, _blocks(tc.spec), activation)
    assert np.allclose(st, sr, rtol=2e-2, atol=1e-4), (st, sr)


@pytest.mark.gpu
def test_tc_training_run_is_sane():
    """A bf16 training run (tcgen05 rollout policy + tcgen05 update): finite
    metrics, no divergence, the value loss falls like the fp32 run's."""
    tr = _trainer("MPE_simple_spread_v3", {}, 256, 32, precision="bf16")
    tr.n_updates = 4
    res = tr.train(O.key_from_seed(8))
    m = res.metrics.as_array()
    assert not res.diverged and np.isfinite(m).all() and m.shape[0] == 4
    assert m[-1, 6] < m[0, 6]  # v_loss
    assert np.isfinite(res.actor).all() and np.isfinite(res.critic).all()


@pytest.mark.gpu
def test_divergence_rolls_back_the_update():
    """A non-finite loss is the reference's DivergenceError (actor_critic.hpp:403-405):
    the update's parameters are restored, the row counts no minibatch and the
    run stops (ppo.cpp:630-650)."""
    import paper_2311_10090_b200 as m
    from paper_2311_10090_b200.ppo import PpoTrainer
    v = m.VectorEnv(m.make_env("MPE_simple_spread_v3", {}), 16, device=0)
    tr = PpoTrainer(v, {"n_envs": 16, "n_rollout_steps": 8, "total_timesteps": 5 * 16 * 8})
    tr.begin(O.key_from_seed(4))
    a, c = tr.params()
    c = c.copy()
    c[-1] = np.inf  # the critic head bias: every value is inf -> non-finite v_loss
    tr.set_params(a, c)
    tr.collect()
    row, diverged = tr.update()
    assert diverged
    a2, c2 = tr.params()
    assert np.array_equal(a2, a) and np.array_equal(c2[:-1], c[:-1]) and np.isinf(c2[-1])
    assert np.all(row[4:11] == 0.0)  # no minibatch completed: the sums are empty
