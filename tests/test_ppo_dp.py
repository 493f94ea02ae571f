"""Data-parallel PPO update (the gradient all-reduce).

Each rank owns a contiguous env shard (dist.shard_range), collects its rows,
draws the same global permutation, keeps the minibatch rows it owns and sums
advantage statistics, gradient, loss sums and episode counts over the ranks.
That is the single-device update's arithmetic split by rows, so a W-rank run
must reproduce the single-device trainer (and hence the reference trainer,
tests/test_ppo.py) up to float summation order.

* GPU: two ranks emulated by two threads on one B200, exchanging through a
  pairwise-sum hook -- vs the unsharded trainer: step / update / n_episodes /
  lr exact, losses and final parameters within 1e-3 relative (fp32; 1e-2 for
  the bf16 tcgen05 step).
* GPU: the native NCCL exchange at world size 1 is the identity: bitwise the
  unsharded, hook-free run.
* CPU (gloo, 2 processes): the torch.distributed hook sums in place.
"""
from __future__ import annotations

import os
import socket
import threading

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as O


def _trainer(venv, n_envs, T, precision="fp32", updates=2):
    from paper_2311_10090_b200.ppo import PpoTrainer
    cfg = {"n_envs": n_envs, "n_rollout_steps": T, "total_timesteps": updates * n_envs * T}
    return PpoTrainer(venv, cfg, False, precision)


class _PairSum:
    """Two in-process ranks: each hook call publishes its buffer, waits for the
    other, and both write back buf0 + buf1 (the same order on both)."""

    def __init__(self):
        self.barrier = threading.Barrier(2, timeout=120)
        self.bufs = [None, None]

    def hook(self, rank):
        import torch

        def fn(t):
            self.bufs[rank] = t.clone()
            self.barrier.wait()
            total = self.bufs[0] + self.bufs[1]
            self.barrier.wait()
            t.copy_(total)
            torch.cuda.synchronize()
        return fn


def _close(x, y, rel=1e-3, absf=1e-4):
    return np.all(np.abs(x - y) <= rel * np.abs(y) + absf * max(np.abs(y).max(), 1e-30))


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("env_id,cfg,n,T", [("MPE_simple_spread_v3", {}, 64, 16),
                                            ("SMAX_5m_vs_6m", {"ally_units": ["marine"] * 3,
                                                               "enemy_units": ["marine"] * 3}, 32, 32)])
def test_two_rank_update_matches_single_device(env_id, cfg, n, T, precision):
    """fp32: the CUDA-core minibatch kernels; bf16: the tcgen05 step over each
    shard's packed rows (the sharded minibatch is compacted to local slots)."""
    import paper_2311_10090_b200 as m
    from paper_2311_10090_b200 import dist as D
    env = m.make_env(env_id, cfg)
    key = O.key_from_seed(12)
    single = _trainer(m.VectorEnv(env, n, device=0), n, T, precision).train(key)

    pair = _PairSum()
    trainers = [_trainer(D.make_sharded(env, n, r, 2, device=0), n, T, precision) for r in range(2)]
    assert all(tr.tensor_core_update == (precision == "bf16") for tr in trainers)
    for r, tr in enumerate(trainers):
        tr.set_allreduce(pair.hook(r))
    out, err = [None, None], []

    def run(r):
        try:
            out[r] = trainers[r].train(key)
        except Exception as e:  # surface in the main thread
            err.append(e)
            pair.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    assert not err, err
    a, b = out
    # the ranks agree exactly (same all-reduced sums, same Adam arithmetic)
    assert np.array_equal(a.actor, b.actor) and np.array_equal(a.critic, b.critic)
    assert np.array_equal(a.metrics.as_array(), b.metrics.as_array())
    m1, m2 = single.metrics.as_array(), a.metrics.as_array()
    assert m1.shape == m2.shape
    for col in (0, 1, 3, 11):  # step, update, n_episodes, lr
        assert np.array_equal(m1[:, col], m2[:, col]), col
    assert np.allclose(m2[:, 2], m1[:, 2], rtol=1e-5, atol=1e-5)
    # bf16 operands turn the float reassociation of the sharded sums into occasional
    # rounding flips from the second update on: a 1e-2 bar there, 1e-3 for fp32
    rel = 1e-3 if precision == "fp32" else 1e-2
    for col in range(4, 11):
        assert np.allclose(m2[:, col], m1[:, col], rtol=rel, atol=1e-5), (col, m2[:, col], m1[:, col])
    assert _close(a.actor, single.actor, rel) and _close(a.critic, single.critic, rel)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_two_rank_wide_gradient_matches_single_device(precision):
    """The wide-input update (Overcooked, 3xTF32 GEMM chain) under the
    data-parallel hook: each rank's gradient over its own rows of a global
    minibatch, summed by the hook, equals the single device's gradient over
    the whole minibatch (fp32 summation-order bar), and so do the loss sums.
    (Whole training trajectories are not compared here: Adam's first step moves
    every parameter by +-lr whatever its gradient's size, so entries that
    cancel to ~0 take the sign of their summation-order noise.)"""
    import paper_2311_10090_b200 as m
    from paper_2311_10090_b200 import dist as D
    env = m.make_env("overcooked_cramped_room_v0", {"max_steps": 40})
    n, T = 16, 32
    key = O.key_from_seed(12)
    single = _trainer(m.VectorEnv(env, n, device=0), n, T, precision)
    pair = _PairSum()
    ranks = [_trainer(D.make_sharded(env, n, r, 2, device=0), n, T, precision) for r in range(2)]
    for r, tr in enumerate(ranks):
        tr.set_allreduce(pair.hook(r))
    for tr in [single] + ranks:
        assert not tr.tensor_core_update
    single.begin(key)
    single.collect()
    R, Rl = single.rollout.R, ranks[0].rollout.R
    assert ranks[1].rollout.R == Rl and 2 * Rl == R
    idx = np.random.default_rng(5).choice(T * R, size=T * R // 2, replace=False).astype(np.int32)
    t, row = idx // R, idx % R
    local = [(t * Rl + (row - r * Rl))[(row >= r * Rl) & (row < (r + 1) * Rl)].astype(np.int32) for r in range(2)]
    assert all(len(x) > 0 for x in local)
    g1, s1 = single.minibatch_grad(idx)
    out, err = [None, None], []

    def run(r):  # the ranks' collect all-reduces episode counts: both ranks run concurrently
        try:
            ranks[r].begin(key)
            ranks[r].collect()
            out[r] = ranks[r].minibatch_grad(local[r])
        except Exception as e:
            err.append(e)
            pair.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join(300)
    assert not err, err
    (ga, sa), (gb, sb) = out
    assert np.array_equal(ga, gb) and np.array_equal(sa, sb)
    assert _close(ga, g1, 2e-3), np.abs(ga - g1).max()
    assert np.allclose(sa, s1, rtol=2e-3, atol=1e-7), (sa, s1)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_nccl_world_of_one_is_identity(precision):
    import paper_2311_10090_b200 as m
    from paper_2311_10090_b200.ppo import nccl_unique_id
    env = m.make_env("MPE_simple_spread_v3", {})
    key = O.key_from_seed(13)
    ref = _trainer(m.VectorEnv(env, 48, device=0), 48, 16, precision).train(key)
    tr = _trainer(m.VectorEnv(env, 48, device=0), 48, 16, precision)
    tr.use_nccl(nccl_unique_id(), 0, 1)
    got = tr.train(key)
    assert np.array_equal(got.metrics.as_array(), ref.metrics.as_array())
    assert np.array_equal(got.actor, ref.actor) and np.array_equal(got.critic, ref.critic)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _hook_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2311_10090_b200.ppo import torch_allreduce
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fn = torch_allreduce()
    for dt in (torch.float32, torch.float64, torch.int64):
        t = torch.arange(5, dtype=dt) * (rank + 1)
        fn(t)
        q.put((rank, str(dt), t.tolist()))
    dist.destroy_process_group()


def test_torch_allreduce_hook_sums_in_place_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_hook_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(6)]
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    for rank, dt, vals in res:
        assert vals == [3 * i for i in range(5)], (rank, dt, vals)


def test_shard_ownership_partitions_every_minibatch():
    """The compaction's ownership rule (ppo.cu shard_map_kernel) restated: over
    W ranks every global minibatch slot is kept by exactly one rank, in order."""
    from paper_2311_10090_b200 import dist as D
    rng = np.random.default_rng(0)
    for n_envs, A, T, W in ((13, 3, 5, 2), (64, 3, 8, 3), (40, 6, 4, 4)):
        Rg = n_envs * A
        mb = rng.permutation(T * Rg)[: T * Rg // 2]
        seen = []
        for r in range(W):
            off, n_local = D.shard_range(n_envs, r, W)
            row0, Rl = off * A, n_local * A
            t, rr = mb // Rg, mb % Rg - row0
            own = (rr >= 0) & (rr < Rl)
            local = t[own] * Rl + rr[own]
            assert np.all(np.diff(np.nonzero(own)[0]) > 0)
            seen.append(np.stack([t[own], rr[own] + row0], 1))
            assert local.max(initial=-1) < T * Rl
        allrows = np.concatenate(seen)
        assert len(allrows) == len(mb) and len({tuple(x) for x in allrows}) == len(mb)
