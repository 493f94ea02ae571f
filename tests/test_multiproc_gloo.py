"""N>1 host logic on CPU: two gloo ranks each own a contiguous shard
(dist.shard_range, the parallel.cpp:61-65 chunk rule), step it with the
oracle as the stand-in for the per-GPU engine, and reduce the exact integer
episode statistics with one all-reduce.  The concatenated shard outputs and
the reduced totals must equal a single full-batch run bit for bit -- the
multi-rank analogue of test_vector_env.cpp:117-154."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as O
from _util import STEP_FIELDS, THREE_M
from paper_2311_10090_b200 import dist as D

CASES = [("SMAX_5m_vs_6m", THREE_M, 13, 40), ("MPE_simple_spread_v3", {}, 9, 60),
         ("overcooked_cramped_room_v0", {"max_steps": 20}, 7, 50)]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _episode_stats(outs):
    """[episodes, sum lengths, sum fixed-point returns] over a run's outputs."""
    eps = lens = rets = 0
    for o in outs:
        fin = o["finished"].astype(bool)
        eps += int(fin.sum())
        lens += int(o["final_lengths"][fin].astype(np.int64).sum())
        rets += sum(D.fixed_point_return(r) for r in o["final_returns"][fin])
    return [eps, lens, rets]


def _run(env_id, cfg, n, T, offset=0, local=None):
    v = O.PortVenv(env_id, cfg, local if local is not None else n, global_offset=offset, global_n=n)
    key = O.key_from_seed(11)
    ak = O.split(O.fold_in(key, 2), T + 1)
    v.reset(key)
    return [v.step_random(ak[t]) for t in range(T)]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        for env_id, cfg, n, T in CASES:
            off, local = D.shard_range(n, rank, world)
            outs = _run(env_id, cfg, n, T, off, local)
            raw = D.all_reduce_episode_stats(_episode_stats(outs))
            elapsed = D.max_over_ranks(float(rank + 1))
            res[env_id] = (off, local, {f: np.stack([o[f] for o in outs]) for f in STEP_FIELDS}, raw, elapsed)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_shard_range_is_the_threadpool_chunk_rule():
    assert [D.shard_range(10, r, 4) for r in range(4)] == [(0, 2), (2, 3), (5, 2), (7, 3)]
    assert sum(D.shard_range(1 << 20, r, 8)[1] for r in range(8)) == 1 << 20
    with pytest.raises(ValueError):
        D.shard_range(3, 0, 4)
    with pytest.raises(ValueError):
        D.shard_range(8, 2, 2)


def test_two_rank_gloo_shards_equal_full_batch():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get() for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for env_id, cfg, n, T in CASES:
        full = _run(env_id, cfg, n, T)
        expect = _episode_stats(full)
        (o0, n0, s0, raw0, t0), (o1, n1, s1, raw1, t1) = got[0][env_id], got[1][env_id]
        assert (o0, o1, n0 + n1) == (0, n0, n)
        assert raw0 == raw1 == expect, env_id          # one SUM all-reduce, exact
        assert t0 == t1 == 2.0                          # max over ranks
        for f in STEP_FIELDS:
            whole = np.stack([o[f] for o in full])
            assert np.array_equal(whole, np.concatenate([s0[f], s1[f]], axis=1)), (env_id, f)
