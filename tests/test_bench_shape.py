"""Bench-shape parity on sampled shards (the persistent kernels' steady state
at the sizes the bench runs them).

The GPU steps the whole bench-size batch; the oracle replays a few small
shards at their global offsets (every key derives from the global env index,
vector_env.cpp:52-55,171, so a shard of the oracle is the same computation as
those rows of the full batch).  Every field of every step must be bit-exact.

* Overcooked cramped_room, 262 144 envs (configs[2]), default max_steps 400,
  ~430 steps: the grid-stride loop of oc_step_kernel runs ~7 iterations per
  warp, and rewards > 0 (deliveries) are asserted to occur in the shards.
* SMAX 27m_vs_30m, 4096 envs (configs[3]), default max_steps 100, 110 steps:
  battles decided by wipe-out (not only time-outs) are asserted to occur.
"""
import numpy as np
import pytest

import oracle as O
from _util import STEP_FIELDS, probe_keys

pytestmark = pytest.mark.gpu

FIELDS = ["actions", "obs", "rewards", "dones", "finished", "final_returns", "final_lengths", "infos", "keys",
          "episode_returns", "episode_lengths"]


def _shard_outputs(v, off, k, n_info):
    out = {}
    for f in FIELDS + ["final_obs"]:
        t = v.view(f)[off:off + k]
        out[f] = t.cpu().numpy().copy()
    out["infos"] = out["infos"][:, :, :n_info]
    out["keys"] = out["keys"].view(np.uint32)
    out["state_hash"] = v.state_hash()[off:off + k].cpu().numpy().view(np.uint64).copy()
    return out


def _run(env_id, cfg, n, T, shards, k, n_info, seed):
    import paper_2311_10090_b200 as m
    v = m.VectorEnv(m.make_env(env_id, cfg), n, device=0)
    key, ak = probe_keys(seed, T)
    v.reset(key)
    ports = []
    for off in shards:
        p = O.PortVenv(env_id, cfg, k, global_offset=off, global_n=n)
        p.reset(key)
        ports.append(p)
    rewards, finished, ends = 0.0, 0, []
    for t in range(T):
        v.step_random(ak[t])
        for off, p in zip(shards, ports):
            a = _shard_outputs(v, off, k, n_info)
            b = p.step_random(ak[t])
            b.update({f: x for f, x in p.batch_state().items() if f not in b})
            for f in STEP_FIELDS:
                assert np.array_equal(a[f], b[f]), (env_id, t, off, f)
            fin = b["finished"].astype(bool)
            assert np.array_equal(a["final_obs"][fin], b["final_obs"][fin]), (env_id, t, off)
            rewards += float(np.maximum(b["rewards"], 0).sum())
            finished += int(fin.sum())
            ends.append(b)
    return rewards, finished, ends


def test_overcooked_bench_shape_shards():
    n = 262144
    shards = [0, 40_000 * 2 + 13, n // 2 + 77, n - 16]
    rewards, finished, _ = _run("overcooked_cramped_room_v0", {}, n, 430, shards, 16, 3, 0)
    assert rewards > 0, "no delivery in the compared shards"
    assert finished == 4 * 16  # every env times out once at step 400


def test_smax27m_bench_shape_shards():
    n = 4096
    shards = [0, 1500, n - 8]
    _, finished, outs = _run("SMAX_27m_vs_30m", {}, n, 110, shards, 8, 3, 0)
    assert finished >= len(shards) * 8
    # some battles end before the 100-step limit: decided by wipe-out
    early = sum(int(((o["final_lengths"] > 0) & (o["final_lengths"] < 100)).sum()) for o in outs)
    assert early > 0, "no battle decided before the time limit"
