"""CPU: pin the oracle (oracle/marl_oracle.c) before trusting it.

* Threefry-2x32-20 known-answer vectors (test_prng.cpp:27-41),
* split / fold_in purity and disjointness (test_prng.cpp:53-90,183-191),
* the SMAX closed-form marine duel (test_smax.cpp:216-263),
* the golden trajectories dumped from the UNMODIFIED reference
  (tests/golden/, gen_golden.py) -- bit-exact, every field, every step,
* and, where the compiled reference is present (oracle/_ref), a live
  port-vs-reference comparison on fresh seeds.
"""
import numpy as np
import pytest

import oracle as O
from _util import GOLDEN, STEP_FIELDS, THREE_M, digest, golden_manifest


KATS = [((0, 0, 0, 0), (0x6B200159, 0x99BA4EFE)),
        ((0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF), (0x1CB996FC, 0xBB002BE7)),
        ((0x13198A2E, 0x03707344, 0x243F6A88, 0x85A308D3), (0xC4923A9C, 0x483DF7A0))]


@pytest.mark.parametrize("inp,out", KATS)
def test_threefry_kat(inp, out):
    assert O.threefry(*inp) == out


def test_split_purity_and_disjointness():
    k = O.key_from_seed(7)
    assert np.array_equal(O.split(k, 2), O.split(k, 2))
    four = O.split(k, 4)
    assert len({tuple(r) for r in four}) == 4
    # children do not alias the parent; fold_in differs from split children
    assert not any(np.array_equal(r, k) for r in four)
    fi = O.fold_in(k, 0)
    assert not any(np.array_equal(r, fi) for r in four)
    # split is a prefix-stable O(1) function of the index
    assert np.array_equal(O.split(k, 10)[:4], four)
    seen = set()
    for s in range(2000):
        for r in O.split(O.key_from_seed(s), 3):
            seen.add(tuple(r))
    assert len(seen) == 6000


def test_smax_duel_closed_form():
    cfg = {"ally_units": ["marine"], "enemy_units": ["marine"], "map_size": 8.0,
           "enemy_controlled": True, "spawn_jitter": 0.0}
    v = O.PortVenv("SMAX_5m_vs_6m", cfg, 1)
    v.reset(O.key_from_seed(7))
    u = v.smax_units()
    assert u["x"][0] == 2.0 and u["x"][1] == 6.0 and u["y"][0] == u["y"][1]
    hp = [39, 33, 27, 21, 21, 15, 9, 3, 0]
    ret = 0.0
    for step in range(1, 10):
        out = v.step(np.array([[5, 5]], np.int32))
        ret += out["rewards"][0, 0]
        if step < 9:
            u = v.smax_units()
            assert u["health"][0] == hp[step - 1] and u["health"][1] == hp[step - 1]
            assert out["finished"][0] == 0
        else:
            assert out["finished"][0] == 1
            assert out["infos"][0, 0].tolist() == [0.0, 0.0, 1.0]  # alive, battle_won, draw
    assert abs(ret - 0.5) < 1e-12


@pytest.mark.parametrize("name", sorted(golden_manifest()))
def test_oracle_matches_reference_golden(name):
    rec = golden_manifest()[name]
    v = O.PortVenv(rec["env_id"], rec["config"], rec["n_envs"])
    key = O.key_from_seed(rec["seed"])
    assert digest(v.reset(key)) == rec["reset_obs"]
    akeys = O.split(O.fold_in(key, 2), rec["steps"] + 1)
    for t, want in enumerate(rec["digests"]):
        out = v.step_random(akeys[t])
        for f in STEP_FIELDS:
            assert digest(out[f]) == want[f], f"{name}: step {t} field {f}"
        fin = out["finished"].astype(bool)
        assert digest(out["final_obs"][fin]) == want["final_obs"], f"{name}: step {t} final_obs"


@pytest.mark.skipif(not O.ref_available(), reason="compiled reference (oracle/_ref) not present")
@pytest.mark.parametrize("env_id,cfg,n,T", [
    ("MPE_simple_spread_v3", {}, 40, 55),
    ("SMAX_5m_vs_6m", THREE_M, 40, 60),
    ("SMAX_3s5z", {}, 6, 30),
    ("SMAX_10m_vs_11m", {"unit_stats": {"marine": {"range": 3.0, "speed": 4.0}}}, 4, 30),
    ("overcooked_counter_circuit_v0", {"max_steps": 40, "cook_time": 3}, 6, 90),
])
def test_oracle_matches_live_reference(env_id, cfg, n, T):
    p, r = O.PortVenv(env_id, cfg, n), O.RefVenv(env_id, cfg, n)
    key = O.key_from_seed(99)
    assert np.array_equal(p.reset(key), r.reset(key))
    ak = O.split(O.fold_in(key, 2), T + 1)
    for t in range(T):
        a, b = p.step_random(ak[t]), r.step_random(ak[t])
        for f in STEP_FIELDS:
            assert np.array_equal(a[f], b[f]), (env_id, t, f)


def test_sharded_oracle_equals_full_batch():
    """Global-index key derivation: two shards == one batch (the analogue of
    test_vector_env.cpp:117-154's thread-count invariance)."""
    full = O.PortVenv("SMAX_5m_vs_6m", THREE_M, 10)
    a = O.PortVenv("SMAX_5m_vs_6m", THREE_M, 4, global_offset=0, global_n=10)
    b = O.PortVenv("SMAX_5m_vs_6m", THREE_M, 6, global_offset=4, global_n=10)
    key = O.key_from_seed(5)
    assert np.array_equal(full.reset(key), np.concatenate([a.reset(key), b.reset(key)]))
    ak = O.split(O.fold_in(key, 2), 31)
    for t in range(30):
        f, x, y = full.step_random(ak[t]), a.step_random(ak[t]), b.step_random(ak[t])
        for k in STEP_FIELDS:
            assert np.array_equal(f[k], np.concatenate([x[k], y[k]])), (t, k)
