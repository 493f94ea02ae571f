"""CPU: the C-ABI library loads, exports every symbol include/marl_b200.h
declares, and its host logic (registry, strict config schema, spaces, key
helpers) behaves like the reference's -- no GPU compute is called here."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2311_10090_b200 as m
from paper_2311_10090_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "marl_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(marl_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_native.EXPORTS)


def test_registry_lists_hot_path_ids():
    ids = m.registered_envs()
    assert ids == sorted(ids)
    for need in ["MPE_simple_spread_v3", "SMAX_2s3z", "SMAX_27m_vs_30m", "overcooked_cramped_room_v0"]:
        assert need in ids
    assert len([i for i in ids if i.startswith("SMAX_")]) == 11  # smax.cpp:38-41


@pytest.mark.parametrize("env_id,cfg,A,D,nact", [
    ("MPE_simple_spread_v3", {}, 3, 18, 5),                   # test_mpe.cpp:53-64
    ("MPE_simple_speaker_listener_v4", {}, 2, 11, 5),         # test_mpe.cpp:66-74
    ("MPE_simple_tag_v3", {}, 4, 16, 5),                      # test_mpe.cpp:76-84
    ("SMAX_2s3z", {}, 5, 10 + 17 * 9, 10),                    # test_smax.cpp:88-101
    ("SMAX_5m_vs_6m", {"enemy_controlled": True, "max_steps": 7}, 11, 10 + 17 * 10, 11),
    ("SMAX_5m_vs_6m", {"ally_units": ["marine"] * 3, "enemy_units": ["marine"] * 3}, 3, 95, 8),
    ("SMAX_27m_vs_30m", {}, 27, 962, 35),
    ("overcooked_cramped_room_v0", {}, 2, 541, 6),
])
def test_spaces_match_reference(env_id, cfg, A, D, nact):
    e = m.make_env(env_id, cfg)
    assert e.num_agents() == A and e.obs_dim == D and e.n_actions_max == nact
    assert e.id() == env_id


def test_agent_names_and_flags():
    e = m.make_env("MPE_simple_tag_v3")
    assert e.agents() == ["adversary_0", "adversary_1", "adversary_2", "agent_0"]
    assert e.observation_space("agent_0").flat_size() == 14 and not e.cooperative()
    assert m.make_env("MPE_simple_tag_v3", {"cooperative_prey_reward": True}).cooperative()
    s = m.make_env("MPE_simple_speaker_listener_v4")
    assert s.action_space("speaker_0").n == 3 and s.observation_space("speaker_0").flat_size() == 3
    e2 = m.make_env("SMAX_5m_vs_6m", {"enemy_controlled": True})
    assert e2.agents()[5] == "enemy_0" and e2.action_space("enemy_3").n == 10 and not e2.cooperative()
    with pytest.raises(m.ContractError):
        e.observation_space("nobody")


@pytest.mark.parametrize("env_id,cfg,exc", [
    ("SMAX_2s3z", {"max_steps": 0}, m.SchemaError),             # test_smax.cpp:611-642
    ("SMAX_2s3z", {"map_size": 2.0}, m.SchemaError),
    ("SMAX_2s3z", {"spawn_jitter": -0.5}, m.SchemaError),
    ("SMAX_2s3z", {"wibble": 1}, m.SchemaError),
    ("SMAX_2s3z", {"ally_units": ["ghost"]}, m.SchemaError),
    ("SMAX_2s3z", {"ally_units": ["marine", 3]}, m.SchemaError),
    ("SMAX_2s3z", {"unit_stats": 5}, m.SchemaError),
    ("SMAX_smacv2_5_units", {"ally_units": ["marine"]}, m.SchemaError),
    ("SMAX_2s3z", {"unit_stats": {"marine": {"helth": 1}}}, m.SchemaError),
    ("SMAX_2s3z", {"unit_stats": {"ghoul": {"health": 1}}}, m.SchemaError),
    ("SMAX_2s3z", {"unit_stats": {"marine": {"health": 0}}}, m.SchemaError),
    ("MPE_simple_spread_v3", {"bogus": 1}, m.SchemaError),       # test_mpe.cpp:63
    ("MPE_simple_spread_v3", {"cooperative_prey_reward": True}, m.SchemaError),
    ("overcooked_cramped_room_v0", {"max_steps": 0}, m.SchemaError),
    ("overcooked_cramped_room_v0", {"layout": "XX\nXX\n"}, m.SchemaError),
    ("overcooked_cramped_room_v0", {"layout": "XXXX\nX1 X\nXXXX\n"}, m.SchemaError),
    ("overcooked_cramped_room_v0", {"layout": "XXPXX\nO  2O\n 1  X\nXDXSX\n"}, m.SchemaError),
    ("nope_v0", {}, m.NotFoundError),
    ("MPE_simple_v3", {}, m.NotFoundError),                      # reserved ids, registry.cpp:90-92
    ("hanabi_v0", {}, m.NotFoundError),
])
def test_config_errors(env_id, cfg, exc):
    with pytest.raises(exc):
        m.make_env(env_id, cfg)


def test_stat_override_and_roster_accepted():
    e = m.make_env("SMAX_5m_vs_6m", {"ally_units": ["marine"], "enemy_units": ["marine"], "map_size": 8.0,
                                     "unit_stats": {"marine": {"health": 90.0, "damage": 9.0}}})
    assert e.num_agents() == 1 and e.obs_dim == 27
    e = m.make_env("SMAX_smacv2_5_units", {"ally_units": ["stalker"] * 5, "enemy_units": ["zealot"] * 5})
    assert e.num_agents() == 5


def test_host_prng_helpers_match_oracle():
    for seed in [0, 1, 2027, 2**40 + 3]:
        k = m.prng.key_from_seed(seed)
        assert np.array_equal(k, O.key_from_seed(seed))
        assert np.array_equal(m.prng.split(k, 7), O.split(k, 7))
        assert np.array_equal(m.prng.fold_in(k, 123), O.fold_in(k, 123))
        assert m.prng.bits(k, 5) == O.bits(k, 5)
    assert m.prng.threefry2x32(0, 0, 0, 0) == (0x6B200159, 0x99BA4EFE)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(m.CudaError):
        m.VectorEnv("MPE_simple_spread_v3", 4)
