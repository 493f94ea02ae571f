"""TEST INFRASTRUCTURE ONLY -- ctypes front-ends for the two CPU checkers.

* ``PortVenv``: the plain-C restatement ``oracle/liboracle_port.so``
  (``marl_oracle.c``) of the reference's VectorEnv hot path.
* ``RefVenv``: the UNMODIFIED reference library compiled under ``oracle/_ref``
  (``libmarl_ref.so``, see oracle/Makefile) driven through ``ref_driver.cpp``.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module.  The product package never does.

``resolve_params`` restates the reference's env factories
(registry.cpp:39-66, mpe.cpp:396-402, smax.cpp:65-146, overcooked.cpp:163-179)
independently of the product's C++ config parser, so a product config bug
cannot hide behind a shared resolver.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle_port.so")
REF_SO = os.path.join(HERE, "_ref", "libmarl_ref.so")

MPE, SMAX, OVERCOOKED = 0, 1, 2

# smax.cpp:26-33 -- health, damage, cooldown, speed, sight, range, radius
SMAX_STATS = [
    [45.0, 6.0, 0.61, 3.15, 9.0, 5.0, 0.375],
    [160.0, 13.0, 1.34, 4.13, 9.0, 6.0, 0.625],
    [150.0, 16.0, 0.86, 3.15, 9.0, 0.1, 0.5],
    [80.0, 12.0, 0.59, 3.15, 9.0, 5.0, 0.625],
    [35.0, 5.0, 0.497, 4.13, 9.0, 0.1, 0.375],
    [125.0, 10.0, 1.07, 3.15, 9.0, 6.0, 0.5625],
]
SMAX_TYPES = ["marine", "stalker", "zealot", "hydralisk", "zergling", "marauder"]
SMAX_STAT_KEYS = ["health", "damage", "cooldown", "speed", "sight", "range", "radius"]


def _roster(m=0, s=0, z=0, h=0, l=0):  # smax.cpp:43-51: stalkers, zealots, marines, hydras, lings
    return [1] * s + [2] * z + [0] * m + [3] * h + [4] * l


SMAX_SCENARIOS = {  # smax.cpp:66-97
    "2s3z": (_roster(s=2, z=3), None),
    "3s5z": (_roster(s=3, z=5), None),
    "5m_vs_6m": (_roster(m=5), _roster(m=6)),
    "10m_vs_11m": (_roster(m=10), _roster(m=11)),
    "27m_vs_30m": (_roster(m=27), _roster(m=30)),
    "3s5z_vs_3s6z": (_roster(s=3, z=5), _roster(s=3, z=6)),
    "3s_vs_5z": (_roster(s=3), _roster(l=5)),
    "6h_vs_8z": (_roster(h=6), _roster(l=8)),
}

OVERCOOKED_LAYOUTS = {  # overcooked.cpp:28-58
    "cramped_room": "XXPXX\nO  2O\nX1  X\nXDXSX\n",
    "asymmetric_advantages": "XXXXXXXXX\nO XSXOX S\nX   P 1 X\nX 2 P   X\nXXXDXDXXX\n",
    "coordination_ring": "XXXPX\nX 1 P\nD2X X\nO   X\nXOSXX\n",
    "forced_coordination": "XXXPX\nO X1P\nO2X X\nD X X\nXXXSX\n",
    "counter_circuit": "XXXPPXXX\nX 1    X\nD XXXX S\nX     2X\nXXXOOXXX\n",
}


class OrcParams(C.Structure):
    _fields_ = [
        ("family", C.c_int),
        ("mpe_scenario", C.c_int),
        ("mpe_coop_prey", C.c_int),
        ("smax_n_ally", C.c_int),
        ("smax_n_enemy", C.c_int),
        ("smax_types", C.c_int8 * 128),
        ("smax_stats", (C.c_double * 7) * 6),
        ("smax_map", C.c_double),
        ("smax_jitter", C.c_double),
        ("smax_max_steps", C.c_int),
        ("smax_enemy_controlled", C.c_int),
        ("oc_layout", C.c_char * 512),
        ("oc_max_steps", C.c_int),
        ("oc_cook_time", C.c_int),
        ("oc_delivery_reward", C.c_double),
        ("oc_shaping_onion", C.c_double),
        ("oc_shaping_plate", C.c_double),
        ("oc_shaping_soup", C.c_double),
        ("oc_random_conflicts", C.c_int),
    ]


class OracleConfigError(ValueError):
    pass


def _take(cfg, key, default, kind):
    if key not in cfg:
        return default
    v = cfg.pop(key)
    if kind is bool and not isinstance(v, bool):
        raise OracleConfigError(key)
    if kind is int and (isinstance(v, bool) or not isinstance(v, int)):
        raise OracleConfigError(key)
    if kind is float and (isinstance(v, bool) or not isinstance(v, (int, float))):
        raise OracleConfigError(key)
    return kind(v) if kind is not list else list(v)


def resolve_params(env_id: str, config=None) -> OrcParams:
    cfg = dict(config or {})
    p = OrcParams()
    if env_id in ("MPE_simple_spread_v3", "MPE_simple_speaker_listener_v4", "MPE_simple_tag_v3"):
        p.family = MPE
        p.mpe_scenario = {"MPE_simple_spread_v3": 0, "MPE_simple_speaker_listener_v4": 1,
                          "MPE_simple_tag_v3": 2}[env_id]
        if _take(cfg, "continuous_actions", False, bool):
            raise OracleConfigError("continuous_actions unsupported by the oracle port")
        if p.mpe_scenario == 2:
            p.mpe_coop_prey = int(_take(cfg, "cooperative_prey_reward", False, bool))
    elif env_id.startswith("SMAX_"):
        scen = env_id[5:]
        if scen not in SMAX_SCENARIOS:
            raise OracleConfigError("unsupported SMAX scenario for the oracle: " + scen)
        ally, enemy = SMAX_SCENARIOS[scen]
        enemy = enemy if enemy is not None else ally
        p.family = SMAX
        p.smax_max_steps = _take(cfg, "max_steps", 100, int)
        p.smax_map = _take(cfg, "map_size", 32.0, float)
        p.smax_enemy_controlled = int(_take(cfg, "enemy_controlled", False, bool))
        p.smax_jitter = _take(cfg, "spawn_jitter", 0.5, float)
        ao = cfg.pop("ally_units", None)
        eo = cfg.pop("enemy_units", None)
        stats = [row[:] for row in SMAX_STATS]
        for tname, over in (cfg.pop("unit_stats", None) or {}).items():
            t = SMAX_TYPES.index(tname)
            for k, val in over.items():
                stats[t][SMAX_STAT_KEYS.index(k)] = float(val)
        if ao:
            ally = [SMAX_TYPES.index(x) for x in ao]
        if eo:
            enemy = [SMAX_TYPES.index(x) for x in eo]
        p.smax_n_ally = len(ally)
        p.smax_n_enemy = len(enemy)
        for i, t in enumerate(ally + enemy):
            p.smax_types[i] = t
        for t in range(6):
            for k in range(7):
                p.smax_stats[t][k] = stats[t][k]
    elif env_id.startswith("overcooked_") and env_id.endswith("_v0"):
        name = env_id[len("overcooked_"):-3]
        if name not in OVERCOOKED_LAYOUTS:
            raise OracleConfigError("unknown layout " + name)
        p.family = OVERCOOKED
        text = _take(cfg, "layout", "", str) or OVERCOOKED_LAYOUTS[name]
        p.oc_layout = text.encode()
        p.oc_max_steps = _take(cfg, "max_steps", 400, int)
        p.oc_cook_time = _take(cfg, "cook_time", 20, int)
        p.oc_delivery_reward = _take(cfg, "delivery_reward", 20.0, float)
        p.oc_shaping_onion = _take(cfg, "shaping_onion", 3.0, float)
        p.oc_shaping_plate = _take(cfg, "shaping_plate", 3.0, float)
        p.oc_shaping_soup = _take(cfg, "shaping_soup", 5.0, float)
        p.oc_random_conflicts = int(_take(cfg, "random_conflict_resolution", False, bool))
    else:
        raise OracleConfigError("env id not covered by the oracle: " + env_id)
    if cfg:
        raise OracleConfigError("unknown keys " + ",".join(cfg))
    return p


_P = C.POINTER
_u32p, _f32p, _f64p, _u8p, _i32p, _u64p = (_P(C.c_uint32), _P(C.c_float), _P(C.c_double),
                                         _P(C.c_uint8), _P(C.c_int32), _P(C.c_uint64))


def _ptr(a, ct):
    return None if a is None else a.ctypes.data_as(_P(ct))


def _key(k):
    return np.ascontiguousarray(np.asarray(k, dtype=np.uint32).reshape(4))


_port = None


def port_lib():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            raise RuntimeError("oracle port not built: run `make -C oracle port`")
        L = C.CDLL(PORT_SO)
        L.orc_create.argtypes = [_P(OrcParams), C.c_int64, C.c_int64, C.c_int64, _P(C.c_void_p)]
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_spec.argtypes = [C.c_void_p] + [_P(C.c_int)] * 4
        L.orc_last_error.restype = C.c_char_p
        L.orc_reset.argtypes = [C.c_void_p, _u32p, _f32p]
        L.orc_random_actions.argtypes = [C.c_void_p, _u32p, _i32p]
        L.orc_legal.argtypes = [C.c_void_p, _u8p]
        L.orc_step.argtypes = [C.c_void_p, _i32p, _f32p, _f64p, _u8p, _u8p, _f32p, _f64p, _i32p, _f64p]
        L.orc_keys.argtypes = [C.c_void_p, _u32p]
        L.orc_episode.argtypes = [C.c_void_p, _f64p, _i32p]
        L.orc_state_hash.argtypes = [C.c_void_p, _u64p]
        L.orc_smax_units.argtypes = [C.c_void_p, C.c_int64] + [_f64p] * 4
        L.orc_smax_winner.argtypes = [C.c_void_p, C.c_int64]
        L.orc_threefry.argtypes = [C.c_uint32] * 4 + [_u32p]
        L.orc_split.argtypes = [_u32p, C.c_uint64, _u32p]
        L.orc_split_child.argtypes = [_u32p, C.c_uint64, _u32p]
        L.orc_fold_in.argtypes = [_u32p, C.c_uint64, _u32p]
        L.orc_bits.argtypes = [_u32p, C.c_uint64]
        L.orc_bits.restype = C.c_uint64
        L.orc_uniform1.argtypes = [_u32p, C.c_double, C.c_double]
        L.orc_uniform1.restype = C.c_double
        _port = L
    return _port


# --------------------------------------------------------------- PRNG helpers
def key_from_seed(seed: int):
    """prng.cpp:116-118"""
    return np.array([seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF, 0, 0], dtype=np.uint32)


def threefry(k0, k1, x0, x1):
    y = np.zeros(2, np.uint32)
    port_lib().orc_threefry(k0, k1, x0, x1, _ptr(y, C.c_uint32))
    return int(y[0]), int(y[1])


def split(key, n):
    out = np.zeros((n, 4), np.uint32)
    port_lib().orc_split(_ptr(_key(key), C.c_uint32), n, _ptr(out, C.c_uint32))
    return out


def fold_in(key, d):
    out = np.zeros(4, np.uint32)
    port_lib().orc_fold_in(_ptr(_key(key), C.c_uint32), d, _ptr(out, C.c_uint32))
    return out


def bits(key, i):
    return int(port_lib().orc_bits(_ptr(_key(key), C.c_uint32), i))


class StepOut(dict):
    """Flattened VectorEnv::step outputs (same layout as the B200 C-ABI views)."""


def _alloc_step(n, A, D, n_info):
    return StepOut(
        obs=np.zeros((n, A, D), np.float32), rewards=np.zeros((n, A), np.float64),
        dones=np.zeros((n, A + 1), np.uint8), finished=np.zeros(n, np.uint8),
        final_obs=np.zeros((n, A, D), np.float32), final_returns=np.zeros(n, np.float64),
        final_lengths=np.zeros(n, np.int32), infos=np.zeros((n, A, max(n_info, 1)), np.float64))


class PortVenv:
    """The C restatement as a batched env (shardable by global index)."""

    def __init__(self, env_id, config=None, n_envs=1, global_offset=0, global_n=None):
        L = port_lib()
        self.params = resolve_params(env_id, config)
        self.n = n_envs
        gn = n_envs if global_n is None else global_n
        h = C.c_void_p()
        rc = L.orc_create(C.byref(self.params), n_envs, global_offset, gn, C.byref(h))
        if rc:
            raise RuntimeError(f"orc_create rc={rc}: {L.orc_last_error().decode()}")
        self.h = h
        a, d, na, ni = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        L.orc_spec(h, C.byref(a), C.byref(d), C.byref(na), C.byref(ni))
        self.n_agents, self.obs_dim, self.n_actions, self.n_info = a.value, d.value, na.value, ni.value

    def __del__(self):
        if getattr(self, "h", None):
            port_lib().orc_destroy(self.h)
            self.h = None

    def _chk(self, rc):
        if rc:
            raise RuntimeError(f"oracle rc={rc}: {port_lib().orc_last_error().decode()}")

    def reset(self, key):
        obs = np.zeros((self.n, self.n_agents, self.obs_dim), np.float32)
        self._chk(port_lib().orc_reset(self.h, _ptr(_key(key), C.c_uint32), _ptr(obs, C.c_float)))
        return obs

    def random_actions(self, step_key):
        act = np.zeros((self.n, self.n_agents), np.int32)
        self._chk(port_lib().orc_random_actions(self.h, _ptr(_key(step_key), C.c_uint32),
                                                _ptr(act, C.c_int32)))
        return act

    def legal(self):
        m = np.zeros((self.n, self.n_agents, self.n_actions), np.uint8)
        self._chk(port_lib().orc_legal(self.h, _ptr(m, C.c_uint8)))
        return m

    def step(self, actions):
        actions = np.ascontiguousarray(actions, dtype=np.int32)
        o = _alloc_step(self.n, self.n_agents, self.obs_dim, self.n_info)
        self._chk(port_lib().orc_step(
            self.h, _ptr(actions, C.c_int32), _ptr(o["obs"], C.c_float), _ptr(o["rewards"], C.c_double),
            _ptr(o["dones"], C.c_uint8), _ptr(o["finished"], C.c_uint8), _ptr(o["final_obs"], C.c_float),
            _ptr(o["final_returns"], C.c_double), _ptr(o["final_lengths"], C.c_int32),
            _ptr(o["infos"], C.c_double)))
        o["infos"] = o["infos"][:, :, : self.n_info]
        o.update(self.batch_state())
        return o

    def step_random(self, step_key):
        a = self.random_actions(step_key)
        o = self.step(a)
        o["actions"] = a
        return o

    def batch_state(self):
        keys = np.zeros((self.n, 4), np.uint32)
        ret = np.zeros(self.n, np.float64)
        ln = np.zeros(self.n, np.int32)
        hs = np.zeros(self.n, np.uint64)
        L = port_lib()
        L.orc_keys(self.h, _ptr(keys, C.c_uint32))
        L.orc_episode(self.h, _ptr(ret, C.c_double), _ptr(ln, C.c_int32))
        L.orc_state_hash(self.h, _ptr(hs, C.c_uint64))
        return dict(keys=keys, episode_returns=ret, episode_lengths=ln, state_hash=hs)

    def smax_units(self, env=0):
        U = self.params.smax_n_ally + self.params.smax_n_enemy
        arrs = [np.zeros(U, np.float64) for _ in range(4)]
        self._chk(port_lib().orc_smax_units(self.h, env, *[_ptr(a, C.c_double) for a in arrs]))
        return dict(zip(["x", "y", "health", "cooldown"], arrs))

    def smax_winner(self, env=0):
        return int(port_lib().orc_smax_winner(self.h, env))


# ------------------------------------------------------- compiled reference
_ref = None


def ref_available():
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError("reference not built: run `make -C oracle ref` (needs /root/reference)")
        L = C.CDLL(REF_SO)
        L.mref_last_error.restype = C.c_char_p
        L.mref_create.argtypes = [C.c_char_p, C.c_char_p, C.c_int, _P(C.c_void_p)]
        L.mref_destroy.argtypes = [C.c_void_p]
        L.mref_spec.argtypes = [C.c_void_p] + [_P(C.c_int)] * 3
        L.mref_set_threads.argtypes = [C.c_int]
        L.mref_reset.argtypes = [C.c_void_p, _u32p, _f32p, _u32p, _u64p]
        L.mref_legal.argtypes = [C.c_void_p, _u8p]
        L.mref_world_state.argtypes = [C.c_void_p, _f32p, _P(C.c_int)]
        L.mref_random_actions.argtypes = [C.c_void_p, _u32p, _i32p]
        L.mref_random_actions_box.argtypes = [C.c_void_p, _u32p, C.c_int, _f32p]
        L.mref_step.argtypes = [C.c_void_p, _i32p, _f32p, _f64p, _u8p, _u8p, _f32p, _f64p, _i32p,
                                _f64p, C.c_int, _f64p, _i32p, _u32p, _u64p]
        L.mref_step_box.argtypes = [C.c_void_p, _f32p, C.c_int, _f32p, _f64p, _u8p, _u8p, _f32p, _f64p, _i32p,
                                    _f64p, C.c_int, _f64p, _i32p, _u32p, _u64p]
        L.mref_probe.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, _u32p, _f64p, _f64p]
        L.mref_threefry.argtypes = [C.c_uint32] * 4 + [_u32p]
        L.mref_split.argtypes = [_u32p, C.c_uint64, _u32p]
        L.mref_fold_in.argtypes = [_u32p, C.c_uint64, _u32p]
        L.mref_hypot.argtypes = [C.c_double, C.c_double]
        L.mref_hypot.restype = C.c_double
        L.mref_rollout_last_error.restype = C.c_char_p
        L.mref_ppo_spec.argtypes = [C.c_char_p, C.c_char_p, C.c_int] + [_P(C.c_int)] * 5
        L.mref_ppo_init.argtypes = [C.c_char_p, C.c_char_p, C.c_int, _u32p, _f32p, _f32p]
        L.mref_collect.argtypes = [C.c_char_p, C.c_char_p, C.c_int, _f32p, C.c_int, C.c_int, C.c_int, _u32p,
                                   _f32p, _f32p,
                                   C.c_double, C.c_double, C.c_double, _f32p, _i32p, _f32p, _u8p, _u8p, _f32p,
                                   _f32p, _u8p, _f32p, _f32p, _f32p, _f64p, _P(C.c_int64)]
        L.mref_permutation.argtypes = [_u32p, C.c_int, _i32p]
        L.mref_ppo_init_rnn.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_int, _u32p, _f32p, _f32p,
                                        _P(C.c_int), _P(C.c_int)]
        L.mref_ff_minibatch.argtypes = [C.c_char_p, C.c_char_p, C.c_int, _f32p, _f32p, _f32p, _f32p, _i32p, _f32p,
                                        _f32p, _f32p, _f32p, _f32p, _u8p, _i32p, C.c_int, C.c_double, C.c_double,
                                        C.c_double, _f32p, _f64p]
        L.mref_train.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, _u32p, _f64p, C.c_int,
                                 _P(C.c_int), _f32p, _P(C.c_int), _f32p, _P(C.c_int), _P(C.c_int), _P(C.c_int64)]
        _ref = L
    return _ref


N_INFO = {MPE: 0, SMAX: 3, OVERCOOKED: 2}


class RefVenv:
    """marl::VectorEnv from the compiled reference, flattened like the C-ABI."""

    def __init__(self, env_id, config=None, n_envs=1):
        L = ref_lib()
        h = C.c_void_p()
        rc = L.mref_create(env_id.encode(), json.dumps(config or {}).encode(), n_envs, C.byref(h))
        if rc:
            raise RuntimeError(f"mref_create rc={rc}: {L.mref_last_error().decode()}")
        self.h = h
        self.n = n_envs
        a, d, na = C.c_int(), C.c_int(), C.c_int()
        L.mref_spec(h, C.byref(a), C.byref(d), C.byref(na))
        self.n_agents, self.obs_dim, self.n_actions = a.value, d.value, na.value
        fam = MPE if env_id.startswith("MPE") else SMAX if env_id.startswith("SMAX") else OVERCOOKED
        self.n_info = N_INFO[fam]
        self.keys = np.zeros((n_envs, 4), np.uint32)
        self.hash = np.zeros(n_envs, np.uint64)

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().mref_destroy(self.h)
            self.h = None

    def _chk(self, rc):
        if rc:
            raise RuntimeError(f"reference rc={rc}: {ref_lib().mref_last_error().decode()}")

    def reset(self, key):
        obs = np.zeros((self.n, self.n_agents, self.obs_dim), np.float32)
        self._chk(ref_lib().mref_reset(self.h, _ptr(_key(key), C.c_uint32), _ptr(obs, C.c_float),
                                       _ptr(self.keys, C.c_uint32), _ptr(self.hash, C.c_uint64)))
        return obs

    def random_actions(self, step_key):
        act = np.zeros((self.n, self.n_agents), np.int32)
        self._chk(ref_lib().mref_random_actions(self.h, _ptr(_key(step_key), C.c_uint32),
                                                _ptr(act, C.c_int32)))
        return act

    def legal(self):
        m = np.zeros((self.n, self.n_agents, self.n_actions), np.uint8)
        self._chk(ref_lib().mref_legal(self.h, _ptr(m, C.c_uint8)))
        return m

    def world_state(self):
        """Env::world_state of every env's current state, [N][W] f32."""
        w = C.c_int()
        self._chk(ref_lib().mref_world_state(self.h, None, C.byref(w)))
        out = np.zeros((self.n, w.value), np.float32)
        self._chk(ref_lib().mref_world_state(self.h, _ptr(out, C.c_float), C.byref(w)))
        return out

    BOX_DIM = 5  # the engine's padded box-action row (continuous MPE)

    def random_actions_box(self, step_key):
        act = np.zeros((self.n, self.n_agents, self.BOX_DIM), np.float32)
        self._chk(ref_lib().mref_random_actions_box(self.h, _ptr(_key(step_key), C.c_uint32), self.BOX_DIM,
                                                    _ptr(act, C.c_float)))
        return act

    def step(self, actions):
        actions = np.asarray(actions)
        box = actions.dtype.kind == "f"
        actions = np.ascontiguousarray(actions, dtype=np.float32 if box else np.int32)
        o = _alloc_step(self.n, self.n_agents, self.obs_dim, self.n_info)
        ret = np.zeros(self.n, np.float64)
        ln = np.zeros(self.n, np.int32)
        fn = ref_lib().mref_step_box if box else ref_lib().mref_step
        head = [self.h, _ptr(actions, C.c_float), self.BOX_DIM] if box else [self.h, _ptr(actions, C.c_int32)]
        self._chk(fn(
            *head, _ptr(o["obs"], C.c_float), _ptr(o["rewards"], C.c_double),
            _ptr(o["dones"], C.c_uint8), _ptr(o["finished"], C.c_uint8), _ptr(o["final_obs"], C.c_float),
            _ptr(o["final_returns"], C.c_double), _ptr(o["final_lengths"], C.c_int32),
            _ptr(o["infos"], C.c_double), self.n_info, _ptr(ret, C.c_double), _ptr(ln, C.c_int32),
            _ptr(self.keys, C.c_uint32), _ptr(self.hash, C.c_uint64)))
        o["infos"] = o["infos"][:, :, : self.n_info]
        o.update(keys=self.keys.copy(), episode_returns=ret, episode_lengths=ln,
                 state_hash=self.hash.copy())
        return o

    def step_random(self, step_key):
        a = self.random_actions(step_key)
        o = self.step(a)
        o["actions"] = a
        return o


def ref_probe(env_id, config, n_envs, n_steps, key, threads=None):
    """throughput_probe (vector_env.cpp:191-222) of the compiled reference."""
    L = ref_lib()
    if threads:
        L.mref_set_threads(int(threads))
    s, cold = C.c_double(), C.c_double()
    rc = L.mref_probe(env_id.encode(), json.dumps(config or {}).encode(), n_envs, n_steps,
                      _ptr(_key(key), C.c_uint32), C.byref(s), C.byref(cold))
    if rc:
        raise RuntimeError(f"probe rc={rc}: {L.mref_last_error().decode()}")
    return s.value, cold.value


# --------------------------------------------------------- IPPO rollout (C5)
def ref_ppo_spec(env_id, config=None, centralized=False):
    """ppo_net_spec + packed parameter counts from the reference (ppo.cpp:80-124);
    centralized: the MAPPO critic on world_state (train_mappo, ppo.hpp:99)."""
    L = ref_lib()
    v = [C.c_int() for _ in range(5)]
    rc = L.mref_ppo_spec(env_id.encode(), json.dumps(config or {}).encode(), int(centralized),
                         *[C.byref(x) for x in v])
    if rc:
        raise RuntimeError(L.mref_rollout_last_error().decode())
    return {"in_dim": v[0].value, "critic_in": v[1].value, "n_actions": v[2].value, "n_actor": v[3].value,
            "n_critic": v[4].value}


def ref_ppo_init(env_id, config, key, centralized=False):
    """ppo_init_nets(key, spec) packed (pack_actor, pack_critic)."""
    L = ref_lib()
    sp = ref_ppo_spec(env_id, config, centralized)
    a = np.zeros(sp["n_actor"], np.float32)
    c = np.zeros(sp["n_critic"], np.float32)
    rc = L.mref_ppo_init(env_id.encode(), json.dumps(config or {}).encode(), int(centralized),
                         _ptr(_key(key), C.c_uint32), _ptr(a, C.c_float), _ptr(c, C.c_float))
    if rc:
        raise RuntimeError(L.mref_rollout_last_error().decode())
    return a, c


def ref_collect(env_id, config, n_envs, T, key, actor, critic, n_windows=1, gamma=0.99, lam=1.0, shaping=0.0,
                centralized=False):
    """The reference Collector (restated over its public pieces, ref_rollout.cpp):
    buffers of the last window, [T][R]."""
    L = ref_lib()
    sp = ref_ppo_spec(env_id, config, centralized)
    v = RefVenv(env_id, config, 1)  # agents per env (TeamLayout rows)
    A = v.n_agents
    R = n_envs * A
    out = {"obs": np.zeros((T, R, sp["in_dim"]), np.float32), "actions": np.zeros((T, R), np.int32),
           "rewards": np.zeros((T, R), np.float32), "dones": np.zeros((T, R), np.uint8),
           "resets": np.zeros((T, R), np.uint8), "logp": np.zeros((T, R), np.float32),
           "value": np.zeros((T, R), np.float32), "legal": np.zeros((T, R, sp["n_actions"]), np.uint8),
           "active": np.zeros((T, R), np.float32), "adv": np.zeros((T, R), np.float32),
           "vtarg": np.zeros((T, R), np.float32), "critic_in": np.zeros((T, R, sp["critic_in"]), np.float32)}
    ep_sum = C.c_double()
    eps = C.c_int64()
    a = np.ascontiguousarray(actor, np.float32)
    c = np.ascontiguousarray(critic, np.float32)
    rc = L.mref_collect(env_id.encode(), json.dumps(config or {}).encode(), int(centralized),
                        _ptr(out["critic_in"], C.c_float), n_envs, T, n_windows,
                        _ptr(_key(key), C.c_uint32), _ptr(a, C.c_float), _ptr(c, C.c_float), gamma, lam, shaping,
                        _ptr(out["obs"], C.c_float), _ptr(out["actions"], C.c_int32), _ptr(out["rewards"], C.c_float),
                        _ptr(out["dones"], C.c_uint8), _ptr(out["resets"], C.c_uint8), _ptr(out["logp"], C.c_float),
                        _ptr(out["value"], C.c_float), _ptr(out["legal"], C.c_uint8), _ptr(out["active"], C.c_float),
                        _ptr(out["adv"], C.c_float), _ptr(out["vtarg"], C.c_float), C.byref(ep_sum), C.byref(eps))
    if rc:
        raise RuntimeError(L.mref_rollout_last_error().decode())
    out["episode_return_sum"] = ep_sum.value
    out["episodes"] = eps.value
    return out


# ------------------------------------------------------------- PPO update
PPO_COLUMNS = ["step", "update", "mean_return", "n_episodes", "loss", "pg_loss", "v_loss", "entropy", "approx_kl",
               "clip_frac", "grad_norm", "lr"]


def ref_permutation(key, n):
    """prng::permutation(key, n) (prng.cpp:151-159)."""
    L = ref_lib()
    out = np.zeros(max(n, 1), np.int32)
    rc = L.mref_permutation(_ptr(_key(key), C.c_uint32), int(n), _ptr(out, C.c_int32))
    if rc:
        raise RuntimeError(L.mref_rollout_last_error().decode())
    return out[:n]


def ref_ff_minibatch(env_id, config, actor, critic, buf, idx, clip_eps=0.3, ent_coef=0.01, vf_coef=1.0,
                     centralized=False):
    """ff_minibatch (ppo.cpp:409-441) over a [T][R] buffer dict -> (flat grad, stats[6])."""
    L = ref_lib()
    sp = ref_ppo_spec(env_id, config, centralized)
    g = np.zeros(sp["n_actor"] + sp["n_critic"], np.float32)
    st = np.zeros(6, np.float64)
    f = {k: np.ascontiguousarray(buf[k]) for k in ("obs", "actions", "logp", "adv", "vtarg", "value", "active",
                                                    "legal")}
    ci = np.ascontiguousarray(buf.get("critic_in", f["obs"]), np.float32)
    ix = np.ascontiguousarray(idx, np.int32)
    a = np.ascontiguousarray(actor, np.float32)
    c = np.ascontiguousarray(critic, np.float32)
    rc = L.mref_ff_minibatch(env_id.encode(), json.dumps(config or {}).encode(), int(centralized),
                             _ptr(a, C.c_float), _ptr(c, C.c_float), _ptr(f["obs"], C.c_float), _ptr(ci, C.c_float),
                             _ptr(f["actions"], C.c_int32), _ptr(f["logp"], C.c_float), _ptr(f["adv"], C.c_float),
                             _ptr(f["vtarg"], C.c_float), _ptr(f["value"], C.c_float), _ptr(f["active"], C.c_float),
                             _ptr(f["legal"], C.c_uint8), _ptr(ix, C.c_int32), len(ix), clip_eps, ent_coef, vf_coef,
                             _ptr(g, C.c_float), _ptr(st, C.c_double))
    if rc:
        raise RuntimeError(L.mref_rollout_last_error().decode())
    return g, st


def ref_train(env_id, config, ppo_config, key, centralized=False, max_rows=4096):
    """The reference's train_ippo / train_mappo (ppo.cpp:518-651)."""
    L = ref_lib()
    m = np.zeros((max_rows, 12), np.float64)
    a = np.zeros(1 << 20, np.float32)  # capacities; the reference reports the true sizes
    c = np.zeros(1 << 20, np.float32)
    na, nc = C.c_int(a.size), C.c_int(c.size)
    nr, dv, sd = C.c_int(), C.c_int(), C.c_int64()
    rc = L.mref_train(env_id.encode(), json.dumps(config or {}).encode(), json.dumps(ppo_config).encode(),
                      int(centralized), _ptr(_key(key), C.c_uint32), _ptr(m, C.c_double), max_rows, C.byref(nr),
                      _ptr(a, C.c_float), C.byref(na), _ptr(c, C.c_float), C.byref(nc), C.byref(dv), C.byref(sd))
    if rc:
        raise RuntimeError(L.mref_rollout_last_error().decode())
    if na.value > a.size or nc.value > c.size:
        raise RuntimeError("ref_train: parameter buffers too small")
    a, c = a[: na.value].copy(), c[: nc.value].copy()
    return {"metrics": m[:nr.value], "actor": a, "critic": c, "diverged": bool(dv.value), "steps_done": sd.value}


def ref_ppo_init_rnn(env_id, config, key, fc_width=64, hidden_width=128, centralized=False):
    """ppo_init_nets for a recurrent spec, packed (pack_actor, pack_critic)."""
    L = ref_lib()
    na, nc = C.c_int(), C.c_int()
    args = (env_id.encode(), json.dumps(config or {}).encode(), int(centralized), fc_width, hidden_width,
            _ptr(_key(key), C.c_uint32))
    rc = L.mref_ppo_init_rnn(*args, None, None, C.byref(na), C.byref(nc))
    if rc:
        raise RuntimeError(L.mref_rollout_last_error().decode())
    a = np.zeros(na.value, np.float32)
    c = np.zeros(nc.value, np.float32)
    rc = L.mref_ppo_init_rnn(*args, _ptr(a, C.c_float), _ptr(c, C.c_float), C.byref(na), C.byref(nc))
    if rc:
        raise RuntimeError(L.mref_rollout_last_error().decode())
    return a, c
