"""Python mirror of the reference's batched env API over the C-ABI.

Mirrors ``marl::make_env`` / ``registered_envs`` (registry.hpp:16-28),
``marl::Env`` metadata (env.hpp:39-89), ``marl::VectorEnv`` (vector_env.hpp:74-89)
and ``throughput_probe`` (vector_env.hpp:96-99) with the same names, argument
meaning and exception types, so code and tests written against the reference
read the same here.  Per-agent dictionaries are flattened to fixed-width device
arrays (see include/marl_b200.h); results are zero-copy torch views of the
engine's device buffers, valid until the next call on the VectorEnv.

Deliberate difference: the reference's ``BatchedState`` is an immutable value
(step never mutates its input, env.hpp:36-38).  The engine keeps exactly one
live state per VectorEnv in HBM, so ``step`` accepts only the latest state
(``reset``'s or the previous result's ``.next``) and raises ContractError for a
stale one rather than silently copying gigabytes of state.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import Any, Dict, List, Optional, Sequence

import numpy as np

from . import _native as N
from .errors import ContractError


def _cfg(config) -> bytes:
    if config is None:
        return b""
    if isinstance(config, (str, bytes)):
        return config.encode() if isinstance(config, str) else config
    return json.dumps(config).encode()


def _key_arr(key) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(key, dtype=np.uint32).reshape(4))
    return a


def _u32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def registered_envs() -> List[str]:
    """registered_envs() (registry.cpp:99-106): implemented ids, sorted."""
    L = N.lib()
    return [L.marl_registered_env(i).decode() for i in range(L.marl_registered_count())]


@dataclass
class SpaceDescriptor:
    """The subset of SpaceDescriptor (spaces.hpp:13-29) the batched engine uses."""
    kind: str
    n: int = 0
    shape: tuple = ()

    def flat_size(self) -> int:
        return self.n if self.kind == "discrete" else int(np.prod(self.shape))


class Env:
    """make_env(id, config) (registry.cpp:83-97): validated id + config and the
    env's static metadata.  Instances are immutable, like marl::Env."""

    def __init__(self, env_id: str, config: Optional[Dict[str, Any]] = None):
        L = N.lib()
        self._id = env_id
        self.config = dict(config or {}) if not isinstance(config, (str, bytes)) else json.loads(config)
        spec = N.Spec()
        N.check(L.marl_env_describe(env_id.encode(), _cfg(self.config), C.byref(spec)))
        self.family = spec.family
        self._max_steps = spec.max_steps
        self._cooperative = bool(spec.cooperative)
        self.obs_dim = spec.obs_dim
        self.n_actions_max = spec.n_actions
        self.n_info = spec.n_info
        self._agents, self._obs_sizes, self._n_actions = [], [], []
        buf = C.create_string_buffer(128)
        for i in range(spec.n_agents):
            o, a = C.c_int32(), C.c_int32()
            N.check(L.marl_env_agent(env_id.encode(), _cfg(self.config), i, buf, 128, C.byref(o), C.byref(a)))
            self._agents.append(buf.value.decode())
            self._obs_sizes.append(o.value)
            self._n_actions.append(a.value)

    def id(self) -> str:
        return self._id

    def agents(self) -> List[str]:
        return list(self._agents)

    def num_agents(self) -> int:
        return len(self._agents)

    def max_steps(self) -> int:
        return self._max_steps

    def cooperative(self) -> bool:
        return self._cooperative

    def observation_space(self, agent: str) -> SpaceDescriptor:
        return SpaceDescriptor("box", shape=(self._obs_sizes[self._index(agent)],))

    def action_space(self, agent: str) -> SpaceDescriptor:
        return SpaceDescriptor("discrete", n=self._n_actions[self._index(agent)])

    def _index(self, agent: str) -> int:
        try:
            return self._agents.index(agent)
        except ValueError:
            raise ContractError(f"{self._id}: unknown agent '{agent}'") from None


def make_env(env_id: str, config: Optional[Dict[str, Any]] = None) -> Env:
    return Env(env_id, config)


class _DevArray:
    """__cuda_array_interface__ wrapper so torch can view engine buffers zero-copy."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(int(s) for s in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


@dataclass
class BatchedState:
    """Handle on the engine's live BatchedState (vector_env.hpp:13-20)."""
    venv: "VectorEnv"
    version: int
    keys: Any = None              # [N,4] carry keys (int32 view of the u32 words)
    episode_returns: Any = None   # [N] f64
    episode_lengths: Any = None   # [N] i32

    def size(self) -> int:
        return self.venv.n_envs()


@dataclass
class StepBatchResult:
    """StepBatchResult (vector_env.hpp:22-36), flattened; tensors are views."""
    obs: Any
    rewards: Any
    dones: Any
    infos: Any
    finished: Any
    final_obs: Any
    final_returns: Any
    final_lengths: Any
    actions: Any
    next: BatchedState
    info_names: List[str] = field(default_factory=list)


class VectorEnv:
    """VectorEnv(env, n_envs) (vector_env.cpp:45-49) on one CUDA device.

    ``global_offset`` / ``global_n`` make this handle one shard of a multi-GPU
    batch: env i here is global env ``global_offset + i`` and draws exactly the
    keys it would in a single ``global_n``-env VectorEnv."""

    def __init__(self, env, n_envs: int, device: int = 0, global_offset: int = 0,
                 global_n: Optional[int] = None, config=None, stream="torch"):
        if isinstance(env, str):
            env = Env(env, config)
        self._env = env
        self._n = int(n_envs)
        self._device = int(device)
        L = N.lib()
        h = C.c_void_p()
        gn = self._n if global_n is None else int(global_n)
        N.check(L.marl_venv_create_shard(env.id().encode(), _cfg(env.config), self._n, int(global_offset),
                                         gn, self._device, C.byref(h)))
        self._h = h
        self._version = -1
        self.global_offset, self.global_n = int(global_offset), gn
        self._torch = None
        if stream == "torch":
            try:
                import torch
                self._torch = torch
                s = torch.cuda.current_stream(self._device)
                N.check(L.marl_venv_set_stream(self._h, C.c_void_p(s.cuda_stream)))
            except ImportError:
                pass
        elif stream is not None:
            N.check(L.marl_venv_set_stream(self._h, C.c_void_p(int(stream))))
        v = N.Views()
        N.check(L.marl_venv_views(self._h, C.byref(v)))
        self._views = v
        A, D, I = env.num_agents(), env.obs_dim, env.n_info
        n = self._n
        self._shapes = {
            "obs": ((n, A, D), "<f4"), "final_obs": ((n, A, D), "<f4"), "rewards": ((n, A), "<f8"),
            "dones": ((n, A + 1), "|u1"), "finished": ((n,), "|u1"), "final_returns": ((n,), "<f8"),
            "final_lengths": ((n,), "<i4"), "infos": ((n, A, I), "<f8"), "actions": ((n, A), "<i4"),
            "keys": ((n, 4), "<i4"), "episode_returns": ((n,), "<f8"), "episode_lengths": ((n,), "<i4"),
        }
        ad = C.c_int32()
        N.check(L.marl_venv_action_dim(self._h, C.byref(ad)))
        self.action_dim = int(ad.value)  # > 0: box action spaces ([N, A, action_dim] f32 actions)
        if self.action_dim:
            pf = C.POINTER(C.c_float)()
            N.check(L.marl_venv_actions_f32(self._h, C.byref(pf)))
            self._actions_f_ptr = C.cast(pf, C.c_void_p).value
            self._shapes["actions_f"] = ((n, A, self.action_dim), "<f4")
        self.info_names = []
        buf = C.create_string_buffer(64)
        for k in range(I):
            N.check(L.marl_venv_info_name(self._h, k, buf, 64))
            self.info_names.append(buf.value.decode())

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                N.lib().marl_venv_destroy(h)
            except Exception:  # interpreter shutdown: module globals already torn down
                pass
            self._h = None

    # ---- metadata
    def env(self) -> Env:
        return self._env

    def n_envs(self) -> int:
        return self._n

    def spec(self) -> N.Spec:
        s = N.Spec()
        N.check(N.lib().marl_venv_spec(self._h, C.byref(s)))
        return s

    # ---- views
    def view(self, name: str):
        """Zero-copy torch tensor over one engine buffer (the buffers never move
        for the life of the handle, so each view is built once)."""
        cache = self.__dict__.setdefault("_view_cache", {})
        t = cache.get(name)
        if t is None:
            shape, ts = self._shapes[name]
            ptr = self._actions_f_ptr if name == "actions_f" else getattr(self._views, name)
            t = cache[name] = self._torch.as_tensor(_DevArray(ptr, shape, ts), device=f"cuda:{self._device}")
        return t

    def _state(self) -> BatchedState:
        return BatchedState(self, self._version, self.view("keys"), self.view("episode_returns"),
                            self.view("episode_lengths"))

    def _result(self) -> StepBatchResult:
        g = self.view
        return StepBatchResult(g("obs"), g("rewards"), g("dones"), g("infos"), g("finished"), g("final_obs"),
                               g("final_returns"), g("final_lengths"),
                               g("actions_f") if self.action_dim else g("actions"), self._state(),
                               list(self.info_names))

    # ---- hot path
    def reset(self, key):
        """VectorEnv::reset (vector_env.cpp:51-70) -> (obs [N,A,D], BatchedState)."""
        N.check(N.lib().marl_venv_reset(self._h, _u32p(_key_arr(key))))
        self._version += 1
        return self.view("obs"), self._state()

    def _check_state(self, state: Optional[BatchedState]):
        if self._version < 0:
            raise ContractError("VectorEnv::step: call reset() before step()")
        if state is not None and (state.venv is not self or state.version != self._version):
            raise ContractError("VectorEnv::step: stale BatchedState (the engine keeps one live state; "
                                "pass the latest reset()/step().next)")

    def step(self, state: Optional[BatchedState], actions, sync: bool = True) -> StepBatchResult:
        """VectorEnv::step (vector_env.cpp:72-129).  ``actions``: [N, A] int32
        as a CUDA tensor (device path) or anything numpy accepts (host path)."""
        self._check_state(state)
        L = N.lib()
        t = self._torch
        if self.action_dim:
            return self._step_box(actions, sync)
        if t is not None and isinstance(actions, t.Tensor) and actions.is_cuda:
            if tuple(actions.shape) != (self._n, self._env.num_agents()):
                raise ContractError(f"VectorEnv::step: expected actions of shape {(self._n, self._env.num_agents())}")
            a = actions.to(t.int32).contiguous()
            N.check(L.marl_venv_step(self._h, C.c_void_p(a.data_ptr())))
            if sync:
                N.check(L.marl_venv_sync(self._h))
        else:
            a = np.ascontiguousarray(np.asarray(actions, dtype=np.int32))
            if a.shape != (self._n, self._env.num_agents()):
                raise ContractError(f"VectorEnv::step: expected {self._n} action rows of "
                                    f"{self._env.num_agents()} agents, got shape {a.shape}")
            N.check(L.marl_venv_step_host(self._h, C.c_void_p(a.ctypes.data), None))
        self._version += 1
        return self._result()

    def _step_box(self, actions, sync: bool) -> StepBatchResult:
        """Box action spaces: [N, A, action_dim] float32, agent a's first
        n_actions[a] entries in [0, 1] (spaces.cpp:36-46)."""
        L = N.lib()
        t = self._torch
        shape = (self._n, self._env.num_agents(), self.action_dim)
        if t is not None and isinstance(actions, t.Tensor) and actions.is_cuda:
            if tuple(actions.shape) != shape:
                raise ContractError(f"VectorEnv::step: expected box actions of shape {shape}")
            a = actions.to(t.float32).contiguous()
            N.check(L.marl_venv_step_continuous(self._h, C.c_void_p(a.data_ptr())))
            if sync:
                N.check(L.marl_venv_sync(self._h))
        else:
            a = np.ascontiguousarray(np.asarray(actions, dtype=np.float32))
            if a.shape != shape:
                raise ContractError(f"VectorEnv::step: expected box actions of shape {shape}, got {a.shape}")
            N.check(L.marl_venv_step_continuous_host(self._h, C.c_void_p(a.ctypes.data), None))
        self._version += 1
        return self._result()

    def step_random(self, step_key, state: Optional[BatchedState] = None) -> StepBatchResult:
        """random_legal_actions(state, step_key) + VectorEnv::step, fused
        (vector_env.cpp:169-187, 214-217).  Asynchronous."""
        self._check_state(state)
        N.check(N.lib().marl_venv_step_random(self._h, _u32p(_key_arr(step_key))))
        self._version += 1
        return self._result()

    def probe_steps(self, parent_key, t0: int, n_steps: int, state: Optional[BatchedState] = None) -> StepBatchResult:
        """n_steps iterations of throughput_probe's loop (vector_env.cpp:202-217):
        step k uses split(parent_key, t0 + k) as its action key, parent_key =
        fold_in(key, 2).  Same outputs as n_steps step_random calls (the views
        hold the last step's); MPE fuses them into one launch.  Asynchronous."""
        self._check_state(state)
        N.check(N.lib().marl_venv_probe_steps(self._h, _u32p(_key_arr(parent_key)), int(t0), int(n_steps)))
        self._version += 1
        return self._result()

    def legal_actions(self):
        """Env::legal_actions for every env/agent: uint8 [N, A, n_actions]."""
        out = self._torch.zeros((self._n, self._env.num_agents(), self._env.n_actions_max),
                                dtype=self._torch.uint8, device=f"cuda:{self._device}")
        N.check(N.lib().marl_venv_legal(self._h, C.c_void_p(out.data_ptr())))
        return out

    def world_state(self):
        """Env::world_state of every env (smax.cpp:272-289, mpe.cpp:229-242,
        overcooked.cpp:315-319): float32 [N, world_state_size]."""
        w = C.c_int32()
        N.check(N.lib().marl_venv_world_state_size(self._h, C.byref(w)))
        out = self._torch.empty((self._n, w.value), dtype=self._torch.float32, device=f"cuda:{self._device}")
        N.check(N.lib().marl_venv_world_state(self._h, C.c_void_p(out.data_ptr())))
        return out

    def state_hash(self):
        """Env::state_hash of every env (int64 tensor holding the u64 bits)."""
        out = self._torch.zeros(self._n, dtype=self._torch.int64, device=f"cuda:{self._device}")
        N.check(N.lib().marl_venv_state_hash(self._h, C.c_void_p(out.data_ptr())))
        return out

    def episode_stats(self, clear: bool = False):
        """(episodes, sum of final_lengths, sum of final_returns) since the last clear."""
        out = (C.c_int64 * 3)()
        N.check(N.lib().marl_venv_episode_stats(self._h, out, int(clear)))
        return int(out[0]), int(out[1]), out[2] / float(1 << 24)

    def episode_stats_raw(self, clear: bool = False):
        out = (C.c_int64 * 3)()
        N.check(N.lib().marl_venv_episode_stats(self._h, out, int(clear)))
        return [int(x) for x in out]

    def sync(self):
        N.check(N.lib().marl_venv_sync(self._h))

    def download(self, fields: Sequence[str] = ("obs", "rewards", "dones", "finished", "final_obs",
                                                 "final_returns", "final_lengths", "infos", "actions")):
        """Copy the current step views to fresh numpy arrays (synchronising)."""
        out = {}
        hs = N.HostStep()
        for f in fields:
            shape, ts = self._shapes[f]
            arr = np.zeros(shape, dtype=np.dtype(ts))
            out[f] = arr
            setattr(hs, f, arr.ctypes.data)
        N.check(N.lib().marl_venv_download(self._h, C.byref(hs)))
        return out

    def host_step_random(self, step_key, out: Dict[str, np.ndarray]):
        """End-to-end call with host buffers: fused random step + D2H of ``out``'s fields."""
        hs = N.HostStep()
        for f, arr in out.items():
            setattr(hs, f, arr.ctypes.data)
        N.check(N.lib().marl_venv_step_random_host(self._h, _u32p(_key_arr(step_key)), C.byref(hs)))
        self._version += 1

    def host_step(self, actions: np.ndarray, out: Dict[str, np.ndarray]):
        hs = N.HostStep()
        for f, arr in out.items():
            setattr(hs, f, arr.ctypes.data)
        if self.action_dim:
            a = np.ascontiguousarray(actions, dtype=np.float32)
            N.check(N.lib().marl_venv_step_continuous_host(self._h, C.c_void_p(a.ctypes.data), C.byref(hs)))
        else:
            a = np.ascontiguousarray(actions, dtype=np.int32)
            N.check(N.lib().marl_venv_step_host(self._h, C.c_void_p(a.ctypes.data), C.byref(hs)))
        self._version += 1

    def keys_numpy(self) -> np.ndarray:
        return self.view("keys").cpu().numpy().view(np.uint32)


@dataclass
class ThroughputResult:
    """ThroughputResult (vector_env.hpp:150-160)."""
    env_id: str
    n_envs: int
    steps: int
    seconds: float
    sps: float
    cold_seconds: float

    def csv_row(self) -> str:  # vector_env.cpp:36-43
        return "%s,%d,%d,%.6f,%.2f" % (self.env_id, self.n_envs, self.steps, self.seconds, self.sps)

    @staticmethod
    def csv_header() -> str:
        return "env_id,n_envs,steps,seconds,sps"


def throughput_probe(env_id: str, n_envs: int, n_steps: int, key, config=None, device: int = 0) -> ThroughputResult:
    """throughput_probe (vector_env.cpp:191-222), device-timed."""
    s, cold = C.c_double(), C.c_double()
    N.check(N.lib().marl_throughput_probe(env_id.encode(), _cfg(config), int(n_envs), int(n_steps),
                                          _u32p(_key_arr(key)), int(device), C.byref(s), C.byref(cold)))
    return ThroughputResult(env_id, n_envs, n_steps, s.value, n_envs * n_steps / s.value, cold.value)


@dataclass
class TrajectoryBatch:
    """marl::TrajectoryBatch (vector_env.hpp:45-57) as device tensors indexed
    [step][env][agent]; log_probs / values are None when the policy gave none."""
    n_steps: int
    n_envs: int
    obs: Any
    actions: Any
    rewards: Any
    dones: Any
    log_probs: Any
    values: Any
    final_obs: Any
    final_state: BatchedState


def rollout(venv: VectorEnv, policy, n_steps: int, key) -> TrajectoryBatch:
    """rollout(venv, policy, n_steps, key) (vector_env.cpp:131-165): reset with
    `key`, then n_steps of policy -> VectorEnv::step.  `policy(obs)` takes the
    [N, A, D] observation tensor and returns (actions [N, A] (or [N, A, dim]
    for box spaces), log_probs or None, values or None)."""
    import torch
    if n_steps < 1:
        raise ContractError("rollout: n_steps must be >= 1")
    obs, state = venv.reset(key)
    N = venv.n_envs()
    cols = {k: [] for k in ("obs", "actions", "rewards", "dones", "log_probs", "values")}
    for _ in range(n_steps):
        actions, log_probs, values = policy(obs)
        if len(actions) != N:
            raise ContractError(f"rollout: policy returned {len(actions)} action maps for {N} envs")
        for name, x in (("log_probs", log_probs), ("values", values)):
            if x is not None and len(x) != N:
                raise ContractError(f"rollout: policy {name} batch size mismatch")
        cols["obs"].append(obs.clone())
        cols["actions"].append(torch.as_tensor(actions).clone())
        cols["log_probs"].append(None if log_probs is None else torch.as_tensor(log_probs).clone())
        cols["values"].append(None if values is None else torch.as_tensor(values).clone())
        r = venv.step(state, actions)
        cols["rewards"].append(r.rewards.clone())
        cols["dones"].append(r.dones.clone())
        obs, state = r.obs, r.next

    def stack(xs):
        return None if any(x is None for x in xs) else torch.stack([x.to(xs[0].device) for x in xs])

    return TrajectoryBatch(n_steps, N, stack(cols["obs"]), stack(cols["actions"]), stack(cols["rewards"]),
                           stack(cols["dones"]), stack(cols["log_probs"]), stack(cols["values"]), obs.clone(),
                           state)
