"""IPPO rollout collection on the device (BASELINE configs[4]).

Python face of the C-ABI ``marl_rollout_*`` (include/marl_b200.h): the
reference's private ``Collector`` (proj/core/src/algo/ppo.cpp:178-374) --
``begin(key)`` is its constructor (ppo.cpp:189-192) and ``collect(...)`` its
``collect(nets, T, seq_base, shaping_at)`` (ppo.cpp:206-323) including the
bootstrap values and GAE (ppo.cpp:285-321).  Parameters are the flat vectors
of ``PpoNets::pack_actor()/pack_critic()`` (nn::pack order, nn.hpp:326-341).

``precision="fp32"`` evaluates the nets in the reference's accumulation order
(the parity path); ``precision="bf16"`` runs the three layers of actor and
critic on the tcgen05 tensor cores with fp32 accumulation.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, Optional

import numpy as np

from . import _native as N
from .venv import VectorEnv, _DevArray, _key_arr, _u32p

_PREC = {"fp32": 0, "bf16": 1}


def policy_spec(venv: VectorEnv, fc_width: int = 64, n_fc_layers: int = 2, activation: str = "tanh",
                centralized: bool = False) -> N.PolicySpec:
    """ppo_net_spec(env, cfg, centralized) (ppo.cpp:80-107)."""
    ps = N.PolicySpec()
    N.check(N.lib().marl_rollout_policy_spec(venv._h, fc_width, n_fc_layers, int(activation == "relu"),
                                             int(centralized), C.byref(ps)))
    return ps


def orthogonal_init(key_seed: int, spec: N.PolicySpec):
    """A deterministic orthogonal initialisation with the reference's gains
    (hidden sqrt(2), actor head 0.01, critic head 1; ppo.cpp:109-124,
    actor_critic.hpp:38-46) for runs that do not load reference parameters.
    Not bit-identical to ppo_init_nets (that uses the reference's own normal
    stream and Gram-Schmidt); parity tests pass the reference's vectors."""
    rng = np.random.default_rng(key_seed)

    def orth(rows, cols, gain):
        a = rng.standard_normal((max(rows, cols), min(rows, cols)))
        q, r = np.linalg.qr(a)
        q = q * np.sign(np.diag(r))
        w = q if rows >= cols else q.T
        return (gain * w[:rows, :cols]).astype(np.float32)

    def branch(out, head_gain):
        W = spec.width
        parts = [orth(W, spec.in_dim, np.sqrt(2)), np.zeros(W, np.float32),
                 orth(W, W, np.sqrt(2)), np.zeros(W, np.float32),
                 orth(out, W, head_gain), np.zeros(out, np.float32)]
        return np.concatenate([p.ravel() for p in parts]).astype(np.float32)

    def critic():
        W = spec.width
        parts = [orth(W, spec.critic_in, np.sqrt(2)), np.zeros(W, np.float32),
                 orth(W, W, np.sqrt(2)), np.zeros(W, np.float32), orth(1, W, 1.0), np.zeros(1, np.float32)]
        return np.concatenate([p.ravel() for p in parts]).astype(np.float32)

    return branch(spec.n_actions, 0.01), critic()


class IppoRollout:
    """Device rollout buffer + collector over one VectorEnv (or shard)."""

    FIELDS = {"obs": "<f4", "actions": "<i4", "rewards": "<f4", "dones": "|u1", "resets": "|u1", "logp": "<f4",
              "value": "<f4", "legal": "|u1", "active": "<f4", "adv": "<f4", "vtarg": "<f4", "last_value": "<f4",
              "critic_in": "<f4"}

    def __init__(self, venv: VectorEnv, n_rollout_steps: int, fc_width: int = 64, n_fc_layers: int = 2,
                 activation: str = "tanh", precision: str = "fp32", centralized: bool = False, _borrowed=None):
        """centralized=True is train_mappo's collector: the critic reads
        Env::world_state (ppo.cpp:341-346) instead of the agent's row."""
        import torch
        self._torch = torch
        self.venv = venv
        self.spec = policy_spec(venv, fc_width, n_fc_layers, activation, centralized)
        if _borrowed is not None:  # a collector owned by a PpoTrainer (marl_ppo_rollout)
            h, self._owned = _borrowed, False
        else:
            h = C.c_void_p()
            N.check(N.lib().marl_rollout_create(venv._h, n_rollout_steps, fc_width, n_fc_layers,
                                                int(activation == "relu"), int(centralized), _PREC[precision],
                                                C.byref(h)))
            self._owned = True
        self._h = h
        v = N.RolloutViews()
        N.check(N.lib().marl_rollout_get_views(self._h, C.byref(v)))
        self.T, self.R = int(v.T), int(v.R)
        shapes = {"obs": (self.T, self.R, self.spec.in_dim), "legal": (self.T, self.R, self.spec.n_actions),
                  "last_value": (self.R,), "critic_in": (self.T, self.R, int(v.critic_dim))}
        self._views = {}
        for name, ts in self.FIELDS.items():
            if name == "critic_in" and not v.critic_in:
                continue
            shape = shapes.get(name, (self.T, self.R))
            self._views[name] = torch.as_tensor(_DevArray(getattr(v, name), shape, ts), device=f"cuda:{venv._device}")

    def __del__(self):
        try:
            if getattr(self, "_h", None) and getattr(self, "_owned", False):
                N.lib().marl_rollout_destroy(self._h)
        except Exception:
            pass

    def set_params(self, actor: np.ndarray, critic: np.ndarray) -> None:
        a = np.ascontiguousarray(actor, dtype=np.float32)
        c = np.ascontiguousarray(critic, dtype=np.float32)
        if a.size != self.spec.n_actor_params or c.size != self.spec.n_critic_params:
            from .errors import ContractError
            raise ContractError(f"rollout: expected {self.spec.n_actor_params}/{self.spec.n_critic_params} "
                                f"parameters, got {a.size}/{c.size}")
        N.check(N.lib().marl_rollout_set_params(self._h, a.ctypes.data_as(C.c_void_p), c.ctypes.data_as(C.c_void_p)))

    def begin(self, key) -> None:
        N.check(N.lib().marl_rollout_begin(self._h, _u32p(_key_arr(key))))

    def collect(self, seq_base: int = 0, gamma: float = 0.99, gae_lambda: float = 1.0,
                shaping: float = 0.0) -> Dict[str, "object"]:
        """One window of n_rollout_steps batch steps; returns zero-copy device
        views of the buffer (valid until the next collect).  Defaults are
        PpoConfig's (ppo.hpp:43-50)."""
        N.check(N.lib().marl_rollout_collect(self._h, int(seq_base), float(gamma), float(gae_lambda), float(shaping)))
        return dict(self._views)

    def view(self, name: str):
        return self._views[name]
