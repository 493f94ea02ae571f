"""IPPO / MAPPO training on the device: the reference's ``train_ippo`` /
``train_mappo`` (proj/core/include/marl/algo/ppo.hpp:96-99,
proj/core/src/algo/ppo.cpp:518-651) over the C-ABI ``marl_ppo_*``
(include/marl_b200.h).

Per update: the rollout window (rollout.py, ppo.cpp:587-588), then
``update_epochs`` x ``n_minibatches`` minibatches, each a device permutation
slice (prng::permutation, prng.cpp:151-159), advantage normalisation,
forward + PPO row loss + backward of actor and critic (ff_minibatch,
ppo.cpp:409-441), clip_global_norm and Adam (nn.hpp:417-452).  A non-finite
loss or gradient is the reference's DivergenceError: the update's parameters
are rolled back and training stops (ppo.cpp:630-650).
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N
from .rollout import IppoRollout, _PREC
from .venv import VectorEnv, _key_arr, _u32p

COLUMNS = ["step", "update", "mean_return", "n_episodes", "loss", "pg_loss", "v_loss", "entropy", "approx_kl",
           "clip_frac", "grad_norm", "lr"]  # ppo.cpp:524-527

_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)


def _fp(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


@dataclass
class MetricTable:
    """marl::MetricTable (metrics.hpp:8-17)."""
    columns: List[str] = field(default_factory=lambda: list(COLUMNS))
    rows: List[List[float]] = field(default_factory=list)

    def add_row(self, row) -> None:
        if len(row) != len(self.columns):
            from .errors import ContractError
            raise ContractError("MetricTable: row width disagrees with the header")
        self.rows.append([float(x) for x in row])

    def at(self, row: int, column: str) -> float:
        if column not in self.columns:
            from .errors import NotFoundError
            raise NotFoundError(f"MetricTable: no column '{column}'")
        return self.rows[row][self.columns.index(column)]

    def to_csv(self) -> str:
        out = [",".join(self.columns)]
        out += [",".join(repr(v) for v in r) for r in self.rows]
        return "\n".join(out) + "\n"

    def as_array(self) -> np.ndarray:
        return np.asarray(self.rows, np.float64).reshape(len(self.rows), len(self.columns))


@dataclass
class PpoRunResult:
    """marl::PpoRunResult (ppo.hpp:88-94); actor / critic are the packed
    parameter vectors (PpoNets::pack_actor / pack_critic)."""
    actor: np.ndarray
    critic: np.ndarray
    metrics: MetricTable
    diverged: bool = False
    steps_done: int = 0


def init_nets(in_dim: int, critic_in: int, n_actions: int, key, fc_width: int = 64, n_fc_layers: int = 2):
    """ppo_init_nets(key, spec) (ppo.cpp:109-124) for a feed-forward spec, packed."""
    W = fc_width

    def count(i, o):
        n, prev = 0, i
        for _ in range(n_fc_layers):
            n += W * prev + W
            prev = W
        return n + o * W + o

    a = np.zeros(count(in_dim, n_actions), np.float32)
    c = np.zeros(count(critic_in, 1), np.float32)
    N.check(N.lib().marl_ppo_init_nets(in_dim, critic_in, n_actions, fc_width, n_fc_layers, _u32p(_key_arr(key)),
                                       _fp(a, C.c_float), _fp(c, C.c_float)))
    return a, c


def init_rnn(in_dim: int, critic_in: int, n_actions: int, key, fc_width: int = 64, hidden_width: int = 128):
    """ppo_init_nets(key, spec) for a recurrent spec (rnn_init, actor_critic.hpp:82-90), packed."""
    return _init_rnn(in_dim, critic_in, n_actions, key, fc_width, hidden_width)


def _rnn_count(i, F, H, o):
    return F * i + F + 3 * H * F + 3 * H * H + 6 * H + F * H + F + o * F + o


def _init_rnn(in_dim, critic_in, n_actions, key, fc_width, hidden_width):
    a = np.zeros(_rnn_count(in_dim, fc_width, hidden_width, n_actions), np.float32)
    c = np.zeros(_rnn_count(critic_in, fc_width, hidden_width, 1), np.float32)
    N.check(N.lib().marl_ppo_init_rnn(in_dim, critic_in, n_actions, fc_width, hidden_width, _u32p(_key_arr(key)),
                                      _fp(a, C.c_float), _fp(c, C.c_float)))
    return a, c


def permutation(key, n: int, device: int = 0):
    """prng::permutation(key, n) computed on the device; returns a cuda int32 tensor."""
    import torch
    out = torch.empty(max(int(n), 1), dtype=torch.int32, device=f"cuda:{device}")
    N.check(N.lib().marl_ppo_permutation(_u32p(_key_arr(key)), int(n), C.c_void_p(out.data_ptr()), device))
    return out[:n]


class PpoTrainer:
    """The device trainer over one VectorEnv (n_envs must equal config['n_envs'])."""

    def __init__(self, venv: VectorEnv, config: Optional[dict] = None, centralized: bool = False,
                 precision: str = "fp32"):
        self.venv = venv
        self.config = dict(config or {})
        h = C.c_void_p()
        N.check(N.lib().marl_ppo_create(venv._h, json.dumps(self.config).encode(), int(centralized),
                                        _PREC[precision], C.byref(h)))
        self._h = h
        n = C.c_int64()
        N.check(N.lib().marl_ppo_n_updates(self._h, C.byref(n)))
        self.n_updates = int(n.value)
        tcu = C.c_int()
        N.check(N.lib().marl_ppo_tensor_core_update(self._h, C.byref(tcu)))
        self.tensor_core_update = bool(tcu.value)  # the minibatch step runs on tcgen05
        r = C.c_void_p()
        N.check(N.lib().marl_ppo_rollout(self._h, C.byref(r)))
        self.rollout = IppoRollout(venv, int(self.config.get("n_rollout_steps", 128)),
                                   int(self.config.get("fc_width", 64)), int(self.config.get("n_fc_layers", 2)),
                                   self.config.get("activation", "tanh"), precision, centralized, _borrowed=r)
        self.spec = self.rollout.spec
        na, nc = C.c_int32(), C.c_int32()
        N.check(N.lib().marl_ppo_param_counts(self._h, C.byref(na), C.byref(nc)))
        self.n_actor_params, self.n_critic_params = int(na.value), int(nc.value)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                N.lib().marl_ppo_destroy(self._h)
        except Exception:
            pass

    def begin(self, key) -> None:
        """train_ppo_impl setup: nets from fold_in(key,10), collector fold_in(key,11)."""
        N.check(N.lib().marl_ppo_begin(self._h, _u32p(_key_arr(key))))

    def params(self):
        a = np.zeros(self.n_actor_params, np.float32)
        c = np.zeros(self.n_critic_params, np.float32)
        N.check(N.lib().marl_ppo_get_params(self._h, _fp(a, C.c_float), _fp(c, C.c_float)))
        return a, c

    def set_params(self, actor, critic) -> None:
        a = np.ascontiguousarray(actor, dtype=np.float32)
        c = np.ascontiguousarray(critic, dtype=np.float32)
        if a.size != self.n_actor_params or c.size != self.n_critic_params:
            from .errors import ContractError
            raise ContractError(f"ppo: expected {self.n_actor_params}/{self.n_critic_params} parameters, "
                                f"got {a.size}/{c.size}")
        N.check(N.lib().marl_ppo_set_params(self._h, _fp(a, C.c_float), _fp(c, C.c_float)))

    def collect(self) -> None:
        N.check(N.lib().marl_ppo_collect(self._h))

    def update(self):
        """Returns (metrics row, diverged)."""
        row = np.zeros(12, np.float64)
        d = C.c_int()
        N.check(N.lib().marl_ppo_update(self._h, _fp(row, C.c_double), C.byref(d)))
        return row, bool(d.value)

    def step(self):
        row = np.zeros(12, np.float64)
        d = C.c_int()
        N.check(N.lib().marl_ppo_step(self._h, _fp(row, C.c_double), C.byref(d)))
        return row, bool(d.value)

    def minibatch_grad(self, idx):
        """ff_minibatch's flat gradient and {loss, pg, v, entropy, kl, clip_frac}
        for buffer slots idx (t*R + r) of the current window."""
        import torch
        ix = torch.as_tensor(np.ascontiguousarray(idx, np.int32), device=f"cuda:{self.venv._device}")
        g = np.zeros(self.spec.n_actor_params + self.spec.n_critic_params, np.float32)
        st = np.zeros(6, np.float64)
        N.check(N.lib().marl_ppo_minibatch_grad(self._h, C.c_void_p(ix.data_ptr()), int(ix.numel()),
                                                _fp(g, C.c_float), _fp(st, C.c_double)))
        return g, st

    # ---- data-parallel update over env shards
    def set_allreduce(self, fn) -> None:
        """fn(buf: torch cuda tensor view) -> None sums the view in place over
        the ranks; called (stream synchronised) at each exchange of the update:
        advantage sums, gradient, loss sums, episode counts."""
        import torch
        dev = self.venv._device
        dts = {N.DTYPE_F32: torch.float32, N.DTYPE_F64: torch.float64, N.DTYPE_I64: torch.int64}

        def cb(ctx, ptr, count, dtype, stream):
            try:
                t = _device_tensor(ptr, int(count), dts[dtype], dev)
                fn(t)
                return 0
            except Exception:  # never unwind through the C frames
                import traceback
                traceback.print_exc()
                return 1

        self._hook = N.ALLREDUCE_FN(cb)  # kept alive with the trainer
        N.check(N.lib().marl_ppo_set_allreduce(self._h, self._hook, None))

    def use_nccl(self, unique_id: bytes, rank: int, world: int) -> None:
        """The native exchange: NCCL all-reduces stream-ordered with the update."""
        buf = (C.c_uint8 * 128).from_buffer_copy(bytes(unique_id))
        N.check(N.lib().marl_ppo_set_nccl(self._h, buf, int(rank), int(world)))

    def train(self, key) -> PpoRunResult:
        self.begin(key)
        table = MetricTable()
        diverged = False
        steps = 0
        for _ in range(self.n_updates):
            row, diverged = self.step()
            table.add_row(row)
            steps = int(row[0])
            if diverged:
                break
        a, c = self.params()
        return PpoRunResult(a, c, table, diverged, steps)


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    N.check(N.lib().marl_nccl_unique_id(buf))
    return bytes(buf)


def _device_tensor(ptr: int, count: int, dtype, device: int):
    """A zero-copy torch view of `count` elements at device address ptr."""
    import torch
    from .venv import _DevArray
    ts = {torch.float32: "<f4", torch.float64: "<f8", torch.int64: "<i8"}[dtype]
    return torch.as_tensor(_DevArray(int(ptr), (count,), ts), device=f"cuda:{device}")


def torch_allreduce(group=None):
    """An exchange through torch.distributed (any backend that reduces CUDA
    tensors): sum in place, then synchronise."""
    import torch
    import torch.distributed as dist

    def fn(t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        if t.is_cuda:
            torch.cuda.synchronize(t.device)
    return fn


def _train(env, config, key, centralized, device, precision):
    cfg = dict(config or {})
    venv = VectorEnv(env, int(cfg.get("n_envs", 16)), device=device)
    return PpoTrainer(venv, cfg, centralized, precision).train(key)


def train_ippo(env, config: Optional[dict], key, device: int = 0, precision: str = "fp32") -> PpoRunResult:
    """train_ippo(env, cfg, key) (ppo.cpp:653-655) on the device."""
    return _train(env, config, key, False, device, precision)


def train_mappo(env, config: Optional[dict], key, device: int = 0, precision: str = "fp32") -> PpoRunResult:
    """train_mappo(env, cfg, key) (ppo.cpp:657-659): the critic reads Env::world_state."""
    return _train(env, config, key, True, device, precision)
