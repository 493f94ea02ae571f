"""ctypes binding of the C-ABI in ``include/marl_b200.h`` (libmarl_b200.so).

The library is built in-tree by ``paper_2311_10090_b200/build.py`` (or
``__graft_entry__.build()``).  There is no fallback: if the library is missing
or cannot be loaded, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import raise_for_status

LIB_PATH = os.environ.get("MARL_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                             "libmarl_b200.so")


class Spec(C.Structure):
    _fields_ = [("family", C.c_int32), ("n_agents", C.c_int32), ("obs_dim", C.c_int32),
                ("n_actions", C.c_int32), ("n_info", C.c_int32), ("max_steps", C.c_int32),
                ("cooperative", C.c_int32), ("device", C.c_int32), ("n_envs", C.c_int64),
                ("global_offset", C.c_int64), ("global_n", C.c_int64)]


class Views(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("obs", "rewards", "dones", "finished", "final_obs",
                                          "final_returns", "final_lengths", "infos", "actions",
                                          "keys", "episode_returns", "episode_lengths")]


class PolicySpec(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("in_dim", "critic_in", "n_actions", "width", "n_layers", "relu",
                                         "n_actor_params", "n_critic_params", "rows_per_env")]


class RolloutViews(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("obs", "actions", "rewards", "dones", "resets", "logp", "value",
                                          "legal", "active", "adv", "vtarg", "last_value", "critic_in")] + \
               [("critic_dim", C.c_int32), ("T", C.c_int32), ("R", C.c_int64), ("in_dim", C.c_int32),
                ("n_actions", C.c_int32)]


class HostStep(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("obs", "rewards", "dones", "finished", "final_obs",
                                          "final_returns", "final_lengths", "infos", "actions")]


EXPORTS = [
    "marl_registered_count", "marl_registered_env", "marl_env_describe", "marl_env_agent",
    "marl_venv_create", "marl_venv_create_shard",
    "marl_venv_destroy", "marl_venv_set_stream", "marl_venv_spec", "marl_venv_agent",
    "marl_venv_info_name", "marl_venv_id", "marl_venv_reset", "marl_venv_step",
    "marl_venv_step_random", "marl_venv_probe_steps", "marl_venv_step_host", "marl_venv_step_random_host",
    "marl_venv_download", "marl_venv_views", "marl_copy_device_to_host", "marl_venv_legal", "marl_venv_state_hash",
    "marl_venv_episode_stats", "marl_venv_sync", "marl_throughput_probe",
    "marl_prng_key_from_seed", "marl_prng_split", "marl_prng_fold_in", "marl_prng_bits",
    "marl_threefry2x32", "marl_gemm_f32", "marl_last_error", "marl_launch_count", "marl_set_grid_cap", "marl_version",
    "marl_venv_world_state_size", "marl_venv_world_state",
    "marl_rollout_policy_spec", "marl_rollout_create", "marl_rollout_set_params", "marl_rollout_begin",
    "marl_rollout_collect", "marl_rollout_get_views", "marl_rollout_destroy",
    "marl_ppo_create", "marl_ppo_init_nets", "marl_ppo_begin", "marl_ppo_n_updates", "marl_ppo_tensor_core_update", "marl_ppo_set_params",
    "marl_ppo_get_params", "marl_ppo_rollout", "marl_ppo_collect", "marl_ppo_update", "marl_ppo_step",
    "marl_ppo_minibatch_grad", "marl_ppo_destroy", "marl_ppo_permutation", "marl_ppo_set_allreduce",
    "marl_nccl_unique_id", "marl_ppo_set_nccl", "marl_venv_action_dim", "marl_venv_actions_f32",
    "marl_venv_step_continuous", "marl_venv_step_continuous_host", "marl_ppo_param_counts", "marl_ppo_init_rnn",
]

# int (*marl_allreduce_fn)(void* ctx, void* dev_buf, int64_t count, int dtype, void* stream)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p)
DTYPE_F32, DTYPE_F64, DTYPE_I64 = 0, 1, 2

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"marl-b200 native library missing at {LIB_PATH}; build it with "
                           "`python paper_2311_10090_b200/build.py` (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, u32p, i32p, i64p = C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_int32), C.POINTER(C.c_int64)
    L.marl_registered_env.restype = C.c_char_p
    L.marl_registered_env.argtypes = [C.c_int]
    L.marl_env_describe.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(Spec)]
    L.marl_env_agent.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_char_p, C.c_size_t, i32p, i32p]
    L.marl_venv_create.argtypes = [C.c_char_p, C.c_char_p, C.c_int64, C.c_int, C.POINTER(vp)]
    L.marl_venv_create_shard.argtypes = [C.c_char_p, C.c_char_p, C.c_int64, C.c_int64, C.c_int64,
                                         C.c_int, C.POINTER(vp)]
    L.marl_venv_destroy.argtypes = [vp]
    L.marl_venv_set_stream.argtypes = [vp, vp]
    L.marl_venv_spec.argtypes = [vp, C.POINTER(Spec)]
    L.marl_venv_agent.argtypes = [vp, C.c_int, C.c_char_p, C.c_size_t, i32p, i32p]
    L.marl_venv_info_name.argtypes = [vp, C.c_int, C.c_char_p, C.c_size_t]
    L.marl_venv_id.argtypes = [vp, C.c_char_p, C.c_size_t]
    L.marl_venv_reset.argtypes = [vp, u32p]
    L.marl_venv_step.argtypes = [vp, vp]
    L.marl_venv_step_random.argtypes = [vp, u32p]
    L.marl_venv_probe_steps.argtypes = [vp, u32p, C.c_uint64, C.c_int]
    L.marl_venv_step_host.argtypes = [vp, vp, C.POINTER(HostStep)]
    L.marl_venv_step_random_host.argtypes = [vp, u32p, C.POINTER(HostStep)]
    L.marl_venv_download.argtypes = [vp, C.POINTER(HostStep)]
    L.marl_venv_views.argtypes = [vp, C.POINTER(Views)]
    L.marl_copy_device_to_host.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
    L.marl_venv_legal.argtypes = [vp, vp]
    L.marl_venv_world_state_size.argtypes = [vp, i32p]
    L.marl_venv_world_state.argtypes = [vp, vp]
    L.marl_venv_state_hash.argtypes = [vp, vp]
    L.marl_venv_episode_stats.argtypes = [vp, i64p, C.c_int]
    L.marl_venv_sync.argtypes = [vp]
    L.marl_throughput_probe.argtypes = [C.c_char_p, C.c_char_p, C.c_int64, C.c_int, u32p, C.c_int,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.marl_prng_key_from_seed.argtypes = [C.c_uint64, u32p]
    L.marl_prng_split.argtypes = [u32p, C.c_uint64, u32p]
    L.marl_prng_fold_in.argtypes = [u32p, C.c_uint64, u32p]
    L.marl_prng_bits.argtypes = [u32p, C.c_uint64]
    L.marl_prng_bits.restype = C.c_uint64
    L.marl_threefry2x32.argtypes = [C.c_uint32] * 4 + [u32p]
    L.marl_rollout_policy_spec.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(PolicySpec)]
    L.marl_rollout_create.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
    L.marl_rollout_set_params.argtypes = [vp, vp, vp]
    L.marl_rollout_begin.argtypes = [vp, u32p]
    L.marl_rollout_collect.argtypes = [vp, C.c_int64, C.c_double, C.c_double, C.c_double]
    L.marl_rollout_get_views.argtypes = [vp, C.POINTER(RolloutViews)]
    L.marl_rollout_destroy.argtypes = [vp]
    f32p, f64p = C.POINTER(C.c_float), C.POINTER(C.c_double)
    L.marl_ppo_create.argtypes = [vp, C.c_char_p, C.c_int, C.c_int, C.POINTER(vp)]
    L.marl_ppo_init_nets.argtypes = [C.c_int] * 5 + [u32p, f32p, f32p]
    L.marl_ppo_begin.argtypes = [vp, u32p]
    L.marl_ppo_n_updates.argtypes = [vp, i64p]
    L.marl_ppo_tensor_core_update.argtypes = [vp, C.POINTER(C.c_int)]
    L.marl_ppo_set_params.argtypes = [vp, f32p, f32p]
    L.marl_ppo_get_params.argtypes = [vp, f32p, f32p]
    L.marl_ppo_rollout.argtypes = [vp, C.POINTER(vp)]
    L.marl_ppo_collect.argtypes = [vp]
    L.marl_ppo_update.argtypes = [vp, f64p, C.POINTER(C.c_int)]
    L.marl_ppo_step.argtypes = [vp, f64p, C.POINTER(C.c_int)]
    L.marl_ppo_minibatch_grad.argtypes = [vp, vp, C.c_int64, f32p, f64p]
    L.marl_ppo_destroy.argtypes = [vp]
    L.marl_ppo_permutation.argtypes = [u32p, C.c_int64, vp, C.c_int]
    L.marl_ppo_set_allreduce.argtypes = [vp, ALLREDUCE_FN, vp]
    L.marl_venv_action_dim.argtypes = [vp, C.POINTER(C.c_int32)]
    L.marl_ppo_param_counts.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.marl_ppo_init_rnn.argtypes = [C.c_int] * 5 + [u32p, C.POINTER(C.c_float), C.POINTER(C.c_float)]
    L.marl_venv_actions_f32.argtypes = [vp, C.POINTER(C.POINTER(C.c_float))]
    L.marl_venv_step_continuous.argtypes = [vp, vp]
    L.marl_venv_step_continuous_host.argtypes = [vp, vp, C.POINTER(HostStep)]
    L.marl_nccl_unique_id.argtypes = [C.POINTER(C.c_uint8)]
    L.marl_ppo_set_nccl.argtypes = [vp, C.POINTER(C.c_uint8), C.c_int, C.c_int]
    L.marl_last_error.restype = C.c_char_p
    L.marl_launch_count.restype = C.c_uint64
    L.marl_set_grid_cap.argtypes = [C.c_int]
    i64 = C.c_int64
    L.marl_gemm_f32.argtypes = [i64, C.c_int, i64, vp, i64, i64, vp, i64, i64, vp, i64, C.c_float, vp]
    L.marl_version.restype = C.c_char_p
    _lib = L
    return L


def check(rc: int) -> None:
    if rc:
        raise_for_status(rc, lib().marl_last_error().decode(errors="replace"))
