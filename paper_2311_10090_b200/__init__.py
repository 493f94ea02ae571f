"""marl-b200: B200-native batched multi-agent environment engine.

The hot path of the reference (marl::VectorEnv::reset/step over MPE, SMAX and
Overcooked, /root/reference/proj/core/src/vector_env.cpp:51-129) as fused
sm_100a CUDA kernels behind a C-ABI (include/marl_b200.h); this package is
the Python mirror of the reference's env API on top of it.
"""
from .errors import ContractError, CudaError, DivergenceError, NotFoundError, SchemaError
from .venv import (BatchedState, Env, StepBatchResult, ThroughputResult, TrajectoryBatch, VectorEnv, make_env,
                   registered_envs, rollout, throughput_probe)
from . import prng

__all__ = [
    "BatchedState", "ContractError", "CudaError", "DivergenceError", "Env", "NotFoundError",
    "SchemaError", "StepBatchResult", "ThroughputResult", "VectorEnv", "make_env", "prng",
    "registered_envs", "rollout", "throughput_probe", "TrajectoryBatch",
]
