"""Shared helpers: run the CUDA engine and the CPU oracle on the same seeded
probe stream and compare the flattened outputs."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
THREE_M = {"ally_units": ["marine"] * 3, "enemy_units": ["marine"] * 3}
STEP_FIELDS = ["actions", "obs", "rewards", "dones", "finished", "final_returns", "final_lengths",
               "infos", "keys", "episode_returns", "episode_lengths", "state_hash"]


def digest(a) -> str:
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()


def golden_manifest():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


def gpu_outputs(venv, n_info):
    """Download one step's outputs + carry views from a marl-b200 VectorEnv."""
    import torch
    out = venv.download()
    out["infos"] = out["infos"][:, :, :n_info]
    out["keys"] = venv.view("keys").cpu().numpy().view(np.uint32).copy()
    out["episode_returns"] = venv.view("episode_returns").cpu().numpy().copy()
    out["episode_lengths"] = venv.view("episode_lengths").cpu().numpy().copy()
    out["state_hash"] = venv.state_hash().cpu().numpy().view(np.uint64).copy()
    torch.cuda.synchronize()
    return out


def probe_keys(seed, T):
    key = O.key_from_seed(seed)
    return key, O.split(O.fold_in(key, 2), T + 1)
