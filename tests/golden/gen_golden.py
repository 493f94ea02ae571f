"""Generate the golden trajectories in tests/golden/ from the UNMODIFIED
reference (oracle/_ref/libmarl_ref.so, built by `make -C oracle ref` from
/root/reference/proj/core/src).  Run here, where /root/reference exists:

    python tests/golden/gen_golden.py

Each case runs VectorEnv::reset(key_from_seed(seed)) then T probe steps with
the reference's random-legal action stream (vector_env.cpp:169-187, action
keys split(fold_in(key, 2), T + 1)[t]) and stores, per step, SHA-1 digests of
every flattened output (bit-exact checks) and, for MPE (tolerance parity),
the full float arrays.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import oracle as O  # noqa: E402

THREE_M = {"ally_units": ["marine"] * 3, "enemy_units": ["marine"] * 3}
CASES = [
    # name, env_id, config, n_envs, steps, seed, store_full
    ("mpe_spread", "MPE_simple_spread_v3", {}, 16, 60, 0, True),
    ("mpe_listener", "MPE_simple_speaker_listener_v4", {}, 8, 30, 1, True),
    ("mpe_tag", "MPE_simple_tag_v3", {}, 8, 30, 2, True),
    ("mpe_tag_coop", "MPE_simple_tag_v3", {"cooperative_prey_reward": True}, 8, 30, 3, True),
    ("smax_3m", "SMAX_5m_vs_6m", THREE_M, 32, 80, 0, False),
    ("smax_2s3z", "SMAX_2s3z", {}, 16, 80, 1, False),
    ("smax_5m_vs_6m", "SMAX_5m_vs_6m", {}, 8, 40, 2, False),
    ("smax_27m_vs_30m", "SMAX_27m_vs_30m", {"max_steps": 12}, 2, 20, 3, False),
    ("smax_3s_vs_5z_ctl", "SMAX_3s_vs_5z", {"enemy_controlled": True, "max_steps": 25}, 8, 40, 4, False),
    ("smax_6h_vs_8z", "SMAX_6h_vs_8z", {"max_steps": 30}, 4, 40, 5, False),
    ("oc_cramped", "overcooked_cramped_room_v0", {"max_steps": 50}, 8, 120, 0, False),
    ("oc_asym", "overcooked_asymmetric_advantages_v0", {"max_steps": 50}, 4, 60, 1, False),
    ("oc_ring", "overcooked_coordination_ring_v0", {"max_steps": 50}, 4, 60, 2, False),
    ("oc_forced", "overcooked_forced_coordination_v0", {"max_steps": 50}, 4, 60, 3, False),
    ("oc_circuit", "overcooked_counter_circuit_v0", {"max_steps": 50}, 4, 60, 4, False),
    ("oc_conflicts", "overcooked_cramped_room_v0", {"max_steps": 30, "random_conflict_resolution": True}, 8, 60, 5, False),
]

FIELDS = ["actions", "obs", "rewards", "dones", "finished", "final_returns", "final_lengths", "infos",
          "keys", "episode_returns", "episode_lengths", "state_hash"]


def digest(a: np.ndarray) -> str:
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()


def final_obs_digest(out) -> str:
    fin = out["finished"].astype(bool)
    return digest(out["final_obs"][fin])


def run_case(env_id, cfg, n, T, seed, make):
    venv = make(env_id, cfg, n)
    key = O.key_from_seed(seed)
    obs0 = venv.reset(key)
    akeys = O.split(O.fold_in(key, 2), T + 1)
    steps = []
    for t in range(T):
        out = venv.step_random(akeys[t])
        steps.append(out)
    return obs0, steps


def main():
    if not O.ref_available():
        sys.exit("build the reference first: make -C oracle ref")
    manifest = {}
    for name, env_id, cfg, n, T, seed, full in CASES:
        obs0, steps = run_case(env_id, cfg, n, T, seed, O.RefVenv)
        rec = {"env_id": env_id, "config": cfg, "n_envs": n, "steps": T, "seed": seed,
               "reset_obs": digest(obs0), "digests": [], "finished_total": 0}
        arrays = {"reset_obs": obs0}
        for t, out in enumerate(steps):
            rec["digests"].append({f: digest(out[f]) for f in FIELDS} | {"final_obs": final_obs_digest(out)})
            rec["finished_total"] += int(out["finished"].sum())
            if full:
                for f in ("obs", "rewards", "final_returns", "final_obs", "finished", "keys", "state_hash",
                          "actions", "dones", "episode_lengths"):
                    arrays.setdefault(f, []).append(out[f])
        if full:
            np.savez_compressed(os.path.join(HERE, name + ".npz"),
                                **{k: (np.stack(v) if isinstance(v, list) else v) for k, v in arrays.items()})
        manifest[name] = rec
        print(f"{name}: {env_id} n={n} T={T} finished={rec['finished_total']}")
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(manifest, f, indent=0)


if __name__ == "__main__":
    main()
