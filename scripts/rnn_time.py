"""Time recurrent (GRU) PPO updates: collect + update, PpoConfig defaults (fc 64, GRU 128)."""
import json
import sys
import time

import torch

import paper_2311_10090_b200 as m
from paper_2311_10090_b200.ppo import PpoTrainer

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 14
T = int(sys.argv[2]) if len(sys.argv) > 2 else 128
v = m.VectorEnv(m.make_env("MPE_simple_spread_v3", {}), n)
tr = PpoTrainer(v, {"n_envs": n, "n_rollout_steps": T, "total_timesteps": 10 * n * T, "recurrent": True})
tr.begin(m.prng.key_from_seed(0))
for it in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    tr.collect(); torch.cuda.synchronize(); t1 = time.perf_counter()
    row, d = tr.update(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(json.dumps({"n": n, "T": T, "collect_ms": (t1 - t0) * 1e3, "update_ms": (t2 - t1) * 1e3,
                      "agent_steps_per_s": n * 3 * T / (t2 - t0), "v_loss": row[6], "mean_return": row[2]}),
          flush=True)
