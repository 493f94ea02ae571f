"""Time one PPO update (collect + update epochs) at a given scale; breakdown by phase."""
import sys, time, json
import torch
import paper_2311_10090_b200 as m
from paper_2311_10090_b200.ppo import PpoTrainer
from paper_2311_10090_b200 import prng

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
T = int(sys.argv[2]) if len(sys.argv) > 2 else 128
prec = sys.argv[3] if len(sys.argv) > 3 else "fp32"
env = sys.argv[4] if len(sys.argv) > 4 else "MPE_simple_spread_v3"
v = m.VectorEnv(m.make_env(env, {}), n, device=0)
cfg = {"n_envs": n, "n_rollout_steps": T, "total_timesteps": 100 * n * T}
tr = PpoTrainer(v, cfg, False, prec)
tr.begin(prng.key_from_seed(0))
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    tr.collect(); torch.cuda.synchronize(); t1 = time.perf_counter()
    row, d = tr.update(); torch.cuda.synchronize(); t2 = time.perf_counter()
    rows = n * 3 * T
    print(json.dumps({"it": it, "n": n, "T": T, "prec": prec, "collect_ms": (t1 - t0) * 1e3, "update_ms": (t2 - t1) * 1e3,
                      "update_rows_per_s": rows * 5 / (t2 - t1), "loss": row[4], "gn": row[10]}), flush=True)
