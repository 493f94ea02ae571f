"""Times one collect + one update of IPPO training on SMAX (args: n_envs [fp32|bf16] [env_id])."""
import json, sys, time, torch
import paper_2311_10090_b200 as m
from paper_2311_10090_b200.ppo import PpoTrainer
n = int(sys.argv[1]); T = 128
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
env_id = sys.argv[3] if len(sys.argv) > 3 else "SMAX_5m_vs_6m"
cfg = {"ally_units": ["marine"] * 3, "enemy_units": ["marine"] * 3} if env_id == "SMAX_5m_vs_6m" else {}
v = m.VectorEnv(m.make_env(env_id, cfg), n)
tr = PpoTrainer(v, {"n_envs": n, "n_rollout_steps": T, "total_timesteps": 10 * n * T}, False, prec)
print("tc", tr.tensor_core_update)
tr.begin(m.prng.key_from_seed(0))
for it in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); tr.collect(); torch.cuda.synchronize(); t1 = time.perf_counter()
    row, d = tr.update(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(json.dumps({"env": env_id, "prec": prec, "n": n, "collect_ms": (t1-t0)*1e3, "update_ms": (t2-t1)*1e3, "agent_steps_per_s": n*3*T/(t2-t0)}))
