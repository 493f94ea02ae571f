"""IPPO training on the device at scale; writes the reference's metrics table
(ppo.cpp:524-527 columns) as CSV.  usage: train_demo.py N_ENVS UPDATES OUT.csv [precision]"""
import sys
import time

import paper_2311_10090_b200 as m
from paper_2311_10090_b200.ppo import PpoTrainer, MetricTable

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
updates = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/train_curve.csv"
prec = sys.argv[4] if len(sys.argv) > 4 else "bf16"
T = 128
cfg = {"n_envs": n, "n_rollout_steps": T, "total_timesteps": updates * n * T}
tr = PpoTrainer(m.VectorEnv(m.make_env("MPE_simple_spread_v3", {}), n), cfg, False, prec)
tr.begin(m.prng.key_from_seed(0))
table = MetricTable()
t0 = time.perf_counter()
for u in range(tr.n_updates):
    row, div = tr.step()
    table.add_row(row)
    print(f"update {u:3d} mean_return {row[2]:9.3f} loss {row[4]:9.4f} v_loss {row[6]:9.4f} "
          f"entropy {row[7]:.4f} kl {row[8]:.5f} grad_norm {row[10]:.3f}", flush=True)
    if div:
        break
sec = time.perf_counter() - t0
with open(out, "w") as f:
    f.write(table.to_csv())
print(f"{tr.n_updates} updates of {n} envs x {T} steps in {sec:.1f} s = "
      f"{tr.n_updates * n * T * 3 / sec:.3e} agent-steps/s (wall, incl. metrics readback)")
