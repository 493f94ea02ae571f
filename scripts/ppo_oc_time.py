"""One train_ippo update on Overcooked cramped_room: collect (bf16 tcgen05 wide-row
policy) + update (fp32 CUDA-core kernels for wide rows) -- where the time goes."""
import sys
import time
import torch
sys.path.insert(0, ".")
import paper_2311_10090_b200 as m
from paper_2311_10090_b200.ppo import PpoTrainer

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
T = 128
cfg = {"n_envs": n, "n_rollout_steps": T, "total_timesteps": 10 * n * T}
tr = PpoTrainer(m.VectorEnv(m.make_env("overcooked_cramped_room_v0", {}), n, device=0), cfg, False, "bf16")
tr.begin(m.prng.key_from_seed(0))
tr.step()
torch.cuda.synchronize()
t0 = time.perf_counter()
tr.collect()
torch.cuda.synchronize()
t1 = time.perf_counter()
tr.step()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"overcooked PPO {n} envs: collect {1e3 * (t1 - t0):.0f} ms, full step (collect + update) {1e3 * (t2 - t1):.0f} ms,"
      f" tensor-core update: {tr.tensor_core_update}")
