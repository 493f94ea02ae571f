"""One recurrent train_ippo run (MPE, small) -> params + metrics to a .npy file,
for comparing the batched and per-step (MARL_RNN_STEPWISE=1) update paths."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2311_10090_b200 as m
from paper_2311_10090_b200.ppo import PpoTrainer
n, T = 64, 32
cfg = {"n_envs": n, "n_rollout_steps": T, "total_timesteps": 3 * n * T, "recurrent": True}
tr = PpoTrainer(m.VectorEnv(m.make_env("MPE_simple_spread_v3", {}), n, device=0), cfg, False, "fp32")
res = tr.train(m.prng.key_from_seed(3))
np.save(sys.argv[1], np.concatenate([res.actor, res.critic, res.metrics.as_array().ravel()]))
