#!/bin/bash
# compute-sanitizer passes over the round's new device paths (small sizes).
export PYTHONPATH=$PWD
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
cat > /tmp/san_ppo.py <<'PY'
import sys
import paper_2311_10090_b200 as m
from paper_2311_10090_b200.ppo import PpoTrainer, permutation
prec = sys.argv[1]
n, T = 512, 16
cfg = {"n_envs": n, "n_rollout_steps": T, "total_timesteps": 2 * n * T}
# MPE (Kx 32: two tiles in flight), SMAX 3m (Kx 96, two X buffers), 5m_vs_6m (Kx 192, one X buffer;
# the policy reads observation rows through L2)
envs = [("MPE_simple_spread_v3", {}), ("SMAX_5m_vs_6m", {"ally_units": ["marine"] * 3,
         "enemy_units": ["marine"] * 3}), ("SMAX_5m_vs_6m", {})]
for env_id, ecfg in envs[:1] if len(sys.argv) > 2 and sys.argv[2] == "mpe" else envs:
    tr = PpoTrainer(m.VectorEnv(m.make_env(env_id, ecfg), n), cfg, False, prec)
    r = tr.train(m.prng.key_from_seed(0))
    print("ppo", env_id, prec, r.metrics.as_array()[-1][:8])
print("perm", permutation(m.prng.key_from_seed(1), 1000).sum().item())
PY
cat > /tmp/san_env.py <<'PY'
import numpy as np
import paper_2311_10090_b200 as m
from paper_2311_10090_b200 import prng as O
for env_id, cfg, n in [("MPE_simple_speaker_listener_v4", {"continuous_actions": True}, 300),
                       ("SMAX_5m_vs_6m", {"ally_units": ["marine"]*3, "enemy_units": ["marine"]*3}, 33000),
                       ("SMAX_2s3z", {}, 5000), ("SMAX_5m_vs_6m", {}, 5000),
                       ("overcooked_cramped_room_v0", {"max_steps": 3}, 33000)]:
    v = m.VectorEnv(env_id, n, config=cfg)
    v.reset(O.key_from_seed(1))
    fields = ("obs", "rewards", "dones", "finished", "final_returns", "final_lengths")
    host = {f: np.zeros(v._shapes[f][0], np.dtype(v._shapes[f][1])) for f in fields}
    for k in range(3):
        v.host_step_random(O.fold_in(O.key_from_seed(2), k), host)
    print(env_id, host["rewards"].sum())
PY
if [ -z "$ENV_ONLY" ]; then
for prec in fp32 bf16; do
  timeout 900 $CS --tool memcheck --leak-check no --error-exitcode 9 python /tmp/san_ppo.py $prec > gpurun_out/san_memcheck_ppo_$prec.log 2>&1
  echo "memcheck ppo $prec rc=$?"; grep -E "ERROR SUMMARY|Invalid|race" gpurun_out/san_memcheck_ppo_$prec.log | head -5
done
timeout 900 $CS --tool racecheck --error-exitcode 9 python /tmp/san_ppo.py fp32 mpe > gpurun_out/san_racecheck_ppo.log 2>&1
echo "racecheck ppo fp32 rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard" gpurun_out/san_racecheck_ppo.log | head -5
timeout 900 $CS --tool racecheck python scripts/race_smax.py > gpurun_out/san_racecheck_smax.log 2>&1
echo "racecheck smax rc=$?"; grep -E "RACECHECK SUMMARY|Race reported" gpurun_out/san_racecheck_smax.log | sort | uniq -c | head -5
fi
timeout 900 $CS --tool memcheck --leak-check no --error-exitcode 9 python /tmp/san_env.py > gpurun_out/san_memcheck_env.log 2>&1
echo "memcheck env rc=$?"; grep -E "ERROR SUMMARY|Invalid" gpurun_out/san_memcheck_env.log | head -5
