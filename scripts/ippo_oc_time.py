"""Collect-window time of the IPPO rollout on wide observation rows (Overcooked
cramped_room: 520 + 2 columns; SMAX 27m_vs_30m: 962 + 27 columns, 35 actions):
the fp32 CUDA-core policy vs the K-chunked bf16 tcgen05 one.
Usage: python scripts/ippo_oc_time.py [n_envs] [env_id]"""
import sys
import time
import torch
sys.path.insert(0, ".")
import paper_2311_10090_b200 as m
from paper_2311_10090_b200.rollout import IppoRollout, orthogonal_init

n, T = int(sys.argv[1]) if len(sys.argv) > 1 else 65536, 128
env_id = sys.argv[2] if len(sys.argv) > 2 else "overcooked_cramped_room_v0"
for prec in ("fp32", "bf16"):
    v = m.VectorEnv(m.make_env(env_id, {}), n, device=0)
    ro = IppoRollout(v, T, precision=prec)
    a, c = orthogonal_init(0, ro.spec)
    ro.set_params(a, c)
    ro.begin(m.prng.key_from_seed(0))
    ro.collect(seq_base=0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for w in range(3):
        ro.collect(seq_base=(w + 1) * T)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"{env_id} IPPO {prec}: {n} envs x {T} steps: {dt * 1e3:.1f} ms per window, "
          f"{n * v.env().num_agents() * T / dt:.3g} agent-steps/s")
