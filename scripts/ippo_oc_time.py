"""Collect-window time of the IPPO rollout on Overcooked cramped_room (520-wide
observation rows): the fp32 CUDA-core policy vs the K-chunked bf16 tcgen05 one."""
import sys
import time
import torch
sys.path.insert(0, ".")
import paper_2311_10090_b200 as m
from paper_2311_10090_b200.rollout import IppoRollout, orthogonal_init

n, T = int(sys.argv[1]) if len(sys.argv) > 1 else 65536, 128
for prec in ("fp32", "bf16"):
    v = m.VectorEnv(m.make_env("overcooked_cramped_room_v0", {}), n, device=0)
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
    print(f"overcooked IPPO {prec}: {n} envs x {T} steps: {dt * 1e3:.1f} ms per window, "
          f"{n * 2 * T / dt:.3g} agent-steps/s")
