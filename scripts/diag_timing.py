"""Diagnostic: per-step device time of the fused step kernel measured three
ways (per-step events with L2 flush, as bench.py; back-to-back events around
K steps; host wall clock) to expose launch gaps."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_10090_b200 as m
import bench

w = sys.argv[1] if len(sys.argv) > 1 else "smax3m"
env_id, cfg, n, _ = bench.WORKLOADS[w]
v = m.VectorEnv(m.make_env(env_id, cfg), n, device=0)
key = m.prng.key_from_seed(0)
ak = m.prng.split(m.prng.fold_in(key, 2), 200)
v.reset(key)
for t in range(10):
    v.step_random(ak[t])
torch.cuda.synchronize()
s = torch.cuda.current_stream()
K = 40
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for t in range(K):
    v.step_random(ak[10 + t])
e1.record(s)
torch.cuda.synchronize()
print(w, "back-to-back per step ms", e0.elapsed_time(e1) / K)
t0 = time.perf_counter()
for t in range(K):
    v.step_random(ak[10 + t])
t1 = time.perf_counter()
torch.cuda.synchronize()
print(w, "host enqueue per step us", (t1 - t0) / K * 1e6)
