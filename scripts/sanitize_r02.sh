#!/bin/bash
# compute-sanitizer passes over round 2's new device paths (small sizes):
# the three-warp MPE probe pipeline (named barriers, shared slots), the 3xTF32
# tcgen05 GEMM (cp.async ring, split-K), the one-thread-per-env SMAX kernel
# and the recurrent trainer on the GEMM.
export PYTHONPATH=$PWD:$PWD/oracle
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
cat > /tmp/san_r02.py <<'PY'
import ctypes as C
import sys
import torch
import paper_2311_10090_b200 as m
from paper_2311_10090_b200 import _native, prng as O
what = sys.argv[1]
if what in ("probe", "all"):
    for env_id, cfg in [("MPE_simple_spread_v3", {}), ("MPE_simple_speaker_listener_v4", {"continuous_actions": True})]:
        v = m.VectorEnv(env_id, 100, config=cfg)
        key = O.key_from_seed(3)
        v.reset(key)
        v.probe_steps(O.fold_in(key, 2), 0, 60)
        v.sync()
        print("probe", env_id, v.episode_stats())
if what in ("gemm", "all"):
    def g(M, N, K, A, sam, sak, B, sbn, sbk, Cm, ldc, beta):
        _native.check(_native.lib().marl_gemm_f32(M, N, K, C.c_void_p(A.data_ptr()), sam, sak, C.c_void_p(B.data_ptr()),
                                                 sbn, sbk, C.c_void_p(Cm.data_ptr()), ldc, C.c_float(beta), None))
    A = torch.randn(300, 18, device="cuda"); B = torch.randn(64, 18, device="cuda"); Cm = torch.zeros(300, 64, device="cuda")
    g(300, 64, 18, A, 18, 1, B, 18, 1, Cm, 64, 0.0)
    D = torch.randn(5000, 96, device="cuda"); X = torch.randn(5000, 40, device="cuda"); G = torch.zeros(96, 40, device="cuda")
    g(96, 40, 5000, D, 1, 96, X, 1, 40, G, 40, 1.0)
    W = torch.randn(128, 384, device="cuda"); Y = torch.zeros(300, 384, device="cuda"); Ain = torch.randn(300, 128, device="cuda")
    g(300, 384, 128, Ain, 128, 1, W, 1, 384, Y, 384, 0.0)
    torch.cuda.synchronize()
    print("gemm ok", float(Cm.sum()), float(G.sum()), float(Y.sum()))
if what in ("smax", "all"):
    for env_id, cfg in [("SMAX_5m_vs_6m", {"ally_units": ["marine"] * 3, "enemy_units": ["marine"] * 3}), ("SMAX_2s3z", {})]:
        v = m.VectorEnv(env_id, 200, config=cfg)
        key = O.key_from_seed(4)
        v.reset(key)
        for t in range(40):
            v.step_random(O.fold_in(key, t))
        v.sync()
        print("smax", env_id, v.episode_stats())
if what in ("policy", "all"):  # tcgen05 rollout policies: wide rows (Overcooked), MAPPO critics, folded MPE
    from paper_2311_10090_b200.rollout import IppoRollout, orthogonal_init
    for env_id, cent in [("overcooked_cramped_room_v0", False), ("MPE_simple_spread_v3", True),
                         ("MPE_simple_spread_v3", False)]:
        v = m.VectorEnv(env_id, 300)
        ro = IppoRollout(v, 4, precision="bf16", centralized=cent)
        a, c = orthogonal_init(0, ro.spec)
        ro.set_params(a, c)
        ro.begin(O.key_from_seed(1))
        out = ro.collect()
        torch.cuda.synchronize()
        print("policy", env_id, cent, float(out["value"].sum()))
if what in ("wide", "all"):  # the wide-input GEMM-chain update (Overcooked, fp32) and the 35-action wide policy (27m)
    from paper_2311_10090_b200.ppo import PpoTrainer
    from paper_2311_10090_b200.rollout import IppoRollout, orthogonal_init
    n, T = 64, 8
    cfg = {"n_envs": n, "n_rollout_steps": T, "total_timesteps": n * T}
    tr = PpoTrainer(m.VectorEnv(m.make_env("overcooked_cramped_room_v0", {}), n), cfg, False, "fp32")
    r = tr.train(O.key_from_seed(0))
    print("wide update", r.metrics.as_array()[-1][:8])
    v = m.VectorEnv("SMAX_27m_vs_30m", 12)
    ro = IppoRollout(v, 3, precision="bf16")
    a, c = orthogonal_init(0, ro.spec)
    ro.set_params(a, c)
    ro.begin(O.key_from_seed(1))
    out = ro.collect()
    torch.cuda.synchronize()
    print("wide policy 27m", float(out["value"].sum()))
if what in ("rnn", "all"):
    from paper_2311_10090_b200.ppo import PpoTrainer
    n, T = 256, 8
    cfg = {"n_envs": n, "n_rollout_steps": T, "total_timesteps": n * T, "recurrent": True}
    tr = PpoTrainer(m.VectorEnv(m.make_env("MPE_simple_spread_v3", {}), n), cfg, False, "fp32")
    r = tr.train(O.key_from_seed(0))
    print("rnn", r.metrics.as_array()[-1][:8])
PY
TAG=${TAG:-r02}
for what in ${MEMCHECK:-probe gemm smax rnn policy wide}; do
  timeout 900 $CS --tool memcheck --leak-check no --error-exitcode 9 python /tmp/san_r02.py $what > gpurun_out/san_${TAG}_memcheck_$what.log 2>&1
  echo "memcheck $what rc=$?"; grep -E "ERROR SUMMARY" gpurun_out/san_${TAG}_memcheck_$what.log | head -2
done
for what in ${RACECHECK:-probe gemm policy wide}; do
  timeout 900 $CS --tool racecheck --error-exitcode 9 python /tmp/san_r02.py $what > gpurun_out/san_${TAG}_racecheck_$what.log 2>&1
  echo "racecheck $what rc=$?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|hazard" gpurun_out/san_${TAG}_racecheck_$what.log | head -3
  timeout 900 $CS --tool synccheck --error-exitcode 9 python /tmp/san_r02.py $what > gpurun_out/san_${TAG}_synccheck_$what.log 2>&1
  echo "synccheck $what rc=$?"; grep -E "ERROR SUMMARY" gpurun_out/san_${TAG}_synccheck_$what.log | head -2
done
