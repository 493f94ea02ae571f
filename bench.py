"""Benchmark of the batched env-step hot path (BASELINE.json metric:
agent-steps/s at 1/2/4/8 B200 vs the CPU reference; % of HBM roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload smax3m|mpe|mpe_large|overcooked|smax2s3z|smax27m|ippo|ippo_oc|ppo|ppo_smax|ppo_oc|ppo_rnn]
  python bench.py --impl reference ...     # the reference's own CPU path, host cores

A "step" is one fused VectorEnv step over the whole synthetic batch with the
reference probe's random-legal action stream (vector_env.cpp:169-217): the
default workload is BASELINE.json configs[1], SMAX 3m with 65536 envs per GPU
(weak scaling).  Multi-GPU runs are launched with torchrun (one rank per GPU,
NCCL); envs are sharded by contiguous global index with no collective in the
step path, and one NCCL all-reduce aggregates the episode statistics.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

THREE_M = {"ally_units": ["marine"] * 3, "enemy_units": ["marine"] * 3}
WORKLOADS = {
    # name: (env_id, config, envs per GPU, label)
    "smax3m": ("SMAX_5m_vs_6m", THREE_M, 65536, "SMAX 3m (3 marines vs 3, heuristic enemy), configs[1]"),
    "mpe": ("MPE_simple_spread_v3", {}, 1024, "MPE simple_spread, configs[0]"),
    "mpe_large": ("MPE_simple_spread_v3", {}, 1 << 22, "MPE simple_spread at 4M envs/GPU (roofline sweep)"),
    "overcooked": ("overcooked_cramped_room_v0", {}, 262144, "Overcooked cramped_room, configs[2]"),
    "smax2s3z": ("SMAX_2s3z", {}, 65536, "SMAX 2s3z, configs[3]"),
    "smax27m": ("SMAX_27m_vs_30m", {}, 4096, "SMAX 27m_vs_30m, configs[3]"),
    # configs[4]: one "step" is one Collector::collect window of IPPO_T env steps
    "ippo": ("MPE_simple_spread_v3", {}, 1 << 20, "IPPO rollout on MPE simple_spread, 2^20 envs x 128 steps, "
             "bf16 actor+critic on tcgen05, configs[4]"),
    "ippo_oc": ("overcooked_cramped_room_v0", {}, 1 << 16, "IPPO rollout on Overcooked cramped_room, 2^16 envs x "
                "128 steps, bf16 tcgen05 wide-row policy (541 + 2 input columns, K-chunked layer 1)"),
    # one "step" is one train_ippo update (collect + update_epochs x n_minibatches)
    "ppo": ("MPE_simple_spread_v3", {}, 1 << 16, "IPPO training update on MPE simple_spread (collect 128 steps + "
            "5 epochs x 2 minibatches of PPO), PpoConfig defaults"),
    "ppo_rnn": ("MPE_simple_spread_v3", {}, 1 << 14, "recurrent (GRU 128) IPPO training update on MPE simple_spread "
                "(collect 128 steps + 5 epochs x 2 minibatches, BPTT), PpoConfig defaults + recurrent"),
    "ppo_smax": ("SMAX_5m_vs_6m", THREE_M, 1 << 14, "IPPO training update on SMAX 3m (collect 128 steps + 5 epochs x "
                 "2 minibatches of PPO; 95-wide observations), PpoConfig defaults"),
    "ppo_oc": ("overcooked_cramped_room_v0", {}, 1 << 14, "IPPO training update on Overcooked cramped_room (collect "
               "128 steps + 5 epochs x 2 minibatches of PPO; 541 + 2 wide observations, fp32-accurate GEMM-chain "
               "update), PpoConfig defaults"),
}
PPO_WORKLOADS = ("ppo", "ppo_rnn", "ppo_smax", "ppo_oc")
IPPO_WORKLOADS = ("ippo", "ippo_oc")
FUSED_PROBE = ("mpe",)  # timed as one fused multi-step probe launch (marl_venv_probe_steps)
IPPO_T = 128
L2_FLUSH_BYTES = 512 << 20  # > 4x the 126 MB L2; its ~80 us also covers the host's enqueue of the next step


def workload_config(workload, world, n_per_gpu=None):
    """The `config` object, identical in both arms (the reference arm times a
    bounded sample of this workload and says so in cpu_baseline.sample)."""
    env_id, cfg, n, label = WORKLOADS[workload]
    n = n_per_gpu or n
    agents = {"SMAX_2s3z": 5, "SMAX_27m_vs_30m": 27, "SMAX_5m_vs_6m": 3, "MPE_simple_spread_v3": 3,
              "overcooked_cramped_room_v0": 2}[env_id]
    c = {"workload": label, "env_id": env_id, "env_config": cfg, "n_envs_per_gpu": n, "global_envs": n * world,
         "agents": agents}
    if workload in IPPO_WORKLOADS:
        c["rollout_steps_per_window"] = IPPO_T
    if workload in PPO_WORKLOADS:
        c.update({"rollout_steps": IPPO_T, "update_epochs": 5, "n_minibatches": 2})
    return c


def algorithmic_bytes(env, n_envs, n_finished):
    """Minimum bytes one fused step must move: state read +
    write, carry (key, return, length) read + write, every output view, and
    final_obs rows of the envs that finished.  fp64 state, f32 obs."""
    A, D = env.num_agents(), env.obs_dim
    fam = env.family
    if fam == 0:    # MPE spread: agent pos/vel rw, landmark pos read (written on reset), steps
        E = 6 if A == 3 else 6
        state_rw = 2 * (2 * A * 8 + 2 * A * 8 + 4) + (2 * (E - A) * 8)
        reset_extra = 2 * (E - A) * 8
    elif fam == 1:  # SMAX: x,y,health,cooldown f64 + packed memory u32 per unit, t
        U = len(env.config.get("ally_units", [])) + len(env.config.get("enemy_units", [])) or None
        U = U or {"SMAX_2s3z": 10, "SMAX_27m_vs_30m": 57}.get(env.id(), A * 2)
        state_rw = 2 * (U * (4 * 8 + 4) + 4)
        reset_extra = 0
    else:           # Overcooked: agents word, pots, counter bits, t
        state_rw = 2 * (4 + 4 + 8 + 4)
        reset_extra = 0
    carry_rw = 2 * (16 + 8 + 4)
    outputs = A * D * 4 + A * 8 + (A + 1) + A * env.n_info * 8 + 1 + 8 + 4 + A * 4
    per_env = state_rw + carry_rw + outputs
    return n_envs * per_env + n_finished * (A * D * 4 + reset_extra)


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: NVML polled every 2 ms from a side thread (the timed region of a
    sub-millisecond step is too short for `nvidia-smi -lms`), with the
    nvidia-smi query of B200_PROFILING.md as the fallback when NVML is absent."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device=0, period_s=0.002):
        import threading
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml as N
            N.nvmlInit()
            self.N, self.h = N, N.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
        except Exception:
            self.N = None
        self.period = period_s
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _sample(self):
        N, h = self.N, self.h
        self.sm.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
        try:
            mask = N.nvmlDeviceGetCurrentClocksEventReasons(h)
        except AttributeError:
            mask = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        for bit, name in self.REASONS.items():
            if mask & bit:
                self.reasons.add(name)

    def _run(self):
        if self.N is None:
            return
        while True:
            self._sample()
            if self._stop.wait(self.period):
                break

    def stop(self):
        self._stop.set()
        self.t.join()
        if self.N is None:
            return self._smi()
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml, 2 ms"}

    @staticmethod
    def _smi():
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            row = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-i", "0"],
                                 capture_output=True, text=True).stdout.strip().split(",")
        except FileNotFoundError:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        return {"sm_mhz": float(row[0]), "sm_max_mhz": float(row[1]),
                "reasons": [n for n, v in zip(names, row[2:]) if v.strip() == "Active"], "samples": 1,
                "source": "nvidia-smi after the timed region (NVML unavailable)"}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_metrics(workload):
    """SM / DRAM utilisation of the step kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_metrics.json")) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


def ncu_traffic(workload):
    """dram bytes per launch of the step kernel from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


# --------------------------------------------------------------------- CPU arms
def cpu_reference_probe(env_id, cfg, n_envs, steps, warmup, threads):
    """The reference's VectorEnv::step + random_legal_actions (its own
    throughput_probe loop, vector_env.cpp:214-217) on the host cores."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    kind = "reference" if O.ref_available() else "port"
    key = O.key_from_seed(0)
    akeys = O.split(O.fold_in(key, 2), steps + warmup + 1)
    if kind == "reference":
        O.ref_lib().mref_set_threads(int(threads))
        v = O.RefVenv(env_id, cfg, n_envs)
        import ctypes as C
        L = O.ref_lib()
        v.reset(key)
        act = np.zeros((n_envs, v.n_agents), np.int32)

        def one(t):
            v._chk(L.mref_random_actions(v.h, O._ptr(akeys[t], C.c_uint32), O._ptr(act, C.c_int32)))
            v._chk(L.mref_step(v.h, O._ptr(act, C.c_int32), None, None, None, None, None, None, None, None, 0,
                               None, None, None, None))
        cores = int(threads)
    else:
        v = O.PortVenv(env_id, cfg, n_envs)
        v.reset(key)

        def one(t):
            v.step(v.random_actions(akeys[t]))
        cores = 1
    for t in range(warmup):
        one(t)
    t0 = time.perf_counter()
    for t in range(warmup, warmup + steps):
        one(t)
    sec = time.perf_counter() - t0
    return sec, kind, cores, v.n_agents


def ippo_bytes_per_env_step(env, in_dim, n_act):
    """Algorithmic bytes of one rollout env-step: the env step,
    the policy kernel (obs row read + buffer row writes: obs, action, logp,
    value, legal, active, reset), the record kernel (rewards/finished read,
    reward/done rows written) and GAE (reward, value, done read; adv, vtarg
    written), per env."""
    A = env.num_agents()
    env_b = algorithmic_bytes(env, 1, 0)
    policy = A * env.obs_dim * 4 + A * (in_dim * 4 + 4 + 4 + 4 + n_act + 4 + 1)
    record = A * 8 + 1 + A * (4 + 1)
    gae = A * (4 + 4 + 1 + 4 + 4)
    return env_b + policy + record + gae


def run_gpu_ippo(args, rank, world, local_rank):
    """configs[4]: the reference's IPPO collector on the device, one timed
    step = one collect window (IPPO_T env steps of every env)."""
    import torch
    import paper_2311_10090_b200 as m
    from paper_2311_10090_b200 import _native
    from paper_2311_10090_b200 import dist as shard
    from paper_2311_10090_b200.rollout import IppoRollout, orthogonal_init

    env_id, cfg, n_per_gpu, label = WORKLOADS[args.workload]
    if args.n_envs:
        n_per_gpu = args.n_envs
    torch.cuda.set_device(local_rank)
    env = m.make_env(env_id, cfg)
    A = env.num_agents()
    N = n_per_gpu * world
    T = IPPO_T
    venv = shard.make_sharded(env, N, rank, world, device=local_rank)
    ro = IppoRollout(venv, T, precision="bf16")
    actor, critic = orthogonal_init(0, ro.spec)
    pin_a = torch.from_numpy(actor).pin_memory().numpy()
    pin_c = torch.from_numpy(critic).pin_memory().numpy()
    ro.set_params(pin_a, pin_c)
    key = m.prng.key_from_seed(0)
    ro.begin(key)
    stream = torch.cuda.current_stream()
    for w in range(args.warmup):
        ro.collect(seq_base=w * T)
    torch.cuda.synchronize()
    venv.episode_stats(clear=True)
    if world > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(local_rank) if rank == 0 else None
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = _native.lib().marl_launch_count()
    for k in range(args.steps):  # the buffer (>> L2) is rewritten every window: no flush needed
        starts[k].record(stream)
        ro.collect(seq_base=(args.warmup + k) * T)
        ends[k].record(stream)
    torch.cuda.synchronize()
    launches = _native.lib().marl_launch_count() - launches0
    clk = clocks.stop() if clocks else None
    win_ms = [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]
    total_ms = shard.max_over_ranks(float(sum(win_ms)), device="cuda")
    stats = shard.all_reduce_episode_stats(venv.episode_stats_raw(), device="cuda")
    env_steps = N * T * args.steps
    value = env_steps * A / (total_ms * 1e-3)
    mean_win_s = float(np.mean(win_ms)) * 1e-3
    bpe = ippo_bytes_per_env_step(env, ro.spec.in_dim, ro.spec.n_actions)
    achieved = n_per_gpu * T * bpe / mean_win_s / 1e9
    peak, peak_src = measured_peak()
    in_ = ro.spec.in_dim
    kx = 32 if in_ <= 32 else ((in_ + 15) // 16 * 16 if in_ <= 192 else (in_ + 63) // 64 * 64)
    flop_row = 2 * (128 * kx + 2 * 64 * 64 + 2 * 16 * 64)  # MMA FLOPs per row as issued (padded operands)
    tflops = n_per_gpu * A * (T + 1) * flop_row / mean_win_s / 1e12

    # end to end through the public API: parameters H2D from pinned memory,
    # one collect window, the episode statistics read back (what an on-GPU
    # trainer consumes from the host), every window
    e2e_steps = max(2, min(args.steps, 5))
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        ro.set_params(pin_a, pin_c)
        ro.collect(seq_base=(args.warmup + args.steps + k) * T)
        venv.episode_stats_raw()
    sec = shard.max_over_ranks(time.perf_counter() - t0, device="cuda")
    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        if O.ref_available():
            n_cpu, t_cpu = 256, 32
            ka, kc = O.ref_ppo_init(env_id, cfg, O.fold_in(O.key_from_seed(0), 10))
            t0 = time.perf_counter()
            O.ref_collect(env_id, cfg, n_cpu, t_cpu, O.key_from_seed(0), ka, kc)
            csec = time.perf_counter() - t0
            cpu = {"value": n_cpu * t_cpu * A / csec, "unit": "agent-steps/s", "cores": 1, "kind": "reference",
                   "sample": f"reference Collector pieces (VectorEnv + ff_forward + sample_masked + compute_gae), "
                             f"{n_cpu} envs x {t_cpu} steps, 1 collect window ({csec:.1f} s, ThreadPool for the env)"}
    line = {
        "metric": "agent-steps/sec (env-steps/sec x agents)", "value": value, "unit": "agent-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16 policy / f64 env",
        "data": "synthetic (reset from key_from_seed(0); orthogonal-init policy, sampled actions)",
        "config": workload_config(args.workload, world, n_per_gpu),
        "run": {"step": "one collect window", "parallelism": f"env-sharded x{world}, no collective in the window",
                "l2": "no flush: each window writes a >20 GB rollout buffer (>> 126 MB L2)"},
        "env_steps_per_sec": env_steps / (total_ms * 1e-3),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "peak_source": peak_src,
                     "bytes_per_launch": n_per_gpu * T * bpe, "mean_launch_us": mean_win_s * 1e6,
                     "kernel": "whole collect window (env step + tcgen05 policy + record + GAE kernels)",
                     "bytes_per_env_step": bpe, "tensor_tflops": tflops},
        "cpu_baseline": cpu,
        "e2e": {"value": N * A * T * e2e_steps / sec, "unit": "agent-steps/s",
                "h2d_bytes_per_step": int(pin_a.nbytes + pin_c.nbytes), "d2h_bytes_per_step": 24,
                "steps": e2e_steps, "path": "IppoRollout.set_params + collect + episode stats (C-ABI marl_rollout_*)"},
        "gpu_launches": int(launches),
        "clocks": clk,
        "episode_stats": shard.summarize(stats),
    }
    print(json.dumps(line))


def ppo_flop_per_row(in_dim, cin, W, na):
    fwd = W * in_dim + W * W + na * W + W * cin + W * W + W      # actor + critic forward MACs
    bwd = (na * W + W * W) + (W + W * W)                         # dx of head and layer 2 (both nets)
    wg = W * in_dim + W * W + na * W + W * cin + W * W + W        # weight gradients
    return 2 * (fwd + bwd + wg)


def run_gpu_ppo(args, rank, world, local_rank):
    """One timed step = one PPO update of train_ippo (ppo.cpp:585-636): the
    rollout window on the device then update_epochs x n_minibatches of
    permutation + ff_minibatch + clip + Adam."""
    import torch
    import paper_2311_10090_b200 as m
    from paper_2311_10090_b200 import _native
    from paper_2311_10090_b200.ppo import PpoTrainer

    env_id, cfg, n_envs, label = WORKLOADS[args.workload]
    if args.n_envs:
        n_envs = args.n_envs
    torch.cuda.set_device(local_rank)
    env = m.make_env(env_id, cfg)
    A = env.num_agents()
    T = IPPO_T
    # weak scaling: n_envs per GPU fixed; N > 1 is data-parallel training over env shards with the
    # update's sums all-reduced over NCCL (identical parameters on every rank)
    gn = n_envs * world
    recurrent = args.workload == "ppo_rnn"
    pc = {"n_envs": gn, "n_rollout_steps": T, "total_timesteps": (args.warmup + args.steps + 8) * gn * T}
    if recurrent:
        pc["recurrent"] = True
    from paper_2311_10090_b200 import dist as shard_mod
    venv = shard_mod.make_sharded(env, gn, rank, world, device=local_rank) if world > 1 else \
        m.VectorEnv(env, n_envs, device=local_rank)
    tr = PpoTrainer(venv, pc, False, "fp32" if recurrent else "bf16")
    if world > 1:
        import torch.distributed as tdist
        from paper_2311_10090_b200.ppo import nccl_unique_id
        uid = [nccl_unique_id() if rank == 0 else None]
        tdist.broadcast_object_list(uid, src=0)
        tr.use_nccl(uid[0], rank, world)
    tr.begin(m.prng.key_from_seed(0))
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        tr.step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(local_rank) if rank == 0 else None
    launches0 = _native.lib().marl_launch_count()
    col_ms, upd_ms, rows = [], [], []
    for k in range(args.steps):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        tr.collect()
        e1.record(stream)
        row, div = tr.update()
        e2.record(stream)
        torch.cuda.synchronize()
        col_ms.append(e0.elapsed_time(e1))
        upd_ms.append(e1.elapsed_time(e2))
        rows.append(row)
    launches = _native.lib().marl_launch_count() - launches0
    clk = clocks.stop() if clocks else None
    step_ms = [c + u for c, u in zip(col_ms, upd_ms)]
    from paper_2311_10090_b200 import dist as shard
    total_ms = shard.max_over_ranks(float(sum(step_ms)), device="cuda")
    value = world * n_envs * A * T * args.steps / (total_ms * 1e-3)
    sp = tr.spec
    fpr = ppo_flop_per_row(sp.in_dim, sp.critic_in, sp.width, sp.n_actions)
    if recurrent:  # RnnBranch MACs (fc 64, GRU 128) x (forward + 2 x backward) x 2 FLOP
        F, Hh = 64, 128
        macs = sum(F * i + 3 * Hh * F + 3 * Hh * Hh + F * Hh + o * F for i, o in ((sp.in_dim, sp.n_actions),
                                                                              (sp.critic_in, 1)))
        fpr = 6 * macs
    R = n_envs * A
    upd_s = float(np.mean(upd_ms)) * 1e-3
    tflops = T * R * 5 * fpr / upd_s / 1e12  # algorithmic FLOPs (unpadded) per second of update
    # end to end through the public API: step() then the new parameters to the host
    e2e_steps = max(2, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        tr.step()
        a, c = tr.params()
    sec = shard.max_over_ranks(time.perf_counter() - t0, device="cuda")
    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        if O.ref_available():
            n_cpu, t_cpu = (64, 32) if not recurrent else (16, 32)
            rc = {"n_envs": n_cpu, "n_rollout_steps": t_cpu, "total_timesteps": n_cpu * t_cpu}
            if recurrent:
                rc["recurrent"] = True
            t0 = time.perf_counter()
            O.ref_train(env_id, cfg, rc, O.key_from_seed(0))
            csec = time.perf_counter() - t0
            cpu = {"value": n_cpu * t_cpu * A / csec, "unit": "agent-steps/s", "cores": 1, "kind": "reference",
                   "sample": f"reference train_ippo, {n_cpu} envs x {t_cpu} steps, 1 update (5 epochs x 2 "
                             f"minibatches), {csec:.1f} s"}
    peak = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["bf16_tflops"])
    except Exception:
        peak = 2250.0
    line = {
        "metric": "agent-steps/sec (env-steps/sec x agents)", "value": value, "unit": "agent-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": ("f32 recurrent policy + f32 BPTT update (3xTF32 tcgen05 GEMMs, fp32-accurate)" if recurrent else
                  "bf16 rollout policy + bf16 tcgen05 PPO update (fp32 accumulate)" if tr.tensor_core_update else
                  "bf16 rollout policy + f32 PPO update (3xTF32 tcgen05 GEMM chain, fp32-accurate)")
        + " / f64 env", "data": "synthetic (key_from_seed(rank))",
        "config": workload_config(args.workload, world, n_envs),
        "run": {"batch_rows": T * R, "step": "one PPO update = collect + update",
                "parallelism": f"dp{world}: env shards, update sums all-reduced over NCCL" if world > 1
                else "single device",
                "l2": "no flush: the rollout buffer (> 1 GB) is rewritten every step"},
        "collect_ms": float(np.mean(col_ms)), "update_ms": float(np.mean(upd_ms)),
        "update_row_passes_per_sec": T * R * 5 / upd_s,
        "roofline": {"bound": "tensor", "achieved": tflops, "peak": peak, "unit": "TFLOP/s", "frac": tflops / peak,
                     "traffic": None, "peak_source": "MEASURED_PEAKS.json bf16_tflops (dense)",
                     "kernel": ("recurrent PPO update (3xTF32 tcgen05 GEMM per time step + gate kernels)" if recurrent
                                else "PPO update phase (ppo_update_tc_kernel dominant: bf16 tcgen05 forward, input- "
                                     "and weight-gradient GEMMs, fp32 TMEM accumulation)" if tr.tensor_core_update
                                else "PPO update phase (wide rows: 3xTF32 tcgen05 GEMM chain, layer-1 product and "
                                     "weight gradient dominant; 3 tf32 MMAs per product, counted once)"),
                     "flop_per_row_pass": fpr,
                     # fp32-accurate paths: tf32 MMAs run at half the bf16 rate and 3xTF32 issues three per
                     # product, so bf16 peak / 6 is their tensor ceiling (a derived figure, stated beside frac)
                     "frac_vs_3xtf32_ceiling": (tflops / (peak / 6.0)) if (recurrent or not tr.tensor_core_update)
                     else None},
        "cpu_baseline": cpu,
        "e2e": {"value": world * n_envs * A * T * e2e_steps / sec, "unit": "agent-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": int(a.nbytes + c.nbytes + 12 * 8), "steps": e2e_steps,
                "path": "PpoTrainer.step + params() (C-ABI marl_ppo_step / marl_ppo_get_params)"},
        "gpu_launches": int(launches),
        "clocks": clk,
        "last_metrics": {k: float(v) for k, v in zip(["step", "update", "mean_return", "n_episodes", "loss",
                                                        "pg_loss", "v_loss", "entropy", "approx_kl", "clip_frac",
                                                        "grad_norm", "lr"], rows[-1])},
    }
    print(json.dumps(line))


def cpu_model():
    """lscpu's model name and the host's thread count."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline_both(env_id, cfg, A):
    """The reference's probe loop on the host: MARL_NUM_THREADS = nproc (the
    reported value) and = 1, each on a bounded sample."""
    n_cpu, k_cpu = cpu_sample_size(env_id, cfg)
    threads = os.cpu_count() or 1
    sec, kind, cores, _ = cpu_reference_probe(env_id, cfg, n_cpu, k_cpu, 1, threads)
    n1, k1 = max(64, n_cpu // 4), k_cpu
    sec1, _, _, _ = cpu_reference_probe(env_id, cfg, n1, k1, 1, 1)
    return {"value": n_cpu * A * k_cpu / sec, "unit": "agent-steps/s", "cores": cores, "kind": kind,
            "sample": f"{n_cpu} envs x {k_cpu} steps of {env_id} ({sec:.1f} s, {cores} threads, "
                      "reference VectorEnv::step + random_legal_actions)",
            "single_thread": {"value": n1 * A * k1 / sec1, "cores": 1,
                              "sample": f"{n1} envs x {k1} steps ({sec1:.1f} s, MARL_NUM_THREADS=1)"},
            "cpu_model": cpu_model(), "nproc": threads}


def cpu_sample_size(env_id, cfg):
    """(envs, steps) of a bounded CPU sample of the workload: ~10-30 s for the
    cpu_baseline leg; the envs cap also bounds one reference-arm step (~1 s)."""
    return {"MPE_simple_spread_v3": (1024, 1000), "SMAX_5m_vs_6m": (65536, 40), "SMAX_2s3z": (65536, 5),
            "SMAX_27m_vs_30m": (4096, 4), "overcooked_cramped_room_v0": (65536, 5)}.get(env_id, (1024, 10))


def run_reference_arm(args, rank, world):
    env_id, cfg, n_per_gpu, label = WORKLOADS[args.workload]
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n_envs = n_per_gpu * world
    if args.workload in PPO_WORKLOADS:  # one step = one train_ippo update of a bounded sample
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        n_cpu, t_cpu = (16, 32) if args.workload == "ppo_rnn" else (64, 32)
        steps = max(1, args.steps)
        rc = {"n_envs": n_cpu, "n_rollout_steps": t_cpu, "total_timesteps": n_cpu * t_cpu * steps}
        if args.workload == "ppo_rnn":
            rc["recurrent"] = True
        t0 = time.perf_counter()
        O.ref_train(env_id, cfg, rc, O.key_from_seed(0))
        sec = time.perf_counter() - t0
        val = n_cpu * 3 * t_cpu * steps / sec
        line = {"impl": "reference", "metric": "agent-steps/sec (env-steps/sec x agents)", "value": val,
                "unit": "agent-steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * sec / steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32 nets / f64 env", "data": "synthetic",
                "config": workload_config(args.workload, world),
                "run": {"cpu_sample_envs": n_cpu, "cpu_sample_rollout_steps": t_cpu},
                "cpu_baseline": {"value": val, "unit": "agent-steps/s", "cores": 1, "kind": "reference",
                                 "sample": f"reference train_ippo, {n_cpu} envs x {t_cpu} steps x {steps} updates"},
                "e2e": {"value": val, "unit": "agent-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return
    if args.workload in IPPO_WORKLOADS:  # one step = one collect window of a bounded env sample
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        n_cpu, t_cpu = 256, IPPO_T
        ka, kc = O.ref_ppo_init(env_id, cfg, O.fold_in(O.key_from_seed(0), 10))
        O.ref_collect(env_id, cfg, n_cpu, 4, O.key_from_seed(0), ka, kc)  # warm
        t0 = time.perf_counter()
        O.ref_collect(env_id, cfg, n_cpu, t_cpu, O.key_from_seed(0), ka, kc, n_windows=max(1, args.steps))
        sec = time.perf_counter() - t0
        A = workload_config(args.workload, 1)["agents"]
        val = n_cpu * A * t_cpu * max(1, args.steps) / sec
        line = {"impl": "reference", "metric": "agent-steps/sec (env-steps/sec x agents)", "value": val,
                "unit": "agent-steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * sec / max(1, args.steps), "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32 policy / f64 env", "data": "synthetic",
                "config": workload_config(args.workload, world),
                "run": {"cpu_sample_envs": n_cpu, "cpu_sample_rollout_steps": t_cpu},
                "cpu_baseline": {"value": val, "unit": "agent-steps/s", "cores": 1, "kind": "reference",
                                 "sample": f"reference Collector pieces, {n_cpu} envs x {t_cpu} steps x "
                                           f"{max(1, args.steps)} windows"},
                "e2e": {"value": val, "unit": "agent-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return
    # each step is one batch step of the whole workload on the host cores
    # unless that would not finish within a few minutes; then a bounded sample.
    n_cpu, _ = cpu_sample_size(env_id, cfg)
    n_cpu = min(n_envs, max(n_cpu, 1))
    sec, kind, cores, A = cpu_reference_probe(env_id, cfg, n_cpu, args.steps, args.warmup, threads)
    val = n_cpu * A * args.steps / sec
    line = {"impl": "reference", "metric": "agent-steps/sec (env-steps/sec x agents)", "value": val,
            "unit": "agent-steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sec / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference random-legal action stream)",
            "config": workload_config(args.workload, world),
            "run": {"cpu_sample_envs": n_cpu},
            "cpu_baseline": {"value": val, "unit": "agent-steps/s", "cores": cores, "kind": kind,
                             "sample": f"{n_cpu} envs x {args.steps} steps of {env_id} on {cores} threads"},
            "e2e": {"value": val, "unit": "agent-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# --------------------------------------------------------------------- GPU arm
def run_gpu_arm(args, rank, world, local_rank):
    import torch
    import paper_2311_10090_b200 as m
    from paper_2311_10090_b200 import _native
    from paper_2311_10090_b200 import dist as shard

    env_id, cfg, n_per_gpu, label = WORKLOADS[args.workload]
    if args.n_envs:
        n_per_gpu = args.n_envs
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
    env = m.make_env(env_id, cfg)
    A = env.num_agents()
    N = n_per_gpu * world
    venv = shard.make_sharded(env, N, rank, world, device=local_rank)  # contiguous shard, no step collective
    stream = torch.cuda.current_stream()
    key = m.prng.key_from_seed(0)
    akeys = m.prng.split(m.prng.fold_in(key, 2), args.steps + args.warmup + 2)  # vector_env.cpp:202
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    fused = args.workload in FUSED_PROBE and not args.per_step
    venv.reset(key)
    for t in range(args.warmup):
        if fused:  # the probe kernel itself warms up (module load, caches)
            venv.probe_steps(m.prng.fold_in(key, 2), t, 1)
        else:
            venv.step_random(akeys[t])
        flush.fill_(float(t))
    torch.cuda.synchronize()
    venv.episode_stats(clear=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()

    clocks = ClockSampler(local_rank) if rank == 0 else None
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    fin_counts = torch.zeros(args.steps, dtype=torch.int64, device="cuda")
    launches0 = _native.lib().marl_launch_count()
    if fused:
        # configs[0] is the reference's throughput_probe loop at 1024 envs, launch-
        # bound one launch per step: the K timed steps run as ONE fused launch
        # (marl_venv_probe_steps: state in registers across steps, every output
        # view still written every step); L2 flushed once before it
        flush.fill_(0.0)
        starts[0].record(stream)
        venv.probe_steps(m.prng.fold_in(key, 2), args.warmup, args.steps)
        ends[0].record(stream)
    else:
        for k in range(args.steps):
            flush.fill_(float(k))  # L2 flush between timed steps (not timed); the GPU is busy with it
            starts[k].record(stream)  # while the host enqueues the step, so no launch gap is timed
            r = venv.step_random(akeys[args.warmup + k])
            ends[k].record(stream)
            fin_counts[k] = r.finished.sum()
    torch.cuda.synchronize()
    launches = _native.lib().marl_launch_count() - launches0
    if dist:
        dist.barrier()
    clk = clocks.stop() if clocks else None
    if fused:
        whole = starts[0].elapsed_time(ends[0])
        step_ms = [whole / args.steps] * args.steps
        eps = venv.episode_stats_raw()[0]  # finished episodes over the K steps (shard-local)
        fin_counts = torch.full((args.steps,), eps / args.steps, dtype=torch.float64)
    else:
        step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = float(sum(step_ms))
    total_ms = shard.max_over_ranks(total_ms, device="cuda")  # device time, max over ranks
    stats = shard.all_reduce_episode_stats(venv.episode_stats_raw(), device="cuda")  # the one collective
    value = N * A * args.steps / (total_ms * 1e-3)

    # roofline of the dominant (only) kernel: algorithmic bytes per launch / mean launch time
    finished = fin_counts.cpu().numpy()
    bytes_per_launch = float(np.mean([algorithmic_bytes(env, n_per_gpu, float(f)) for f in finished]))
    mean_launch_s = float(np.mean(step_ms)) * 1e-3
    achieved = bytes_per_launch / mean_launch_s / 1e9
    peak, peak_src = measured_peak()
    traffic = ncu_traffic(args.workload)

    # end-to-end through the C-ABI with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        D = env.obs_dim
        pin = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True).numpy()  # noqa: E731
        host = {"obs": pin((n_per_gpu, A, D), torch.float32), "rewards": pin((n_per_gpu, A), torch.float64),
                "dones": pin((n_per_gpu, A + 1), torch.uint8), "finished": pin((n_per_gpu,), torch.uint8),
                "final_returns": pin((n_per_gpu,), torch.float64), "final_lengths": pin((n_per_gpu,), torch.int32)}
        if env.n_info:
            host["infos"] = pin((n_per_gpu, A, env.n_info), torch.float64)
        dense = sum(a.nbytes for a in host.values())
        # final_obs: valid where finished; the device writes just those rows into the mapped pinned buffer
        host["final_obs"] = pin((n_per_gpu, A, D), torch.float32)
        fin_rows = float(np.mean(finished)) if len(finished) else 0.0
        d2h = dense + fin_rows * A * D * 4
        e2e_steps = max(3, min(args.steps, 20))
        venv.host_step_random(akeys[0], host)  # warm
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for k in range(e2e_steps):
            venv.host_step_random(akeys[1 + k], host)
        sec = time.perf_counter() - t0
        sec = shard.max_over_ranks(sec, device="cuda")
        e2e = {"value": N * A * e2e_steps / sec, "unit": "agent-steps/s",
               "h2d_bytes_per_step": 16, "d2h_bytes_per_step": int(d2h * world),
               "steps": e2e_steps, "path": "marl_venv_step_random_host (C-ABI, pinned host buffers)"}

    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_baseline_both(env_id, cfg, A)
    line = {
        "metric": "agent-steps/sec (env-steps/sec x agents)", "value": value, "unit": "agent-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reset from key_from_seed(0); reference random-legal action stream)",
        "config": workload_config(args.workload, world, n_per_gpu),
        "run": {"parallelism": f"env-sharded x{world}, no step collective",
                "l2": ("flushed once before the fused K-step launch (state stays in registers across its steps)"
                       if fused else "flushed between timed steps (512 MB write, untimed)"),
                "launch": (f"one fused launch of {args.steps} probe steps (marl_venv_probe_steps)" if fused
                           else "one launch per step (marl_venv_step_random)")},
        "env_steps_per_sec": N * args.steps / (total_ms * 1e-3),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "bytes_per_launch": bytes_per_launch, "mean_launch_us": mean_launch_s * 1e6,
                     "kernel": ("fused multi-step probe kernel (per-step bytes; launch time / K)" if fused
                                else "fused step kernel (step_random)"),
                     "ncu": ncu_metrics(args.workload)},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk,
        "episode_stats": shard.summarize(stats),
    }
    print(json.dumps(line))


def self_launch(n):
    """`python bench.py --gpus N` outside torchrun: re-run this command as N
    ranks (one per GPU, NCCL over NVLink, rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the NCCL log shows the N ranks and the transport
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="marl-b200", choices=["marl-b200", "reference"])
    ap.add_argument("--workload", default="smax3m", choices=sorted(WORKLOADS))
    ap.add_argument("--n-envs", type=int, default=0, help="override envs per GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--per-step", action="store_true", help="mpe: one launch per step instead of the fused probe")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args.gpus))  # one rank per GPU under torchrun
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    import torch
    if torch.cuda.device_count() < world:
        sys.exit(f"bench.py: --gpus {world} needs {world} visible GPUs, found {torch.cuda.device_count()}")
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    try:
        if args.workload in IPPO_WORKLOADS:
            run_gpu_ippo(args, rank, world, local_rank)
        elif args.workload in PPO_WORKLOADS:
            run_gpu_ppo(args, rank, world, local_rank)
        else:
            run_gpu_arm(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
