#!/usr/bin/env python
"""Benchmark: env transitions/s of the stock-trading pod rollout on B200.

Contract (see the task statement): ``python bench.py --gpus N --steps K
--warmup W`` (torchrun for N > 1, one rank per GPU) prints ONE JSON line on
rank 0.  A step is one rollout collection (worker_collect, pod.hpp:95-132) of
BASELINE.json configs[1]: 30-asset stock-trading VecEnv x 65,536 envs per GPU,
horizon 256 (16.8M transitions/GPU/step): actor+critic forward, Philox
sampling, env step, rollout-buffer writes and the bootstrap values.  The same
run also measures the env-step kernel alone, one full PPO update on the
collected buffer (GAE + 4 epochs x 1,024-row minibatches + Adam), the
end-to-end public-API path with host buffers, and the reference CPU path
(oracle/_ref, the unmodified reference headers) on the host cores.

``--impl reference`` times only the reference CPU implementation (rank 0).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ["NCCL_DEBUG"] = "WARN"
# Exactly one line on stdout: native libraries (NCCL banners, ...) write to fd 1,
# so fd 1 is pointed at stderr and the JSON line goes to a saved copy of it.
_JSON_OUT = os.fdopen(os.dup(1), "w")
os.dup2(2, 1)


def emit(obj) -> None:
    _JSON_OUT.write(json.dumps(obj) + "\n")
    _JSON_OUT.flush()

METRIC = "env transitions/sec (1/2/4/8 B200, device-timed) vs host-CPU ref; % HBM roofline"
UNIT = "transitions/s"
K_ASSETS, T_ROWS, MARKET_SEED = 30, 2048, 2112
S_DIM = 1 + 6 * K_ASSETS
# algorithmic work per transition
ENV_BYTES = 36 * K_ASSETS + 41  # action 4K + balance 16 + shares 8K + ep_return 16 + obs 4(1+6K) + reward 4 + done 1
BUF_BYTES = 4 * (1 + K_ASSETS) + 4 * K_ASSETS + 4 * 3 + 1  # compact rollout row: obs 124 + act 120 + logp/val/rew 12 + done 1
MLP_FLOPS = 2 * (181 * 64 + 64 * 64 + 64 * 30) + 2 * (181 * 64 + 64 * 64 + 64 * 1)  # 66,688
# What stock_rollout_tc_kernel actually issues to the tensor cores per transition (rollout_tc.cu
# header): layer 1 of both nets as ONE [32 private features x 128] MMA (the 150 shared features'
# term is computed once per step for the whole VecEnv), layer 2 of each net [64 x 64], the actor
# head [64 x 32]; the critic head is a 64-term fp32 dot product on the SIMT pipes.
TC_EXEC_FLOPS = 2 * 32 * 128 + 2 * (2 * 64 * 64) + 2 * 64 * 32  # 28,672
# dram__bytes_read.sum + dram__bytes_write.sum of stock_rollout_tc_kernel<30> from one `ncu --set full`
# capture (profiles/r2_s2_rollout_full.txt: 65,536 envs x 32 steps), per transition; scaled to the launch below.
TC_DRAM_BYTES_PER_TRANSITION = 263  # ncu dram__bytes_read+write.sum per transition, profiles/r2_s2_rollout_full.txt (551.9 MB / 65,536 x 32)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p["bf16_tflops_sustained"], "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region: NVML
    (nvidia_ml_py) polled every 2 ms from a background thread, so even a 30 ms region gets
    samples; nvidia-smi -lms as the fallback when NVML is unavailable."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        self.device, self.rows, self.proc, self.nvml, self.stop_evt = device, [], None, None, threading.Event()
        self.window = None  # (t0, t1) wall times of the timed region; samples outside it are dropped

    def begin(self):
        self.t_begin = time.perf_counter()

    def end(self):
        self.window = (self.t_begin, time.perf_counter())

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.nvml = pynvml

            def poll():
                while not self.stop_evt.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((sm, mx, rs, time.perf_counter()))
                    except Exception:
                        pass
                    self.stop_evt.wait(0.002)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 6 and p[0].replace(".", "").isdigit():
                rs = {n for n, v in zip(names, p[2:6]) if v.lower().startswith("active")}
                self.rows.append((float(p[0]), float(p[1]) if p[1].replace(".", "").isdigit() else None, rs,
                                  time.perf_counter()))

    def stop(self):
        self.stop_evt.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        elif self.nvml is not None:
            self.thread.join(timeout=1)
        return self.summary()

    def summary(self):
        if self.window is not None:  # the sampler runs from before the warm-up: keep the timed region only
            self.rows = [r for r in self.rows if self.window[0] <= r[3] <= self.window[1]]
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows]
        mx = [float(r[1]) for r in self.rows if r[1]]
        reasons = set()
        for r in self.rows:
            if isinstance(r[2], set):
                reasons |= r[2]
            else:
                reasons |= {n for bit, n in self.REASONS.items() if r[2] & bit}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows), "source": "nvml" if self.nvml is not None else "nvidia-smi"}


class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.torch = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(self.local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.torch, self.dist = torch, dist

    def barrier(self):
        if self.torch:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if not self.torch:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.torch:
            self.dist.destroy_process_group()


def market_arrays():
    from paper_2112_05923_b200 import podracer as pr
    m = pr.synthetic_market(K_ASSETS, T_ROWS, MARKET_SEED)
    ind = pr.compute_indicators(m["high"], m["low"], m["close"])
    return m, ind


def ref_inputs(ref):
    """The reference arm's inputs built by the reference build itself (oracle/_ref shim): the
    BASELINE.md §3 synthetic market, compute_indicators (market.hpp:373-392) and
    artifact_init(S, A, seed=7) (artifact.hpp:91-105) -- libprb.so is never loaded on this arm."""
    from oracle_bind import ptr, SZ
    close, high, low = (np.zeros((K_ASSETS, T_ROWS)) for _ in range(3))
    ref.ref_synthetic_market(MARKET_SEED, K_ASSETS, T_ROWS, ptr(close), ptr(high), ptr(low))
    ind = np.zeros((4, K_ASSETS, T_ROWS))
    assert ref.ref_compute_indicators(ptr(high), ptr(low), ptr(close), T_ROWS, K_ASSETS, ptr(ind)) == 0
    hid = np.array([64, 64], dtype=np.uint64)
    P = ref.ref_artifact_init(S_DIM, K_ASSETS, 7, 1e-3, ptr(hid, SZ), 2, None)
    flat = np.zeros(P)
    ref.ref_artifact_init(S_DIM, K_ASSETS, 7, 1e-3, ptr(hid, SZ), 2, ptr(flat))
    return close, ind, flat, hid


REF_ENVS, REF_HORIZON = 1024, 256  # configs[0]: the reference's own CPU-runnable pod shape


def ref_collect_step(ref, inputs, seed: int):
    """ONE whole worker_collect phase of the reference's pod_train (pod.hpp:408-433) on the host
    cores: W = the largest power of two <= cores threads, each owning a VecEnv of 1,024 / W stock
    envs, horizon 256 -- 262,144 transitions of the configs[1] per-transition work (same env, same
    181-64-64-30 / 181-64-64-1 nets).  Returns (seconds, transitions, threads)."""
    from oracle_bind import ptr, SZ
    close, ind, flat, hid = inputs
    cores = os.cpu_count() or 1
    W = min(1 << (cores.bit_length() - 1), REF_ENVS)
    dt = ref.ref_bench_collect(ptr(close), ptr(ind), T_ROWS, K_ASSETS, 0, T_ROWS - 1, W, REF_ENVS // W, REF_HORIZON,
                               ptr(flat), ptr(hid, SZ), 2, seed)
    return dt, W * (REF_ENVS // W) * REF_HORIZON, W


def ref_sample_desc(W, reps, total_tr, total_s):
    return (f"{reps} whole worker_collect phases (pod.hpp:408-433): {W} threads x {REF_ENVS // W} stock envs x "
            f"horizon {REF_HORIZON} = {REF_ENVS * REF_HORIZON} transitions each ({total_tr} transitions, "
            f"{total_s:.1f} s), 64x64 actor/critic, f64, unmodified reference headers -O3 -march=x86-64-v3")


def cpu_reference_rate(seconds: float):
    """cpu_baseline: whole configs[0]-sized reference collects (ref_collect_step) repeated for
    about `seconds` on the host cores."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import REF_BENCH_SO, load_ref
    ref = load_ref(REF_BENCH_SO)
    if ref is None:
        return None
    inputs = ref_inputs(ref)
    total_s, total_tr, reps = 0.0, 0, 0
    while total_s < seconds or reps < 1:
        dt, tr, W = ref_collect_step(ref, inputs, 2112 + reps)
        total_s += dt
        total_tr += tr
        reps += 1
    return {"value": total_tr / total_s, "unit": UNIT, "cores": W, "kind": "reference",
            "sample": ref_sample_desc(W, reps, total_tr, total_s)}


def run_reference(args, d: Dist):
    """--impl reference: the reference's own CPU path (oracle/_ref/libpodracer_ref_bench.so, the
    unmodified headers) on the host cores, rank 0 only.  A step is one whole worker_collect
    phase of a configs[0]-sized pod (1,024 envs x 256); nothing is projected."""
    if d.rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import REF_BENCH_SO, load_ref
    ref = load_ref(REF_BENCH_SO)
    if ref is None:
        emit({"impl": "reference", "unavailable": "oracle/_ref/libpodracer_ref_bench.so not built"})
        return
    inputs = ref_inputs(ref)
    times, trs = [], []
    for i in range(args.warmup + args.steps):
        dt, tr, W = ref_collect_step(ref, inputs, 2112 + i)
        if i >= args.warmup:
            times.append(dt)
            trs.append(tr)
    total_s, total_tr = float(sum(times)), int(sum(trs))
    value = total_tr / total_s
    cb = {"value": value, "unit": UNIT, "cores": W, "kind": "reference",
          "sample": ref_sample_desc(W, len(times), total_tr, total_s)}
    cfg = config_dict(args)
    cfg.update({"workload": f"reference worker_collect, configs[0]-sized sample of the configs[1] workload: "
                            f"stock-trading VecEnv {K_ASSETS} assets x {REF_ENVS} envs ({W} threads x "
                            f"{REF_ENVS // W}), horizon {REF_HORIZON}, one whole collect per step",
                "envs_per_gpu": None, "envs": REF_ENVS, "horizon": REF_HORIZON,
                "parallelism": f"{W} host threads (rank 0 only)",
                "l2": "host CPU path (no GPU)"})
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_s / len(times) * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (BASELINE.md §3 market and artifact_init weights, built by the reference build)",
           "config": cfg, "cpu_baseline": cb,
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)


def config_dict(args):
    return {"workload": f"configs[1]: single-pod PPO rollout, stock-trading VecEnv {K_ASSETS} assets x "
                        f"{args.envs} envs/GPU, horizon {args.horizon}",
            "assets": K_ASSETS, "envs_per_gpu": args.envs, "horizon": args.horizon, "market_rows": T_ROWS,
            "actor_critic": "181-64-64-30 / 181-64-64-1 tanh", "parallelism": f"replicas x{args.gpus} (one pod per GPU)",
            "l2": "no flush: each step writes a %.1f GB rollout buffer >> 126 MB L2" % (
                args.envs * args.horizon * (4 * (1 + K_ASSETS) + 4 * K_ASSETS + 13) / 1e9)}


def run_ours(args, d: Dist):
    from paper_2112_05923_b200 import podracer as pr
    lib = pr._lib.lib()
    hbm, bf16, bf16_sus, peak_src = load_peaks()
    ctx = pr.Context(d.local)
    m, ind = market_arrays()
    market = pr.MarketData(ctx, m["close"], ind)
    cfg = pr.StockConfig()
    N, H = args.envs, args.horizon
    env = pr.VectorizedEnvironment.stock(ctx, market, cfg, 0, T_ROWS - 1, N)
    env.reset(2112 + d.rank)
    agent = pr.Agent.init(ctx, S_DIM, K_ASSETS, seed=7 + d.rank)
    ro = pr.Rollout.for_env(env, H)

    # ---- warm-up (the clock sampler is already polling, so it is warm when the region starts) ----
    clocks = ClockSampler(d.local)
    clocks.start()
    for i in range(args.warmup):
        ro.collect(agent, env, seed=1000 + i)
    ctx.synchronize()

    # ---- timed region: K rollout collections, CUDA events on the launching stream ----
    lib.prb_ctx_profile(ctx.h, 1)  # per-kernel event pairs inside the region (kernel shares / roofline)
    d.barrier()
    ctx.synchronize()
    clocks.begin()
    dev_ms = time_region(lib, ctx, lambda: [ro.collect(agent, env, seed=2000 + i) for i in range(args.steps)])
    clocks.end()
    clk = clocks.stop()
    prof = {}
    for name, kind in (("policy_fwd_sample", 0), ("env_stock_step", 1), ("stock_rollout_fused", 7)):
        ms, n = C.c_double(), C.c_uint64()
        lib.prb_ctx_profile_read(ctx.h, kind, C.byref(ms), C.byref(n))
        prof[name] = (ms.value, n.value)
    lib.prb_ctx_profile(ctx.h, 0)
    d.barrier()
    dev_ms = d.max(dev_ms)
    transitions = d.world * args.steps * N * H
    value = transitions / (dev_ms / 1e3)

    # ---- roofline of the dominant kernel (algorithmic work per launch / average launch time) ----
    kernels = {}
    region_ms = dev_ms
    for name, (ms, n) in prof.items():
        if n == 0:
            continue
        avg_s = ms / n / 1e3
        if name == "policy_fwd_sample":
            k = {"bound": "tensor", "unit": "TFLOP/s", "achieved": N * MLP_FLOPS / avg_s / 1e12, "peak": bf16_sus,
                 "work_per_launch": f"{N} rows x {MLP_FLOPS} FLOP"}
        elif name == "env_stock_step":
            k = {"bound": "hbm", "unit": "GB/s", "achieved": N * ENV_BYTES / avg_s / 1e9, "peak": hbm,
                 "work_per_launch": f"{N} envs x {ENV_BYTES} B"}
        else:
            # one launch is a ~4 ms collect inside a ~80 ms region: the burst bf16 peak applies
            k = {"bound": "tensor", "unit": "TFLOP/s", "achieved": N * H * MLP_FLOPS / avg_s / 1e12, "peak": bf16,
                 "work_per_launch": f"{N}x{H} transitions x {MLP_FLOPS} FLOP (algorithmic actor+critic fwd)",
                 "executed_tensor_tflops": N * H * TC_EXEC_FLOPS / avg_s / 1e12,
                 "executed_tensor_flop_per_transition": TC_EXEC_FLOPS,
                 "executed_note": "the kernel issues 28,672 tensor FLOP per transition: layer 1 over the 31 "
                                  "private features (K=32), the 150 shared features' term once per step per VecEnv",
                 "hbm_gbs": N * H * BUF_BYTES / avg_s / 1e9, "hbm_frac": N * H * BUF_BYTES / avg_s / 1e9 / hbm,
                 "hbm_bytes_per_transition": BUF_BYTES}
        k.update({"ms_total": ms, "launches": n, "share": ms / region_ms, "frac": k["achieved"] / k["peak"]})
        kernels[name] = k
    dom = max(kernels, key=lambda k: kernels[k]["ms_total"])
    kd = kernels[dom]
    roofline = {"kernel": dom, "bound": kd["bound"], "achieved": kd["achieved"], "peak": kd["peak"],
                "unit": kd["unit"], "frac": kd["frac"],
                "traffic": (N * H * TC_DRAM_BYTES_PER_TRANSITION if dom == "stock_rollout_fused" else None),
                "traffic_source": "ncu dram bytes/transition, profiles/r2_s2_rollout_full.txt, x transitions per launch",
                "peak_source": f"{peak_src} (MEASURED_PEAKS.json "
                               f"{'bf16_tflops (burst)' if kd['bound'] == 'tensor' else 'hbm_gbs'})"}
    if dom == "stock_rollout_fused":
        # neither the tensor nor the HBM roof binds this kernel (both < 20%): per-thread instruction
        # issue does -- the fp64 portfolio chain + sampling + epilogues; ncu of the same kernel
        roofline["limiter"] = ("instruction issue/latency: ~3.2K instructions per transition, ~50% issue-active "
                               "at the 16 warps/SM that TMEM (128 cols/CTA) and registers allow "
                               "(profiles/r2_s2_rollout_full.txt, DESIGN.md section 3)")

    # ---- env step alone (the VecEnv boundary) at configs[4] scale: 1M envs/GPU, > L2 ----
    env_step = env_leg(pr, lib, ctx, market, cfg, args.env_envs, hbm, d)

    # ---- the GAE reverse scan alone on the collected configs[1] buffer (HBM-bound) ----
    gae = gae_leg(lib, ctx, ro, N, H, hbm, d)
    # ---- Adam alone on an agent larger than L2 (HBM-bound) ----
    adam = adam_leg(pr, lib, ctx, hbm, d)

    # ---- one full PPO update on the collected buffer (GAE + epochs x minibatches + Adam) ----
    ppo = None
    if not args.skip_ppo:
        pcfg = pr.PpoConfig(minibatch_size=1024, epochs_per_update=args.ppo_epochs, buffer_size=N * H)
        out_agent = pr.Agent(ctx, S_DIM, K_ASSETS)
        res = {}

        def upd():
            res["stats"] = pr.ppo_update(agent, ro, pcfg, seed=9, out=out_agent)[1]
        ppo_ms = time_region(lib, ctx, upd)
        coll_ms = dev_ms / args.steps
        st = res["stats"]
        ppo = {"update_ms": ppo_ms, "minibatches": st.minibatches, "ms_per_minibatch": ppo_ms / max(st.minibatches, 1),
               "epochs": args.ppo_epochs, "minibatch_size": 1024,
               "iteration_transitions_per_s": N * H / ((coll_ms + ppo_ms) / 1e3),
               "mean_policy_loss": st.mean_policy_loss, "mean_value_loss": st.mean_value_loss}

    # ---- the other BASELINE configs, measured in the same run (not the headline) ----
    other = {}
    if not args.skip_configs:
        other["configs[2]_pointmass"] = leg_pointmass(pr, lib, ctx, args.pm_envs, args.pm_horizon, d)
        other["configs[4]_stock_1M"] = leg_stock_large(pr, lib, ctx, market, cfg, args.c5_envs, H, d)
    if not args.skip_configs:
        other["configs[3]_tournament"] = leg_tournament(pr, ctx, market, cfg, d, args.pods_per_gpu)
    if not args.skip_configs:
        other["configs[0]_iteration"] = leg_c1_iteration(pr, lib, ctx, market, cfg, m, ind, d,
                                                         with_cpu=(d.rank == 0 and d.world == 1 and not args.skip_cpu))

    # ---- end to end through the public API with host buffers ----
    # Every step: pinned h2d of the params, worker_collect, d2h of the step's 16.8M rewards.
    # Two rollout buffers alternate and the reward copy runs on a second context's stream,
    # so the d2h of step i overlaps the collect of step i+1 (prb_rollout_collect returns
    # when its kernels are done; a buffer is reused only after its copy has completed).
    P = agent.param_count
    host_params = np.ascontiguousarray(agent.flatten_params().astype(np.float32))
    d_params = lib.prb_agent_params_device(agent.h)
    ro2 = pr.Rollout.for_env(env, H)
    ro2.set_mode(2)
    ctx_copy = [pr.Context(d.local), pr.Context(d.local)]  # one copy stream per buffer
    d_rw = []
    for r_ in (ro, ro2):
        p_ = C.c_void_p()
        lib.prb_rollout_device_fields(r_.h, None, None, None, C.byref(p_), None, None, None)
        d_rw.append(p_.value)
    nrew = N * H * 4
    pin = pinned(host_params.nbytes + 2 * nrew)
    hp = np.frombuffer(pin, dtype=np.float32, count=P)
    hr = [np.frombuffer(pin, dtype=np.float32, count=N * H, offset=host_params.nbytes + j * nrew) for j in range(2)]
    hp[:] = host_params
    ros = (ro, ro2)

    def e2e_steps():
        for i in range(args.steps):
            j = i % 2
            if i >= 2:
                ctx_copy[j].synchronize()  # buffer j's previous copy (step i-2) has landed
            lib.prb_memcpy_h2d_async(ctx.h, d_params, hp.ctypes.data, hp.nbytes)
            lib.prb_rollout_collect(ros[j].h, agent.h, env.h, 4000 + i)
            lib.prb_memcpy_d2h_async(ctx_copy[j].h, hr[j].ctypes.data, d_rw[j], nrew)
        ctx.synchronize()
        for c_ in ctx_copy:
            c_.synchronize()
    e2e_steps()  # warm the second buffer
    d.barrier()
    t0 = time.perf_counter()
    e2e_steps()
    e2e_s = d.max(time.perf_counter() - t0)
    del ro2
    e2e = {"value": transitions / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(hp.nbytes),
           "d2h_bytes_per_step": int(nrew),
           "note": "host wall clock: pinned h2d params + collect + d2h of all rewards each step; the d2h of "
                   "step i overlaps the collect of step i+1 (two rollout buffers, one copy stream each)"}

    # ---- CPU baseline: the reference path on this box's host cores (rank 0, N=1 only) ----
    cpu = None
    if d.rank == 0 and d.world == 1 and not args.skip_cpu:
        cpu = cpu_reference_rate(seconds=args.cpu_seconds)

    # kernel launches in the timed region: fused collect = shared-layer kernel + fused kernel
    launches = int(prof["policy_fwd_sample"][1] + prof["env_stock_step"][1] + 2 * prof["stock_rollout_fused"][1])
    if d.rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": d.world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "bf16 tcgen05 MLP (fp32 accum) + fp64 accounting",
               "data": "synthetic (BASELINE.md §3 market, random-init artifact_init weights)",
               "config": config_dict(args), "roofline": roofline, "kernels": kernels, "env_step": env_step,
               "gae": gae, "adam": adam, "ppo_update": ppo, "other_configs": other, "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches,
               "clocks": clk}
        emit((out))
    d.close()


def leg_pointmass(pr, lib, ctx, n_envs, horizon, d):
    """configs[2]: PointMass2D (SPEC.md analytic control env) x 262,144 envs, actor/critic 3x256."""
    env = pr.VectorizedEnvironment.pointmass(ctx, n_envs)
    env.reset(7)
    agent = pr.Agent.init(ctx, 6, 2, seed=7, hidden=(256, 256, 256))
    ro = pr.Rollout.for_env(env, horizon)
    ro.collect(agent, env, seed=1)
    ms = d.max(time_region(lib, ctx, lambda: ro.collect(agent, env, seed=2)))
    flops = 2 * (6 * 256 + 256 * 256 * 2 + 256 * 2) + 2 * (6 * 256 + 256 * 256 * 2 + 256)
    rate = n_envs * horizon / (ms / 1e3)
    tflops = rate * flops / 1e12
    return {"value": d.world * rate, "unit": UNIT, "envs_per_gpu": n_envs, "horizon": horizon, "ms_per_collect": ms,
            "mlp_tflops": tflops, "tensor_frac": tflops / load_peaks()[2],
            "flop_per_transition": flops,
            "path": "rollout_pm_tc.cu: persistent tcgen05 3x256 actor/critic, bf16 weights streamed from L2 "
                    "through a 5-slot bulk-copy ring, fp64 PointMass step + mt19937_64 resets in the same kernel"}


def leg_c1_iteration(pr, lib, ctx, market, cfg, m, ind, d, with_cpu: bool):
    """configs[0] (the reference's CPU-runnable case): one full PPO iteration of a pod --
    collect 1,024 stock envs x 256 steps, GAE, 4 epochs x 256 minibatches of 1,024 with Adam
    (pod.hpp:408-461) -- on the GPU, next to the reference on the host cores: its threaded
    worker_collect timed in full and its ppo_update timed on 32 minibatches and scaled."""
    N1, H1, EP, MB = 1024, 256, 4, 1024
    env = pr.VectorizedEnvironment.stock(ctx, market, cfg, 0, T_ROWS - 1, N1)
    env.reset(3)
    agent = pr.Agent.init(ctx, S_DIM, K_ASSETS, seed=7)
    ro = pr.Rollout.for_env(env, H1)
    pcfg = pr.PpoConfig(minibatch_size=MB, epochs_per_update=EP, buffer_size=N1 * H1)

    def iteration(i):
        ro.collect(agent, env, seed=100 + i)
        pr.ppo_update(agent, ro, pcfg, seed=200 + i, out=agent)
    iteration(0)
    ms = d.max(time_region(lib, ctx, lambda: [iteration(i) for i in (1, 2, 3)])) / 3
    # the reference pod's own iteration shape: num_learners = 2 (config.hpp PodConfig) concurrent
    # learners + fuse_parameters (pod.hpp:436-461) -- here both learners in one tensor-core launch
    outs = [pr.Agent(ctx, S_DIM, K_ASSETS), pr.Agent(ctx, S_DIM, K_ASSETS)]

    def pod_iteration(i):
        ro.collect(agent, env, seed=300 + i)
        pr.ppo_update_learners([agent, agent], [ro, ro], pcfg, [400 + i, 500 + i], outs=outs)
        pr.fuse_parameters(outs, out=agent)
    pod_iteration(0)
    ms2 = d.max(time_region(lib, ctx, lambda: [pod_iteration(i) for i in (1, 2, 3)])) / 3
    out = {"workload": "configs[0]: 30 assets x 1,024 envs, horizon 256, 4 epochs x 256 minibatches of 1,024",
           "gpu_ms_per_iteration": ms, "gpu_transitions_per_s": N1 * H1 / (ms / 1e3),
           "gpu_ms_per_iteration_2_learners": ms2,
           "two_learners_note": "collect + 2 concurrent tensor-core learners + fuse (the reference pod's "
                                "num_learners = 2); gpu_ms_per_iteration is collect + 1 fp32 SIMT learner"}
    if with_cpu:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle_bind import REF_BENCH_SO, load_ref, ptr, SZ
        ref = load_ref(REF_BENCH_SO)
        if ref is not None:
            cores = os.cpu_count() or 1
            W = 1 << (cores.bit_length() - 1)
            flat = pr.artifact_init(S_DIM, K_ASSETS, 7)
            hid = np.array([64, 64], dtype=np.uint64)
            close = np.ascontiguousarray(m["close"]); indc = np.ascontiguousarray(ind)
            col_s = ref.ref_bench_collect(ptr(close), ptr(indc), T_ROWS, K_ASSETS, 0, T_ROWS - 1, W, N1 // W, H1,
                                          ptr(flat), ptr(hid, SZ), 2, 2112)
            nmb = 32
            ppo_s = ref.ref_bench_ppo(ptr(flat), S_DIM, K_ASSETS, ptr(hid, SZ), 2, nmb * MB, H1, MB, 1, 7)
            cpu_ms = (col_s + ppo_s / nmb * EP * (N1 * H1 // MB)) * 1e3
            out.update({"cpu_ms_per_iteration": cpu_ms, "cpu_cores": W,
                        "cpu_sample": f"worker_collect {W} threads x {N1 // W} envs x {H1} measured ({col_s:.2f} s); "
                                      f"ppo_update 1 epoch x {nmb} minibatches measured ({ppo_s:.2f} s) and scaled to "
                                      f"{EP * N1 * H1 // MB} (single-threaded, as one learner)",
                        "speedup_gpu_vs_cpu": cpu_ms / ms})
    del ro
    return out


def leg_stock_large(pr, lib, ctx, market, cfg, n_envs, horizon, d):
    """configs[4] per-GPU scale: 1,048,576 stock envs x 256 steps (compact rollout rows, 69 GB)."""
    env = pr.VectorizedEnvironment.stock(ctx, market, cfg, 0, T_ROWS - 1, n_envs)
    env.reset(11)
    agent = pr.Agent.init(ctx, S_DIM, K_ASSETS, seed=7)
    ro = pr.Rollout.for_env(env, horizon)
    ro.collect(agent, env, seed=1)
    ms = d.max(time_region(lib, ctx, lambda: ro.collect(agent, env, seed=2)))
    rate = n_envs * horizon / (ms / 1e3)
    del ro
    return {"value": d.world * rate, "unit": UNIT, "envs_per_gpu": n_envs, "horizon": horizon, "ms_per_collect": ms,
            "rollout_gb_per_gpu": n_envs * horizon * BUF_BYTES / 1e9}


def leg_tournament(pr, ctx, market, cfg, d, pods, learners=2, gens=2):
    """configs[3]: one GPU's pod population, a REAL generation timed end to end: every pod's collect
    in one grouped tcgen05 launch (configs[0]-sized pods: 1,024 stock envs x 256 steps), every pod's
    `learners` PPO learners (4 epochs x 256 minibatches of 1,024) in one tensor-core launch (8
    co-resident CTAs per learner), per-pod fusion, evaluation (10 episodes of 40 steps), the NCCL all-gather
    ranking over every rank's pods and the top-3 elite broadcasts + device mutations
    (tournament.PodPopulation, tournament.hpp:395-506).  Host wall clock around each generation
    (max over ranks); the learners alone are also timed against the fp32 SIMT update run serially."""
    from paper_2112_05923_b200 import tournament as tn
    comm = None
    if d.world > 1:
        def share(b):
            obj = [b]
            d.dist.broadcast_object_list(obj, src=0)
            return obj[0]
        comm = tn.Communicator(ctx, d.rank, d.world, share)
    N, H = 1024, 256
    pcfg = pr.PpoConfig(minibatch_size=1024, epochs_per_update=4, buffer_size=N * H)
    pop = tn.PodPopulation(ctx, market, cfg, pods=pods, envs_per_pod=N, horizon=H, learners=learners, ppo_cfg=pcfg,
                           window=(0, T_ROWS - 1), eval_episodes=10, eval_window=(1900, 1940), capacity=10, top_k=3,
                           seed=2112, rank=d.rank, world=d.world, comm=comm)
    pop.generation()  # warm-up (workspaces, first-touch)
    times = []
    for _ in range(gens):
        d.barrier()
        ctx.synchronize()
        t0 = time.perf_counter()
        out = pop.generation()
        ctx.synchronize()
        times.append(d.max(time.perf_counter() - t0))
    # the learner phase alone: concurrent tensor-core learners vs the SIMT update one after another
    srcs = [a for a in pop.agents for _ in range(learners)]
    ros = [r for r in pop.rollouts for _ in range(learners)]
    outs = [o for lo in pop.learner_out for o in lo]
    pr.ppo_update_learners(srcs, ros, pcfg, list(range(len(srcs))), outs=outs)
    ctx.synchronize()
    t0 = time.perf_counter()
    pr.ppo_update_learners(srcs, ros, pcfg, list(range(len(srcs))), outs=outs)
    ctx.synchronize()
    learn_tc = time.perf_counter() - t0
    for l in range(2):  # warm: the SIMT update's workspace on these destinations (ppo_mode 0: SIMT)
        pr.ppo_update(srcs[l], ros[l], pcfg, l, out=outs[l])
    ctx.synchronize()
    t0 = time.perf_counter()
    for l in range(2):  # two serial SIMT learners, scaled to all of them
        pr.ppo_update(srcs[l], ros[l], pcfg, l, out=outs[l])
    ctx.synchronize()
    learn_simt = (time.perf_counter() - t0) / 2 * len(srcs)
    if comm is not None:
        comm.close()
    gen_s = float(np.median(times))
    trans = pods * N * H
    return {"pods_per_gpu": pods, "pods_total": pods * d.world, "learners_per_pod": learners,
            "pod": f"{N} stock envs x {H} steps, 4 epochs x {N * H // 1024} minibatches of 1,024 per learner",
            "ms_per_generation": 1e3 * gen_s,
            "transitions_per_s": d.world * trans / gen_s,
            "learner_phase_ms": 1e3 * learn_tc, "learner_phase_ms_simt_serial": 1e3 * learn_simt,
            "learner_speedup_vs_simt_serial": learn_simt / learn_tc,
            "board_top3": out["board"][:3], "fresh_inits": out["fresh"],
            "what": "grouped collect + concurrent tcgen05 learners + fusion + evaluation + all-gather ranking + "
                    "elite broadcast/mutation; host-timed per generation (max over ranks)"}


GAE_BYTES = 4 + 4 + 1 + 4 + 4  # read reward, value, done; write advantage, return (stats fused in the pass)


def gae_leg(lib, ctx, ro, N, H, hbm, d, reps=10):
    """buffer_advantages (ppo.hpp:212-244) on the collected N x H buffer: the reverse GAE scan,
    one thread per env walking its time-major column, fp64 recursion, normalisation stats fused."""
    lib.prb_gae(ro.h, 0.99, 0.95, 1)
    lib.prb_ctx_profile(ctx.h, 1)
    region = d.max(time_region(lib, ctx, lambda: [lib.prb_gae(ro.h, 0.99, 0.95, 1) for _ in range(reps)]))
    ms, n = C.c_double(), C.c_uint64()
    lib.prb_ctx_profile_read(ctx.h, 3, C.byref(ms), C.byref(n))  # PRB_PROF_GAE
    lib.prb_ctx_profile(ctx.h, 0)
    avg_s = ms.value / max(n.value, 1) / 1e3
    gbs = N * H * GAE_BYTES / avg_s / 1e9
    return {"transitions_per_s": d.world * N * H / avg_s, "kernel_avg_us": avg_s * 1e6, "achieved_gbs": gbs,
            "frac_hbm": gbs / hbm, "bytes_per_transition": GAE_BYTES, "region_ms_per_call": region / reps,
            "buffer": f"{N} envs x {H} steps ({N * H * GAE_BYTES / 1e6:.0f} MB > L2)"}


def adam_leg(pr, lib, ctx, hbm, d, reps=20):
    """adam_step (nn.hpp:164-182) through prb_adam_step_device on an agent whose
    params + m + v + grads (16 B/param) exceed L2: grid-wide finite gate, then the update."""
    agent = pr.Agent.init(ctx, 4096, 2, seed=1, hidden=(1024, 1024))  # 10.5M params, 168 MB of state
    P = agent.param_count
    g = pr.DeviceArray.from_numpy(ctx, np.random.default_rng(0).normal(size=P).astype(np.float32) * 1e-3)
    agent.adam_step_device(g.ptr)
    lib.prb_ctx_profile(ctx.h, 1)
    region = d.max(time_region(lib, ctx, lambda: [lib.prb_adam_step_device(agent.h, C.c_void_p(g.ptr))
                                                  for _ in range(reps)]))
    ms, n = C.c_double(), C.c_uint64()
    lib.prb_ctx_profile_read(ctx.h, 6, C.byref(ms), C.byref(n))  # PRB_PROF_ADAM
    lib.prb_ctx_profile(ctx.h, 0)
    out = {"params": P, "bytes_per_param": 28, "region_ms_per_step": region / reps,
           "note": "28 B/param = read p, g, m, v + write p, m, v (fp32); the finite check re-reads g (L2)"}
    if n.value:
        avg_s = ms.value / n.value / 1e3
        out.update({"kernel_avg_us": avg_s * 1e6, "achieved_gbs": P * 28 / avg_s / 1e9,
                    "frac_hbm": P * 28 / avg_s / 1e9 / hbm})
    step_s = region / reps / 1e3
    out.update({"step_gbs": P * 28 / step_s / 1e9, "step_frac_hbm": P * 28 / step_s / 1e9 / hbm})
    return out


def env_leg(pr, lib, ctx, market, cfg, n_envs, hbm, d, steps=50):
    """prb_vecenv_step on device buffers: n_envs stock envs, U(-1.2,1.2) fp32 actions resident in HBM."""
    env = pr.VectorizedEnvironment.stock(ctx, market, cfg, 0, T_ROWS - 1, n_envs)
    env.reset(5)
    rng = np.random.default_rng(0)
    acts = [pr.DeviceArray.from_numpy(ctx, rng.uniform(-1.2, 1.2, (n_envs, K_ASSETS)).astype(np.float32))
            for _ in range(2)]
    d_rew, d_done = ctx.alloc((n_envs,)), ctx.alloc((n_envs,), np.uint8)
    for i in range(3):
        env.step_device(acts[i % 2].ptr, d_rew.ptr, d_done.ptr)
    lib.prb_ctx_profile(ctx.h, 1)
    region = time_region(lib, ctx, lambda: [env.step_device(acts[i % 2].ptr, d_rew.ptr, d_done.ptr)
                                            for i in range(steps)])
    ms, n = C.c_double(), C.c_uint64()
    lib.prb_ctx_profile_read(ctx.h, 1, C.byref(ms), C.byref(n))
    lib.prb_ctx_profile(ctx.h, 0)
    region = d.max(region)
    kern_rate = n_envs * n.value / (ms.value / 1e3)
    rate = n_envs * steps / (region / 1e3)
    return {"value": d.world * rate, "unit": UNIT, "envs_per_gpu": n_envs, "steps": steps,
            "kernel_avg_us": ms.value / max(n.value, 1) * 1e3,
            "achieved_gbs": kern_rate * ENV_BYTES / 1e9, "frac_hbm": kern_rate * ENV_BYTES / 1e9 / hbm,
            "bytes_per_transition": ENV_BYTES,
            "note": "obs [N][181] fp32 written every step (VecStepResult.next_states); state/actions > L2"}


def time_region(lib, ctx, fn) -> float:
    """Device milliseconds of everything fn() enqueues on ctx's stream (CUDA events, sync both sides)."""
    cudart = _cudart()
    stream = C.c_void_p(ctx.stream)
    a, b = C.c_void_p(), C.c_void_p()
    cudart.cudaEventCreate(C.byref(a))
    cudart.cudaEventCreate(C.byref(b))
    ctx.synchronize()
    cudart.cudaEventRecord(a, stream)
    fn()
    cudart.cudaEventRecord(b, stream)
    cudart.cudaEventSynchronize(b)
    ms = C.c_float()
    cudart.cudaEventElapsedTime(C.byref(ms), a, b)
    cudart.cudaEventDestroy(a)
    cudart.cudaEventDestroy(b)
    return float(ms.value)


_CUDART = None


def _cudart():
    global _CUDART
    if _CUDART is None:
        for name in ("libcudart.so.12", "libcudart.so", "/usr/local/cuda/lib64/libcudart.so.12"):
            try:
                _CUDART = C.CDLL(name)
                break
            except OSError:
                continue
        if _CUDART is None:
            raise RuntimeError("libcudart not found")
        _CUDART.cudaEventRecord.argtypes = [C.c_void_p, C.c_void_p]
        _CUDART.cudaEventSynchronize.argtypes = [C.c_void_p]
        _CUDART.cudaEventElapsedTime.argtypes = [C.POINTER(C.c_float), C.c_void_p, C.c_void_p]
        _CUDART.cudaEventDestroy.argtypes = [C.c_void_p]
        _CUDART.cudaHostAlloc.argtypes = [C.POINTER(C.c_void_p), C.c_size_t, C.c_uint]
    return _CUDART


def pinned(nbytes: int):
    p = C.c_void_p()
    rc = _cudart().cudaHostAlloc(C.byref(p), nbytes, 0)
    if rc != 0:
        raise RuntimeError(f"cudaHostAlloc failed ({rc})")
    return (C.c_char * nbytes).from_address(p.value)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--envs", type=int, default=65536)
    ap.add_argument("--horizon", type=int, default=256)
    ap.add_argument("--ppo-epochs", type=int, default=4)
    ap.add_argument("--env-envs", type=int, default=1 << 20)
    ap.add_argument("--skip-configs", action="store_true")
    ap.add_argument("--pm-envs", type=int, default=262144)
    ap.add_argument("--pm-horizon", type=int, default=256)
    ap.add_argument("--c5-envs", type=int, default=1 << 20)
    ap.add_argument("--pods-per-gpu", type=int, default=8)
    ap.add_argument("--skip-ppo", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    d = Dist()
    if args.impl == "reference":
        run_reference(args, d)
        d.close()
        return
    run_ours(args, d)


if __name__ == "__main__":
    main()
