#!/usr/bin/env python3
"""Benchmark: whole-box PPO training env-steps/s on B200 (BASELINE.json `metric`).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config configs/at_4096env_3x256.cfg]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1, one rank per GPU)
    python bench.py --impl reference ...                        (CPU reference arm)

A step is one PPO iteration of the data-parallel TCG_EX job: every env of every GMI
advances `horizon` steps (rollout), then `epochs` x `minibatches` PPO updates with the
cross-GMI / cross-GPU gradient reduction.  Default workload = BASELINE configs[1]
(AT-like, 4096 envs per GPU, 3x256 MLP, 1 GMI per B200).  Envs shard across ranks
([N*c/n, N*(c+1)/n)); the only data-path collective is the per-minibatch gradient
all-reduce.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PPO training env-steps/sec (whole box)"
UNIT = "env-steps/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default=os.path.join(ROOT, "configs", "at_4096env_3x256.cfg"))
    p.add_argument("--gmis", type=int, default=0, help="override GMIs per GPU")
    p.add_argument("--envs", type=int, default=0, help="override envs per GPU")
    p.add_argument("--backend", type=int, default=None, help="0 streams, 1 green contexts (default: config)")
    p.add_argument("--decoupled", type=int, default=None,
                   help="1: serving GMI + trainer GMI per GPU with an experience channel (BASELINE config 4)")
    p.add_argument("--serving-sms", type=int, default=0, help="SMs of the serving GMI (decoupled mode)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-multi-gmi", action="store_true",
                   help="skip the decoupled multi-GMI layout measured beside the single-context one")
    p.add_argument("--cpu-sample-envs", type=int, default=64)
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ clocks during the timed region
class ClockSampler:
    """Samples SM clock and throttle reasons every `period` s on a thread (NVML), falling
    back to `nvidia-smi -lms` when NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, device: int = 0, period: float = 0.01):
        import threading
        self.device, self.period = device, period
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._thread = None
        self._nvml = None

    def _run(self):
        nv = self._nvml
        h = nv.nvmlDeviceGetHandleByIndex(self.device)
        self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            mask = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            for name, attr in self.REASONS:
                if mask & getattr(nv, attr, 0):
                    self.reasons.add(name)
            time.sleep(self.period)

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
        except Exception:  # noqa: BLE001 - no NVML: clocks reported as unavailable
            return
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()

    def stop(self):
        if self._thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self._stop.set()
        self._thread.join(timeout=5)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"], "samples": 0}
        loaded = [x for x in self.samples if x > 0.5 * (self.max_mhz or max(self.samples))] or self.samples
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml"}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return j["bf16_tflops_sustained"], j["hbm_gbs"], "measured (MEASURED_PEAKS.json: sustained bf16, HBM copy)"
    except (OSError, KeyError, ValueError):
        return 1400.0, 6650.0, "fallback (B200_PROFILING.md)"


def gemm_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per gemm_tcgen05_kernel launch, from the
    committed ncu --set full capture (profiles/traffic.json); None when absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)["gemm_tcgen05_kernel"]["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


GEMM_PHASES = ("roll_gemm", "roll_head", "val_gemm", "val_head", "fwd_gemm", "head_fwd", "head_dx", "head_dw",
               "dw_gemm", "dx_gemm")


def phase_table(prof: dict, iter_ms: float, peak_tf: float, peak_gbs: float) -> dict:
    """Per-phase device time per iteration (GMI 0 + update stream, CUDA events around every
    launch) with the roofline each phase is bound by: tensor (algorithmic flops / time) or
    HBM (algorithmic bytes / time)."""
    out = {}
    for name, p in prof.items():
        if p["launches"] == 0:
            continue
        row = {"ms": round(p["ms"], 4), "share": round(p["ms"] / iter_ms, 4) if iter_ms else None,
               "launches": p["launches"]}
        ridge = peak_tf * 1e12 / (peak_gbs * 1e9)  # flop per byte where the two roofs meet
        if p["flop"] > 0 and p["ms"] > 0:
            tf = p["flop"] / (p["ms"] / 1e3) / 1e12
            row.update(achieved_tflops=round(tf, 1))
            if p["bytes"] > 0:
                gbs = p["bytes"] / (p["ms"] / 1e3) / 1e9
                row.update(achieved_gbs=round(gbs, 1), intensity=round(p["flop"] / p["bytes"], 1))
            if p["bytes"] > 0 and p["flop"] / p["bytes"] < ridge:
                row.update(bound="hbm", frac=round(gbs / peak_gbs, 4))
            else:
                row.update(bound="tensor", frac=round(tf / peak_tf, 4))
        elif p["bytes"] > 0 and p["ms"] > 0:
            gbs = p["bytes"] / (p["ms"] / 1e3) / 1e9
            row.update(bound="hbm", achieved_gbs=round(gbs, 1), frac=round(gbs / peak_gbs, 4))
        out[name] = row
    return out


# ------------------------------------------------------------------ CPU leg (oracle port)
def cpu_iteration_sample(cfg, envs: int, iters: int, warmup: int):
    """Times the CPU restatement (oracle/ppo_oracle.c, OpenMP, all host threads) on a bounded
    sample of the same workload: `envs` environments, same MLP / horizon / epochs / minibatches."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from golden_util import PpoOracle, make_cfg  # test infrastructure: baseline leg only

    threads = os.cpu_count() or 1
    o = PpoOracle(make_cfg(cfg.obs_dim, cfg.act_dim, cfg.hidden, envs, threads=threads,
                           horizon=cfg.horizon, epochs=cfg.epochs, minibatches=cfg.minibatches))
    for _ in range(warmup):
        o.iteration()
    t0 = time.perf_counter()
    steps = 0
    for _ in range(iters):
        steps += o.iteration().env_steps
    dt = time.perf_counter() - t0
    sample = (f"{iters} PPO iteration(s) of the same workload at {envs} envs "
              f"({steps // max(iters, 1)} env-steps each, {cfg.epochs}x{cfg.minibatches} updates), "
              f"oracle/ppo_oracle.c with {threads} OpenMP threads")
    return steps / dt, threads, sample


def run_reference(args, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    value, threads, sample = cpu_iteration_sample(cfg, args.cpu_sample_envs, args.steps, args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "AT-like locomotion, 3x256 actor-critic MLP (BASELINE configs[1] shapes)",
                       "num_envs": args.cpu_sample_envs, "note": "reference has no PPO code; oracle port timed"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer, nccl_unique_id

    world, rank, local = dist_env()
    cfg = PpoConfig.from_config_file(args.config)
    if args.gmis:
        cfg.gmis_per_gpu = args.gmis
    envs_per_gpu = args.envs or cfg.num_envs // max(1, cfg.num_gpus)
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg.num_gpus, cfg.rank, cfg.device = world, rank, local
    cfg.num_envs = envs_per_gpu * world
    if args.decoupled is not None:
        cfg.decoupled = args.decoupled
        if cfg.decoupled:
            cfg.gmis_per_gpu = 1
            cfg.gmi_backend = 1
    if args.serving_sms:
        cfg.serving_sms = args.serving_sms
    if args.backend is not None:
        cfg.gmi_backend = args.backend
    cfg.instrument = 0  # timed loop runs the plain graph; a separate pass below is instrumented
    nid = None
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    trainer = Trainer(cfg, nid)
    upd = torch.cuda.ExternalStream(trainer.stream(-1))

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    for _ in range(max(3, args.warmup)):
        trainer.iteration()

    # ---- device-timed throughput: K iterations enqueued back to back, inputs resident in HBM
    clocks = ClockSampler(local)
    if rank == 0:
        clocks.start()
    barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(upd)
    for _ in range(args.steps):
        trainer.iteration_async()
    t1.record(upd)
    st = trainer.synchronize()
    barrier()
    clk = clocks.stop() if rank == 0 else None
    ms = t0.elapsed_time(t1)
    launches = st.kernel_launches * args.steps
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = ms_t.item()
    steps_total = st.env_steps * world * args.steps
    value = steps_total / (ms_max / 1e3)

    # ---- end to end through the public API: synchronous gmi_ppo_iteration per step, including
    # the H2D of the iteration control block and the D2H read of the iteration's loss statistics.
    barrier()
    w0 = time.perf_counter()
    for _ in range(args.steps):
        trainer.iteration()
    barrier()
    wall = time.perf_counter() - w0
    wall_t = torch.tensor([wall], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(wall_t, op=dist.ReduceOp.MAX)
    e2e = steps_total / wall_t.item()

    # ---- instrumented pass (not part of the timed numbers): CUDA events around every launch
    # of GMI 0 and the update stream -> per-phase time, flops and bytes for the rooflines.
    trainer.set_instrument(True)
    trainer.iteration()
    t2, t3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    t2.record(upd)
    trainer.iteration_async()
    t3.record(upd)
    ist = trainer.synchronize()
    prof = trainer.profile()
    iter_ms_instr = t2.elapsed_time(t3)
    trainer.set_instrument(False)

    multi = None
    if not cfg.decoupled and not args.no_multi_gmi and world == 1:  # one box, same workload
        trainer.close()
        try:
            multi = time_decoupled(args, cfg, world, rank, barrier)
            multi["vs_single_context"] = multi["value"] / value
        except Exception as e:  # noqa: BLE001 -- the headline line must still print
            multi = {"error": f"{type(e).__name__}: {e}"}

    if rank == 0:
        peak_tf, peak_gbs, peak_src = measured_peaks()
        gemm_ms, gemm_flop, gemm_bytes = ist.gemm_ms, ist.gemm_flop, ist.gemm_bytes
        achieved_tf = gemm_flop / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else 0.0
        achieved_gbs = gemm_bytes / (gemm_ms / 1e3) / 1e9 if gemm_ms > 0 else 0.0
        # K <= 256 layer GEMMs and split-K weight gradients sit below the ridge point
        # (peak_tf / peak_gbs flop per byte): the roof that binds them is HBM bandwidth.
        intensity = gemm_flop / gemm_bytes if gemm_bytes > 0 else float("inf")
        hbm_bound = intensity < peak_tf * 1e12 / (peak_gbs * 1e9)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cv, cores, sample = cpu_iteration_sample(cfg, args.cpu_sample_envs, 1, 0)
            cpu = {"value": cv, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}
        ws = working_set_mb(cfg, envs_per_gpu)
        layout = (f"{cfg.gmis_per_gpu} GMI(s) per B200 (BASELINE configs[1])" if not cfg.decoupled else
                  f"decoupled: 1 serving GMI ({cfg.serving_sms or 16} SMs, simulator+agent) + 1 trainer GMI "
                  f"per B200, device experience channel, one-iteration policy lag (BASELINE configs[3])")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"AT-like locomotion, {envs_per_gpu} envs/GPU, "
                                   f"{'x'.join(map(str, cfg.hidden))} actor-critic MLP, "
                                   f"{layout}",
                       "config_file": os.path.relpath(args.config, ROOT), "envs_per_gpu": envs_per_gpu,
                       "obs_dim": cfg.obs_dim, "act_dim": cfg.act_dim, "hidden": cfg.hidden,
                       "horizon": cfg.horizon, "epochs": cfg.epochs, "minibatches": cfg.minibatches,
                       "gmis_per_gpu": cfg.gmis_per_gpu + (1 if cfg.decoupled else 0),
                       "gmi_backend": ["streams", "green_ctx"][cfg.gmi_backend], "decoupled": bool(cfg.decoupled),
                       "parallelism": f"dp{world * cfg.gmis_per_gpu} ({world} GPU x {cfg.gmis_per_gpu} GMI)",
                       "env_steps_per_step": steps_total // args.steps,
                       "l2": f"no flush: per-iteration working set ~{ws:.0f} MB > 126 MB L2",
                       "cuda_graph": bool(cfg.use_graph)},
            "roofline": {"bound": "hbm" if hbm_bound else "tensor",
                         "kernel": "gemm_tcgen05_kernel (every MLP GEMM of GMI 0, all phases)",
                         "achieved": achieved_gbs if hbm_bound else achieved_tf,
                         "peak": peak_gbs if hbm_bound else peak_tf, "unit": "GB/s" if hbm_bound else "TFLOP/s",
                         "frac": achieved_gbs / peak_gbs if hbm_bound else achieved_tf / peak_tf,
                         "intensity_flop_per_byte": intensity,
                         "ridge_flop_per_byte": peak_tf * 1e12 / (peak_gbs * 1e9),
                         "algorithmic_bytes_per_launch": gemm_bytes / max(1, ist.gemm_launches),
                         "tensor_view": {"achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                                         "frac": achieved_tf / peak_tf},
                         "traffic": gemm_traffic(),
                         "traffic_unit": "DRAM bytes per launch (ncu, profiles/traffic.json)",
                         "peak_source": peak_src,
                         "gemm_share_of_step": gemm_ms / iter_ms_instr if iter_ms_instr else None,
                         "instrumented_ms_per_step": iter_ms_instr},
            "phases": phase_table(prof, iter_ms_instr, peak_tf, peak_gbs),
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 16, "d2h_bytes_per_step": 32,
                    "api": "gmi_ppo_iteration (synchronous C-ABI call per step)"},
            "gpu_launches": launches,
            "clocks": clk,
            "multi_gmi": multi,
        }
        print(json.dumps(line), flush=True)
    if multi is None:
        trainer.close()
    if world > 1:
        dist.destroy_process_group()


def time_decoupled(args, cfg, world, rank, barrier):
    """The same workload in the decoupled multi-GMI layout (BASELINE configs[3] per GPU): a
    16-SM serving GMI (simulator + agent) streams experience to a 132-SM trainer GMI through the
    device channel, one-iteration policy lag. Device-timed like the main number, max over ranks."""
    import copy
    import torch
    import torch.distributed as dist
    from paper_2206_08482_b200.ppo import Trainer, nccl_unique_id

    dc = copy.deepcopy(cfg)
    dc.decoupled, dc.gmis_per_gpu, dc.gmi_backend = 1, 1, 1
    dc.serving_sms = args.serving_sms or 16
    nid = None
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    t = Trainer(dc, nid)
    upd = torch.cuda.ExternalStream(t.stream(-1))
    for _ in range(max(3, args.warmup)):
        t.iteration()
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(upd)
    for _ in range(args.steps):
        t.iteration_async()
    b.record(upd)
    st = t.synchronize()
    barrier()
    ms = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    t.close()
    value = st.env_steps * world * args.steps / (ms.item() / 1e3)
    return {"layout": f"decoupled: serving GMI ({dc.serving_sms} SMs, simulator+agent) + trainer GMI "
                      f"(remaining SMs) per B200, device experience channel (configs/at_4096env_decoupled.cfg)",
            "semantics": "one-iteration policy lag (PAPER.md:378-407); behaviour log-probs recorded",
            "value": value, "unit": UNIT, "ms_per_step": ms.item() / args.steps}


def working_set_mb(cfg, envs):
    S_p = (cfg.obs_dim + 31) // 32 * 32
    T = cfg.horizon
    B = T * envs
    hid = sum((h + 31) // 32 * 32 for h in cfg.hidden)
    byt = (T + 1) * envs * S_p * 2 + B * S_p * 2  # rollout obs + epoch copy
    byt += 2 * (B // cfg.minibatches) * hid * 2 * 2  # activations + grads, both nets
    byt += B * (cfg.act_dim + 6) * 4
    return byt / 1e6


if __name__ == "__main__":
    main()
