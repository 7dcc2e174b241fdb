#!/usr/bin/env python3
"""Benchmark: whole-box PPO training env-steps/s on B200 (BASELINE.json `metric`).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config configs/at_4096env_3x256.cfg]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1, one rank per GPU)
    python bench.py --gpus N ...        (N > 1: re-executes itself under torch.distributed.run)
    python bench.py --impl reference ...                        (CPU reference arm, no libgmi)

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
                   help="1: serving GMI + trainer GMI per GPU with an experience channel (BASELINE config 4); "
                        "2: AsyncDecoupled across GPUs (serving GPUs -> trainer GPUs, even --gpus)")
    p.add_argument("--serving-sms", type=int, default=0, help="SMs of the serving GMI (decoupled mode)")
    p.add_argument("--comm", default="auto", choices=["auto", "peer", "nccl"],
                   help="cross-GPU step: auto = peer exchange for N > 1 (none at N = 1); peer = the fused "
                        "peer exchange even at N = 1 (measures its cost over one rank); nccl = ncclAllReduce")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-multi-gmi", action="store_true",
                   help="skip the decoupled multi-GMI layout measured beside the single-context one")
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
        self._lock = threading.Lock()
        self._thread = None
        self._nvml = None
        self._h = None
        self.error = None

    def _nvml_index(self, nv):
        """NVML index of CUDA device `self.device` (NVML enumerates all GPUs, CUDA only the
        visible ones): matched by UUID."""
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(self.device).uuid).lower()
            for i in range(nv.nvmlDeviceGetCount()):
                u = nv.nvmlDeviceGetUUID(nv.nvmlDeviceGetHandleByIndex(i))
                u = (u.decode() if isinstance(u, bytes) else u).lower()
                if uuid and uuid in u:
                    return i
        except Exception:  # noqa: BLE001 - fall back to the CUDA ordinal
            pass
        return self.device

    def sample(self):
        """One SM-clock + throttle-reason sample (callable from the main thread as well: the
        timed loop polls its end event and samples while the device drains the queue)."""
        if self._nvml is None:
            return
        nv = self._nvml
        with self._lock:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
            try:
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except AttributeError:  # older bindings
                mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
            for name, attr in self.REASONS:
                if mask & getattr(nv, attr, getattr(nv, attr.replace("ClocksEvent", "ClocksThrottle"), 0)):
                    self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.sample()
            except Exception as e:  # noqa: BLE001 - keep the failure visible in the line
                self.error = repr(e)
                return
            time.sleep(self.period)

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self._nvml_index(pynvml))
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._nvml = pynvml
        except Exception as e:  # noqa: BLE001 - no NVML: clocks reported as unavailable
            self.error = repr(e)
            return
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()

    def stop(self):
        if self._thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self._stop.set()
        self._thread.join(timeout=5)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"], "samples": 0,
                    "error": self.error}
        loaded = [x for x in self.samples if x > 0.5 * (self.max_mhz or max(self.samples))] or self.samples
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml"}


def measured_peaks():
    """(burst bf16 TF/s, sustained bf16 TF/s, HBM GB/s, source) from the driver-written
    MEASURED_PEAKS.json, else the B200_PROFILING.md fallbacks."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return (j["bf16_tflops"], j["bf16_tflops_sustained"], j["hbm_gbs"],
                "measured (MEASURED_PEAKS.json):")
    except (OSError, KeyError, ValueError):
        return 2250.0, 1400.0, 6650.0, "fallback (B200_PROFILING.md):"


def gemm_traffic(kind: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the `kind` GEMM (fwd / dx / dw)
    from the committed ncu --set full capture summary (profiles/traffic.json); None when absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)["kernels"][kind]["dram_bytes_per_launch"]
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


# ------------------------------------------------------------------ config without libgmi
# Catalog observation / action widths and default hidden widths (workload.hpp:126-134); the
# reference arm reads the config file with this plain parser so that it never loads libgmi.
CATALOG = {"AT": (60, 8, [256, 128, 64]), "AY": (48, 12, [256, 128, 64]), "BB": (24, 3, [256, 128, 64]),
           "FC": (23, 9, [256, 128, 64]), "HM": (108, 21, [200, 400, 100]), "SH": (211, 20, [512, 512, 512, 256])}
ENV_NAMES = {"AT": "Ant-like locomotion", "AY": "Anymal-like", "BB": "BallBalance-like", "FC": "FrankaCabinet-like",
             "HM": "Humanoid-like", "SH": "ShadowHand-like"}
BASELINE_CONFIG = {"at_512env_2x64.cfg": "configs[0]", "at_4096env_3x256.cfg": "configs[1]",
                   "hm_8192env_4gmi.cfg": "configs[2]", "at_4096env_decoupled.cfg": "configs[3] (one GPU)",
                   "decoupled_8gpu.cfg": "configs[3]", "sh_sweep_8gpu.cfg": "configs[4]"}


def plain_config(path):
    """Sections / keys of a proj/configs-schema file (config.hpp:125-154 syntax), no validation."""
    sec, out = None, {}
    with open(path) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            if line.startswith("["):
                sec = line.strip("[]").strip()
                out.setdefault(sec, {})
            elif "=" in line and sec is not None:
                k, v = (x.strip() for x in line.split("=", 1))
                out[sec].setdefault(k, v)
    return out


def workload_of(path, envs_override=0):
    c = plain_config(path)
    bench = c.get("workload", {}).get("benchmark", "AT")
    S, A, hid = CATALOG[bench]
    ppo = c.get("ppo", {})
    hidden = [int(h) for h in ppo["hidden"].split(",")] if "hidden" in ppo else hid
    ngpu = sum(1 for _ in open(path) if _.split("#", 1)[0].strip().startswith("gpu ")
               or _.split("#", 1)[0].strip().startswith("gpu="))
    num_envs = int(ppo.get("num_envs", 4096))
    envs = envs_override or num_envs // max(1, ngpu)
    return dict(bench=bench, env=ENV_NAMES.get(bench, bench), obs_dim=S, act_dim=A, hidden=hidden,
                envs_per_gpu=envs, horizon=int(ppo.get("horizon", 32)), epochs=int(ppo.get("epochs", 4)),
                minibatches=int(ppo.get("minibatches", 4)),
                gmis_per_gpu=int(c.get("model", {}).get("gmis_per_gpu", 1)),
                decoupled=int(ppo.get("decoupled", 0)),
                baseline=BASELINE_CONFIG.get(os.path.basename(path), "custom"), path=path)


def workload_label(w, n_gpus, layout):
    return (f"{w['env']} ({w['bench']}), {w['envs_per_gpu']} envs/GPU x {n_gpus} GPU, "
            f"{w['obs_dim']}:{':'.join(map(str, w['hidden']))}:{w['act_dim']} actor-critic MLP, {layout} "
            f"(BASELINE {w['baseline']})")


# ------------------------------------------------------------------ CPU leg (oracle port)
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_iteration_sample(w, envs: int, iters: int, warmup: int, threads: int = 0, warmup_envs: int = 0):
    """Times the CPU restatement (oracle/ppo_oracle.c, OpenMP) on `envs` environments of the same
    workload (same MLP / horizon / epochs / minibatches): `warmup` untimed iterations (at
    `warmup_envs` envs when given), then `iters` timed ones. Returns env-steps/s and a sample note."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from golden_util import PpoOracle, make_cfg  # test infrastructure: baseline leg only

    threads = threads or os.cpu_count() or 1
    mk = lambda n: PpoOracle(make_cfg(w["obs_dim"], w["act_dim"], w["hidden"], n, threads=threads,
                                      horizon=w["horizon"], epochs=w["epochs"], minibatches=w["minibatches"]))
    if warmup:
        ow = mk(warmup_envs or envs)
        for _ in range(warmup):
            ow.iteration()
        del ow
    o = mk(envs)
    t0 = time.perf_counter()
    steps = 0
    for _ in range(iters):
        steps += o.iteration().env_steps
    dt = time.perf_counter() - t0
    sample = (f"{iters} PPO iteration(s) at {envs} envs ({steps // max(iters, 1)} env-steps each, "
              f"{w['epochs']}x{w['minibatches']} updates), oracle/ppo_oracle.c, {threads} OpenMP thread(s)")
    return steps / dt, threads, sample


def reduction_vs_reference():
    """The reference's own execute() (reduction.hpp:225-334, oracle/_ref/gmux_ref_bench, one host
    thread as shipped) beside K1 (gmi_reduce_device, fp64, the same fold order, bit-identical
    results) on the BASELINE layouts at the real gradient lengths."""
    exe = os.path.join(ROOT, "oracle", "_ref", "gmux_ref_bench")
    if not os.path.exists(exe):
        return {"unavailable": "oracle/_ref/gmux_ref_bench not built"}
    import ctypes as C
    import torch
    from paper_2206_08482_b200 import _lib
    out = []
    res = subprocess.run([exe, "1"], capture_output=True, text=True, timeout=300)
    codes = {"MPR": 0, "MRR": 1, "HAR": 2}
    for line in res.stdout.splitlines():
        r = json.loads(line)
        g, t, n = r["g"], r["t"], r["len"]
        bufs = [torch.full((n,), 1.0 + 0.001 * i, dtype=torch.float64, device="cuda") for i in range(g * t)]
        dst = torch.empty(n, dtype=torch.float64, device="cuda")
        ptrs = (C.c_void_p * (g * t))(*[b.data_ptr() for b in bufs])
        counts, ids = (C.c_int * g)(*([t] * g)), (C.c_int * (g * t))(*range(g * t))
        st = torch.cuda.current_stream()

        def k1():
            _lib.call("gmi_reduce_device", codes[r["strategy"]], g, counts, ids, ptrs, C.c_void_p(dst.data_ptr()),
                      n, 1, 0, C.c_void_p(st.cuda_stream))
        for _ in range(3):
            k1()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(20):
            k1()
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 20
        out.append({"case": r["case"], "strategy": r["strategy"], "len": n, "ref_execute_s": r["seconds"],
                    "k1_ms": ms, "speedup": r["seconds"] / (ms / 1e3),
                    "k1_gbs": (g * t + 1) * 8.0 * n / (ms / 1e3) / 1e9})
    return {"layouts": out, "note": "reference execute() single host thread (as shipped) vs K1 on one B200, "
                                    "fp64, all g x t GMI buffers resident on the device"}


def run_reference(args):
    """Reference arm: the CPU path of this workload (the reference has no PPO code, so its CPU
    restatement oracle/ppo_oracle.c is timed) on all host threads, same config as our arm;
    every timed step is one full PPO iteration of one GPU's share of envs. No libgmi."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    w = workload_of(args.config, args.envs)
    if args.gmis:
        w["gmis_per_gpu"] = args.gmis
    ngpu = max(1, args.gpus)
    # warm-up steps touch the code/data paths only (a smaller env count keeps the run within minutes)
    value, threads, sample = cpu_iteration_sample(w, w["envs_per_gpu"], args.steps, args.warmup,
                                                  warmup_envs=min(512, w["envs_per_gpu"]))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ngpu,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": bench_config(w, ngpu),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": sample + (f"; warm-up iterations at {min(512, w['envs_per_gpu'])} envs"
                                                 if args.warmup else ""),
                             "nproc": os.cpu_count(), "cpu_model": cpu_model(),
                             "note": "the reference (gmux) has no PPO code; its CPU restatement is timed. "
                                     "Host env-steps/s do not depend on the GPU count, so each step "
                                     "processes one GPU's envs"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def layout_of(w):
    return (f"{w['gmis_per_gpu']} GMI(s) per GPU" if not w["decoupled"] else
            "decoupled: serving GMI + trainer GMI per GPU, device experience channel")


def bench_config(w, ngpu):
    """The workload as named by the config file -- identical in both arms (same_config)."""
    return {"workload": workload_label(w, ngpu, layout_of(w)),
            "config_file": os.path.relpath(os.path.abspath(w["path"]), ROOT),
            "benchmark": w["bench"], "envs_per_gpu": w["envs_per_gpu"], "obs_dim": w["obs_dim"],
            "act_dim": w["act_dim"], "hidden": w["hidden"], "horizon": w["horizon"], "epochs": w["epochs"],
            "minibatches": w["minibatches"], "gmis_per_gpu": w["gmis_per_gpu"],
            "parallelism": f"dp{ngpu * w['gmis_per_gpu']} ({ngpu} GPU x {w['gmis_per_gpu']} GMI)",
            "l2": "no flush: per-iteration working set > 126 MB L2 (run.working_set_mb)"}


def relaunch(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-exec under torch.distributed.run,
    one rank per GPU on this node, rendezvous on 127.0.0.1."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ our arm
def time_trainer(cfg, steps, warmup, world, barrier, instrument=True, tune=None):
    """Device-timed K iterations of one trainer (max over ranks), then one instrumented iteration
    for the per-unit (per-GMI) busy time. Returns (value, ms_per_step, units) and, with `tune`
    (candidate SM splits), the measured split choice of gmi_ppo_tune_shares made first."""
    import torch
    import torch.distributed as dist

    t = make_trainer(cfg, world, cfg.rank)
    upd = torch.cuda.ExternalStream(t.stream(-1))
    for _ in range(max(3, warmup)):
        t.iteration()
    tuning = None
    if tune:
        best, tput = t.tune_shares(tune, iters=3)
        tuning = {"candidates_sms": tune, "env_steps_per_s": tput, "chosen": tune[best]}
        upd = torch.cuda.ExternalStream(t.stream(-1))  # a resize moves the update stream
        for _ in range(2):
            t.iteration()
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(upd)
    for _ in range(steps):
        t.iteration_async()
    b.record(upd)
    st = t.synchronize()
    barrier()
    ms = torch.tensor([a.elapsed_time(b)], dtype=torch.float64,
                      device="cpu" if os.environ.get("GMI_BENCH_SHARE_GPU") == "1" else "cuda")
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    value = st.env_steps * world * steps / (ms.item() / 1e3)
    units = None
    if instrument:
        t.set_instrument(True)
        t.iteration()
        c, d = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c.record(upd)
        t.iteration_async()
        d.record(upd)
        t.synchronize()
        it_ms = c.elapsed_time(d)
        units = unit_report(t.unit_busy(), it_ms, cfg.decoupled)
    t.close()
    if tune:
        return value, ms.item() / steps, units, tuning
    return value, ms.item() / steps, units


def make_trainer(cfg, world, rank):
    """One rank's trainer. N > 1: the peer exchange is wired over CUDA IPC (every rank's window
    handle gathered through torch.distributed), or an NCCL communicator with --comm nccl."""
    import torch.distributed as dist
    from paper_2206_08482_b200.ppo import Trainer, nccl_unique_id

    if world == 1:
        return Trainer(cfg)
    if cfg.decoupled == 2:
        # AsyncDecoupled across GPUs: serving rank s <-> trainer rank world/2 + s over the link
        # windows; the trainer ranks' own data-parallel job over the peer exchange
        t = Trainer(cfg)
        handles = [None] * world
        dist.all_gather_object(handles, t.link_handle())
        t.link_attach(handles[(rank + world // 2) % world])
        serving = rank < world // 2
        comm = [None] * world
        dist.all_gather_object(comm, None if serving or world == 2 else t.comm_handle())
        if not serving and world > 2:
            t.comm_attach(comm[world // 2:])
        dist.barrier()
        return t
    if cfg.comm == 1:
        t = Trainer(cfg)
        handles = [None] * world
        dist.all_gather_object(handles, t.comm_handle())
        t.comm_attach(handles)
        dist.barrier()
        return t
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return Trainer(cfg, obj[0])


def unit_report(busy, it_ms, decoupled):
    names = (["serving GMI (simulator+agent)", "trainer GMI"] if decoupled else
             [f"GMI {i}" for i in range(len(busy) - 1)]) + ["update stream (K1 fold + Adam)"]
    return [{"unit": n, "sms": s, "busy_ms": round(b, 4), "sm_busy_frac": round(b / it_ms, 4) if it_ms else None}
            for n, (b, s) in zip(names, busy)] + [{"instrumented_iteration_ms": round(it_ms, 4)}]


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    world, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    import torch
    import torch.distributed as dist
    from paper_2206_08482_b200.ppo import PpoConfig

    w = workload_of(args.config, args.envs)
    w["path"] = args.config
    cfg = PpoConfig.from_config_file(args.config)
    if args.gmis:
        cfg.gmis_per_gpu = w["gmis_per_gpu"] = args.gmis
    envs_per_gpu = w["envs_per_gpu"]

    # GMI_BENCH_SHARE_GPU=1 (tests only): every rank on cuda:0, one process each (time-sliced),
    # host-side collectives on gloo -- exercises the N > 1 path on a one-GPU box
    share = os.environ.get("GMI_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg.num_gpus, cfg.rank, cfg.device = world, rank, local
    cfg.num_envs = envs_per_gpu * world
    if args.decoupled is not None:
        cfg.decoupled = args.decoupled
        if cfg.decoupled:
            cfg.gmis_per_gpu = 1
            cfg.gmi_backend = 1 if cfg.decoupled == 1 else 0
    split = cfg.decoupled == 2
    if split:  # AsyncDecoupled across GPUs: envs live on the serving half (envs_per_gpu each)
        if world < 2 or world % 2:
            raise SystemExit("bench.py: --decoupled 2 needs an even --gpus >= 2")
        cfg.num_envs = envs_per_gpu * (world // 2)
    if args.serving_sms:
        cfg.serving_sms = args.serving_sms
    if args.backend is not None:
        cfg.gmi_backend = args.backend
    cfg.instrument = 0  # timed loop runs the plain graph; a separate pass below is instrumented
    cfg.comm = 1 if args.comm == "peer" or (args.comm == "auto" and world > 1) else 0
    trainer = make_trainer(cfg, world, rank)
    serving_rank = split and rank < world // 2
    # the stream the rank's last work of an iteration lands on (a serving rank: its serving stream)
    upd = torch.cuda.ExternalStream(trainer.stream(-2 if serving_rank else -1))

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
    while rank == 0 and not t1.query():  # sample clocks while the device drains the timed queue
        clocks.sample()
        time.sleep(0.002)
    st = trainer.synchronize()
    barrier()
    clk = clocks.stop() if rank == 0 else None
    ms = t0.elapsed_time(t1)
    launches = st.kernel_launches * args.steps
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cpu" if share else "cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = ms_t.item()
    steps_t = torch.tensor([st.env_steps * args.steps], dtype=torch.float64, device="cpu" if share else "cuda")
    if world > 1:  # decoupled = 2: only the serving ranks count env-steps
        dist.all_reduce(steps_t, op=dist.ReduceOp.SUM)
    steps_total = int(steps_t.item())
    value = steps_total / (ms_max / 1e3)

    # ---- end to end through the public API: synchronous gmi_ppo_iteration per step, including
    # the H2D of the iteration control block and the D2H read of the iteration's loss statistics.
    barrier()
    w0 = time.perf_counter()
    for _ in range(args.steps):
        trainer.iteration()
    barrier()
    wall = time.perf_counter() - w0
    wall_t = torch.tensor([wall], dtype=torch.float64, device="cpu" if share else "cuda")
    if world > 1:
        dist.all_reduce(wall_t, op=dist.ReduceOp.MAX)
    e2e = steps_total / wall_t.item()

    # ---- instrumented pass (not part of the timed numbers): CUDA events around every launch
    # -> per-phase time / flops / bytes for the rooflines and per-GMI busy time.
    trainer.set_instrument(True)
    trainer.iteration()
    t2, t3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    t2.record(upd)
    trainer.iteration_async()
    t3.record(upd)
    trainer.synchronize()
    prof = trainer.profile()
    iter_ms_instr = t2.elapsed_time(t3)
    units = unit_report(trainer.unit_busy(), iter_ms_instr, cfg.decoupled)
    if split:  # the roofline / phases / units of the first trainer rank, reported by rank 0
        got = [None] * world
        dist.all_gather_object(got, (prof, iter_ms_instr, units))
        prof, iter_ms_instr, units = got[world // 2]
        units = [{"unit": "trainer GPU (whole GPU; the serving GPU rolls out concurrently)"}] + units[1:]
    trainer.set_instrument(False)
    barrier()
    trainer.close()

    extra = {}
    if world == 1 and not args.no_multi_gmi and not cfg.decoupled:
        extra = other_layouts(args, cfg, w, value, world, barrier)

    if rank == 0:
        peak_burst, peak_sust, peak_gbs, peak_src = measured_peaks()
        at_max = bool(clk and clk.get("sm_mhz") and clk.get("sm_max_mhz") and clk["sm_mhz"] >= 0.97 * clk["sm_max_mhz"])
        peak_tf = peak_burst if at_max else peak_sust
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cv, cores, sample = cpu_iteration_sample(w, envs_per_gpu, 1, 0)
            c1, _, s1 = cpu_iteration_sample(w, max(64, envs_per_gpu // 16), 1, 0, threads=1)
            cpu = {"value": cv, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                   "single_thread": {"value": c1, "sample": s1}, "nproc": os.cpu_count(), "cpu_model": cpu_model(),
                   "reduction": reduction_vs_reference()}
        layout = (f"{cfg.gmis_per_gpu} GMI(s) per B200 ({['CUDA streams', 'green contexts'][cfg.gmi_backend]})"
                  if not cfg.decoupled else
                  f"AsyncDecoupled across GPUs: {world // 2} serving B200(s) (simulator+agent) -> {world // 2} trainer "
                  f"B200(s), experience pulled over NVLink, one-iteration policy lag" if split else
                  f"decoupled: serving GMI ({cfg.serving_sms or 16} SMs, simulator+agent) + trainer GMI per B200, "
                  f"device experience channel, one-iteration policy lag")
        run = {"layout": layout, "comm": (["ncclAllReduce" if world > 1 else "none (one GPU)",
                                           "peer exchange (fused RS + sharded Adam + AG)"][cfg.comm]),
               "gmis_per_gpu": cfg.gmis_per_gpu + (1 if cfg.decoupled == 1 else 0),
               "gmi_backend": ["streams", "green_ctx"][cfg.gmi_backend], "sm_per_gmi": cfg.sm_per_gmi,
               "decoupled": bool(cfg.decoupled),
               "decoupled_mode": ["off", "per GPU (serving + trainer GMI)", "across GPUs (AsyncDecoupled)"][cfg.decoupled],
               "env_steps_per_step": steps_total // args.steps,
               "cuda_graph": bool(cfg.use_graph),
               "working_set_mb": round(working_set_mb(cfg, envs_per_gpu), 1)}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": bench_config(w, world),
            "run": run,
            "roofline": roofline(prof, peak_tf, peak_gbs, peak_src, at_max, iter_ms_instr),
            "phases": phase_table(prof, iter_ms_instr, peak_tf, peak_gbs),
            "gmi_units": units,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 16, "d2h_bytes_per_step": 32,
                    "api": "gmi_ppo_iteration (synchronous C-ABI call per step)"},
            "gpu_launches": launches,
            "clocks": clk,
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


GEMM_FAMILY = {"fwd_gemm": ("fwd", "gemm_tcgen05_kernel<256,0,0,0,1,0> (training forward, all hidden layers of both "
                                   "nets chained in one launch)"),
               "dx_gemm": ("dx", "gemm_tcgen05_kernel<128,0,1,1,1,0> (input gradients, elu' fused, weight-stationary "
                                 "128-column parts)"),
               "dw_gemm": ("dw", "gemm_tcgen05_kernel<256,1,1,2,0,1> (split-K weight gradients of every layer, bias "
                                 "column sums fused)")}


def roofline(prof, peak_tf, peak_gbs, peak_src, at_max, iter_ms):
    """Dominant kernel = the GEMM family (training forward / input gradient / weight gradient,
    one template each) with the largest measured time in the instrumented iteration (CUDA events
    around each launch on the GMI stream). Its bound follows from its arithmetic intensity
    against the ridge point (peak bf16 TF/s / peak HBM GB/s): algorithmic bytes (every operand
    read once, outputs written once: gemm_bytes() in host/trainer.cpp) / time for HBM-bound,
    algorithmic flops (2 M N K at the real widths) / time for tensor-bound, against the burst
    peaks when the SM clock sat at its maximum. The tensor view of the same kernel and the
    training-forward GEMM's numbers are kept beside it."""
    fam = {k: prof[k] for k in GEMM_FAMILY if k in prof and prof[k].get("ms", 0) > 0}
    if not fam:
        return None
    dom = max(fam, key=lambda k: fam[k]["ms"])
    d = fam[dom]
    ms, flop, byt = d["ms"], d["flop"], d["bytes"]
    n = max(1, d.get("launches", 0))
    tf = flop / (ms / 1e3) / 1e12
    gbs = byt / (ms / 1e3) / 1e9 if byt else 0.0
    ridge = peak_tf * 1e12 / (peak_gbs * 1e9)
    hbm = byt > 0 and flop / byt < ridge
    fms = sum(v["ms"] for v in fam.values())
    ffl = sum(v["flop"] for v in fam.values())
    fby = sum(v["bytes"] for v in fam.values())
    f = prof.get("fwd_gemm", {})
    fwd = None
    if f.get("ms"):
        ftf = f["flop"] / (f["ms"] / 1e3) / 1e12
        fwd = {"kernel": GEMM_FAMILY["fwd_gemm"][1], "achieved_tflops": ftf,
               "frac_tensor": ftf / peak_tf if peak_tf else None,
               "achieved_gbs": f["bytes"] / (f["ms"] / 1e3) / 1e9 if f.get("bytes") else 0.0,
               "launches_per_step": f.get("launches", 0), "traffic": gemm_traffic("fwd")}
    return {"bound": "hbm" if hbm else "tensor", "kernel": GEMM_FAMILY[dom][1],
            "achieved": gbs if hbm else tf, "peak": peak_gbs if hbm else peak_tf,
            "unit": "GB/s" if hbm else "TFLOP/s",
            "frac": (gbs / peak_gbs if hbm else tf / peak_tf) if (peak_gbs if hbm else peak_tf) else None,
            "traffic": gemm_traffic(GEMM_FAMILY[dom][0]),
            "traffic_unit": "DRAM bytes per launch (ncu launch list, profiles/traffic.json)",
            "algorithmic_flop_per_launch": flop / n, "algorithmic_bytes_per_launch": byt / n,
            "intensity_flop_per_byte": flop / byt if byt else None, "ridge_flop_per_byte": ridge,
            "launches_per_step": d.get("launches", 0), "avg_launch_us": 1e3 * ms / n,
            "share_of_step": ms / iter_ms if iter_ms else None,
            "peak_source": peak_src + (" burst (SM clock at max during the timed region)" if at_max else " sustained"),
            "tensor_view": {"achieved": tf, "peak": peak_tf, "unit": "TFLOP/s", "frac": tf / peak_tf if peak_tf else None},
            "training_forward": fwd,
            "gemm_family": {"kernels": "forward + input-gradient + weight-gradient GEMMs", "ms": fms,
                            "achieved_tflops": ffl / (fms / 1e3) / 1e12 if fms else 0.0,
                            "frac": (ffl / (fms / 1e3) / 1e12) / peak_tf if fms else None,
                            "achieved_gbs": fby / (fms / 1e3) / 1e9 if fms else 0.0}}


def other_layouts(args, cfg, w, value, world, barrier):
    """Extra keys, N = 1 only: the decoupled multi-GMI layout of the same workload (BASELINE
    configs[3] per GPU) and BASELINE configs[2] (HM, 8192 envs, 4 green-context GMIs) beside HM
    with one GMI on the same box -- the north_star's multi-GMI vs single-context check -- each
    with per-GMI busy fractions from an instrumented iteration."""
    import copy
    out = {}
    try:
        dc = copy.deepcopy(cfg)
        dc.decoupled, dc.gmis_per_gpu, dc.gmi_backend, dc.sm_per_gmi = 1, 1, 1, 0
        dc.serving_sms = args.serving_sms or 16
        v, msps, units = time_trainer(dc, args.steps, args.warmup, world, barrier)
        out["multi_gmi"] = {"layout": f"decoupled: serving GMI ({dc.serving_sms} SMs) + trainer GMI (remaining SMs), "
                                      "device experience channel (configs/at_4096env_decoupled.cfg)",
                            "semantics": "one-iteration policy lag (PAPER.md:378-407); behaviour log-probs recorded",
                            "value": v, "unit": UNIT, "ms_per_step": msps, "vs_single_context": v / value,
                            "gmi_units": units}
    except Exception as e:  # noqa: BLE001 -- the headline line must still print
        out["multi_gmi"] = {"error": f"{type(e).__name__}: {e}"}
    try:
        from paper_2206_08482_b200.ppo import PpoConfig
        hm_path = os.path.join(ROOT, "configs", "hm_8192env_4gmi.cfg")
        hm = PpoConfig.from_config_file(hm_path)
        hm.num_gpus, hm.rank, hm.device = 1, 0, cfg.device
        v4, ms4, u4 = time_trainer(hm, args.steps, args.warmup, world, barrier)
        one = copy.deepcopy(hm)
        one.gmis_per_gpu, one.gmi_backend, one.sm_per_gmi = 1, 0, 0
        v1, ms1, u1 = time_trainer(one, args.steps, args.warmup, world, barrier)
        hw = workload_of(hm_path)
        out["config2_hm_4gmi"] = {
            "workload": workload_label(hw, 1, f"4 GMIs per B200 (green contexts, {hm.sm_per_gmi} SMs each)"),
            "value": v4, "unit": UNIT, "ms_per_step": ms4, "gmi_units": u4,
            "single_context": {"value": v1, "ms_per_step": ms1, "gmi_units": u1},
            "vs_single_context": v4 / v1}
        # the same HM workload in the decoupled layout; the serving / trainer split is chosen by
        # the adaptive manager on the live trainer (gmi_ppo_tune_shares over measured candidates)
        dec = copy.deepcopy(one)
        dec.decoupled, dec.gmi_backend, dec.serving_sms = 1, 1, 16
        vd, msd, ud, tuning = time_trainer(dec, args.steps, args.warmup, world, barrier,
                                           tune=[[16, 0], [24, 0], [32, 0], [40, 0]])
        out["config2_hm_4gmi"]["decoupled"] = {
            "layout": "serving GMI (simulator+agent: fused wide rollout + critic + GAE on its partition) + trainer GMI, "
                      "device experience channel, one-iteration policy lag",
            "value": vd, "ms_per_step": msd, "gmi_units": ud, "vs_single_context": vd / v1, "tuning": tuning}
    except Exception as e:  # noqa: BLE001
        out["config2_hm_4gmi"] = {"error": f"{type(e).__name__}: {e}"}
    return out


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
