"""Per-GMI SM utilisation (BASELINE metric): active SM cycles of each GMI's kernels
divided by (SMs of the GMI's partition x elapsed cycles of an iteration).

    # 1. on the GPU box: ncu over ITERS profiled iterations (cudaProfilerStart/Stop window)
    ncu --profile-from-start off --clock-control none --csv \
        --metrics gpu__time_duration.sum,sm__cycles_active.sum,sm__cycles_elapsed.avg.per_second \
        --log-file gpurun_out/util.csv python tools/sm_util.py probe CONFIG ITERS /tmp/x.json
    python tools/sm_util.py probe CONFIG ITERS gpurun_out/util_probe.json   # no profiler: slot time
    # 2. aggregate (here or there):
    python tools/sm_util.py report gpurun_out/util.csv gpurun_out/util_probe.json

The probe also times the iteration without the profiler (CUDA events, graph replay) and writes
the partition sizes; kernels are attributed to GMIs by the CUDA context ncu reports (one green
context per GMI; the trainer's update stream lives in the primary context and is booked to the
trainer GMI).
"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def probe(config, iters=2, out=os.path.join(ROOT, "gpurun_out", "util_probe.json")):
    """Times the iteration (run it WITHOUT ncu for slot_ms) and brackets `iters` iterations with
    cudaProfilerStart/Stop (run it under ncu --profile-from-start off for the kernel metrics)."""
    import torch
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer

    cfg = PpoConfig.from_config_file(config)
    t = Trainer(cfg)
    for _ in range(4):
        t.iteration()
    upd = torch.cuda.ExternalStream(t.stream(-1))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(upd)
    for _ in range(10):
        t.iteration_async()
    b.record(upd)
    st = t.synchronize()
    slot_ms = a.elapsed_time(b) / 10
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(iters):
        t.iteration()
    torch.cuda.cudart().cudaProfilerStop()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    serving = (cfg.serving_sms or 16) if cfg.decoupled else 0
    gmis = ([{"gmi": "serving (simulator+agent)", "sms": serving if cfg.gmi_backend else sms},
             {"gmi": "trainer", "sms": sms - serving if cfg.gmi_backend else sms}] if cfg.decoupled else
            [{"gmi": f"holistic {i}", "sms": (cfg.sm_per_gmi or (sms // cfg.gmis_per_gpu) // 8 * 8)
              if cfg.gmi_backend else sms} for i in range(cfg.gmis_per_gpu)])
    info = {"config": os.path.relpath(config, ROOT), "iters": iters, "slot_ms": slot_ms, "sms": sms,
            "backend": cfg.gmi_backend, "decoupled": bool(cfg.decoupled), "gmis": gmis,
            "launches_per_iteration": st.kernel_launches}
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(info, f)
    print(json.dumps(info))


def report(csv_path, probe_path):
    with open(probe_path) as f:
        info = json.load(f)
    rows = defaultdict(dict)
    with open(csv_path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        v = r["Metric Value"].replace(",", "")
        rows[r["ID"]].update(ctx=r["Context"], stream=r["Stream"], name=r["Kernel Name"])
        rows[r["ID"]][r["Metric Name"]] = float(v) if v else 0.0
    by_ctx = defaultdict(lambda: {"active_s": 0.0, "busy_ms": 0.0, "launches": 0, "kernels": defaultdict(float)})
    for r in rows.values():
        c = by_ctx[r["ctx"]]
        hz = r.get("sm__cycles_elapsed.avg.per_second", 0.0) or 1.9e9
        c["active_s"] += r.get("sm__cycles_active.sum", 0.0) / hz
        c["busy_ms"] += r.get("gpu__time_duration.sum", 0.0) / 1e6
        c["launches"] += 1
        c["kernels"][r["name"].split("(")[0][:60]] += r.get("gpu__time_duration.sum", 0.0) / 1e6
    iters, slot_s = info["iters"], info["slot_ms"] / 1e3
    ctxs = sorted(by_ctx, key=lambda k: by_ctx[k]["launches"])
    gmis = info["gmis"]
    out = []
    if info["decoupled"] and len(ctxs) >= 2:
        # fewest launches = serving GMI; everything else (trainer green ctx + primary ctx) = trainer
        groups = {"serving (simulator+agent)": [ctxs[0]], "trainer": ctxs[1:]}
    elif info["backend"] and len(ctxs) >= len(gmis) + 1:
        # green-context GMIs: the context with the fewest launches is the primary context (the
        # update stream: K1 fold + Adam, booked separately); the others are the GMIs in creation
        # order (ncu context ids increase with creation)
        upd = ctxs[0]
        green = sorted(ctxs[1:], key=lambda k: int(k) if str(k).isdigit() else str(k))
        groups = {g["gmi"]: [c] for g, c in zip(gmis, green)}
        gmis = gmis + [{"gmi": "update stream (primary context)", "sms": info["sms"]}]
        groups["update stream (primary context)"] = [upd]
    else:
        groups = {g["gmi"]: [] for g in gmis}
        groups[gmis[0]["gmi"]] = ctxs
    for g in gmis:
        cs = groups.get(g["gmi"], [])
        act = sum(by_ctx[c]["active_s"] for c in cs) / iters
        busy = sum(by_ctx[c]["busy_ms"] for c in cs) / iters
        kern = defaultdict(float)
        for c in cs:
            for k, v in by_ctx[c]["kernels"].items():
                kern[k] += v / iters
        top = sorted(kern.items(), key=lambda kv: -kv[1])[:4]
        out.append({"gmi": g["gmi"], "sms": g["sms"], "sm_utilisation": act / (g["sms"] * slot_s),
                    "kernel_ms_per_iteration": busy, "slot_ms": info["slot_ms"],
                    "top_kernels_ms": {k: round(v, 4) for k, v in top}})
    res = {"definition": "sum over the GMI's kernels of sm__cycles_active.sum / SM clock, divided by "
                         "(GMI partition SMs x device-timed iteration); ncu times are serialised replays",
           "config": info["config"], "per_gmi": out}
    print(json.dumps(res, indent=1))
    return res


if __name__ == "__main__":
    if sys.argv[1] == "probe":
        probe(sys.argv[2], int(sys.argv[3]), sys.argv[4])
    else:
        report(sys.argv[2], sys.argv[3])
