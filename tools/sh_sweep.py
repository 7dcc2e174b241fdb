#!/usr/bin/env python3
"""BASELINE configs[4]: the adaptive GMI manager's sweep on the ShadowHand-like workload
(SH 211:512:512:512:256:20, 32768 envs in total), 1 / 2 / 4 / 7 GMIs per GPU x 2 / 4 / 8 GPUs.

Every (GPUs g, GMIs per GPU t) point splits the job's 32768 envs as 32768 / g per GPU and
32768 / (g t) per GMI (rounded down to the minibatch tiling, a multiple of 8). Each point is
MEASURED on this B200 through the real PPO iteration (gmux.GpuProfiler -> gmi_gpu_profile:
t SM-partitioned green-context GMIs; t = 1 also on plain streams, the single-context layout),
written as a recorded trace in the reference's TSV format (search.hpp:136-171), and the
reference's unmodified Alg. 2 (gmux.explore = search.hpp:198-249) then picks (t, envs per GMI)
for each g from those measurements with the reference ThroughputEstimator (per-GPU throughput
x g, damped by the predicted all-reduce latency). One GPU measures every per-GPU point (the
per-GPU work of g GPUs is identical; the cross-GPU step is the estimator's term).

    python tools/sh_sweep.py [--out profiles/r2/sh_sweep]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2", "sh_sweep"))
    ap.add_argument("--total-envs", type=int, default=32768)
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    from paper_2206_08482_b200 import gmux

    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    prof = gmux.GpuProfiler(iters=a.iters, backend=1)
    single = gmux.GpuProfiler(iters=a.iters, backend=0)
    points, rows = [], []
    for g in (2, 4, 8):
        for t in (1, 2, 4, 7):
            env = a.total_envs // (g * t) // 8 * 8
            t0 = time.time()
            r = prof.profile("SH", t, env)
            p = {"gpus": g, "gmis_per_gpu": t, "num_env_per_gmi": env, "backend": "green_ctx",
                 "runnable": r.runnable, "top_per_gmi": r.top, "mem_gb_per_gmi": r.mem,
                 "gpu_env_steps_per_s": r.top * t, "probe_s": round(time.time() - t0, 2)}
            points.append(p)
            rows.append(f"SH {t} {env} {int(r.runnable)} {r.top:.6f} {r.mem:.6f}")
            print(json.dumps(p), flush=True)
            if t == 1:
                r1 = single.profile("SH", 1, env)
                points.append({"gpus": g, "gmis_per_gpu": 1, "num_env_per_gmi": env, "backend": "streams",
                               "runnable": r1.runnable, "top_per_gmi": r1.top, "mem_gb_per_gmi": r1.mem,
                               "gpu_env_steps_per_s": r1.top})
                print(json.dumps(points[-1]), flush=True)
    trace = a.out + "_trace.tsv"
    with open(trace, "w") as f:
        f.write("# bench gmis_per_gpu num_env runnable top mem -- measured on one B200 (green-context GMIs)\n")
        f.write("\n".join(rows) + "\n")
    rec = gmux.RecordedTraceProfiler.from_file(trace)
    est = gmux.ThroughputEstimator(gmux.load_benchmark("SH"))
    grid = sorted({p["num_env_per_gmi"] for p in points})
    decisions = {}
    for g in (2, 4, 8):
        res = gmux.explore(rec, est, "SH", g, gmux.SearchConfig(num_env_grid=grid, max_gmis_per_gpu=7))
        decisions[g] = {"feasible": res.feasible, "reason": res.reason, "gmis_per_gpu": res.gmis_per_gpu,
                        "num_env_per_gmi": res.num_env, "est_throughput": res.est_throughput,
                        "visited": [v.__dict__ for v in res.visited]}
        print(json.dumps({"gpus": g, "choice": {k: v for k, v in decisions[g].items() if k != "visited"}}),
              flush=True)
    with open(a.out + ".json", "w") as f:
        json.dump({"workload": "SH 211:512:512:512:256:20, 32768 envs total", "points": points,
                   "explore": decisions, "trace": os.path.relpath(trace, ROOT)}, f, indent=1)


if __name__ == "__main__":
    main()
