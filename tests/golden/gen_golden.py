#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs oracle/_ref/gmux_ref (the reference's header-only planner compiled in place by
oracle/Makefile against /root/reference/proj/include) on a fixed request set and stores
request/response pairs.  Re-run after changing the request set:

    make -C oracle ref && python tests/golden/gen_golden.py

Large fp64 result vectors are stored as the SHA-256 of their little-endian bytes (the
product must match bit-for-bit); small ones are stored in full.  Buffer contents are
never stored: both sides regenerate them from ``buffer_values`` below, which mirrors
``buffer_value`` in oracle/ref_driver.cpp exactly.
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import struct
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.path.join(ROOT, "oracle", "_ref", "gmux_ref")
CONFIG_DIR = os.path.join(ROOT, "configs")

M64 = (1 << 64) - 1


def buffer_values(kind: str, seed: int, gid: int, length: int) -> list[float]:
    if kind == "cli":
        return [1.0 + 0.001 * gid + 1e-6 * float(e) for e in range(length)]
    out = []
    for e in range(length):
        z = (seed * 0x9E3779B97F4A7C15 + (gid & M64) * 0xBF58476D1CE4E5B9 + e * 0x94D049BB133111EB) & M64
        z = (z + 0x9E3779B97F4A7C15) & M64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        z ^= z >> 31
        out.append(0.1 + 0.9 * (float(z >> 11) * (1.0 / 9007199254740992.0)))
    return out


def f64_digest(values) -> str:
    return hashlib.sha256(b"".join(struct.pack("<d", v) for v in values)).hexdigest()


def trace_digest(trace) -> str:
    s = "\n".join(f"{a} {b} {c} {d!r} {k}" for a, b, c, d, k in trace)
    return hashlib.sha256(s.encode()).hexdigest()


def uniform(g: int, t: int, start: int = 0) -> list[list[int]]:
    return [[start + i * t + j for j in range(t)] for i in range(g)]


def run_ref(requests: list[dict]) -> list[dict]:
    proc = subprocess.run([REF], input=json.dumps(requests), capture_output=True, text=True, check=True)
    out = json.loads(proc.stdout)
    assert len(out) == len(requests)
    return out


def count_vectors(gmax: int, tmax: int):
    for g in range(1, gmax + 1):
        counts = [1] * g
        while True:
            yield list(counts)
            i = g - 1
            while i >= 0 and counts[i] == tmax:
                counts[i] = 1
                i -= 1
            if i < 0:
                break
            counts[i] += 1


def layout_from_counts(counts, start=0):
    mpl, nxt = [], start
    for c in counts:
        mpl.append(list(range(nxt, nxt + c)))
        nxt += c
    return mpl


def gen_selection():
    reqs = []
    for counts in count_vectors(5, 5):
        mpl = layout_from_counts(counts)
        reqs.append({"op": "select", "mpl": mpl})
        reqs.append({"op": "leaders", "mpl": mpl})
    extra = [[[0, 1], [2, 3]], [[5], [7]], [[1, 3], [5, 7]], [[0], [1, 2]], [[0, 1, 2], [3, 4, 5]],
             [[9, 4, 2], [3, 8, 1], [7, 6, 5]], [[12, 13, 14, 15, 16, 17, 18]] * 1,
             [], [[0, 1], []], [[0, 1], [1, 2]]]
    for mpl in extra:
        reqs.append({"op": "select", "mpl": mpl})
        reqs.append({"op": "leaders", "mpl": mpl})
    for g in range(1, 9):
        for t in range(1, 10):
            reqs.append({"op": "rings", "mpl": uniform(g, t, 100)})
    for mpl in ([[0], [1, 2]], [[3, 1], [0, 2]], [[4, 5, 6], [1, 2, 3], [7, 8, 9]]):
        reqs.append({"op": "rings", "mpl": mpl})
    return reqs


def gen_predict():
    reqs = []
    for s in ("MPR", "MRR", "HAR"):
        for g in range(0, 9):
            for t in range(0, 10):
                for m_p, b1, b2 in ((240.0, 1.0, 30.0), (128.0, 1.3, 41.0), (1e6, 1.0, 30.0), (0.0, 1.0, 30.0)):
                    reqs.append({"op": "predict", "s": s, "g": g, "t": t, "m_p": m_p, "b1": b1, "b2": b2})
    return reqs


def execute_requests():
    reqs = []
    # CLI example (README "reduce --layout [[0,1],[2,3]] --payload 240").
    for s in ("MPR", "MRR", "HAR"):
        reqs.append({"op": "execute", "strategy": s, "mpl": [[0, 1], [2, 3]], "len": 30, "gen": "cli"})
    # Acceptance criterion 3 shape: uniform g in [1,8], t in [1,9], len 16, b1 = 1, b2 = 30.
    for g in range(1, 9):
        for t in range(1, 10):
            for s in ("MPR", "MRR", "HAR"):
                if s == "MRR" and t > g:
                    continue
                reqs.append({"op": "execute", "strategy": s, "mpl": uniform(g, t), "len": 16,
                             "gen": "hash", "seed": 7})
    # Random layouts (criterion 1 style): ids offset, ragged, len 1..300, b1 = 1.3, b2 = 41.
    rng = random.Random(20240811)
    for trial in range(160):
        g = rng.randint(1, 4)
        nxt = 10 * trial + rng.randint(0, 3)
        mpl = []
        for _ in range(g):
            t = rng.randint(1, 4)
            mpl.append(list(range(nxt, nxt + t)))
            nxt += t
        if rng.random() < 0.3:  # shuffle ids within/between GPUs: placement order matters
            flat = [i for l in mpl for i in l]
            rng.shuffle(flat)
            it = iter(flat)
            mpl = [[next(it) for _ in l] for l in mpl]
        length = rng.choice([1, 2, 3, 5, 7, 16, 31, 64, 100, 257, 300])
        uni = all(len(l) == len(mpl[0]) for l in mpl)
        for s in ("MPR", "HAR", "MRR"):
            if s == "MRR" and not (uni and len(mpl[0]) <= g):
                continue
            reqs.append({"op": "execute", "strategy": s, "mpl": mpl, "len": length, "gen": "hash",
                         "seed": trial, "b1": 1.3, "b2": 41.0})
    # MRR on inapplicable layouts must raise MultiStreamError.
    reqs.append({"op": "execute", "strategy": "MRR", "mpl": [[0, 1, 2], [3, 4, 5]], "len": 8, "gen": "hash", "seed": 5})
    reqs.append({"op": "execute", "strategy": "MRR", "mpl": [[0], [1, 2]], "len": 8, "gen": "hash", "seed": 5})
    # BASELINE.json layouts at the real gradient lengths (P fp32 words reduced as fp64 here).
    for name, s, mpl, length in (
        ("AT-1x4 MPR", "MPR", uniform(1, 4), 114121),
        ("HM-2x4 HAR", "HAR", uniform(2, 4), 286822),
        ("HM-4x4 MRR", "MRR", uniform(4, 4), 286822),
        ("SH-2x7 HAR", "HAR", uniform(2, 7), 1535765),
        ("SH-8x2 MRR", "MRR", uniform(8, 2), 1535765),
        ("AT3x256-8x1 MRR", "MRR", uniform(8, 1), 296713),
    ):
        reqs.append({"op": "execute", "strategy": s, "mpl": mpl, "len": length, "gen": "hash",
                     "seed": 42, "label": name})
    return reqs


def compact_execute(rq, rs):
    if "error" in rs:
        return rs
    out = {k: rs[k] for k in ("strategy", "latency", "broadcast_latency")}
    out["trace_len"] = len(rs["trace"])
    out["trace_sha256"] = trace_digest(rs["trace"])
    if len(rs["trace"]) <= 64:
        out["trace"] = rs["trace"]
    out["result_sha256"] = f64_digest(rs["result"])
    if rq["len"] <= 64:
        out["result"] = rs["result"]
    return out


def topo(gpus, parts=(), b1=1.0, b2=30.0):
    return {"b1": b1, "b2": b2, "gpus": gpus, "partitions": list(parts)}


def gpus(n, arch="sm80"):
    return [{"id": i, "arch": arch} for i in range(n)]


def mps(gid, gpu, share, mem=None):
    return {"gmi_id": gid, "gpu_id": gpu, "backend": "mps", "sm_share": share,
            "mem_gb": 40.0 * share if mem is None else mem}


def mig(gid, gpu, units, mem):
    return {"gmi_id": gid, "gpu_id": gpu, "backend": "mig", "sm_share": units / 8.0, "mem_gb": mem}


def gen_plans():
    reqs = []
    for tpl in ("TCG", "TCG_EX", "TDG", "TDG_EX", "async_decoupled"):
        for n in (1, 2, 3, 4, 8):
            for gpg in (0, 1, 2, 3, 4, 7):
                reqs.append({"op": "plan", "template": tpl, "topology": topo(gpus(n)), "gmis_per_gpu": gpg})
    # unsorted GPU ids, partitions ignored for ids, invalid topologies
    reqs.append({"op": "plan", "template": "TCG_EX", "topology": topo([{"id": 5}, {"id": 2}, {"id": 9}]), "gmis_per_gpu": 2})
    reqs.append({"op": "plan", "template": "TCG_EX", "topology": topo(gpus(2), [mps(7, 0, 0.5), mps(3, 0, 0.5), mps(11, 1, 1.0)]), "gmis_per_gpu": 2})
    reqs.append({"op": "plan", "template": "TCG_EX", "topology": topo(gpus(1), [mps(0, 0, 0.7), mps(1, 0, 0.7)]), "gmis_per_gpu": 2})
    reqs.append({"op": "plan", "template": "TCG_EX", "topology": topo([]), "gmis_per_gpu": 2})
    reqs.append({"op": "plan", "template": "async_decoupled", "topology": topo([{"id": 3}, {"id": 1}, {"id": 2}]), "gmis_per_gpu": 3})
    return reqs


def gen_validate():
    T = []
    T.append(topo(gpus(1), [mig(0, 0, 3, 20.0), mig(1, 0, 3, 20.0), mig(2, 0, 1, 5.0)]))
    T.append(topo(gpus(1), [mig(0, 0, 4, 20.0), mig(1, 0, 4, 20.0)]))
    T.append(topo(gpus(1), [mig(0, 0, 7, 40.0)]))
    T.append(topo(gpus(1), [mig(0, 0, 3, 40.0)]))
    T.append(topo(gpus(1), [mps(0, 0, 0.5), mps(1, 0, 0.5)]))
    T.append(topo(gpus(1), [mps(0, 0, 0.5), mps(1, 0, 0.6)]))
    T.append(topo(gpus(1), [mps(0, 0, 0.5), mig(1, 0, 3, 20.0)]))
    T.append(topo(gpus(1, "sm70"), [mig(0, 0, 3, 20.0)]))
    T.append(topo(gpus(1), [mps(0, 3, 0.5)]))
    T.append(topo(gpus(2), [mps(0, 0, 0.5), mps(0, 1, 0.5)]))
    T.append(topo(gpus(1), [mps(0, 0, 0.0), mps(1, 0, 1.5, 0.0)]))
    T.append(topo(gpus(1), [mps(0, 0, 0.5)], b1=0.0, b2=-1.0))
    T.append(topo([{"id": 0, "sm_units": 10}], [mig(0, 0, 3, 20.0)]))
    T.append(topo(gpus(2), [mig(i, i // 3, u, m) for i, (u, m) in enumerate([(1, 5.0), (2, 10.0), (4, 20.0), (3, 20.0), (3, 20.0), (2, 10.0)])]))
    T.append(topo(gpus(1), [mps(i, 0, 1.0 / 3.0) for i in range(3)]))
    return [{"op": "validate", "topology": t} for t in T]


def gen_workload_costs():
    reqs = []
    for b in ("AT", "AY", "BB", "FC", "HM", "SH"):
        reqs.append({"op": "workload", "bench": b})
        for n in (1, 2, 8, 16):
            reqs.append({"op": "costs", "bench": b, "n_gmis": n})
    reqs.append({"op": "workload", "bench": "XX"})
    return reqs


def gen_explore():
    reqs = []
    for g in (1, 2, 4, 8):
        for bench in ("AT", "HM", "SH"):
            reqs.append({"op": "explore", "num_gpu": g, "bench": bench, "estimator": {"bench": bench},
                         "comm_discount": True})
    knee = [[g, 4096 if g == 2 else 8192] for g in range(1, 11)]
    cap = [[g, 1.0 if g == 2 else 0.1] for g in range(1, 11)]
    reqs.append({"op": "explore", "num_gpu": 2, "model": {"knee_override": knee, "cap_scale": cap}})
    reqs.append({"op": "explore", "num_gpu": 2, "model": {"knee_override": [[2, 2048]]}})
    reqs.append({"op": "explore", "num_gpu": 2, "model": {"min_runnable_share": 2.0}})
    reqs.append({"op": "explore", "num_gpu": 2, "trace_rows": [
        "# bench gpg env runnable top mem", "AT 2 512 1 1000 4.0", "AT 2 1024 1 1900 6.0",
        "AT 2 2048 1 2100 12.0", "AT 2 4096 0 0 0"]})
    reqs.append({"op": "explore", "num_gpu": 2, "trace_rows": ["AT 1 128 1 500 2.0"]})
    reqs.append({"op": "explore", "num_gpu": 2, "trace_rows": [
        "AT 3 128 1 100 2.0", "AT 3 256 1 100 2.0", "AT 3 512 1 150 2.0", "AT 3 1024 1 300 3.0"]})
    # random concave-past-knee models (test_search.cpp:43-61 family), fixed seed
    rng = random.Random(424242)
    for i in range(24):
        u = rng.random
        m = {"peak_top": 5e4 + u() * 2e5, "mem_base": 0.25 + u() * 2.0, "mem_per_env": 0.0005 + u() * 0.004,
             "min_runnable_share": 0.05 + u() * 0.3}
        m["mem_capacity"] = 1e9 if u() < 0.5 else 10.0 * (m["mem_base"] + 512.0 * m["mem_per_env"]) * (1.0 + u() * 20.0)
        m["knee_override"] = [[g, 1 << (9 + int(u() * 4.99))] for g in range(1, 11)]
        m["cap_scale"] = [[g, 0.8 + u() * 0.4] for g in range(1, 11)]
        reqs.append({"op": "explore", "num_gpu": rng.choice([1, 2, 4, 8]), "model": m,
                     "sat_threshold": rng.choice([0.05, 0.1, 0.2])})
    reqs.append({"op": "explore", "num_gpu": 2, "sat_threshold": 0.0})
    reqs.append({"op": "explore", "num_gpu": 0})
    reqs.append({"op": "explore", "num_gpu": 2, "grid": [100, 300, 900], "max_gmis_per_gpu": 3})
    return reqs


def gen_pipeline():
    reqs = []
    tiny = {"bench": "AT", "state_bytes": 4, "action_bytes": 2, "reward_bytes": 1}
    for g in (2, 3, 4):
        for gpg in (1, 2):
            for k in (1, 3, 8):
                for mode in ("stack", "slice"):
                    for seed in (0, 99):
                        reqs.append({"op": "pipeline", "duration": 500.0, "workload": {"bench": "SH"},
                                     "plan": {"template": "async_decoupled", "topology": {"default_gpus": g},
                                              "gmis_per_gpu": gpg},
                                     "topology": {"default_gpus": g},
                                     "config": {"compress_threshold": k, "batch_mode": mode, "seed": seed}})
    coloc = {"kind": "async_decoupled", "gpu_layout": [[0, [0, 1]], [1, [2]]],
             "roles": [[0, ["simulator", "agent"]], [1, ["trainer"]], [2, ["trainer"]]]}
    for ov in (1.0, 0.0):
        reqs.append({"op": "pipeline", "duration": 200.0, "workload": tiny, "plan": coloc,
                     "config": {"compress_threshold": 4, "per_message_overhead": ov}})
    reqs.append({"op": "pipeline", "duration": 0.0, "plan": coloc})
    reqs.append({"op": "pipeline", "duration": 100.0, "plan": coloc, "config": {"compress_threshold": 0}})
    reqs.append({"op": "pipeline", "duration": 100.0, "plan": {"kind": "async_decoupled",
                 "gpu_layout": [[0, [0]]], "roles": [[0, ["trainer"]]]}})
    return reqs


def gen_config():
    reqs = []
    for name in sorted(os.listdir(CONFIG_DIR)):
        if name.endswith(".cfg"):
            with open(os.path.join(CONFIG_DIR, name)) as f:
                reqs.append({"op": "config", "text": f.read(), "origin": name})
    bad = [
        "[topology]\nb1 = 1.0\nbogus = 2\n",
        "[topology\nb1 = 1\n",
        "b1 = 1\n",
        "[]\n",
        "[topology]\njust words\n",
        "[topology]\ngpu = arch=sm80\n",
        "[topology]\ngpu = id=0 arch=sm90\n",
        "[topology]\ngpu = id=x\n",
        "[topology]\ngmi = id=0 gpu=0 backend=tpu\n",
        "[topology]\ngmi = id=0 gpu=0 backend=mig profile=9g.99gb\n",
        "[topology]\ngmi = id=0 gpu=0 backend=mps\n",
        "[topology]\ngpu = id=0 badtoken\n",
        "[workload]\nbenchmark = HM\nalpha = 0.5\nsteps_per_train = 16\n",
        "[workload]\nnope = 1\n",
        "[workload]\nalpha = 2.0\n",
        "[model]\nbatch_mode = zigzag\n",
        "[model]\ngmis_per_gpu = 4\nlatency_scale = 250\nseed = 17\nbatch_mode = slice\n",
        "[search]\nnum_env_min = 256\nnum_env_max = 4096\nprofile_trace = run.tsv\n",
        "[search]\nnum_env_min = 512\nnum_env_max = 256\n",
        "[search]\nwhat = 1\n",
        "# only comments\n\n",
        "[ppo]\nanything = goes\n[topology]\nb2 = 45\n",
    ]
    for text in bad:
        reqs.append({"op": "config", "text": text})
    return reqs


def main():
    if not os.path.exists(REF):
        sys.exit(f"{REF} missing: run `make -C oracle ref` in the build container first")
    suites = {
        "selection": gen_selection(),
        "predict": gen_predict(),
        "execute": execute_requests(),
        "plans": gen_plans(),
        "validate": gen_validate(),
        "workload": gen_workload_costs(),
        "explore": gen_explore(),
        "pipeline": gen_pipeline(),
        "config": gen_config(),
    }
    for name, reqs in suites.items():
        res = run_ref(reqs)
        if name == "execute":
            res = [compact_execute(q, r) for q, r in zip(reqs, res)]
        path = os.path.join(HERE, f"ref_{name}.json")
        with open(path, "w") as f:
            json.dump({"generator": "tests/golden/gen_golden.py via oracle/_ref/gmux_ref",
                       "cases": [{"request": q, "response": r} for q, r in zip(reqs, res)]}, f,
                      separators=(",", ":"))
        print(f"{path}: {len(reqs)} cases, {os.path.getsize(path) // 1024} KiB")


if __name__ == "__main__":
    main()
