"""Product planner (libgmi C-ABI via the gmux mirror) vs the reference's own outputs.

Every fixture under tests/golden/ref_*.json was produced by running the reference
planner (oracle/_ref/gmux_ref, compiled from /root/reference headers) on the request;
see tests/golden/gen_golden.py.  Integer contracts and fp64 closed forms must match
exactly (the same IEEE operation sequence), including exception type and message.
"""
import hashlib
import json
import os

import pytest

from paper_2206_08482_b200 import gmux as G

HERE = os.path.dirname(os.path.abspath(__file__))
ERR = {"invalid_argument": ValueError, "MultiStreamError": G.MultiStreamError,
       "PlanError": G.PlanError, "PipelineError": G.PipelineError, "ConfigError": G.ConfigError,
       "runtime_error": RuntimeError}


def cases(name):
    with open(os.path.join(HERE, "golden", f"ref_{name}.json")) as f:
        return json.load(f)["cases"]


def expect_error(resp, fn):
    with pytest.raises(ERR[resp["type"]]) as ei:
        fn()
    assert str(ei.value) == resp["error"]


def run(resp, fn):
    if "error" in resp:
        expect_error(resp, fn)
        return None
    return fn()


# ------------------------------------------------------------------ reduction.hpp
def test_selection_leaders_rings():
    n = 0
    for c in cases("selection"):
        rq, rs = c["request"], c["response"]
        if rq["op"] == "select":
            got = run(rs, lambda: G.select_strategy(rq["mpl"]))
            if got is not None:
                assert got.name == rs["strategy"], rq
        elif rq["op"] == "leaders":
            got = run(rs, lambda: G.leader_gmis(rq["mpl"]))
            if got is not None:
                assert got == rs["leaders"], rq
        else:
            got = run(rs, lambda: G.mrr_rings(rq["mpl"]))
            if got is not None:
                assert got == rs["rings"], rq
        n += 1
    assert n > 7000


def test_predict_latency_exact():
    for c in cases("predict"):
        rq, rs = c["request"], c["response"]
        got = run(rs, lambda: G.predict_latency(G.Strategy[rq["s"]], rq["g"], rq["t"], rq["m_p"], rq["b1"], rq["b2"]))
        if got is not None:
            assert got == rs["latency"], rq


def _trace_digest(events):
    s = "\n".join(f"{e.step} {e.src} {e.dst} {e.bytes!r} {G.to_string(e.kind)}" for e in events)
    return hashlib.sha256(s.encode()).hexdigest()


def test_execute_schedule_and_latency():
    """Trace (step/src/dst/bytes/kind), latency and broadcast latency of execute()."""
    for c in cases("execute"):
        rq, rs = c["request"], c["response"]
        fn = lambda: G.reduction_schedule(G.Strategy[rq["strategy"]], rq["mpl"], rq["len"],
                                          rq.get("b1", 1.0), rq.get("b2", 30.0))
        got = run(rs, fn)
        if got is None:
            continue
        info, trace = got
        assert info.latency == rs["latency"], rq
        assert info.broadcast_latency == rs["broadcast_latency"], rq
        assert len(trace) == rs["trace_len"], rq
        if "trace" in rs:
            assert [[e.step, e.src, e.dst, e.bytes, G.to_string(e.kind)] for e in trace] == rs["trace"]
        assert _trace_digest(trace) == rs["trace_sha256"], rq


def test_cli_example_latencies():
    """README: reduce --layout [[0,1],[2,3]] --payload 240 -> MRR 24 (MPR 360, HAR 248)."""
    lay = [[0, 1], [2, 3]]
    assert G.select_strategy(lay) == G.Strategy.MRR
    assert [G.predict_latency(s, 2, 2, 240, 1, 30) for s in G.Strategy] == [360.0, 24.0, 248.0]


def test_layout_validation_errors():
    for bad, msg in (([], "layout needs at least one GPU"), ([[0, 1], []], "layout has an empty per-GPU list"),
                     ([[0, 1], [1, 2]], "duplicate gmi id 1 in layout")):
        with pytest.raises(ValueError, match=msg):
            G.GmiLayout(bad).validate()


# ------------------------------------------------------------------ topology / mapping / workload
def _topology(j):
    if "default_gpus" in j:
        t = G.default_topology(j["default_gpus"])
    else:
        t = G.Topology()
    t.b1, t.b2 = j.get("b1", t.b1), j.get("b2", t.b2)
    for g in j.get("gpus", []):
        t.gpus.append(G.GpuSpec(g["id"], G.GpuArch.SM70 if g.get("arch") == "sm70" else G.GpuArch.SM80,
                                g.get("sm_units", 8), g.get("mem_gb", 40.0)))
    for p in j.get("partitions", []):
        t.partitions.append(G.GmiPartition(p["gmi_id"], p["gpu_id"],
                                           G.Backend.MIG if p.get("backend") == "mig" else G.Backend.MPS,
                                           p["sm_share"], p["mem_gb"]))
    return t


TPL = {"TDG": G.TemplateKind.TDG, "TCG": G.TemplateKind.TCG, "TDG_EX": G.TemplateKind.TDG_EX,
       "TCG_EX": G.TemplateKind.TCG_EX, "async_decoupled": G.TemplateKind.AsyncDecoupled}
ROLE = {"simulator": G.Role.Simulator, "agent": G.Role.Agent, "trainer": G.Role.Trainer}


def _plan_json(p):
    return {"template": G.to_string(p.template_kind),
            "gpu_layout": [[g, p.gpu_layout[g]] for g in sorted(p.gpu_layout)],
            "roles": [[i, sorted((G.to_string(r) for r in p.gmi_assignments[i]),
                                 key=lambda n: ["simulator", "agent", "trainer"].index(n))]
                      for i in sorted(p.gmi_assignments)],
            "serving_gpus": p.serving_gpus, "training_gpus": p.training_gpus}


def test_build_plan():
    for c in cases("plans"):
        rq, rs = c["request"], c["response"]
        got = run(rs, lambda: G.build_plan(TPL[rq["template"]], _topology(rq["topology"]),
                                           G.load_benchmark("AT"), rq["gmis_per_gpu"]))
        if got is not None:
            assert _plan_json(got) == rs, rq


def test_validate_layout():
    for c in cases("validate"):
        rq, rs = c["request"], c["response"]
        got = [[v.gpu_id, v.rule] for v in G.validate_layout(_topology(rq["topology"]))]
        assert got == rs["violations"], rq


def _workload_json(w):
    return {"name": w.name, "state_bytes": w.state_bytes, "action_bytes": w.action_bytes,
            "reward_bytes": w.reward_bytes, "model_bytes": w.model_bytes,
            "steps_per_train": w.steps_per_train, "alpha": w.alpha, "beta": w.beta,
            "policy_dims": w.policy_dims, "param_count": G.policy_value_param_count(w.policy_dims),
            "sim": [w.simulator.r_sm, w.simulator.r_mem, w.simulator.t_iter],
            "agent": [w.agent.r_sm, w.agent.r_mem, w.agent.t_iter],
            "trainer": [w.trainer.r_sm, w.trainer.r_mem, w.trainer.t_iter]}


def test_workload_and_costs():
    for c in cases("workload"):
        rq, rs = c["request"], c["response"]
        if rq["op"] == "workload":
            got = run(rs, lambda: G.load_benchmark(rq["bench"]))
            if got is not None:
                assert _workload_json(got) == rs
            continue
        w = G.load_benchmark(rq["bench"])
        n = rq["n_gmis"]
        tdg, tcg = G.training_cost(G.TemplateKind.TDG_EX, w, n), G.training_cost(G.TemplateKind.TCG_EX, w, n)
        sd, sc = G.serving_cost(G.TemplateKind.TDG, w), G.serving_cost(G.TemplateKind.TCG, w)
        assert [tdg.resource_size, tdg.comm_bytes] == rs["train_dedicated"]
        assert [tcg.resource_size, tcg.comm_bytes] == rs["train_colocated"]
        assert [sd.resource_size, sd.comm_bytes] == rs["serve_dedicated"]
        assert [sc.resource_size, sc.comm_bytes] == rs["serve_colocated"]
        assert G.serving_throughput_ratio(w) == rs["serving_ratio"]
        assert G.training_throughput_ratio(w) == rs["training_ratio"]
        assert G.serving_colocation_penalty(w) == rs["serving_penalty"]
        assert G.training_colocation_penalty(w) == rs["training_penalty"]
        assert G.allreduce_bytes(n, w.model_bytes) == rs["allreduce_bytes"]
        assert G.training_throughput(tcg, w, 8.0, 1000.0) == rs["training_throughput"]


def test_headline_ratios():
    """test_mapping.cpp:89-95: 2.58 / 5.458 / 0.16279 / 0.46580."""
    w = G.load_benchmark("AT")
    assert abs(G.serving_throughput_ratio(w) - 2.58) < 1e-2
    assert abs(G.training_throughput_ratio(w) - 5.458) < 1e-3
    assert abs(G.serving_colocation_penalty(w) - 0.16279) < 1e-5
    assert abs(G.training_colocation_penalty(w) - 0.46580) < 1e-5
    assert [G.policy_value_param_count(G.load_benchmark(b).policy_dims) for b in ("AT", "HM", "SH")] == \
        [114121, 286822, 1535765]


# ------------------------------------------------------------------ search.hpp
def _visited(r):
    return [[v.gmis_per_gpu, v.num_env, v.runnable, v.top, v.mem, v.sat, v.acc_top, v.pruned_here]
            for v in r.visited]


def test_explore(tmp_path):
    for i, c in enumerate(cases("explore")):
        rq, rs = c["request"], c["response"]
        if "trace_rows" in rq:
            p = tmp_path / f"trace{i}.tsv"
            p.write_text("\n".join(rq["trace_rows"]) + "\n")
            prof = G.RecordedTraceProfiler.from_file(str(p))
        else:
            m = rq.get("model", {})
            prof = G.SyntheticCostModel(**{k: v for k, v in m.items() if k not in ("knee_override", "cap_scale")})
            prof.knee_override = {k: v for k, v in m.get("knee_override", [])}
            prof.cap_scale = {k: v for k, v in m.get("cap_scale", [])}
        ej = rq.get("estimator", {})
        est = G.ThroughputEstimator(G.load_benchmark(ej.get("bench", "AT")), ej.get("b1", 1.0), ej.get("b2", 30.0),
                                    ej.get("latency_scale", 1000.0))
        cfg = G.SearchConfig(rq.get("grid", G.SearchConfig().num_env_grid), rq.get("max_gmis_per_gpu", 10),
                             rq.get("sat_threshold", 0.1))
        got = run(rs, lambda: G.explore(prof, est, rq.get("bench", "AT"), rq["num_gpu"], cfg))
        if got is None:
            continue
        assert (got.feasible, got.reason, got.num_env, got.gmis_per_gpu, got.est_throughput) == \
            (rs["feasible"], rs["reason"], rs["num_env"], rs["gmis_per_gpu"], rs["est_throughput"]), rq
        assert _visited(got) == rs["visited"], rq
        if rq.get("comm_discount"):
            assert [est.comm_discount(g, rq["num_gpu"]) for g in range(1, 11)] == rs["comm_discount"]


def test_explore_profiler_exception_propagates():
    class Boom(G.Profiler):
        def profile(self, bench, gpg, env):
            raise KeyError("boom")

    with pytest.raises(KeyError):
        G.explore(Boom(), G.ThroughputEstimator(G.load_benchmark("AT")), "AT", 2)


# ------------------------------------------------------------------ channels.hpp
def _plan_from(j):
    if "template" in j:
        return G.build_plan(TPL[j["template"]], _topology(j["topology"]), G.load_benchmark(j.get("bench", "AT")),
                            j["gmis_per_gpu"])
    p = G.MappingPlan(TPL[j.get("kind", "async_decoupled")])
    for g, ids in j["gpu_layout"]:
        p.gpu_layout[g] = ids
    for i, names in j["roles"]:
        p.gmi_assignments[i] = {ROLE[n] for n in names}
    return p


def test_simulate_pipeline():
    for c in cases("pipeline"):
        rq, rs = c["request"], c["response"]
        wj = rq.get("workload", {})
        w = G.load_benchmark(wj.get("bench", "AT"))
        for k in ("state_bytes", "action_bytes", "reward_bytes"):
            if k in wj:
                setattr(w, k, wj[k])
        cj = rq.get("config", {})
        cfg = G.PipelineConfig(cj.get("compress_threshold", 8),
                               G.BatchMode.Slice if cj.get("batch_mode") == "slice" else G.BatchMode.Stack,
                               cj.get("target_batch", 32), cj.get("per_message_overhead", 1.0), cj.get("seed", 0))
        topo = _topology(rq.get("topology", {"default_gpus": 2}))
        got = run(rs, lambda: G.simulate_pipeline(w, _plan_from(rq["plan"]), topo, cfg, rq["duration"]))
        if got is None:
            continue
        for k in ("pps", "ttop", "records_produced", "records_delivered", "units_sent", "batches_emitted",
                  "bytes_moved", "transfer_busy_time", "delivery_makespan", "training_makespan"):
            assert getattr(got, k) == rs[k], (k, rq)
        assert [[t, n] for t, n in sorted(got.trainer_records.items())] == rs["trainer_records"]
        assert [[b.trainer_gmi, b.emit_time, [[r.agent_gmi, r.seq] for r in b.records]] for b in got.batches] == \
            rs["batches"]


# ------------------------------------------------------------------ config.hpp
def test_config_schema():
    for c in cases("config"):
        rq, rs = c["request"], c["response"]

        def load():
            cfg = G.parse_config(rq["text"], rq.get("origin", "<config>"))
            t = G.topology_from_config(cfg)
            w = G.workload_from_config(cfg)
            m = G.model_from_config(cfg)
            s = G.search_from_config(cfg)
            return t, w, m, s

        got = run(rs, load)
        if got is None:
            continue
        t, w, m, s = got
        assert {"b1": t.b1, "b2": t.b2,
                "gpus": [[g.id, "sm70" if g.arch == G.GpuArch.SM70 else "sm80", g.sm_units, g.mem_gb] for g in t.gpus],
                "partitions": [[p.gmi_id, p.gpu_id, "mig" if p.backend == G.Backend.MIG else "mps", p.sm_share, p.mem_gb]
                               for p in t.partitions]} == rs["topology"]
        assert _workload_json(w) == rs["workload"]
        assert {"serving_combw_factor": m.calibration.serving_combw_factor,
                "training_combw_factor": m.calibration.training_combw_factor,
                "gmis_per_gpu": m.gmis_per_gpu, "latency_scale": m.latency_scale,
                "compress_threshold": m.pipeline.compress_threshold, "target_batch": m.pipeline.target_batch,
                "message_overhead": m.pipeline.per_message_overhead, "seed": m.pipeline.seed,
                "batch_mode": "slice" if m.pipeline.batch_mode == G.BatchMode.Slice else "stack"} == rs["model"]
        assert {"sat_threshold": s.config.sat_threshold, "max_gmis_per_gpu": s.config.max_gmis_per_gpu,
                "grid": s.config.num_env_grid, "profile_trace": s.profile_trace} == rs["search"]


def test_config_missing_file():
    with pytest.raises(G.ConfigError, match="config not found: /no/such.cfg"):
        G.load_config("/no/such.cfg")


def test_config_extension_sections_visible_to_b200_only():
    cfg = G.load_config(os.path.join(os.path.dirname(HERE), "configs", "at_4096env_3x256.cfg"))
    assert cfg.get("ppo", "num_envs") == "4096"
    assert cfg.get("ppo", "hidden") == "256,256,256"
    assert G.topology_from_config(G.parse_config("[topology]\ngpu = id=0 arch=sm100\n")).gpus[0].arch == G.GpuArch.SM100
