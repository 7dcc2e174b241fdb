// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// Golden-vector driver for the reference planner/simulator. Compiled by
// oracle/Makefile directly against the read-only reference headers under
// /root/reference/proj/include (nothing is copied), producing oracle/_ref/gmux_ref.
// It reads a JSON array of requests on stdin and writes a JSON array of responses,
// one per request, so tests/golden/gen_golden.py can pin the product's integer and
// fp64 contracts to the reference's own outputs:
//   select/leaders/rings  reduction.hpp:98-139      predict  reduction.hpp:142-152
//   execute               reduction.hpp:225-334      plan     mapping.hpp:216-279
//   validate              topology.hpp:134-212       workload workload.hpp:95-134
//   costs                 mapping.hpp:95-178          explore  search.hpp:54-249
//   pipeline              channels.hpp:110-397        config   config.hpp:125-301
#include <cstdint>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "gmux/channels.hpp"
#include "gmux/config.hpp"
#include "gmux/mapping.hpp"
#include "gmux/reduction.hpp"
#include "gmux/search.hpp"
#include "gmux/topology.hpp"
#include "gmux/workload.hpp"

using nlohmann::json;
using namespace gmux;

namespace {

// Deterministic buffer values shared with tests (see tests/golden/gen_golden.py):
// "cli":  1.0 + 0.001*id + 1e-6*e            (tools/gmux.cpp:228)
// "hash": 0.1 + 0.9*u53(splitmix64(seed,id,e)) (U(0.1,1.0) like test_reduction.cpp:25)
double buffer_value(const std::string& kind, uint64_t seed, int id, std::size_t e) {
  if (kind == "cli") return 1.0 + 0.001 * id + 1e-6 * double(e);
  uint64_t z = seed * 0x9E3779B97F4A7C15ull + uint64_t(int64_t(id)) * 0xBF58476D1CE4E5B9ull +
               uint64_t(e) * 0x94D049BB133111EBull;
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  const double u = double(z >> 11) * (1.0 / 9007199254740992.0);
  return 0.1 + 0.9 * u;
}

GmiLayout layout_of(const json& j) {
  GmiLayout l;
  for (const auto& g : j) l.mpl.push_back(g.get<std::vector<int>>());
  return l;
}

Strategy strategy_of(const std::string& s) {
  if (s == "MPR") return Strategy::MPR;
  if (s == "MRR") return Strategy::MRR;
  if (s == "HAR") return Strategy::HAR;
  throw std::invalid_argument("bad strategy " + s);
}

TemplateKind template_of(const std::string& s) {
  if (s == "TDG") return TemplateKind::TDG;
  if (s == "TCG") return TemplateKind::TCG;
  if (s == "TDG_EX") return TemplateKind::TDG_EX;
  if (s == "TCG_EX") return TemplateKind::TCG_EX;
  if (s == "async_decoupled") return TemplateKind::AsyncDecoupled;
  throw std::invalid_argument("bad template " + s);
}

Topology topology_of(const json& j) {
  Topology t = default_topology(0);
  if (j.contains("default_gpus")) t = default_topology(j["default_gpus"].get<int>());
  if (j.contains("b1")) t.b1 = j["b1"];
  if (j.contains("b2")) t.b2 = j["b2"];
  for (const auto& g : j.value("gpus", json::array())) {
    GpuSpec s;
    s.id = g["id"];
    s.arch = g.value("arch", std::string("sm80")) == "sm70" ? GpuArch::SM70 : GpuArch::SM80;
    s.sm_units = g.value("sm_units", kSmUnitsPerGpu);
    s.mem_gb = g.value("mem_gb", 40.0);
    t.gpus.push_back(s);
  }
  for (const auto& p : j.value("partitions", json::array())) {
    GmiPartition q;
    q.gmi_id = p["gmi_id"];
    q.gpu_id = p["gpu_id"];
    q.backend = p.value("backend", std::string("mps")) == "mig" ? Backend::MIG : Backend::MPS;
    q.sm_share = p["sm_share"];
    q.mem_gb = p["mem_gb"];
    t.partitions.push_back(q);
  }
  return t;
}

std::string role_name(Role r) { return to_string(r); }

json plan_json(const MappingPlan& p) {
  json out;
  out["template"] = to_string(p.template_kind);
  json layout = json::array();
  for (const auto& [gpu, ids] : p.gpu_layout) layout.push_back({gpu, ids});
  out["gpu_layout"] = layout;
  json roles = json::array();
  for (const auto& [gmi, rs] : p.gmi_assignments) {
    std::vector<std::string> names;
    for (Role r : rs) names.push_back(role_name(r));
    roles.push_back({gmi, names});
  }
  out["roles"] = roles;
  out["serving_gpus"] = p.serving_gpus;
  out["training_gpus"] = p.training_gpus;
  return out;
}

MappingPlan plan_of(const json& j) {
  if (j.contains("template") && j.contains("topology"))
    return build_plan(template_of(j["template"]), topology_of(j["topology"]),
                      load_benchmark(j.value("bench", std::string("AT"))), j["gmis_per_gpu"]);
  MappingPlan p;  // explicit plan (test_channels.cpp:27-36 style)
  p.template_kind = template_of(j.value("kind", std::string("async_decoupled")));
  for (const auto& e : j["gpu_layout"]) p.gpu_layout[e[0].get<int>()] = e[1].get<std::vector<int>>();
  for (const auto& e : j["roles"]) {
    std::set<Role> rs;
    for (const auto& n : e[1]) {
      const std::string s = n;
      rs.insert(s == "simulator" ? Role::Simulator : s == "agent" ? Role::Agent : Role::Trainer);
    }
    p.gmi_assignments[e[0].get<int>()] = rs;
  }
  return p;
}

DrlWorkload workload_of(const json& j) {
  DrlWorkload w = load_benchmark(j.value("bench", std::string("AT")));
  if (j.contains("state_bytes")) w.state_bytes = j["state_bytes"];
  if (j.contains("action_bytes")) w.action_bytes = j["action_bytes"];
  if (j.contains("reward_bytes")) w.reward_bytes = j["reward_bytes"];
  if (j.contains("trainer_t_iter")) w.trainer.t_iter = j["trainer_t_iter"];
  return w;
}

json workload_json(const DrlWorkload& w) {
  return {{"name", w.name},
          {"state_bytes", w.state_bytes},
          {"action_bytes", w.action_bytes},
          {"reward_bytes", w.reward_bytes},
          {"model_bytes", w.model_bytes},
          {"steps_per_train", w.steps_per_train},
          {"alpha", w.alpha},
          {"beta", w.beta},
          {"policy_dims", w.policy_dims},
          {"param_count", policy_value_param_count(w.policy_dims)},
          {"sim", {w.simulator.r_sm, w.simulator.r_mem, w.simulator.t_iter}},
          {"agent", {w.agent.r_sm, w.agent.r_mem, w.agent.t_iter}},
          {"trainer", {w.trainer.r_sm, w.trainer.r_mem, w.trainer.t_iter}}};
}

json opt_json(const std::optional<double>& v) { return v ? json(*v) : json(nullptr); }

json handle(const json& rq) {
  const std::string op = rq["op"];
  json out;
  if (op == "select") {
    out["strategy"] = to_string(select_strategy(layout_of(rq["mpl"])));
  } else if (op == "leaders") {
    out["leaders"] = leader_gmis(layout_of(rq["mpl"]));
  } else if (op == "rings") {
    out["rings"] = mrr_rings(layout_of(rq["mpl"]));
  } else if (op == "predict") {
    out["latency"] = predict_latency(strategy_of(rq["s"]), rq["g"], rq["t"], rq["m_p"], rq["b1"],
                                     rq["b2"]);
  } else if (op == "execute") {
    const GmiLayout layout = layout_of(rq["mpl"]);
    const std::size_t len = rq["len"];
    const std::string kind = rq.value("gen", std::string("hash"));
    const uint64_t seed = rq.value("seed", uint64_t(0));
    std::vector<GradientBuffer> bufs;
    for (int id : layout.all_gmis()) {
      GradientBuffer b{id, std::vector<double>(len)};
      for (std::size_t e = 0; e < len; ++e) b.values[e] = buffer_value(kind, seed, id, e);
      bufs.push_back(std::move(b));
    }
    Topology topo = default_topology(4);
    topo.b1 = rq.value("b1", 1.0);
    topo.b2 = rq.value("b2", 30.0);
    const ReductionRun run = execute(strategy_of(rq["strategy"]), layout, bufs, topo);
    out["strategy"] = to_string(run.strategy);
    out["latency"] = run.latency;
    out["broadcast_latency"] = run.broadcast_latency;
    json trace = json::array();
    for (const auto& e : run.trace) trace.push_back({e.step, e.src, e.dst, e.bytes, to_string(e.kind)});
    out["trace"] = trace;
    out["result"] = run.result;
  } else if (op == "plan") {
    out = plan_json(plan_of(rq));
  } else if (op == "validate") {
    const ValidationReport r = validate_layout(topology_of(rq["topology"]));
    json v = json::array();
    for (const auto& x : r.violations) v.push_back({x.gpu_id, x.rule});
    out["violations"] = v;
  } else if (op == "workload") {
    out = workload_json(load_benchmark(rq["bench"].get<std::string>()));
  } else if (op == "costs") {
    const DrlWorkload w = workload_of(rq);
    const int n = rq.value("n_gmis", 1);
    const CostEstimate tdg = training_cost(TemplateKind::TDG_EX, w, n);
    const CostEstimate tcg = training_cost(TemplateKind::TCG_EX, w, n);
    const CostEstimate sd = serving_cost(TemplateKind::TDG, w);
    const CostEstimate sc = serving_cost(TemplateKind::TCG, w);
    out["train_dedicated"] = {tdg.resource_size, tdg.comm_bytes};
    out["train_colocated"] = {tcg.resource_size, tcg.comm_bytes};
    out["serve_dedicated"] = {sd.resource_size, sd.comm_bytes};
    out["serve_colocated"] = {sc.resource_size, sc.comm_bytes};
    out["serving_ratio"] = serving_throughput_ratio(w);
    out["training_ratio"] = training_throughput_ratio(w);
    out["serving_penalty"] = serving_colocation_penalty(w);
    out["training_penalty"] = training_colocation_penalty(w);
    out["allreduce_bytes"] = allreduce_bytes(n, w.model_bytes);
    const double bw = rq.value("bandwidth", 1000.0);
    out["training_throughput"] = training_throughput(tcg, w, rq.value("r_all", 8.0), bw);
  } else if (op == "explore") {
    std::unique_ptr<Profiler> prof;
    if (rq.contains("trace_rows")) {
      const std::string path = "/tmp/gmux_ref_trace_" + std::to_string(::getpid()) + ".tsv";
      {
        std::ofstream f(path);
        for (const auto& r : rq["trace_rows"]) f << r.get<std::string>() << "\n";
      }
      prof = std::make_unique<RecordedTraceProfiler>(RecordedTraceProfiler::from_file(path));
      std::remove(path.c_str());
    } else {
      auto m = std::make_unique<SyntheticCostModel>();
      const json& mj = rq.value("model", json::object());
      if (mj.contains("peak_top")) m->peak_top = mj["peak_top"];
      if (mj.contains("mem_base")) m->mem_base = mj["mem_base"];
      if (mj.contains("mem_per_env")) m->mem_per_env = mj["mem_per_env"];
      if (mj.contains("mem_capacity")) m->mem_capacity = mj["mem_capacity"];
      if (mj.contains("min_runnable_share")) m->min_runnable_share = mj["min_runnable_share"];
      if (mj.contains("knee_base")) m->knee_base = mj["knee_base"];
      for (const auto& e : mj.value("knee_override", json::array())) m->knee_override[e[0]] = e[1];
      for (const auto& e : mj.value("cap_scale", json::array())) m->cap_scale[e[0]] = e[1];
      prof = std::move(m);
    }
    const json& ej = rq.value("estimator", json::object());
    ThroughputEstimator est{load_benchmark(ej.value("bench", std::string("AT"))),
                            ej.value("b1", 1.0), ej.value("b2", 30.0),
                            ej.value("latency_scale", 1000.0)};
    SearchConfig cfg;
    if (rq.contains("grid")) cfg.num_env_grid = rq["grid"].get<std::vector<int>>();
    cfg.max_gmis_per_gpu = rq.value("max_gmis_per_gpu", 10);
    cfg.sat_threshold = rq.value("sat_threshold", 0.1);
    const SearchResult r = explore(*prof, est, rq.value("bench", std::string("AT")), rq["num_gpu"], cfg);
    out["feasible"] = r.feasible;
    out["reason"] = r.reason;
    out["num_env"] = r.num_env;
    out["gmis_per_gpu"] = r.gmis_per_gpu;
    out["est_throughput"] = r.est_throughput;
    json vis = json::array();
    for (const auto& v : r.visited)
      vis.push_back({v.gmis_per_gpu, v.num_env, v.runnable, v.top, v.mem, opt_json(v.sat),
                     opt_json(v.acc_top), v.pruned_here});
    out["visited"] = vis;
    if (rq.value("comm_discount", false)) {
      json cd = json::array();
      for (int gpg = 1; gpg <= 10; ++gpg) cd.push_back(est.comm_discount(gpg, rq["num_gpu"]));
      out["comm_discount"] = cd;
    }
  } else if (op == "pipeline") {
    const DrlWorkload w = workload_of(rq.value("workload", json::object()));
    const MappingPlan plan = plan_of(rq["plan"]);
    const Topology topo = topology_of(rq.value("topology", json{{"default_gpus", 2}}));
    PipelineConfig c;
    const json& cj = rq.value("config", json::object());
    c.compress_threshold = cj.value("compress_threshold", 8);
    c.batch_mode = cj.value("batch_mode", std::string("stack")) == "slice" ? BatchMode::Slice
                                                                          : BatchMode::Stack;
    c.target_batch = cj.value("target_batch", 32);
    c.per_message_overhead = cj.value("per_message_overhead", 1.0);
    c.seed = cj.value("seed", 0u);
    const PipelineMetrics m = simulate_pipeline(w, plan, topo, c, rq["duration"]);
    out["pps"] = m.pps;
    out["ttop"] = m.ttop;
    out["records_produced"] = m.records_produced;
    out["records_delivered"] = m.records_delivered;
    out["units_sent"] = m.units_sent;
    out["batches_emitted"] = m.batches_emitted;
    out["bytes_moved"] = m.bytes_moved;
    out["transfer_busy_time"] = m.transfer_busy_time;
    out["delivery_makespan"] = m.delivery_makespan;
    out["training_makespan"] = m.training_makespan;
    json tr = json::array();
    for (const auto& [t, n] : m.trainer_records) tr.push_back({t, n});
    out["trainer_records"] = tr;
    json bs = json::array();
    for (const auto& b : m.batches) {
      json recs = json::array();
      for (const auto& r : b.records) recs.push_back({r.agent_gmi, r.seq});
      bs.push_back({b.trainer_gmi, b.emit_time, recs});
    }
    out["batches"] = bs;
  } else if (op == "config") {
    std::istringstream in(rq["text"].get<std::string>());
    const ConfigFile cfg = parse_config(in, rq.value("origin", std::string("<config>")));
    const Topology t = topology_from_config(cfg);
    json gpus = json::array();
    for (const auto& g : t.gpus) gpus.push_back({g.id, to_string(g.arch), g.sm_units, g.mem_gb});
    json parts = json::array();
    for (const auto& p : t.partitions)
      parts.push_back({p.gmi_id, p.gpu_id, to_string(p.backend), p.sm_share, p.mem_gb});
    out["topology"] = {{"b1", t.b1}, {"b2", t.b2}, {"gpus", gpus}, {"partitions", parts}};
    out["workload"] = workload_json(workload_from_config(cfg));
    const ModelParams m = model_from_config(cfg);
    out["model"] = {{"serving_combw_factor", m.calibration.serving_combw_factor},
                    {"training_combw_factor", m.calibration.training_combw_factor},
                    {"gmis_per_gpu", m.gmis_per_gpu},
                    {"latency_scale", m.latency_scale},
                    {"compress_threshold", m.pipeline.compress_threshold},
                    {"target_batch", m.pipeline.target_batch},
                    {"message_overhead", m.pipeline.per_message_overhead},
                    {"seed", m.pipeline.seed},
                    {"batch_mode", m.pipeline.batch_mode == BatchMode::Slice ? "slice" : "stack"}};
    const SearchSettings s = search_from_config(cfg);
    out["search"] = {{"sat_threshold", s.config.sat_threshold},
                     {"max_gmis_per_gpu", s.config.max_gmis_per_gpu},
                     {"grid", s.config.num_env_grid},
                     {"profile_trace", s.profile_trace ? json(*s.profile_trace) : json(nullptr)}};
  } else {
    throw std::invalid_argument("unknown op " + op);
  }
  return out;
}

}  // namespace

int main() {
  json requests = json::parse(std::cin);
  json responses = json::array();
  for (const auto& rq : requests) {
    json r;
    try {
      r = handle(rq);
    } catch (const MultiStreamError& e) {
      r = {{"error", e.what()}, {"type", "MultiStreamError"}};
    } catch (const PlanError& e) {
      r = {{"error", e.what()}, {"type", "PlanError"}};
    } catch (const PipelineError& e) {
      r = {{"error", e.what()}, {"type", "PipelineError"}};
    } catch (const ConfigError& e) {
      r = {{"error", e.what()}, {"type", "ConfigError"}};
    } catch (const std::invalid_argument& e) {
      r = {{"error", e.what()}, {"type", "invalid_argument"}};
    } catch (const std::exception& e) {
      r = {{"error", e.what()}, {"type", "runtime_error"}};
    }
    responses.push_back(r);
  }
  std::cout << responses.dump() << "\n";
  return 0;
}
