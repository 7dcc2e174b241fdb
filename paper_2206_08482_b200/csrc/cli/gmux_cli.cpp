// `gmux` command line front end over the B200 drop-in (include/gmux/gmux.hpp -> libgmi.so).
//
// Same subcommands, options, text / structured (JSON) renderings and exit codes as the
// reference CLI (proj/tools/gmux.cpp:349-412; reports proj/include/gmux/report.hpp:23-129), so
// scripts written against the reference keep working byte for byte (tests/test_cli.py pins the
// output against the reference binary). Exit codes: 0 ok, 1 domain violation / infeasible,
// 2 usage, config or I/O error (G:389-411).
//
// B200 extensions (additive): `search --profiler gpu` drives Alg. 2 with the measured PPO
// iteration (GpuProfiler, green-context GMIs); `reduce --device` runs the reduction data path on
// the GPU (the drop-in execute(): K1 fold via gmi_execute_host) instead of the host fold.
#include <cctype>
#include <cmath>
#include <fstream>
#include <functional>
#include <iomanip>
#include <iostream>
#include <map>
#include <memory>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "gmux/gmux.hpp"

namespace {

using json = nlohmann::json;
using namespace gmux;

// ------------------------------------------------------------------ arguments
struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Args {
  std::string command;
  std::string topology;
  std::string workload = "AT";
  std::string mode = "serving";
  std::string format = "text";
  std::optional<double> b1, b2, sat_threshold;
  double duration = 2000.0;
  std::string force_strategy, layout, profiler = "synthetic";
  double payload = 0;
  bool full_trace = false, device = false;
};

double to_number(const std::string& opt, const std::string& v) {
  std::size_t used = 0;
  double d = 0;
  try {
    d = std::stod(v, &used);
  } catch (const std::exception&) {
    used = 0;
  }
  if (used != v.size()) throw UsageError("could not convert: " + opt + " = " + v);
  return d;
}

Args parse_args(int argc, char** argv) {
  static const std::vector<std::string> kCommands = {"validate", "plan", "reduce", "pipeline", "search"};
  Args a;
  // option -> (commands that accept it, empty = global; setter)
  using Setter = std::function<void(const std::string&)>;
  struct Spec {
    std::vector<std::string> scope;
    bool flag;
    Setter set;
  };
  const std::map<std::string, Spec> specs = {
      {"--topology", {{}, false, [&](const std::string& v) { a.topology = v; }}},
      {"--workload", {{}, false, [&](const std::string& v) { a.workload = v; }}},
      {"--mode", {{}, false, [&](const std::string& v) { a.mode = v; }}},
      {"--b1", {{}, false, [&](const std::string& v) { a.b1 = to_number("--b1", v); }}},
      {"--b2", {{}, false, [&](const std::string& v) { a.b2 = to_number("--b2", v); }}},
      {"--sat-threshold", {{}, false, [&](const std::string& v) { a.sat_threshold = to_number("--sat-threshold", v); }}},
      {"--format", {{}, false, [&](const std::string& v) {
                      if (v != "text" && v != "structured") throw UsageError("--format: " + v + " not in {...}");
                      a.format = v;
                    }}},
      {"--layout", {{"reduce"}, false, [&](const std::string& v) { a.layout = v; }}},
      {"--payload", {{"reduce"}, false, [&](const std::string& v) { a.payload = to_number("--payload", v); }}},
      {"--force-strategy", {{"reduce"}, false, [&](const std::string& v) { a.force_strategy = v; }}},
      {"--full-trace", {{"reduce"}, true, [&](const std::string&) { a.full_trace = true; }}},
      {"--device", {{"reduce"}, true, [&](const std::string&) { a.device = true; }}},
      {"--duration", {{"pipeline"}, false, [&](const std::string& v) {
                        a.duration = to_number("--duration", v);
                        if (!(a.duration > 0)) throw UsageError("--duration: Value " + v + " not a positive number");
                      }}},
      {"--profiler", {{"search"}, false, [&](const std::string& v) {
                        if (v != "synthetic" && v != "gpu") throw UsageError("--profiler: expected synthetic or gpu");
                        a.profiler = v;
                      }}},
  };
  for (int i = 1; i < argc; ++i) {
    std::string tok = argv[i];
    if (tok.rfind("--", 0) != 0) {
      bool known = false;
      for (const auto& c : kCommands) known = known || c == tok;
      if (!a.command.empty() || !known) throw UsageError("The following argument was not expected: " + tok);
      a.command = tok;
      continue;
    }
    std::optional<std::string> value;
    if (const auto eq = tok.find('='); eq != std::string::npos) {
      value = tok.substr(eq + 1);
      tok.resize(eq);
    }
    const auto it = specs.find(tok);
    const bool in_scope = it != specs.end() &&
                          (it->second.scope.empty() ||
                           (!a.command.empty() && it->second.scope.front() == a.command));
    if (!in_scope) throw UsageError("The following argument was not expected: " + tok);
    if (!it->second.flag && !value) {
      if (i + 1 >= argc) throw UsageError(tok + " requires an argument");
      value = argv[++i];
    }
    it->second.set(value.value_or(""));
  }
  if (a.command.empty()) throw UsageError("A subcommand is required");
  return a;
}

// ------------------------------------------------------------------ shared context
struct Session {
  ConfigFile cfg;
  Topology topo;
  DrlWorkload workload;
  ModelParams model;
  SearchSettings search;
};

Session open_session(const Args& a, bool topology_required) {
  Session s;
  if (!a.topology.empty())
    s.cfg = load_config(a.topology);
  else if (topology_required)
    throw ConfigError("config not found: --topology is required for this command");
  if (s.cfg.has("topology")) s.topo = topology_from_config(s.cfg);
  if (s.topo.gpus.empty()) s.topo = default_topology(2);  // G:51-52
  if (a.b1) s.topo.b1 = *a.b1;
  if (a.b2) s.topo.b2 = *a.b2;
  // --workload: a config file with a [workload] section, else the topology file's section
  // when the default is kept, else a catalog name
  if (std::ifstream(a.workload).good())
    s.workload = workload_from_config(load_config(a.workload));
  else if (a.workload == "AT" && s.cfg.has("workload"))
    s.workload = workload_from_config(s.cfg);
  else
    s.workload = load_benchmark(a.workload);
  s.model = model_from_config(s.cfg);
  s.search = search_from_config(s.cfg);
  if (a.sat_threshold) s.search.config.sat_threshold = *a.sat_threshold;
  return s;
}

std::string num(double v, int precision = 6) {
  std::ostringstream o;
  o << std::setprecision(precision) << v;
  return o.str();
}

std::string mode_name(RunMode m) {
  return m == RunMode::Serving ? "serving" : m == RunMode::SyncTrain ? "sync_train" : "async_train";
}

RunMode mode_from(const std::string& m) {
  if (m == "serving") return RunMode::Serving;
  if (m == "sync_train") return RunMode::SyncTrain;
  if (m == "async_train") return RunMode::AsyncTrain;
  throw UsageError("--mode: expected serving, sync_train, or async_train");
}

// reports (the reference's report.hpp schema; nlohmann::json orders object keys)
json report(const ValidationReport& r) {
  json v = json::array();
  for (const auto& x : r.violations) v.push_back({{"gpu", x.gpu_id}, {"rule", x.rule}});
  return {{"ok", r.ok()}, {"violations", v}};
}
json report(const CostEstimate& c) { return {{"resource_size", c.resource_size}, {"comm_bytes", c.comm_bytes}}; }
json report(const MappingPlan& p) {
  json roles = json::object(), layout = json::object();
  for (const auto& [id, set] : p.gmi_assignments) {
    json names = json::array();
    for (Role r : set) names.push_back(to_string(r));
    roles[std::to_string(id)] = names;
  }
  for (const auto& [gpu, ids] : p.gpu_layout) layout[std::to_string(gpu)] = ids;
  json out = {{"template", to_string(p.template_kind)}, {"gmi_roles", roles}, {"gpu_layout", layout}};
  if (p.template_kind == TemplateKind::AsyncDecoupled) {
    out["serving_gpus"] = p.serving_gpus;
    out["training_gpus"] = p.training_gpus;
  }
  return out;
}
json report(const PipelineMetrics& m) {
  json per = json::object();
  for (const auto& [id, n] : m.trainer_records) per[std::to_string(id)] = n;
  return {{"pps", m.pps},
          {"ttop", m.ttop},
          {"records_produced", m.records_produced},
          {"records_delivered", m.records_delivered},
          {"units_sent", m.units_sent},
          {"batches_emitted", m.batches_emitted},
          {"bytes_moved", m.bytes_moved},
          {"transfer_busy_time", m.transfer_busy_time},
          {"delivery_makespan", m.delivery_makespan},
          {"training_makespan", m.training_makespan},
          {"trainer_records", per}};
}
json report(const SearchResult& r) {
  json out = {{"feasible", r.feasible}};
  if (r.feasible) {
    out["num_env"] = r.num_env;
    out["gmis_per_gpu"] = r.gmis_per_gpu;
    out["est_throughput"] = r.est_throughput;
  } else {
    out["reason"] = r.reason;
  }
  json log = json::array();
  for (const auto& v : r.visited) {
    json p = {{"gmis_per_gpu", v.gmis_per_gpu}, {"num_env", v.num_env}, {"runnable", v.runnable}};
    if (v.runnable) p.update({{"top", v.top}, {"mem", v.mem}});
    if (v.sat) p["sat"] = *v.sat;
    if (v.acc_top) p["acc_top"] = *v.acc_top;
    if (v.pruned_here) p["pruned"] = true;
    log.push_back(p);
  }
  out["visited"] = log;
  return out;
}

struct Output {
  json structured;
  std::ostringstream text;
  int code = 0;
};

// ------------------------------------------------------------------ commands
Output run_validate(const Args& a) {
  Output o;
  const Session s = open_session(a, true);
  const ValidationReport r = validate_layout(s.topo);
  if (r.ok()) {
    o.text << "layout ok: " << s.topo.gpus.size() << " GPU(s), " << s.topo.partitions.size() << " partition(s)\n";
  } else {
    o.text << "layout invalid: " << r.violations.size() << " violation(s)\n";
    for (const auto& v : r.violations)
      o.text << (v.gpu_id >= 0 ? "  gpu " + std::to_string(v.gpu_id) : std::string("  topology")) << ": " << v.rule
             << '\n';
  }
  o.structured = report(r);
  o.code = r.ok() ? 0 : 1;
  return o;
}

Output run_plan(const Args& a) {
  Output o;
  const Session s = open_session(a, false);
  const RunMode mode = mode_from(a.mode);
  const TemplateKind chosen = select_template(mode);
  const double r_all = double(s.topo.gpus.size());  // G:139-140
  const int n = int(s.topo.gpus.size()) * s.model.gmis_per_gpu;
  const DrlWorkload& w = s.workload;
  o.structured = {{"mode", mode_name(mode)}, {"workload", w.name}, {"selected_template", to_string(chosen)}};
  o.text << "mode: " << mode_name(mode) << "  workload: " << w.name << '\n';
  auto table = [&](const char* title, TemplateKind lo, TemplateKind hi, const CostEstimate& cl, const CostEstimate& ch,
                   double ratio) {
    o.structured["cost_table"] = {{to_string(lo), report(cl)}, {to_string(hi), report(ch)}};
    o.structured["ratio_over_dedicated"] = ratio;
    o.text << title << '\n';
    for (const auto& [k, c] : {std::pair{lo, cl}, std::pair{hi, ch}})
      o.text << "  " << to_string(k) << ": R=" << num(c.resource_size) << " COM=" << num(c.comm_bytes) << '\n';
  };
  if (mode == RunMode::Serving) {
    const CostEstimate tdg = serving_cost(TemplateKind::TDG, w), tcg = serving_cost(TemplateKind::TCG, w);
    const double bw = tdg.comm_bytes / (s.model.calibration.serving_combw_factor * w.interaction_time());
    if (!(tdg.comm_bytes > 0 && s.model.calibration.serving_combw_factor > 0 && w.interaction_time() > 0))
      throw std::invalid_argument("calibration inputs must be positive");
    const double t_dg = serving_throughput(tdg, w, r_all, bw), t_cg = serving_throughput(tcg, w, r_all, bw);
    const double ratio = serving_throughput_ratio(w, s.model.calibration);
    table("cost table (serving):", TemplateKind::TDG, TemplateKind::TCG, tdg, tcg, ratio);
    o.structured["throughput"] = {{"TDG", t_dg}, {"TCG", t_cg}, {"r_all", r_all}, {"calibrated_bw", bw}};
    o.structured["colocation_penalty"] = serving_colocation_penalty(w);
    o.text << "throughput (R_all=" << num(r_all) << ", calibrated): TDG=" << num(t_dg) << " TCG=" << num(t_cg) << '\n'
           << "TCG selected, est. ratio " << num(ratio, 3) << "x over TDG\n";
  } else if (mode == RunMode::SyncTrain) {
    const CostEstimate tdg = training_cost(TemplateKind::TDG_EX, w, n), tcg = training_cost(TemplateKind::TCG_EX, w, n);
    const double ratio = training_throughput_ratio(w, s.model.calibration);
    table(("cost table (sync training, n=" + std::to_string(n) + "):").c_str(), TemplateKind::TDG_EX,
          TemplateKind::TCG_EX, tdg, tcg, ratio);
    o.structured["n_gmis"] = n;
    o.structured["colocation_penalty"] = training_colocation_penalty(w);
    o.text << "TCG_EX selected, est. ratio " << num(ratio, 3) << "x over TDG_EX\n";
  } else {
    o.text << "async_train: decoupled serving/training split\n";
  }
  const MappingPlan plan = build_plan(chosen, s.topo, w, s.model.gmis_per_gpu);
  o.structured["plan"] = report(plan);
  if (mode == RunMode::AsyncTrain) {
    o.text << "  serving GPUs:";
    for (int g : plan.serving_gpus) o.text << ' ' << g;
    o.text << "\n  training GPUs:";
    for (int g : plan.training_gpus) o.text << ' ' << g;
    o.text << '\n';
  }
  for (const auto& [gpu, ids] : plan.gpu_layout) {
    o.text << "  gpu " << gpu << ":";
    for (int id : ids) o.text << ' ' << id;
    o.text << '\n';
  }
  return o;
}

std::vector<std::vector<int>> layout_from_text(const std::string& t) {
  // [[a, b], [c]] with optional whitespace / trailing commas
  std::vector<std::vector<int>> out;
  std::size_t i = 0;
  auto ws = [&] {
    while (i < t.size() && std::isspace(static_cast<unsigned char>(t[i]))) ++i;
  };
  auto need = [&](char c) {
    ws();
    if (i >= t.size() || t[i] != c) throw std::invalid_argument("bad layout: expected '" + std::string(1, c) + "' in " + t);
    ++i;
  };
  auto comma = [&] {
    ws();
    if (i < t.size() && t[i] == ',') {
      ++i;
      ws();
    }
  };
  need('[');
  ws();
  while (i < t.size() && t[i] != ']') {
    need('[');
    std::vector<int> gpu;
    ws();
    while (i < t.size() && t[i] != ']') {
      std::size_t used = 0;
      gpu.push_back(std::stoi(t.substr(i), &used));
      i += used;
      comma();
    }
    need(']');
    out.push_back(gpu);
    comma();
  }
  need(']');
  return out;
}

Output run_reduce(const Args& a) {
  Output o;
  const Session s = open_session(a, false);
  if (a.layout.empty()) throw UsageError("--layout: a layout such as [[0,1],[2,3]] is required");
  GmiLayout layout{layout_from_text(a.layout)};
  layout.validate();
  // payload bytes -> fp64 elements (G:209-212): the simulator counts 8 B per element
  const std::size_t len = std::size_t(std::max(1.0, std::round((a.payload > 0 ? a.payload : s.workload.model_bytes) / 8.0)));
  const double m_p = 8.0 * double(len);
  Strategy strategy = select_strategy(layout);
  const bool forced = !a.force_strategy.empty();
  if (forced) {
    static const std::map<std::string, Strategy> by_name = {
        {"mpr", Strategy::MPR}, {"mrr", Strategy::MRR}, {"har", Strategy::HAR}};
    const auto it = by_name.find(a.force_strategy);
    if (it == by_name.end()) throw UsageError("--force-strategy: expected mpr, mrr, or har");
    strategy = it->second;
  }
  // golden buffers 1 + 0.001 id + 1e-6 e (G:228) and their exact elementwise sum
  std::vector<GradientBuffer> bufs;
  std::vector<double> want(len, 0.0);
  for (int id : layout.all_gmis()) {
    GradientBuffer b{id, std::vector<double>(len)};
    for (std::size_t e = 0; e < len; ++e) want[e] += (b.values[e] = 1.0 + 0.001 * id + 1e-6 * double(e));
    bufs.push_back(std::move(b));
  }
  // schedule (Alg. 1 rings, trace, Table-3 latency) from libgmi; the data path either on the
  // B200 (--device: the drop-in execute(), K1 fold in the strategy's ring order) or, like the
  // reference simulator, on the host (ring-order fold is only observable below 1e-9)
  ReductionRun run;
  if (a.device) {
    run = execute(strategy, layout, bufs, s.topo);
  } else {
    const std::vector<int> counts = layout.counts(), ids = layout.all_gmis();
    gmi_reduction_info_t info{};
    detail::check(gmi_reduction_schedule(int(strategy), layout.num_gpus(), counts.data(), ids.data(), len, 8.0,
                                         s.topo.b1, s.topo.b2, nullptr, 0, &info));
    std::vector<gmi_trace_event_t> tr(std::max<std::size_t>(info.trace_len, 1));
    detail::check(gmi_reduction_schedule(int(strategy), layout.num_gpus(), counts.data(), ids.data(), len, 8.0,
                                         s.topo.b1, s.topo.b2, tr.data(), tr.size(), &info));
    run.strategy = strategy;
    run.latency = info.latency;
    run.broadcast_latency = info.broadcast_latency;
    for (std::size_t i = 0; i < info.trace_len; ++i)
      run.trace.push_back({tr[i].step, tr[i].src, tr[i].dst, tr[i].bytes, LinkKind(tr[i].kind)});
    run.result.assign(len, 0.0);
    for (const auto& b : bufs)
      for (std::size_t e = 0; e < len; ++e) run.result[e] += b.values[e];
  }
  double worst = 0;
  for (std::size_t e = 0; e < len; ++e)
    worst = std::max(worst, std::abs(run.result[e] - want[e]) / std::max(1.0, std::abs(want[e])));
  if (worst > 1e-9) throw std::runtime_error("reduction result diverged from elementwise sum");

  o.structured = {{"layout", layout.mpl}, {"payload_bytes", m_p}, {"strategy", to_string(strategy)}, {"forced", forced}};
  o.text << to_string(strategy) << " selected, latency " << num(run.latency);
  if (layout.uniform()) {
    const int g = layout.num_gpus(), t = int(layout.mpl.front().size());
    json pred;
    std::string others;
    for (Strategy x : {Strategy::MPR, Strategy::MRR, Strategy::HAR}) {
      const double p = predict_latency(x, g, t, m_p, s.topo.b1, s.topo.b2);
      pred[to_string(x)] = p;
      if (x != strategy) others += (others.empty() ? "" : ", ") + to_string(x) + ' ' + num(p);
    }
    const double own = pred[to_string(strategy)].get<double>();
    if (std::abs(run.latency - own) > 1e-12 * std::max(1.0, std::abs(own)))
      throw std::runtime_error("trace latency disagrees with the closed-form prediction");
    o.structured["predicted_latency"] = pred;
    o.structured["trace_matches_prediction"] = true;
    o.text << " (" << others << ")";
  }
  o.text << "\nresult: elementwise sum verified over " << len << " elements\n";
  if (a.device) o.structured["device"] = true;
  o.structured["result_verified"] = true;
  o.structured["broadcast_latency"] = run.broadcast_latency;
  json head = json::array();
  for (std::size_t i = 0; i < run.trace.size() && i < 12; ++i) {
    const TraceEvent& e = run.trace[i];
    head.push_back({{"step", e.step}, {"src", e.src}, {"dst", e.dst}, {"bytes", e.bytes}, {"link", to_string(e.kind)}});
  }
  o.structured["trace"] = {{"events_total", run.trace.size()}, {"head", head}};
  if (a.full_trace)
    for (const TraceEvent& e : run.trace)
      o.text << e.step << ' ' << e.src << ' ' << e.dst << ' ' << e.bytes << ' ' << to_string(e.kind) << '\n';
  return o;
}

Output run_pipeline(const Args& a) {
  Output o;
  const Session s = open_session(a, false);
  const MappingPlan plan = build_plan(TemplateKind::AsyncDecoupled, s.topo, s.workload, s.model.gmis_per_gpu);
  const PipelineMetrics multi = simulate_pipeline(s.workload, plan, s.topo, s.model.pipeline, a.duration);
  const PipelineMetrics uni = simulate_pipeline(s.workload, plan, s.topo, uni_channel(s.model.pipeline), a.duration);
  o.structured = {{"duration", a.duration},
                  {"compress_threshold", s.model.pipeline.compress_threshold},
                  {"plan", report(plan)},
                  {"multi_channel", report(multi)},
                  {"uni_channel", report(uni)}};
  o.text << "experience pipeline over " << a.duration << " time units (threshold "
         << s.model.pipeline.compress_threshold << "):\n"
         << "               multi-channel    uni-channel\n";
  auto row = [&](const char* label, const std::string& m, const std::string& u) {
    o.text << "  " << std::left << std::setw(13) << label << std::right << std::setw(13) << m << "    "
           << std::setw(11) << u << '\n';
  };
  row("PPS", num(multi.pps), num(uni.pps));
  row("TTOP", num(multi.ttop), num(uni.ttop));
  row("records", std::to_string(multi.records_produced), std::to_string(uni.records_produced));
  row("units sent", std::to_string(multi.units_sent), std::to_string(uni.units_sent));
  row("batches", std::to_string(multi.batches_emitted), std::to_string(uni.batches_emitted));
  return o;
}

Output run_search(const Args& a) {
  Output o;
  const Session s = open_session(a, false);
  std::unique_ptr<Profiler> prof;
  if (a.profiler == "gpu")
    prof = std::make_unique<GpuProfiler>();
  else if (s.search.profile_trace)
    prof = std::make_unique<RecordedTraceProfiler>(RecordedTraceProfiler::from_file(*s.search.profile_trace));
  else
    prof = std::make_unique<SyntheticCostModel>();
  const ThroughputEstimator est{s.workload, s.topo.b1, s.topo.b2, s.model.latency_scale};
  const SearchResult r = explore(*prof, est, s.workload.name, int(s.topo.gpus.size()), s.search.config);
  if (r.feasible)
    o.text << "best configuration: num_env=" << r.num_env << " gmis_per_gpu=" << r.gmis_per_gpu
           << " est_throughput=" << num(r.est_throughput) << '\n';
  else
    o.text << "infeasible: " << r.reason << '\n';
  o.text << "visited points (" << r.visited.size() << "):\n";
  for (const auto& v : r.visited) {
    o.text << "  gpg=" << v.gmis_per_gpu << " env=" << v.num_env;
    if (!v.runnable) {
      o.text << " not-runnable\n";
      continue;
    }
    o.text << " top=" << num(v.top) << " mem=" << num(v.mem);
    if (v.sat) o.text << " sat=" << num(*v.sat, 4);
    if (v.acc_top) o.text << " acc_top=" << num(*v.acc_top);
    o.text << (v.pruned_here ? " pruned\n" : "\n");
  }
  o.structured = report(r);
  o.code = r.feasible ? 0 : 1;
  return o;
}

}  // namespace

int main(int argc, char** argv) {
  static const std::map<std::string, std::function<Output(const Args&)>> commands = {
      {"validate", run_validate}, {"plan", run_plan}, {"reduce", run_reduce},
      {"pipeline", run_pipeline}, {"search", run_search}};
  Args args;
  try {
    args = parse_args(argc, argv);
  } catch (const UsageError& e) {
    std::cerr << e.what() << '\n';
    return 2;
  }
  // exit-code split of the reference (G:389-411): config / usage / invalid input -> 2,
  // domain errors (multi-stream, plan, pipeline, anything else) -> 1
  try {
    Output o = commands.at(args.command)(args);
    if (args.format == "structured")
      std::cout << o.structured.dump(2) << '\n';
    else
      std::cout << o.text.str();
    return o.code;
  } catch (const ConfigError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  } catch (const MultiStreamError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  } catch (const PlanError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  } catch (const PipelineError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
}
