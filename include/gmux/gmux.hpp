// gmux.hpp — C++ drop-in for the reference's `namespace gmux` (proj/include/gmux/*.hpp),
// backed by libgmi.so through the C-ABI in gmi.h. Same type names, signatures, argument
// meaning and exception classes; every algorithm runs inside libgmi (execute() on the
// B200 through the K1 reduction kernel). Link with -lgmi; no CUDA headers needed.
//
// Replaced reference interfaces (paths under proj/include/gmux/):
//   reduction.hpp  Strategy GmiLayout GradientBuffer TraceEvent ReductionRun MultiStreamError
//                  select_strategy leader_gmis mrr_rings predict_latency execute
//   topology.hpp   GpuArch Backend TaskMode GpuSpec GmiPartition Topology default_topology
//                  Violation ValidationReport validate_layout select_backend LinkKind path_bandwidth
//   workload.hpp   Role RoleProfile DrlWorkload validate_workload dense_param_count
//                  policy_value_param_count benchmark_names load_benchmark
//   mapping.hpp    TemplateKind RunMode CostEstimate serving_cost training_cost allreduce_bytes
//                  serving_throughput training_throughput CalibrationParams *_ratio *_penalty
//                  select_template MappingPlan PlanError build_plan
//   search.hpp     ProfileResult Profiler SearchConfig validate_config saturation ThroughputEstimator
//                  SyntheticCostModel RecordedTraceProfiler VisitedPoint SearchResult explore
//   channels.hpp   BatchMode PipelineConfig RecordId TrainingBatch PipelineMetrics PipelineError
//                  simulate_pipeline uni_channel
//   config.hpp     ConfigError ConfigFile parse_config load_config topology_from_config
//                  workload_from_config ModelParams model_from_config SearchSettings search_from_config
#pragma once

#include <cstring>
#include <exception>
#include <istream>
#include <iterator>
#include <limits>
#include <map>
#include <memory>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "gmi.h"

namespace gmux {

// ------------------------------------------------------------------ errors
struct MultiStreamError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct PlanError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct PipelineError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int rc) {
  if (rc == GMI_OK) return;
  const std::string msg = gmi_last_error();
  switch (rc) {
    case GMI_ERR_INVALID: throw std::invalid_argument(msg);
    case GMI_ERR_MULTISTREAM: throw MultiStreamError(msg);
    case GMI_ERR_PLAN: throw PlanError(msg);
    case GMI_ERR_PIPELINE: throw PipelineError(msg);
    case GMI_ERR_CONFIG: throw ConfigError(msg);
    default: throw std::runtime_error(msg);
  }
}
}  // namespace detail

// ------------------------------------------------------------------ topology.hpp
enum class GpuArch { SM70, SM80, SM100 };
enum class Backend { MPS, MIG };
enum class TaskMode { Training, Serving };
enum class LinkKind { Intra, HostBounce, Ring, LocalReduce };

inline std::string to_string(GpuArch a) { return a == GpuArch::SM70 ? "sm70" : a == GpuArch::SM80 ? "sm80" : "sm100"; }
inline std::string to_string(Backend b) { return b == Backend::MPS ? "mps" : "mig"; }
inline std::string to_string(LinkKind k) {
  switch (k) {
    case LinkKind::Intra: return "intra";
    case LinkKind::HostBounce: return "host_bounce";
    case LinkKind::Ring: return "ring";
    case LinkKind::LocalReduce: return "local_reduce";
  }
  return "?";
}

inline constexpr int kSmUnitsPerGpu = 8;

struct GpuSpec {
  int id = 0;
  GpuArch arch = GpuArch::SM80;
  int sm_units = kSmUnitsPerGpu;
  double mem_gb = 40.0;
};

struct GmiPartition {
  int gmi_id = 0;
  int gpu_id = 0;
  Backend backend = Backend::MPS;
  double sm_share = 1.0;
  double mem_gb = 0.0;
};

struct Topology {
  std::vector<GpuSpec> gpus;
  std::vector<GmiPartition> partitions;
  double b1 = 1.0;
  double b2 = 30.0;
};

struct MigProfile {
  std::string_view name;
  int units;
  double mem_gb;
};

inline constexpr int kUsableMigUnits = 7;

inline const std::vector<MigProfile>& mig_profiles() {
  static const std::vector<MigProfile> p = {
      {"1g.5gb", 1, 5.0}, {"2g.10gb", 2, 10.0}, {"3g.20gb", 3, 20.0}, {"4g.20gb", 4, 20.0}, {"7g.40gb", 7, 40.0}};
  return p;
}

// B200 extension: NVIDIA's published 180 GB B200 profiles (compute slices of 7, label memory).
inline const std::vector<MigProfile>& mig_profiles_sm100() {
  static const std::vector<MigProfile> p = {{"1g.23gb", 1, 23.0}, {"1g.45gb", 1, 45.0}, {"2g.45gb", 2, 45.0},
                                            {"3g.90gb", 3, 90.0}, {"4g.90gb", 4, 90.0}, {"7g.180gb", 7, 180.0}};
  return p;
}

inline const MigProfile* find_mig_profile(std::string_view name) {
  for (const auto* tab : {&mig_profiles(), &mig_profiles_sm100()})
    for (const auto& p : *tab)
      if (p.name == name) return &p;
  return nullptr;
}

inline GmiPartition mig_partition(int gmi_id, int gpu_id, std::string_view profile) {
  const MigProfile* p = find_mig_profile(profile);
  if (!p) throw std::invalid_argument("unknown MIG profile: " + std::string(profile));
  return {gmi_id, gpu_id, Backend::MIG, double(p->units) / kSmUnitsPerGpu, p->mem_gb};
}

inline GmiPartition mps_partition(int gmi_id, int gpu_id, double sm_share, double mem_gb) {
  return {gmi_id, gpu_id, Backend::MPS, sm_share, mem_gb};
}

inline Topology default_topology(int num_gpus = 2) {
  Topology t;
  for (int i = 0; i < num_gpus; ++i) t.gpus.push_back({i});
  return t;
}

struct Violation {
  int gpu_id;
  std::string rule;
};
struct ValidationReport {
  std::vector<Violation> violations;
  bool ok() const { return violations.empty(); }
};

namespace detail {
struct CTopology {
  std::vector<gmi_gpu_t> g;
  std::vector<gmi_partition_t> p;
  gmi_topology_t t{};
  explicit CTopology(const Topology& topo) {
    for (const auto& x : topo.gpus)
      g.push_back({x.id, x.arch == GpuArch::SM70 ? 70 : x.arch == GpuArch::SM80 ? 80 : 100, x.sm_units, x.mem_gb});
    for (const auto& x : topo.partitions)
      p.push_back({x.gmi_id, x.gpu_id, x.backend == Backend::MIG ? 1 : 0, x.sm_share, x.mem_gb});
    t = {g.data(), int(g.size()), p.data(), int(p.size()), topo.b1, topo.b2};
  }
};
}  // namespace detail

inline ValidationReport validate_layout(const Topology& topo) {
  detail::CTopology c(topo);
  int n = 0;
  detail::check(gmi_validate_layout(&c.t, nullptr, 0, &n));
  std::vector<gmi_violation_t> v(std::max(n, 1));
  detail::check(gmi_validate_layout(&c.t, v.data(), n, &n));
  ValidationReport r;
  for (int i = 0; i < n; ++i) r.violations.push_back({v[i].gpu_id, v[i].rule});
  return r;
}

inline Backend select_backend(GpuArch arch, TaskMode mode) {
  int b = 0;
  detail::check(gmi_select_backend(arch == GpuArch::SM70 ? 70 : arch == GpuArch::SM80 ? 80 : 100,
                                   mode == TaskMode::Training, &b));
  return b == 1 ? Backend::MIG : Backend::MPS;
}

struct LinkPath {
  LinkKind kind;
  double bandwidth;
};

inline LinkPath path_bandwidth(const Topology& topo, int src_gmi, int dst_gmi) {
  detail::CTopology c(topo);
  int kind = 0;
  double bw = 0;
  detail::check(gmi_path_bandwidth(&c.t, src_gmi, dst_gmi, &kind, &bw));
  return {LinkKind(kind), bw};
}

// ------------------------------------------------------------------ reduction.hpp
enum class Strategy { MPR, MRR, HAR };

inline std::string to_string(Strategy s) {
  switch (s) {
    case Strategy::MPR: return "MPR";
    case Strategy::MRR: return "MRR";
    case Strategy::HAR: return "HAR";
  }
  return "?";
}

struct GmiLayout {
  std::vector<std::vector<int>> mpl;

  int num_gpus() const { return int(mpl.size()); }
  std::size_t total_gmis() const {
    std::size_t n = 0;
    for (const auto& l : mpl) n += l.size();
    return n;
  }
  bool uniform() const {
    for (const auto& l : mpl)
      if (l.size() != mpl.front().size()) return false;
    return true;
  }
  std::vector<int> all_gmis() const {
    std::vector<int> out;
    for (const auto& l : mpl) out.insert(out.end(), l.begin(), l.end());
    return out;
  }
  std::vector<int> counts() const {
    std::vector<int> c;
    for (const auto& l : mpl) c.push_back(int(l.size()));
    return c;
  }
  void validate() const {
    int s = 0;
    const auto c = counts();
    const auto ids = all_gmis();
    detail::check(gmi_select_strategy(num_gpus(), c.data(), ids.data(), &s));
  }
};

struct GradientBuffer {
  int gmi_id = 0;
  std::vector<double> values;
};

struct TraceEvent {
  int step = 0;
  int src = 0;
  int dst = 0;
  double bytes = 0;
  LinkKind kind = LinkKind::HostBounce;
};

struct ReductionRun {
  Strategy strategy = Strategy::MPR;
  std::vector<double> result;
  double latency = 0;
  double broadcast_latency = 0;
  std::vector<TraceEvent> trace;
};

inline Strategy select_strategy(const GmiLayout& layout) {
  int s = 0;
  const auto c = layout.counts();
  const auto ids = layout.all_gmis();
  detail::check(gmi_select_strategy(layout.num_gpus(), c.data(), ids.data(), &s));
  return Strategy(s);
}

inline std::vector<int> leader_gmis(const GmiLayout& layout) {
  std::vector<int> out(layout.mpl.size());
  const auto c = layout.counts();
  const auto ids = layout.all_gmis();
  detail::check(gmi_leader_gmis(layout.num_gpus(), c.data(), ids.data(), out.data()));
  return out;
}

inline std::vector<std::vector<int>> mrr_rings(const GmiLayout& layout) {
  const auto c = layout.counts();
  const auto ids = layout.all_gmis();
  std::vector<int> flat(std::max<std::size_t>(ids.size(), 1));
  int t = 0;
  detail::check(gmi_mrr_rings(layout.num_gpus(), c.data(), ids.data(), flat.data(), &t));
  const int g = layout.num_gpus();
  std::vector<std::vector<int>> rings(t);
  for (int r = 0; r < t; ++r) rings[r].assign(flat.begin() + r * g, flat.begin() + (r + 1) * g);
  return rings;
}

inline double predict_latency(Strategy s, int g, int t, double m_p, double b1, double b2) {
  double out = 0;
  detail::check(gmi_predict_latency(int(s), g, t, m_p, b1, b2, &out));
  return out;
}

// Device-backed: the elementwise sum runs on the B200 (K1) in the reference's fold order.
inline ReductionRun execute(Strategy strategy, const GmiLayout& layout, const std::vector<GradientBuffer>& buffers,
                            const Topology& topo) {
  layout.validate();
  const std::vector<int> members = layout.all_gmis();
  if (buffers.size() != members.size()) throw std::invalid_argument("need exactly one buffer per GMI in the layout");
  const std::size_t len = buffers.empty() ? 0 : buffers.front().values.size();
  std::map<int, const GradientBuffer*> by_id;
  for (const auto& b : buffers) {
    if (b.values.size() != len) throw std::invalid_argument("mismatched buffer lengths");
    if (!by_id.emplace(b.gmi_id, &b).second)
      throw std::invalid_argument("duplicate buffer for gmi " + std::to_string(b.gmi_id));
  }
  for (int id : members)
    if (!by_id.count(id)) throw std::invalid_argument("missing buffer for gmi " + std::to_string(id));
  const auto c = layout.counts();
  gmi_reduction_info_t info{};
  detail::check(gmi_reduction_schedule(int(strategy), layout.num_gpus(), c.data(), members.data(), len, 8.0,
                                       topo.b1, topo.b2, nullptr, 0, &info));
  std::vector<gmi_trace_event_t> tr(std::max<std::size_t>(info.trace_len, 1));
  detail::check(gmi_reduction_schedule(int(strategy), layout.num_gpus(), c.data(), members.data(), len, 8.0,
                                       topo.b1, topo.b2, tr.data(), tr.size(), &info));
  ReductionRun run;
  run.strategy = strategy;
  run.latency = info.latency;
  run.broadcast_latency = info.broadcast_latency;
  for (std::size_t i = 0; i < info.trace_len; ++i)
    run.trace.push_back({tr[i].step, tr[i].src, tr[i].dst, tr[i].bytes, LinkKind(tr[i].kind)});
  run.result.resize(len);
  if (len > 0) {
    std::vector<const void*> ptrs;
    for (int id : members) ptrs.push_back(by_id[id]->values.data());
    detail::check(gmi_execute_host(int(strategy), layout.num_gpus(), c.data(), members.data(), ptrs.data(), len,
                                   GMI_F64, run.result.data()));
  }
  return run;
}

// ------------------------------------------------------------------ workload.hpp
enum class Role { Simulator, Agent, Trainer };
enum class ResourceKind { SM, Memory };

inline std::string to_string(Role r) {
  return r == Role::Simulator ? "simulator" : r == Role::Agent ? "agent" : "trainer";
}

struct RoleProfile {
  Role role = Role::Simulator;
  double r_sm = 1.0;
  double r_mem = 0.5;
  double t_iter = 1.0;
};

struct DrlWorkload {
  std::string name;
  double state_bytes = 0;
  double action_bytes = 0;
  double reward_bytes = 0;
  double model_bytes = 0;
  int steps_per_train = 1;
  double alpha = 0.2;
  double beta = 0.3;
  std::vector<int> policy_dims;
  RoleProfile simulator{Role::Simulator, 1.0, 0.5, 6.0};
  RoleProfile agent{Role::Agent, 0.1, 0.05, 1.0};
  RoleProfile trainer{Role::Trainer, 0.2, 0.1, 2.0};

  const RoleProfile& profile(Role r) const {
    return r == Role::Simulator ? simulator : r == Role::Agent ? agent : trainer;
  }
  double record_bytes() const { return state_bytes + action_bytes + reward_bytes; }
  double interaction_time() const { return simulator.t_iter + agent.t_iter; }
  double iteration_time() const { return interaction_time() + trainer.t_iter; }
};

namespace detail {
inline gmi_workload_t to_c(const DrlWorkload& w) {
  gmi_workload_t c{};
  std::strncpy(c.name, w.name.c_str(), sizeof(c.name) - 1);
  c.state_bytes = w.state_bytes;
  c.action_bytes = w.action_bytes;
  c.reward_bytes = w.reward_bytes;
  c.model_bytes = w.model_bytes;
  c.steps_per_train = w.steps_per_train;
  c.alpha = w.alpha;
  c.beta = w.beta;
  if (w.policy_dims.size() > GMI_MAX_DIMS) throw std::invalid_argument("too many policy dims");
  c.num_dims = int(w.policy_dims.size());
  for (std::size_t i = 0; i < w.policy_dims.size(); ++i) c.policy_dims[i] = w.policy_dims[i];
  c.simulator = {w.simulator.r_sm, w.simulator.r_mem, w.simulator.t_iter};
  c.agent = {w.agent.r_sm, w.agent.r_mem, w.agent.t_iter};
  c.trainer = {w.trainer.r_sm, w.trainer.r_mem, w.trainer.t_iter};
  return c;
}
inline DrlWorkload from_c(const gmi_workload_t& c) {
  DrlWorkload w;
  w.name = c.name;
  w.state_bytes = c.state_bytes;
  w.action_bytes = c.action_bytes;
  w.reward_bytes = c.reward_bytes;
  w.model_bytes = c.model_bytes;
  w.steps_per_train = c.steps_per_train;
  w.alpha = c.alpha;
  w.beta = c.beta;
  w.policy_dims.assign(c.policy_dims, c.policy_dims + c.num_dims);
  w.simulator = {Role::Simulator, c.simulator.r_sm, c.simulator.r_mem, c.simulator.t_iter};
  w.agent = {Role::Agent, c.agent.r_sm, c.agent.r_mem, c.agent.t_iter};
  w.trainer = {Role::Trainer, c.trainer.r_sm, c.trainer.r_mem, c.trainer.t_iter};
  return w;
}
}  // namespace detail

inline void validate_workload(const DrlWorkload& w) {
  const auto c = detail::to_c(w);
  detail::check(gmi_validate_workload(&c));
}

inline ResourceKind dominant_resource(double r_sm, double r_mem) {
  if (!(r_sm > 0 && r_sm <= 1) || !(r_mem > 0 && r_mem <= 1))
    throw std::invalid_argument("resource fractions must lie in (0,1]");
  return r_sm >= r_mem ? ResourceKind::SM : ResourceKind::Memory;
}

inline std::size_t dense_param_count(const std::vector<int>& dims) {
  std::size_t n = 0;
  detail::check(gmi_dense_param_count(dims.data(), int(dims.size()), &n));
  return n;
}

inline std::size_t policy_value_param_count(const std::vector<int>& dims) {
  std::size_t n = 0;
  detail::check(gmi_policy_value_param_count(dims.data(), int(dims.size()), &n));
  return n;
}

inline const std::vector<std::string>& benchmark_names() {
  static const std::vector<std::string> names = {"AT", "AY", "BB", "FC", "HM", "SH"};
  return names;
}

inline DrlWorkload load_benchmark(std::string_view name) {
  gmi_workload_t c{};
  detail::check(gmi_load_benchmark(std::string(name).c_str(), &c));
  return detail::from_c(c);
}

// ------------------------------------------------------------------ mapping.hpp
enum class TemplateKind { TDG, TCG, TDG_EX, TCG_EX, AsyncDecoupled };
enum class RunMode { Serving, SyncTrain, AsyncTrain };

inline std::string to_string(TemplateKind t) {
  switch (t) {
    case TemplateKind::TDG: return "TDG";
    case TemplateKind::TCG: return "TCG";
    case TemplateKind::TDG_EX: return "TDG_EX";
    case TemplateKind::TCG_EX: return "TCG_EX";
    case TemplateKind::AsyncDecoupled: return "async_decoupled";
  }
  return "?";
}

struct CostEstimate {
  double resource_size = 0;
  double comm_bytes = 0;
  double throughput = 0;
};

inline CostEstimate serving_cost(TemplateKind tpl, const DrlWorkload& w) {
  const auto c = detail::to_c(w);
  CostEstimate e;
  detail::check(gmi_serving_cost(int(tpl), &c, &e.resource_size, &e.comm_bytes));
  return e;
}

inline CostEstimate training_cost(TemplateKind tpl, const DrlWorkload& w, int n_gmis) {
  const auto c = detail::to_c(w);
  CostEstimate e;
  detail::check(gmi_training_cost(int(tpl), &c, n_gmis, &e.resource_size, &e.comm_bytes));
  return e;
}

inline double allreduce_bytes(int n_gmis, double model_bytes) {
  double out = 0;
  detail::check(gmi_allreduce_bytes(n_gmis, model_bytes, &out));
  return out;
}

inline double serving_throughput(const CostEstimate& cost, const DrlWorkload& w, double r_all, double bandwidth) {
  const auto c = detail::to_c(w);
  double out = 0;
  detail::check(gmi_throughput(0, cost.resource_size, cost.comm_bytes, &c, r_all, bandwidth, &out));
  return out;
}

inline double training_throughput(const CostEstimate& cost, const DrlWorkload& w, double r_all, double bandwidth) {
  const auto c = detail::to_c(w);
  double out = 0;
  detail::check(gmi_throughput(1, cost.resource_size, cost.comm_bytes, &c, r_all, bandwidth, &out));
  return out;
}

struct CalibrationParams {
  double serving_combw_factor = 2.0;
  double training_combw_factor = 7.0;
};

inline double serving_throughput_ratio(const DrlWorkload& w, const CalibrationParams& cal = {}) {
  const auto c = detail::to_c(w);
  double out = 0;
  detail::check(gmi_throughput_ratio(0, &c, cal.serving_combw_factor, &out));
  return out;
}

inline double training_throughput_ratio(const DrlWorkload& w, const CalibrationParams& cal = {}) {
  const auto c = detail::to_c(w);
  double out = 0;
  detail::check(gmi_throughput_ratio(1, &c, cal.training_combw_factor, &out));
  return out;
}

inline double serving_colocation_penalty(const DrlWorkload& w) {
  const auto c = detail::to_c(w);
  double out = 0;
  detail::check(gmi_colocation_penalty(0, &c, &out));
  return out;
}

inline double training_colocation_penalty(const DrlWorkload& w) {
  const auto c = detail::to_c(w);
  double out = 0;
  detail::check(gmi_colocation_penalty(1, &c, &out));
  return out;
}

inline TemplateKind select_template(RunMode mode) {
  return mode == RunMode::Serving ? TemplateKind::TCG
         : mode == RunMode::SyncTrain ? TemplateKind::TCG_EX
                                      : TemplateKind::AsyncDecoupled;
}

struct MappingPlan {
  TemplateKind template_kind = TemplateKind::TCG;
  std::map<int, std::set<Role>> gmi_assignments;
  std::map<int, std::vector<int>> gpu_layout;
  std::vector<int> serving_gpus;
  std::vector<int> training_gpus;

  std::vector<std::vector<int>> mpl() const {
    std::vector<std::vector<int>> out;
    for (const auto& [gpu, gmis] : gpu_layout) out.push_back(gmis);
    return out;
  }
  std::vector<int> gmis_with_role(Role r) const {
    std::vector<int> out;
    for (const auto& [gmi, roles] : gmi_assignments)
      if (roles.count(r)) out.push_back(gmi);
    return out;
  }
};

namespace detail {
inline std::set<Role> roles_of(int mask) {
  std::set<Role> s;
  if (mask & GMI_ROLE_SIM) s.insert(Role::Simulator);
  if (mask & GMI_ROLE_AGENT) s.insert(Role::Agent);
  if (mask & GMI_ROLE_TRAINER) s.insert(Role::Trainer);
  return s;
}
inline int mask_of(const std::set<Role>& s) {
  int m = 0;
  for (Role r : s) m |= r == Role::Simulator ? GMI_ROLE_SIM : r == Role::Agent ? GMI_ROLE_AGENT : GMI_ROLE_TRAINER;
  return m;
}
}  // namespace detail

inline MappingPlan build_plan(TemplateKind tpl, const Topology& topo, const DrlWorkload& w, int gmis_per_gpu) {
  (void)w;
  detail::CTopology c(topo);
  const std::size_t ng = std::max<std::size_t>(topo.gpus.size(), 1);
  const std::size_t total = std::max<std::size_t>(topo.gpus.size() * std::size_t(std::max(gmis_per_gpu, 0)), 1);
  std::vector<int> gpu_ids(ng), gmi_ids(total), roles(total), serving(ng);
  detail::check(gmi_build_plan(int(tpl), &c.t, gmis_per_gpu, gpu_ids.data(), gmi_ids.data(), roles.data(),
                               serving.data()));
  MappingPlan plan;
  plan.template_kind = tpl;
  for (std::size_t g = 0; g < topo.gpus.size(); ++g) {
    auto& ids = plan.gpu_layout[gpu_ids[g]];
    for (int j = 0; j < gmis_per_gpu; ++j) {
      const int id = gmi_ids[g * gmis_per_gpu + j];
      ids.push_back(id);
      plan.gmi_assignments[id] = detail::roles_of(roles[id]);
    }
    if (serving[g] == 1) plan.serving_gpus.push_back(gpu_ids[g]);
    if (serving[g] == 0) plan.training_gpus.push_back(gpu_ids[g]);
  }
  return plan;
}

// ------------------------------------------------------------------ search.hpp
struct ProfileResult {
  bool runnable = false;
  double top = 0;
  double mem = 0;
};

class Profiler {
 public:
  virtual ~Profiler() = default;
  virtual ProfileResult profile(const std::string& bench, int gmis_per_gpu, int num_env) const = 0;
};

struct SearchConfig {
  std::vector<int> num_env_grid = {128, 256, 512, 1024, 2048, 4096, 8192, 16384};
  int max_gmis_per_gpu = 10;
  double sat_threshold = 0.1;
};

inline void validate_config(const SearchConfig& c) {
  if (c.num_env_grid.empty()) throw std::invalid_argument("num_env grid must not be empty");
  if (c.max_gmis_per_gpu < 1) throw std::invalid_argument("max_gmis_per_gpu must be >= 1");
  if (!(c.sat_threshold > 0 && c.sat_threshold < 1)) throw std::invalid_argument("sat_threshold must lie in (0,1)");
}

inline double saturation(double top, double pre_top, double mem, double pre_mem) {
  double out = 0;
  detail::check(gmi_saturation(top, pre_top, mem, pre_mem, &out));
  return out;
}

struct ThroughputEstimator {
  DrlWorkload workload;
  double b1 = 1.0;
  double b2 = 30.0;
  double latency_scale = 1000.0;

  gmi_estimator_t c() const { return {detail::to_c(workload), b1, b2, latency_scale}; }
  double comm_discount(int gmis_per_gpu, int num_gpu) const {
    const auto e = c();
    double out = 0;
    detail::check(gmi_comm_discount(&e, gmis_per_gpu, num_gpu, &out));
    return out;
  }
  double estimate(int gmis_per_gpu, int num_gpu, double per_gmi_top) const {
    const auto e = c();
    double out = 0;
    detail::check(gmi_estimate(&e, gmis_per_gpu, num_gpu, per_gmi_top, &out));
    return out;
  }
};

struct SyntheticCostModel final : Profiler {
  double peak_top = 120000.0;
  double mem_base = 1.0;
  double mem_per_env = 0.002;
  double mem_capacity = 40.0;
  double min_runnable_share = 0.1;
  int knee_base = 8192;
  std::map<int, int> knee_override;
  std::map<int, double> cap_scale;

  ProfileResult profile(const std::string& bench, int gmis_per_gpu, int num_env) const override {
    std::vector<int> kk, kv, ck;
    std::vector<double> cv;
    for (const auto& [k, v] : knee_override) kk.push_back(k), kv.push_back(v);
    for (const auto& [k, v] : cap_scale) ck.push_back(k), cv.push_back(v);
    const gmi_synthetic_model_t m{peak_top, mem_base, mem_per_env, mem_capacity, min_runnable_share, knee_base,
                                  int(kk.size()), kk.data(), kv.data(), int(ck.size()), ck.data(), cv.data()};
    int ok = 0;
    ProfileResult r;
    detail::check(gmi_synthetic_profile(&m, bench.c_str(), gmis_per_gpu, num_env, &ok, &r.top, &r.mem));
    r.runnable = ok != 0;
    return r;
  }
};

class RecordedTraceProfiler final : public Profiler {
 public:
  static RecordedTraceProfiler from_file(const std::string& path) {
    void* h = nullptr;
    detail::check(gmi_trace_profiler_load(path.c_str(), &h));
    return RecordedTraceProfiler(h);
  }
  ProfileResult profile(const std::string& bench, int gmis_per_gpu, int num_env) const override {
    int ok = 0;
    ProfileResult r;
    detail::check(gmi_trace_profiler_profile(h_.get(), bench.c_str(), gmis_per_gpu, num_env, &ok, &r.top, &r.mem));
    r.runnable = ok != 0;
    return r;
  }

 private:
  explicit RecordedTraceProfiler(void* h) : h_(h, gmi_trace_profiler_free) {}
  std::shared_ptr<void> h_;
};

/// B200 extension: the on-device Profiler the reference's explore() was written for
/// (search.hpp:32-37) -- runs the real PPO iteration with gmis_per_gpu GMIs (green contexts
/// by default) of num_env envs each and reports per-GMI env-steps/s and device GB.
class GpuProfiler final : public Profiler {
 public:
  explicit GpuProfiler(int device = 0, int backend = 1, int iters = 3)
      : device_(device), backend_(backend), iters_(iters) {}
  ProfileResult profile(const std::string& bench, int gmis_per_gpu, int num_env) const override {
    int ok = 0;
    ProfileResult r;
    detail::check(gmi_gpu_profile(bench.c_str(), gmis_per_gpu, num_env, device_, backend_, iters_, &ok, &r.top,
                                  &r.mem));
    r.runnable = ok != 0;
    return r;
  }

 private:
  int device_, backend_, iters_;
};

struct VisitedPoint {
  int gmis_per_gpu = 0;
  int num_env = 0;
  bool runnable = false;
  double top = 0;
  double mem = 0;
  std::optional<double> sat;
  std::optional<double> acc_top;
  bool pruned_here = false;
};

struct SearchResult {
  bool feasible = false;
  std::string reason;
  int num_env = 0;
  int gmis_per_gpu = 0;
  double est_throughput = 0;
  std::vector<VisitedPoint> visited;
};

inline SearchResult explore(const Profiler& profiler, const ThroughputEstimator& estimator, const std::string& bench,
                            int num_gpu, const SearchConfig& config) {
  struct Ctx {
    const Profiler* p;
    std::exception_ptr err;
  } ctx{&profiler, nullptr};
  auto probe = [](void* user, const char* b, int gpg, int env, int* ok, double* top, double* mem) -> int {
    auto* c = static_cast<Ctx*>(user);
    try {
      const ProfileResult r = c->p->profile(b, gpg, env);
      *ok = r.runnable;
      *top = r.top;
      *mem = r.mem;
      return GMI_OK;
    } catch (...) {
      c->err = std::current_exception();
      return GMI_ERR_DOMAIN;
    }
  };
  const auto est = estimator.c();
  const gmi_search_config_t cfg{config.num_env_grid.data(), int(config.num_env_grid.size()), config.max_gmis_per_gpu,
                                config.sat_threshold};
  const std::size_t cap = std::max<std::size_t>(1, config.num_env_grid.size() * std::size_t(std::max(config.max_gmis_per_gpu, 0)));
  std::vector<gmi_visit_t> v(cap);
  gmi_search_result_t r{};
  const int rc = gmi_explore(probe, &ctx, &est, bench.c_str(), num_gpu, &cfg, &r, v.data(), cap);
  if (ctx.err) std::rethrow_exception(ctx.err);
  detail::check(rc);
  SearchResult out;
  out.feasible = r.feasible != 0;
  out.reason = r.reason;
  out.num_env = r.num_env;
  out.gmis_per_gpu = r.gmis_per_gpu;
  out.est_throughput = r.est_throughput;
  for (std::size_t i = 0; i < r.num_visited; ++i)
    out.visited.push_back({v[i].gmis_per_gpu, v[i].num_env, v[i].runnable != 0, v[i].top, v[i].mem,
                           v[i].has_sat ? std::optional<double>(v[i].sat) : std::nullopt,
                           v[i].has_acc_top ? std::optional<double>(v[i].acc_top) : std::nullopt,
                           v[i].pruned_here != 0});
  return out;
}

// ------------------------------------------------------------------ channels.hpp
enum class BatchMode { Slice, Stack };

struct PipelineConfig {
  int compress_threshold = 8;
  BatchMode batch_mode = BatchMode::Stack;
  int target_batch = 32;
  double per_message_overhead = 1.0;
  unsigned seed = 0;
};

inline PipelineConfig uni_channel(PipelineConfig config) {
  config.compress_threshold = 1;
  return config;
}

struct RecordId {
  int agent_gmi = 0;
  long seq = 0;
  bool operator==(const RecordId&) const = default;
  auto operator<=>(const RecordId&) const = default;
};

struct TrainingBatch {
  int trainer_gmi = 0;
  double emit_time = 0;
  std::vector<RecordId> records;
};

struct PipelineMetrics {
  double pps = 0;
  double ttop = 0;
  long records_produced = 0;
  long records_delivered = 0;
  long units_sent = 0;
  long batches_emitted = 0;
  double bytes_moved = 0;
  double transfer_busy_time = 0;
  double delivery_makespan = 0;
  double training_makespan = 0;
  std::map<int, long> trainer_records;
  std::vector<TrainingBatch> batches;
};

inline PipelineMetrics simulate_pipeline(const DrlWorkload& w, const MappingPlan& plan, const Topology& topo,
                                         const PipelineConfig& config, double duration) {
  const auto wc = detail::to_c(w);
  detail::CTopology tc(topo);
  std::vector<int> gpu_ids, counts, ids, masks;
  for (const auto& [gpu, g] : plan.gpu_layout) {
    gpu_ids.push_back(gpu);
    counts.push_back(int(g.size()));
    for (int id : g) {
      ids.push_back(id);
      auto it = plan.gmi_assignments.find(id);
      masks.push_back(it == plan.gmi_assignments.end() ? 0 : detail::mask_of(it->second));
    }
  }
  const gmi_plan_t pc{int(plan.template_kind), int(gpu_ids.size()), gpu_ids.data(), counts.data(), ids.data(),
                      masks.data()};
  const gmi_pipeline_config_t cc{config.compress_threshold, config.batch_mode == BatchMode::Slice ? 0 : 1,
                                 config.target_batch, config.per_message_overhead, config.seed};
  void* h = nullptr;
  gmi_pipeline_metrics_t m{};
  detail::check(gmi_simulate_pipeline(&wc, &pc, &tc.t, &cc, duration, &h, &m));
  std::unique_ptr<void, void (*)(void*)> guard(h, gmi_pipeline_free);
  PipelineMetrics out;
  out.pps = m.pps;
  out.ttop = m.ttop;
  out.records_produced = m.records_produced;
  out.records_delivered = m.records_delivered;
  out.units_sent = m.units_sent;
  out.batches_emitted = m.batches_emitted;
  out.bytes_moved = m.bytes_moved;
  out.transfer_busy_time = m.transfer_busy_time;
  out.delivery_makespan = m.delivery_makespan;
  out.training_makespan = m.training_makespan;
  std::vector<int> tr(std::max<std::size_t>(m.num_trainers, 1));
  std::vector<long> rec(tr.size());
  detail::check(gmi_pipeline_trainer_records(h, tr.data(), rec.data()));
  for (std::size_t i = 0; i < m.num_trainers; ++i) out.trainer_records[tr[i]] = rec[i];
  const std::size_t nb = gmi_pipeline_num_batches(h);
  for (std::size_t i = 0; i < nb; ++i) {
    TrainingBatch b;
    std::size_t n = 0;
    detail::check(gmi_pipeline_batch(h, i, &b.trainer_gmi, &b.emit_time, &n));
    std::vector<int> ag(std::max<std::size_t>(n, 1));
    std::vector<long> sq(ag.size());
    detail::check(gmi_pipeline_batch_records(h, i, ag.data(), sq.data()));
    for (std::size_t j = 0; j < n; ++j) b.records.push_back({ag[j], sq[j]});
    out.batches.push_back(std::move(b));
  }
  return out;
}

// ------------------------------------------------------------------ config.hpp
struct ModelParams {
  CalibrationParams calibration;
  int gmis_per_gpu = 2;
  double latency_scale = 1000.0;
  PipelineConfig pipeline;
};

struct SearchSettings {
  SearchConfig config;
  std::optional<std::string> profile_trace;
};

class ConfigFile {
 public:
  ConfigFile() {
    void* h = nullptr;
    detail::check(gmi_config_parse("", "<config>", &h));
    h_.reset(h, gmi_config_free);
  }
  explicit ConfigFile(void* h) : h_(h, gmi_config_free) {}
  bool has(const std::string& section) const {
    int out = 0;
    detail::check(gmi_config_has(h_.get(), section.c_str(), &out));
    return out != 0;
  }
  std::optional<std::string> get(const std::string& section, const std::string& key) const {
    std::vector<char> buf(4096);
    int found = 0;
    detail::check(gmi_config_get(h_.get(), section.c_str(), key.c_str(), buf.data(), buf.size(), &found));
    return found ? std::optional<std::string>(buf.data()) : std::nullopt;
  }
  void* handle() const { return h_.get(); }

 private:
  std::shared_ptr<void> h_;
};

inline ConfigFile parse_config(std::istream& in, const std::string& origin = "<config>") {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  void* h = nullptr;
  detail::check(gmi_config_parse(text.c_str(), origin.c_str(), &h));
  return ConfigFile(h);
}

inline ConfigFile load_config(const std::string& path) {
  void* h = nullptr;
  detail::check(gmi_config_load(path.c_str(), &h));
  return ConfigFile(h);
}

inline Topology topology_from_config(const ConfigFile& cfg) {
  int ng = 0, np = 0;
  double b1 = 0, b2 = 0;
  detail::check(gmi_config_topology(cfg.handle(), nullptr, 0, &ng, nullptr, 0, &np, &b1, &b2));
  std::vector<gmi_gpu_t> g(std::max(ng, 1));
  std::vector<gmi_partition_t> p(std::max(np, 1));
  detail::check(gmi_config_topology(cfg.handle(), g.data(), ng, &ng, p.data(), np, &np, &b1, &b2));
  Topology t;
  t.b1 = b1;
  t.b2 = b2;
  for (int i = 0; i < ng; ++i)
    t.gpus.push_back({g[i].id, g[i].arch == 70 ? GpuArch::SM70 : g[i].arch == 80 ? GpuArch::SM80 : GpuArch::SM100,
                      g[i].sm_units, g[i].mem_gb});
  for (int i = 0; i < np; ++i)
    t.partitions.push_back({p[i].gmi_id, p[i].gpu_id, p[i].backend == 1 ? Backend::MIG : Backend::MPS, p[i].sm_share,
                            p[i].mem_gb});
  return t;
}

inline DrlWorkload workload_from_config(const ConfigFile& cfg, const std::string& fallback = "AT") {
  gmi_workload_t c{};
  detail::check(gmi_config_workload(cfg.handle(), fallback.c_str(), &c));
  return detail::from_c(c);
}

inline ModelParams model_from_config(const ConfigFile& cfg) {
  gmi_model_params_t c{};
  detail::check(gmi_config_model(cfg.handle(), &c));
  ModelParams m;
  m.calibration = {c.serving_combw_factor, c.training_combw_factor};
  m.gmis_per_gpu = c.gmis_per_gpu;
  m.latency_scale = c.latency_scale;
  m.pipeline = {c.pipeline.compress_threshold, c.pipeline.batch_mode == 0 ? BatchMode::Slice : BatchMode::Stack,
                c.pipeline.target_batch, c.pipeline.per_message_overhead, c.pipeline.seed};
  return m;
}

inline SearchSettings search_from_config(const ConfigFile& cfg) {
  gmi_search_settings_t c{};
  detail::check(gmi_config_search(cfg.handle(), &c));
  SearchSettings s;
  s.config.num_env_grid.assign(c.grid, c.grid + c.grid_len);
  s.config.max_gmis_per_gpu = c.max_gmis_per_gpu;
  s.config.sat_threshold = c.sat_threshold;
  if (c.has_profile_trace) s.profile_trace = c.profile_trace;
  return s;
}

}  // namespace gmux
