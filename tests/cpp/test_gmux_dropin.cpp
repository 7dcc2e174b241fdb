// Drop-in parity suite for include/gmux/gmux.hpp (C++ over libgmi's C-ABI), written in the
// style of the reference's Catch2 suites (proj/tests/test_*.cpp) with a minimal CHECK shim
// (Catch2 is not available in this image). Built and run by tests/test_cpp_dropin.py.
// Device cases (execute) run only when argv[1] == "gpu".
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "gmux/gmux.hpp"

using namespace gmux;

static int g_checks = 0, g_failed = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    ++g_checks;                                                              \
    if (!(cond)) {                                                           \
      ++g_failed;                                                            \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                        \
  } while (0)
#define CHECK_THROWS_AS(expr, type)   \
  do {                                \
    bool caught = false;              \
    try {                             \
      (void)(expr);                   \
    } catch (const type&) {           \
      caught = true;                  \
    } catch (...) {                   \
    }                                 \
    CHECK(caught && #type);           \
  } while (0)

static std::string selection_oracle(const std::vector<std::vector<int>>& mpl) {
  std::set<std::size_t> per;
  if (mpl.size() <= 1) return "MPR";
  for (const auto& l : mpl) per.insert(l.size());
  if (per.size() > 1) return "HAR";
  if (*per.begin() > mpl.size()) return "HAR";
  return "MRR";
}

static void reduction_cases() {
  CHECK(select_strategy({{{0, 1, 2}}}) == Strategy::MPR);
  CHECK(select_strategy({{{0, 1}, {2, 3}}}) == Strategy::MRR);
  CHECK(select_strategy({{{0, 1, 2}, {3, 4, 5}}}) == Strategy::HAR);
  CHECK(select_strategy({{{0}, {1, 2}}}) == Strategy::HAR);
  for (int g = 1; g <= 5; ++g) {
    std::vector<int> counts(g, 1);
    while (true) {
      GmiLayout layout;
      int next = 0;
      for (int c : counts) {
        layout.mpl.emplace_back();
        for (int i = 0; i < c; ++i) layout.mpl.back().push_back(next++);
      }
      CHECK(to_string(select_strategy(layout)) == selection_oracle(layout.mpl));
      int i = g - 1;
      while (i >= 0 && counts[i] == 5) counts[i--] = 1;
      if (i < 0) break;
      ++counts[i];
    }
  }
  CHECK_THROWS_AS(GmiLayout{}.validate(), std::invalid_argument);
  CHECK_THROWS_AS((GmiLayout{{{0, 1}, {}}}).validate(), std::invalid_argument);
  CHECK_THROWS_AS((GmiLayout{{{0, 1}, {1, 2}}}).validate(), std::invalid_argument);
  CHECK(leader_gmis({{{0, 1}, {2, 3}}}) == (std::vector<int>{0, 2}));
  CHECK(leader_gmis({{{5}, {7}}}) == (std::vector<int>{5, 7}));
  CHECK(leader_gmis({{{1, 3}, {5, 7}}}) == (std::vector<int>{1, 5}));
  CHECK(predict_latency(Strategy::MPR, 2, 2, 240, 1, 30) == 360.0);
  CHECK(predict_latency(Strategy::MRR, 2, 2, 240, 1, 30) == 24.0);
  CHECK(predict_latency(Strategy::HAR, 2, 2, 240, 1, 30) == 248.0);
  CHECK_THROWS_AS(predict_latency(Strategy::MPR, 0, 1, 240, 1, 30), std::invalid_argument);
  CHECK_THROWS_AS(mrr_rings({{{0}, {1, 2}}}), MultiStreamError);
  CHECK_THROWS_AS(mrr_rings({{{0, 1, 2}, {3, 4, 5}}}), MultiStreamError);
  for (int g = 2; g <= 5; ++g)
    for (int t = 1; t <= g; ++t) {
      GmiLayout layout;
      int next = 100;
      for (int i = 0; i < g; ++i) {
        layout.mpl.emplace_back();
        for (int j = 0; j < t; ++j) layout.mpl.back().push_back(next++);
      }
      auto gpu_of = [&](int id) {
        for (int i = 0; i < g; ++i)
          for (int x : layout.mpl[i])
            if (x == id) return i;
        return -1;
      };
      const auto rings = mrr_rings(layout);
      CHECK(int(rings.size()) == t);
      std::set<int> seen, ends;
      for (const auto& ring : rings) {
        std::set<int> gpus;
        for (int id : ring) {
          CHECK(seen.insert(id).second);
          gpus.insert(gpu_of(id));
        }
        CHECK(int(gpus.size()) == g);
        CHECK(ends.insert(gpu_of(ring.back())).second);
      }
    }
  for (int g = 2; g <= 8; ++g)
    for (int t = 1; t <= 9; ++t)
      CHECK(predict_latency(Strategy::HAR, g, t, 1e6, 1.0, 30.0) < predict_latency(Strategy::MPR, g, t, 1e6, 1.0, 30.0));
}

static void execute_cases() {  // device
  const Topology topo = default_topology(2);
  const GmiLayout layout{{{0, 1}, {2, 3}}};
  std::vector<GradientBuffer> bufs;
  for (int id : layout.all_gmis()) {
    GradientBuffer b{id, std::vector<double>(30)};
    for (std::size_t e = 0; e < 30; ++e) b.values[e] = 1.0 + 0.001 * id + 1e-6 * double(e);
    bufs.push_back(b);
  }
  const ReductionRun mrr = execute(Strategy::MRR, layout, bufs, topo);
  CHECK(mrr.latency == 24.0);
  CHECK(mrr.trace.size() == 15);
  for (std::size_t e = 0; e < 30; ++e) {
    double want = 0;
    for (const auto& b : bufs) want += b.values[e];
    CHECK(std::abs(mrr.result[e] - want) <= 1e-9 * std::max(1.0, std::abs(want)));
  }
  CHECK(execute(Strategy::HAR, layout, bufs, topo).latency == 248.0);
  CHECK(execute(Strategy::MPR, layout, bufs, topo).latency == 360.0);
  std::vector<GradientBuffer> bad = {{0, {1.0, 2.0}}, {1, {1.0}}};
  CHECK_THROWS_AS(execute(Strategy::MPR, GmiLayout{{{0}, {1}}}, bad, topo), std::invalid_argument);
  std::mt19937 rng(101);
  std::uniform_real_distribution<double> val(0.1, 1.0);
  for (int trial = 0; trial < 30; ++trial) {
    GmiLayout lay;
    int next = trial;
    const int g = 1 + trial % 4;
    for (int i = 0; i < g; ++i) {
      lay.mpl.emplace_back();
      for (int j = 0; j <= (trial + i) % 4; ++j) lay.mpl.back().push_back(next++);
    }
    std::vector<GradientBuffer> bb;
    for (int id : lay.all_gmis()) {
      GradientBuffer b{id, std::vector<double>(1 + trial * 7)};
      for (auto& v : b.values) v = val(rng);
      bb.push_back(b);
    }
    const ReductionRun r = execute(select_strategy(lay), lay, bb, topo);
    for (std::size_t e = 0; e < r.result.size(); ++e) {
      double want = 0;
      for (const auto& b : bb) want += b.values[e];
      CHECK(std::abs(r.result[e] - want) <= 1e-9 * std::max(1.0, want));
    }
  }
}

static void mapping_cases() {
  const DrlWorkload w = load_benchmark("AT");
  CHECK(std::abs(serving_throughput_ratio(w) - 2.58) < 1e-2);
  CHECK(std::abs(training_throughput_ratio(w) - 5.458) < 1e-3);
  CHECK(std::abs(serving_colocation_penalty(w) - 0.16279) < 1e-5);
  CHECK(std::abs(training_colocation_penalty(w) - 0.46580) < 1e-5);
  CHECK(policy_value_param_count(load_benchmark("AT").policy_dims) == 114121);
  CHECK(policy_value_param_count(load_benchmark("HM").policy_dims) == 286822);
  CHECK(policy_value_param_count(load_benchmark("SH").policy_dims) == 1535765);
  CHECK_THROWS_AS(load_benchmark("XX"), std::invalid_argument);
  const MappingPlan plan = build_plan(TemplateKind::TCG_EX, default_topology(2), w, 2);
  CHECK(plan.gpu_layout.at(0) == (std::vector<int>{0, 1}));
  CHECK(plan.gpu_layout.at(1) == (std::vector<int>{2, 3}));
  for (const auto& [gmi, roles] : plan.gmi_assignments)
    CHECK(roles == (std::set<Role>{Role::Simulator, Role::Agent, Role::Trainer}));
  const MappingPlan tdg = build_plan(TemplateKind::TDG, default_topology(1), w, 2);
  CHECK(tdg.gmi_assignments.at(0) == std::set<Role>{Role::Simulator});
  CHECK(tdg.gmi_assignments.at(1) == std::set<Role>{Role::Agent});
  CHECK_THROWS_AS(build_plan(TemplateKind::TDG, default_topology(1), w, 3), PlanError);
  CHECK_THROWS_AS(build_plan(TemplateKind::AsyncDecoupled, default_topology(1), w, 2), PlanError);
  const MappingPlan async = build_plan(TemplateKind::AsyncDecoupled, default_topology(3), w, 2);
  CHECK(async.serving_gpus == (std::vector<int>{0, 1}));
  CHECK(async.training_gpus == (std::vector<int>{2}));
  Topology bad = default_topology(1);
  bad.partitions.push_back(mig_partition(0, 0, "4g.20gb"));
  bad.partitions.push_back(mig_partition(1, 0, "4g.20gb"));
  CHECK_THROWS_AS(build_plan(TemplateKind::TCG, bad, w, 1), PlanError);
  CHECK(!validate_layout(bad).ok());
  CHECK(select_backend(GpuArch::SM80, TaskMode::Serving) == Backend::MIG);
  CHECK(select_backend(GpuArch::SM70, TaskMode::Serving) == Backend::MPS);
}

static void search_cases() {
  const ThroughputEstimator est{load_benchmark("AT"), 1.0, 30.0, 1000.0};
  const SyntheticCostModel model;
  const SearchResult r = explore(model, est, "AT", 2, SearchConfig{});
  CHECK(r.feasible);
  CHECK(r.num_env == 8192 && r.gmis_per_gpu == 1);
  CHECK(r.visited.size() == 58);
  CHECK(std::abs(r.est_throughput - 54777.47496128383) < 1e-9);
  SyntheticCostModel peaked;
  for (int g = 1; g <= 10; ++g) {
    peaked.cap_scale[g] = g == 2 ? 1.0 : 0.1;
    peaked.knee_override[g] = g == 2 ? 4096 : 8192;
  }
  const SearchResult p = explore(peaked, est, "AT", 2, SearchConfig{});
  CHECK(p.num_env == 4096 && p.gmis_per_gpu == 2);
  SyntheticCostModel dead;
  dead.min_runnable_share = 2.0;
  const SearchResult d = explore(dead, est, "AT", 2, SearchConfig{});
  CHECK(!d.feasible && d.reason == "no runnable configuration");
  SearchConfig bad;
  bad.sat_threshold = 0.0;
  CHECK_THROWS_AS(explore(model, est, "AT", 2, bad), std::invalid_argument);
}

static void channel_cases() {
  const DrlWorkload w = load_benchmark("AT");
  const Topology topo = default_topology(2);
  const MappingPlan plan = build_plan(TemplateKind::AsyncDecoupled, topo, w, 2);
  PipelineConfig cfg;
  const PipelineMetrics mcc = simulate_pipeline(w, plan, topo, cfg, 3000.0);
  const PipelineMetrics ucc = simulate_pipeline(w, plan, topo, uni_channel(cfg), 3000.0);
  CHECK(mcc.records_delivered == mcc.records_produced);
  CHECK(mcc.pps > ucc.pps);
  std::set<std::pair<int, long>> seen;
  for (const auto& b : mcc.batches)
    for (const auto& r : b.records) CHECK(seen.insert({r.agent_gmi, r.seq}).second);
  CHECK(long(seen.size()) == mcc.records_produced);
}

static void config_cases() {
  std::istringstream in("[topology]\nb1 = 2\ngpu = id=0 arch=sm100\ngmi = id=0 gpu=0 backend=mps share=0.5\n"
                        "[workload]\nbenchmark = HM\n[ppo]\nnum_envs = 8192\n");
  const ConfigFile cfg = parse_config(in);
  const Topology t = topology_from_config(cfg);
  CHECK(t.b1 == 2.0 && t.gpus.size() == 1 && t.gpus[0].arch == GpuArch::SM100);
  CHECK(t.partitions.size() == 1 && t.partitions[0].mem_gb == 20.0);
  CHECK(workload_from_config(cfg).name == "HM");
  CHECK(cfg.get("ppo", "num_envs") == std::optional<std::string>("8192"));
  std::istringstream bad("[topology]\nbogus = 1\n");
  const ConfigFile b = parse_config(bad);
  CHECK_THROWS_AS(topology_from_config(b), ConfigError);
  std::istringstream bad2("b1 = 1\n");
  CHECK_THROWS_AS(parse_config(bad2), ConfigError);
  CHECK_THROWS_AS(load_config("/no/such.cfg"), ConfigError);
}

int main(int argc, char** argv) {
  reduction_cases();
  mapping_cases();
  search_cases();
  channel_cases();
  config_cases();
  if (argc > 1 && std::strcmp(argv[1], "gpu") == 0) execute_cases();
  std::printf("%d checks, %d failed\n", g_checks, g_failed);
  return g_failed == 0 ? 0 : 1;
}
