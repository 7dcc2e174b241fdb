// Internal model of the GMI planner (host C++). These are libgmi's own types; the
// extern "C" layer (capi_plan.cpp) flattens them and include/gmux/gmux.hpp rebuilds
// the reference's public types on top of that ABI.
//
// Behavioural contract (reference, proj/include/gmux/):
//   reduction schedule  reduction.hpp:98-334     workload catalog  workload.hpp:61-134
//   topology rules      topology.hpp:134-252     placement          mapping.hpp:95-279
//   adaptive search     search.hpp:45-249        channel pipeline   channels.hpp:93-397
//   config schema       config.hpp:125-301
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <map>
#include <optional>
#include <set>
#include <string>
#include <vector>

namespace gmi::plan {

// ------------------------------------------------------------------ layout / reduction
enum class Algo : int { MPR = 0, MRR = 1, HAR = 2 };
enum class Link : int { Intra = 0, HostBounce = 1, Ring = 2, LocalReduce = 3 };

// Per-GPU GMI id lists in placement order (the reference's "MPL").
struct Placement {
  std::vector<std::vector<int>> per_gpu;

  int gpus() const { return int(per_gpu.size()); }
  std::vector<int> flat() const;
  bool same_width() const;
  void check() const;  // throws invalid_argument like GmiLayout::validate
};

Algo choose_algo(const Placement& p);
std::vector<int> gpu_leaders(const Placement& p);
std::vector<std::vector<int>> disjoint_rings(const Placement& p);  // throws MULTISTREAM
double closed_form_latency(Algo a, int g, int t, double m_p, double b1, double b2);

struct Hop {
  int step, src, dst;
  double bytes;
  Link link;
};

// Communication schedule of one reduction over `len` elements of `elem_bytes`
// (8 for the reference's fp64 buffers): the hop list, its ideal-link latency and the
// final broadcast. Element values never enter; the fold order that the device kernel
// reproduces is described by FoldPlan below.
struct Schedule {
  Algo algo;
  std::vector<Hop> hops;
  double latency = 0;
  double broadcast_latency = 0;
  int result_holder = 0;
};
Schedule build_schedule(Algo a, const Placement& p, std::size_t len, double elem_bytes, double b1,
                        double b2);

// Chunk bounds of the ring schedule: [len*c/n, len*(c+1)/n).
inline std::size_t chunk_lo(std::size_t len, int n, int c) {
  return len * std::size_t(c) / std::size_t(n);
}

// ------------------------------------------------------------------ topology
enum class Arch : int { SM70 = 70, SM80 = 80, SM100 = 100 };
enum class Backend : int { MPS = 0, MIG = 1 };

struct Gpu {
  int id = 0;
  Arch arch = Arch::SM80;
  int sm_units = 8;
  double mem_gb = 40.0;
};

struct Partition {
  int gmi_id = 0;
  int gpu_id = 0;
  Backend backend = Backend::MPS;
  double sm_share = 1.0;
  double mem_gb = 0.0;
};

struct Machine {
  std::vector<Gpu> gpus;
  std::vector<Partition> parts;
  double b1 = 1.0;
  double b2 = 30.0;
};

struct MigShape {
  const char* name;
  int units;
  double mem_gb;
};
const std::vector<MigShape>& mig_table();
const MigShape* mig_by_name(const std::string& name);

Machine default_machine(int num_gpus);
std::vector<std::pair<int, std::string>> check_machine(const Machine& m);  // violations
int green_sms(double share, const Gpu& gpu);  // sm100: SMs of the green context realising an MPS share
Backend backend_for(Arch a, bool training);
Link link_between(const Machine& m, int src_gmi, int dst_gmi, double* bandwidth);

// ------------------------------------------------------------------ workload
struct RoleCost {
  double r_sm, r_mem, t_iter;
};

struct Workload {
  std::string name;
  double S = 0, A = 0, W = 0, Mp = 0;
  int m = 1;
  double alpha = 0.2, beta = 0.3;
  std::vector<int> dims;
  RoleCost sim{1.0, 0.5, 6.0};
  RoleCost agent{0.1, 0.05, 1.0};
  RoleCost trainer{0.2, 0.1, 2.0};

  double interaction() const { return sim.t_iter + agent.t_iter; }
  double iteration() const { return interaction() + trainer.t_iter; }
};

Workload catalog(const std::string& name);
const std::vector<std::string>& catalog_names();
void check_workload(const Workload& w);
std::size_t mlp_params(const std::vector<int>& dims);
std::size_t actor_critic_params(const std::vector<int>& dims);

// ------------------------------------------------------------------ placement / costs
enum class Tpl : int { TDG = 0, TCG = 1, TDG_EX = 2, TCG_EX = 3, Async = 4 };
enum RoleBit : int { kSim = 1, kAgent = 2, kTrainer = 4 };

struct Assignment {
  Tpl tpl = Tpl::TCG;
  std::map<int, int> roles;                   // gmi -> RoleBit mask
  std::map<int, std::vector<int>> per_gpu;    // gpu -> gmi ids
  std::vector<int> serving, training;
};

Assignment assign(Tpl tpl, const Machine& m, int gmis_per_gpu);

struct Cost {
  double resource = 0, comm = 0;
};
Cost serving_cost(Tpl tpl, const Workload& w);
Cost training_cost(Tpl tpl, const Workload& w, int n_gmis);
double allreduce_volume(int n_gmis, double model_bytes);
double training_rate(const Cost& c, const Workload& w, double r_all, double bw);
double serving_rate(const Cost& c, const Workload& w, double r_all, double bw);
double serving_gain(const Workload& w, double factor);
double training_gain(const Workload& w, double factor);
double serving_penalty(const Workload& w);
double training_penalty(const Workload& w);

// ------------------------------------------------------------------ adaptive search
struct Probe {
  bool runnable = false;
  double top = 0, mem = 0;
};
using ProbeFn = std::function<Probe(const std::string& bench, int gpg, int num_env)>;

struct SearchGrid {
  std::vector<int> envs = {128, 256, 512, 1024, 2048, 4096, 8192, 16384};
  int max_gpg = 10;
  double sat = 0.1;
};
void check_grid(const SearchGrid& g);

struct Projection {
  Workload w;
  double b1 = 1.0, b2 = 30.0, latency_scale = 1000.0;
  double discount(int gpg, int gpus) const;
  double project(int gpg, int gpus, double per_gmi_top) const;
};

double saturation_ratio(double top, double pre_top, double mem, double pre_mem);

struct Visit {
  int gpg, env;
  bool runnable;
  double top, mem;
  std::optional<double> sat, acc;
  bool pruned;
};
struct SearchOutcome {
  bool feasible = false;
  std::string reason;
  int env = 0, gpg = 0;
  double est = 0;
  std::vector<Visit> visits;
};
SearchOutcome search(const ProbeFn& probe, const Projection& proj, const std::string& bench,
                     int gpus, const SearchGrid& grid);

struct SyntheticProbe {
  double peak_top = 120000.0, mem_base = 1.0, mem_per_env = 0.002, mem_capacity = 40.0;
  double min_share = 0.1;
  int knee_base = 8192;
  std::map<int, int> knee_override;
  std::map<int, double> cap_scale;
  int knee(int gpg) const;
  Probe operator()(const std::string& bench, int gpg, int num_env) const;
};

struct TableProbe {
  std::map<std::tuple<std::string, int, int>, Probe> rows;
  static TableProbe from_file(const std::string& path);
  Probe operator()(const std::string& bench, int gpg, int num_env) const;
};

// ------------------------------------------------------------------ channel pipeline
enum class Stream : int { State = 0, Action = 1, Reward = 2 };
enum class BatchKind : int { Slice = 0, Stack = 1 };

struct RecordKey {
  int agent = 0;
  long seq = 0;
};
struct Batch {
  int trainer = 0;
  double emit = 0;
  std::vector<RecordKey> recs;
};
struct ChannelConfig {
  int k = 8;
  BatchKind mode = BatchKind::Stack;
  int target = 32;
  double overhead = 1.0;
  unsigned seed = 0;
};
void check_channels(const ChannelConfig& c);
struct FlowStats {
  double pps = 0, ttop = 0;
  long produced = 0, delivered = 0, units = 0, batches = 0;
  double bytes = 0, busy = 0, delivery_span = 0, training_span = 0;
  std::map<int, long> per_trainer;
  std::vector<Batch> out;
};
FlowStats run_channels(const Workload& w, const Assignment& a, const Machine& m,
                       const ChannelConfig& c, double duration);
// The same pipeline executed on the GPU over real payloads (cuda/channels.cu): agent_buf holds
// 3 x agents device pointers [channel * agents + agent] (state / action / reward records of each
// agent in ascending gmi-id order), trainer_buf 3 x trainers receive buffers of
// trainer_capacity records each; stream = cudaStream_t.
FlowStats run_channels_device(const Workload& w, const Assignment& a, const Machine& m, const ChannelConfig& c,
                              double duration, const std::vector<const void*>& agent_buf,
                              const std::vector<void*>& trainer_buf, long trainer_capacity, void* stream,
                              std::vector<int>* key_agent_out = nullptr, std::vector<long>* key_seq_out = nullptr);

// ------------------------------------------------------------------ config schema
struct CfgLine {
  std::string key, value;
  int line = 0;
};
struct CfgFile {
  std::map<std::string, std::vector<CfgLine>> sections;
  const std::vector<CfgLine>& lines(const std::string& s) const;
  std::optional<std::string> get(const std::string& s, const std::string& k) const;
  bool has(const std::string& s) const { return sections.count(s) > 0; }
};
CfgFile parse_cfg(const std::string& text, const std::string& origin);
Machine cfg_machine(const CfgFile& f);
Workload cfg_workload(const CfgFile& f, const std::string& fallback);

struct CfgModel {
  double serving_factor = 2.0, training_factor = 7.0;
  int gmis_per_gpu = 2;
  double latency_scale = 1000.0;
  ChannelConfig channels;
};
CfgModel cfg_model(const CfgFile& f);

struct CfgSearch {
  SearchGrid grid;
  std::optional<std::string> trace;
};
CfgSearch cfg_search(const CfgFile& f);

}  // namespace gmi::plan
