// Workload catalog, GPU/partition model, GMI placement templates and the analytical
// cost tables (reference: workload.hpp:61-134, topology.hpp:27-252, mapping.hpp:51-279).
#include <algorithm>
#include <cmath>
#include <limits>
#include <map>
#include <string>

#include "errors.hpp"
#include "planner.hpp"

namespace gmi::plan {

// ------------------------------------------------------------------ workload
std::size_t mlp_params(const std::vector<int>& dims) {
  std::size_t n = 0;
  for (std::size_t i = 1; i < dims.size(); ++i) n += std::size_t(dims[i - 1] + 1) * std::size_t(dims[i]);
  return n;
}

// Policy MLP plus a value MLP over the same hidden stack with a scalar head.
std::size_t actor_critic_params(const std::vector<int>& dims) {
  if (dims.size() < 2) invalid("policy needs at least two layer widths");
  std::vector<int> critic = dims;
  critic.back() = 1;
  return mlp_params(dims) + mlp_params(critic);
}

const std::vector<std::string>& catalog_names() {
  static const std::vector<std::string> names = {"AT", "AY", "BB", "FC", "HM", "SH"};
  return names;
}

Workload catalog(const std::string& name) {
  static const std::map<std::string, std::vector<int>> dims = {
      {"AT", {60, 256, 128, 64, 8}},   {"AY", {48, 256, 128, 64, 12}},
      {"BB", {24, 256, 128, 64, 3}},   {"FC", {23, 256, 128, 64, 9}},
      {"HM", {108, 200, 400, 100, 21}}, {"SH", {211, 512, 512, 512, 256, 20}},
  };
  auto it = dims.find(name);
  if (it == dims.end()) invalid("unknown benchmark: " + name);
  Workload w;
  w.name = name;
  w.dims = it->second;
  const double fp32 = 4.0;
  w.S = w.dims.front() * fp32;
  w.A = w.dims.back() * fp32;
  w.W = fp32;
  w.Mp = double(actor_critic_params(w.dims)) * fp32;
  w.m = 32;
  return w;
}

void check_workload(const Workload& w) {
  auto need = [](bool ok, const char* what) {
    if (!ok) invalid(std::string("workload: ") + what);
  };
  need(w.S > 0 && w.A > 0 && w.W > 0, "S, A, W must be positive");
  need(w.Mp > 0, "model size must be positive");
  need(w.m >= 1, "steps_per_train must be >= 1");
  need(w.alpha > 0 && w.alpha <= 1, "alpha outside (0,1]");
  need(w.beta > 0 && w.beta <= 1, "beta outside (0,1]");
  for (const RoleCost* r : {&w.sim, &w.agent, &w.trainer}) {
    need(r->r_sm > 0 && r->r_sm <= 1, "r_sm outside (0,1]");
    need(r->r_mem > 0 && r->r_mem <= 1, "r_mem outside (0,1]");
    need(r->t_iter > 0, "t_iter must be positive");
  }
}

// ------------------------------------------------------------------ topology
const std::vector<MigShape>& mig_table() {
  static const std::vector<MigShape> t = {
      {"1g.5gb", 1, 5.0}, {"2g.10gb", 2, 10.0}, {"3g.20gb", 3, 20.0}, {"4g.20gb", 4, 20.0}, {"7g.40gb", 7, 40.0}};
  return t;
}

// B200 extension of topology.hpp:37-43: the MIG profiles NVIDIA publishes for the 180 GB B200
// (7 compute slices, 8 memory slices of ~22.5 GB; label sizes). Units count compute slices in
// the reference's 8-unit model with one unit reserved (topology.hpp:34-35), so the same
// "7 usable units" rule applies; B200 adds the memory-slice budget (8) that the A100-40GB
// table never needed (every A100 profile there has memory slices == compute units + 0..1).
const std::vector<MigShape>& mig_table_sm100() {
  static const std::vector<MigShape> t = {{"1g.23gb", 1, 23.0}, {"1g.45gb", 1, 45.0}, {"2g.45gb", 2, 45.0},
                                          {"3g.90gb", 3, 90.0}, {"4g.90gb", 4, 90.0}, {"7g.180gb", 7, 180.0}};
  return t;
}

int mig_memory_slices_sm100(double mem_gb) { return int(mem_gb / 22.5 + 0.5); }

const MigShape* mig_by_name(const std::string& name) {
  for (const auto* tab : {&mig_table(), &mig_table_sm100()})
    for (const auto& s : *tab)
      if (name == s.name) return &s;
  return nullptr;
}

static const MigShape* mig_by_shape(double share, double mem, Arch arch) {
  for (const auto& s : arch == Arch::SM100 ? mig_table_sm100() : mig_table())
    if (std::abs(share - double(s.units) / 8.0) < 1e-9 && std::abs(mem - s.mem_gb) < 1e-9) return &s;
  return nullptr;
}

Machine default_machine(int num_gpus) {
  Machine m;
  for (int i = 0; i < num_gpus; ++i) m.gpus.push_back(Gpu{i});
  return m;
}

static const Gpu* gpu_by_id(const Machine& m, int id) {
  for (const auto& g : m.gpus)
    if (g.id == id) return &g;
  return nullptr;
}

// SMs of the green context realising an MPS share on an sm100 GPU: whole 8-SM groups
// (cuDevSmResourceSplitByCount granularity, cuda.h:25262) of the physical SM count (148 on
// B200 unless the config gives sm_units > 8).
int green_sms(double share, const Gpu& gpu) {
  const int sms = gpu.sm_units > 8 ? gpu.sm_units : 148;
  return int(share * sms + 1e-9) / 8 * 8;
}

std::vector<std::pair<int, std::string>> check_machine(const Machine& m) {
  std::vector<std::pair<int, std::string>> bad;
  auto flag = [&](int gpu, std::string why) { bad.emplace_back(gpu, std::move(why)); };

  if (m.b1 <= 0 || m.b2 <= 0) flag(-1, "bandwidths must be positive");
  std::map<int, int> seen;
  for (const auto& p : m.parts) ++seen[p.gmi_id];
  for (const auto& [id, n] : seen)
    if (n > 1) flag(-1, "duplicate gmi id " + std::to_string(id));

  std::map<int, std::vector<const Partition*>> on_gpu;
  for (const auto& p : m.parts) {
    if (!gpu_by_id(m, p.gpu_id)) {
      flag(p.gpu_id, "partition gmi " + std::to_string(p.gmi_id) + " references unknown GPU");
      continue;
    }
    on_gpu[p.gpu_id].push_back(&p);
  }

  for (auto& [gid, parts] : on_gpu) {
    const Gpu& gpu = *gpu_by_id(m, gid);
    std::sort(parts.begin(), parts.end(), [](auto* a, auto* b) { return a->gmi_id < b->gmi_id; });
    const Backend be = parts.front()->backend;
    if (std::any_of(parts.begin(), parts.end(), [&](auto* p) { return p->backend != be; })) {
      flag(gid, "mixed MPS and MIG backends on one GPU");
      continue;
    }
    bool fields = true;
    for (const auto* p : parts) {
      if (!(p->sm_share > 0 && p->sm_share <= 1.0)) {
        flag(gid, "gmi " + std::to_string(p->gmi_id) + " sm_share outside (0,1]");
        fields = false;
      }
      if (p->mem_gb <= 0) {
        flag(gid, "gmi " + std::to_string(p->gmi_id) + " mem_gb not positive");
        fields = false;
      }
    }
    if (!fields) continue;
    if (be == Backend::MIG) {
      if (gpu.arch == Arch::SM70) {
        flag(gid, "MIG unavailable on sm70 (only MPS)");
        continue;
      }
      if (gpu.sm_units != 8) {
        flag(gid, "MIG profiles require an 8-unit GPU");
        continue;
      }
      int units = 0, mem_slices = 0;
      bool shapes = true;
      for (const auto* p : parts) {
        const MigShape* s = mig_by_shape(p->sm_share, p->mem_gb, gpu.arch);
        if (!s) {
          flag(gid, "gmi " + std::to_string(p->gmi_id) + " not an allowed MIG profile");
          shapes = false;
          continue;
        }
        units += s->units;
        mem_slices += mig_memory_slices_sm100(s->mem_gb);
      }
      const int usable = gpu.arch == Arch::SM70 ? gpu.sm_units : gpu.sm_units - 1;
      if (shapes && units > usable)
        flag(gid, "exceeds 7 usable units (" + std::to_string(units) + "/8 allocated)");
      if (shapes && gpu.arch == Arch::SM100 && mem_slices > 8)
        flag(gid, "exceeds 8 memory slices (" + std::to_string(mem_slices) + "/8 allocated)");
    } else {
      double sum = 0;
      for (const auto* p : parts) sum += p->sm_share;
      if (sum > 1.0 + 1e-9) flag(gid, "MPS shares exceed 1.0");
      if (gpu.arch == Arch::SM100)  // B200: each share is realised as a green context of 8-SM groups
        for (const auto* p : parts)
          if (green_sms(p->sm_share, gpu) < 8)
            flag(gid, "gmi " + std::to_string(p->gmi_id) + " share below one 8-SM green-context group");
    }
  }
  return bad;
}

Backend backend_for(Arch a, bool training) {
  if (a == Arch::SM70) return Backend::MPS;
  return training ? Backend::MPS : Backend::MIG;
}

Link link_between(const Machine& m, int src, int dst, double* bw) {
  const Partition *a = nullptr, *b = nullptr;
  for (const auto& p : m.parts) {
    if (p.gmi_id == src && !a) a = &p;
    if (p.gmi_id == dst && !b) b = &p;
  }
  if (!a) invalid("unknown gmi id " + std::to_string(src));
  if (!b) invalid("unknown gmi id " + std::to_string(dst));
  if (src == dst) {
    *bw = std::numeric_limits<double>::infinity();
    return Link::Intra;
  }
  if (a->gpu_id == b->gpu_id) {
    *bw = m.b1;
    return Link::HostBounce;
  }
  *bw = m.b2;
  return Link::Ring;
}

// ------------------------------------------------------------------ placement
Assignment assign(Tpl tpl, const Machine& m, int gpg) {
  if (gpg < 1) invalid("gmis_per_gpu must be >= 1");
  const auto bad = check_machine(m);
  if (!bad.empty()) fail(GMI_ERR_PLAN, "topology does not validate: " + bad.front().second);
  if (m.gpus.empty()) fail(GMI_ERR_PLAN, "topology has no GPUs");

  std::vector<int> ids;
  for (const auto& g : m.gpus) ids.push_back(g.id);
  std::sort(ids.begin(), ids.end());

  Assignment out;
  out.tpl = tpl;
  int next = 0;
  auto place = [&](int gpu, int roles) {
    out.per_gpu[gpu].push_back(next);
    out.roles[next] = roles;
    ++next;
  };

  if (tpl == Tpl::TCG || tpl == Tpl::TCG_EX) {
    const int roles = tpl == Tpl::TCG ? (kSim | kAgent) : (kSim | kAgent | kTrainer);
    for (int gpu : ids)
      for (int i = 0; i < gpg; ++i) place(gpu, roles);
  } else if (tpl == Tpl::TDG || tpl == Tpl::TDG_EX) {
    const std::vector<int> cycle = tpl == Tpl::TDG ? std::vector<int>{kSim, kAgent}
                                                   : std::vector<int>{kSim, kAgent, kTrainer};
    const std::size_t total = ids.size() * std::size_t(gpg);
    if (total % cycle.size() != 0)
      fail(GMI_ERR_PLAN, "dedicated template needs the GMI count divisible by " + std::to_string(cycle.size()));
    std::size_t k = 0;
    for (int gpu : ids)
      for (int i = 0; i < gpg; ++i) place(gpu, cycle[k++ % cycle.size()]);
  } else {
    if (ids.size() < 2) fail(GMI_ERR_PLAN, "not enough GPUs for the decoupled serving/training split");
    const std::size_t serving = (ids.size() + 1) / 2;  // serving takes the odd GPU
    for (std::size_t i = 0; i < ids.size(); ++i) {
      const bool serve = i < serving;
      (serve ? out.serving : out.training).push_back(ids[i]);
      for (int j = 0; j < gpg; ++j) place(ids[i], serve ? (kSim | kAgent) : kTrainer);
    }
  }
  return out;
}

// ------------------------------------------------------------------ cost tables
double allreduce_volume(int n, double mb) { return 2.0 * (n - 1) * mb / n; }

Cost serving_cost(Tpl tpl, const Workload& w) {
  if (tpl == Tpl::TDG) {
    const double r = (w.sim.t_iter * w.sim.r_sm + w.agent.t_iter * w.alpha * w.agent.r_sm) /
                     (w.sim.t_iter + w.agent.t_iter);
    return {r, 2 * w.S + w.A + w.W};
  }
  if (tpl == Tpl::TCG) return {std::max(w.sim.r_sm, w.agent.r_sm), 0.0};
  invalid("serving_cost expects TDG or TCG");
}

Cost training_cost(Tpl tpl, const Workload& w, int n) {
  if (n < 1) invalid("n_gmis must be >= 1");
  if (tpl == Tpl::TDG_EX) {
    const double r = (w.sim.t_iter * w.sim.r_sm + w.agent.t_iter * w.alpha * w.agent.r_sm +
                      w.trainer.t_iter * w.beta * w.trainer.r_sm) /
                     (w.sim.t_iter + w.agent.t_iter + w.trainer.t_iter);
    return {r, w.m * (w.S + w.A + w.W) + w.Mp + allreduce_volume(n, w.Mp)};
  }
  if (tpl == Tpl::TCG_EX) return {std::max({w.sim.r_sm, w.agent.r_sm, w.trainer.r_sm}), allreduce_volume(n, w.Mp)};
  invalid("training_cost expects TDG_EX or TCG_EX");
}

double serving_rate(const Cost& c, const Workload& w, double r_all, double bw) {
  if (bw <= 0 || r_all <= 0) invalid("r_all and bandwidth must be positive");
  return (r_all / c.resource) / (w.interaction() + c.comm / bw);
}

double training_rate(const Cost& c, const Workload& w, double r_all, double bw) {
  if (bw <= 0 || r_all <= 0) invalid("r_all and bandwidth must be positive");
  return (r_all / c.resource) / (w.iteration() + c.comm / bw);
}

static double calibrate(double com, double factor, double t_ref) {
  if (com <= 0 || factor <= 0 || t_ref <= 0) invalid("calibration inputs must be positive");
  return com / (factor * t_ref);
}

double serving_gain(const Workload& w, double factor) {
  const Cost d = serving_cost(Tpl::TDG, w), c = serving_cost(Tpl::TCG, w);
  const double bw = calibrate(d.comm, factor, w.interaction());
  return serving_rate(c, w, 1.0, bw) / serving_rate(d, w, 1.0, bw);
}

double training_gain(const Workload& w, double factor) {
  const Cost d = training_cost(Tpl::TDG_EX, w, 1), c = training_cost(Tpl::TCG_EX, w, 1);
  const double bw = calibrate(d.comm, factor, w.iteration());
  return training_rate(c, w, 1.0, bw) / training_rate(d, w, 1.0, bw);
}

double serving_penalty(const Workload& w) {
  return serving_cost(Tpl::TCG, w).resource / serving_cost(Tpl::TDG, w).resource - 1.0;
}

double training_penalty(const Workload& w) {
  return training_cost(Tpl::TCG_EX, w, 1).resource / training_cost(Tpl::TDG_EX, w, 1).resource - 1.0;
}

}  // namespace gmi::plan
