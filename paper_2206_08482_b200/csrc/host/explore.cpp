// Adaptive GMI manager (Alg. 2): saturation-pruned sweep over (GMIs per GPU,
// num_env) behind a pluggable probe. Reference behaviour: search.hpp:45-249.
// The probe is where the measured B200 iteration plugs in (host/gpu_profiler.cpp).
#include <cmath>
#include <fstream>
#include <limits>
#include <sstream>

#include "errors.hpp"
#include "planner.hpp"

namespace gmi::plan {

void check_grid(const SearchGrid& g) {
  if (g.envs.empty()) invalid("num_env grid must not be empty");
  if (g.max_gpg < 1) invalid("max_gmis_per_gpu must be >= 1");
  if (!(g.sat > 0 && g.sat < 1)) invalid("sat_threshold must lie in (0,1)");
}

double saturation_ratio(double top, double pre_top, double mem, double pre_mem) {
  if (pre_top <= 0 || pre_mem <= 0) invalid("saturation needs positive previous trackers");
  const double gain = (top - pre_top) / pre_top;
  const double growth = (mem - pre_mem) / pre_mem;
  if (growth == 0) return gain == 0 ? 0.0 : std::copysign(std::numeric_limits<double>::infinity(), gain);
  return gain / growth;
}

// Linear scaling over GMIs and GPUs, damped by the predicted synchronization
// latency of the strategy Alg. 1 picks for a uniform GPU-major layout.
double Projection::discount(int gpg, int gpus) const {
  Placement p;
  int id = 0;
  p.per_gpu.resize(gpus);
  for (auto& g : p.per_gpu)
    for (int t = 0; t < gpg; ++t) g.push_back(id++);
  const Algo a = choose_algo(p);
  const double lat = closed_form_latency(a, gpus, gpg, w.Mp, b1, b2);
  const double it = w.iteration();
  return it / (it + lat / latency_scale);
}

double Projection::project(int gpg, int gpus, double per_gmi_top) const {
  if (gpg < 1 || gpus < 1 || per_gmi_top < 0) invalid("estimate needs positive inputs");
  return per_gmi_top * gpg * gpus * discount(gpg, gpus);
}

SearchOutcome search(const ProbeFn& probe, const Projection& proj, const std::string& bench, int gpus,
                     const SearchGrid& grid) {
  check_grid(grid);
  if (gpus < 1) invalid("num_gpu must be >= 1");
  SearchOutcome out;
  bool any = false;
  double best = -std::numeric_limits<double>::infinity();
  for (int gpg = grid.max_gpg; gpg >= 1; --gpg) {
    double last_top = 0, last_mem = 0;
    for (int env : grid.envs) {
      const Probe pr = probe(bench, gpg, env);
      Visit v{gpg, env, pr.runnable, pr.top, pr.mem, std::nullopt, std::nullopt, false};
      if (!pr.runnable) {
        out.visits.push_back(v);
        continue;
      }
      any = true;
      if (last_top == 0 && last_mem == 0) {  // first runnable point seeds, never estimated
        last_top = pr.top;
        last_mem = pr.mem;
        out.visits.push_back(v);
        continue;
      }
      const double sat = saturation_ratio(pr.top, last_top, pr.mem, last_mem);
      v.sat = sat;
      last_top = pr.top;
      last_mem = pr.mem;
      if (sat < grid.sat) {
        v.pruned = true;
        out.visits.push_back(v);
        break;
      }
      const double acc = proj.project(gpg, gpus, pr.top);
      v.acc = acc;
      out.visits.push_back(v);
      if (acc > best) {
        best = acc;
        out.feasible = true;
        out.env = env;
        out.gpg = gpg;
        out.est = acc;
      }
    }
  }
  if (!out.feasible)
    out.reason = any ? "no point passed the saturation gate to be estimated" : "no runnable configuration";
  return out;
}

int SyntheticProbe::knee(int gpg) const {
  if (auto it = knee_override.find(gpg); it != knee_override.end()) return it->second;
  int k = 512;
  while (2 * k <= knee_base / gpg && k < 8192) k *= 2;
  return k;
}

Probe SyntheticProbe::operator()(const std::string& bench, int gpg, int num_env) const {
  catalog(bench);  // unknown names throw
  if (gpg < 1 || num_env < 1) invalid("profile needs gmis_per_gpu >= 1 and num_env >= 1");
  const double share = 1.0 / gpg;
  const double mem = mem_base + mem_per_env * num_env;
  if (share < min_share || mem > mem_capacity * share) return {false, 0, 0};
  double scale = 1.0;
  if (auto it = cap_scale.find(gpg); it != cap_scale.end()) scale = it->second;
  const double cap = peak_top * share * scale;
  const int kn = knee(gpg);
  return {true, cap * std::min(double(num_env), double(kn)) / double(kn), mem};
}

TableProbe TableProbe::from_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(GMI_ERR_DOMAIN, "cannot open trace file: " + path);
  TableProbe t;
  std::string line;
  int n = 0;
  while (std::getline(in, line)) {
    ++n;
    if (auto h = line.find('#'); h != std::string::npos) line.erase(h);
    std::istringstream ss(line);
    std::string bench;
    int gpg = 0, env = 0, ok = 0;
    double top = 0, mem = 0;
    if (!(ss >> bench)) continue;
    if (!(ss >> gpg >> env >> ok >> top >> mem))
      fail(GMI_ERR_DOMAIN, "trace file " + path + ": malformed row at line " + std::to_string(n));
    t.rows[{bench, gpg, env}] = {ok != 0, top, mem};
  }
  return t;
}

Probe TableProbe::operator()(const std::string& bench, int gpg, int num_env) const {
  auto it = rows.find({bench, gpg, num_env});
  return it == rows.end() ? Probe{false, 0, 0} : it->second;
}

}  // namespace gmi::plan
