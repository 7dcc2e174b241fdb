// Layout-aware gradient-reduction planning: Alg. 1 strategy choice, leader GMIs,
// disjoint multi-rings, Table 3 closed forms, and the hop schedule + ideal-link
// latency of each strategy. Behaviour follows reduction.hpp:39-334 of the reference
// (see planner.hpp); the element arithmetic runs on the device (cuda/reduce.cu).
#include <algorithm>
#include <map>
#include <set>
#include <string>

#include "errors.hpp"
#include "planner.hpp"

namespace gmi::plan {

std::vector<int> Placement::flat() const {
  std::vector<int> out;
  for (const auto& g : per_gpu) out.insert(out.end(), g.begin(), g.end());
  return out;
}

bool Placement::same_width() const {
  for (const auto& g : per_gpu)
    if (g.size() != per_gpu.front().size()) return false;
  return true;
}

void Placement::check() const {
  if (per_gpu.empty()) invalid("layout needs at least one GPU");
  std::set<int> ids;
  for (const auto& g : per_gpu) {
    if (g.empty()) invalid("layout has an empty per-GPU list");
    for (int id : g)
      if (!ids.insert(id).second) invalid("duplicate gmi id " + std::to_string(id) + " in layout");
  }
}

// Alg. 1 (reduction.hpp:98-106): one GPU -> host-path ring; ragged or
// oversubscribed (t > g) -> hierarchical; otherwise disjoint multi-ring.
Algo choose_algo(const Placement& p) {
  p.check();
  const int g = p.gpus();
  if (g <= 1) return Algo::MPR;
  if (!p.same_width()) return Algo::HAR;
  if (int(p.per_gpu.front().size()) > g) return Algo::HAR;
  return Algo::MRR;
}

// reduction.hpp:110-122: smallest id with id % (GMIs on that GPU) == 0, else min id.
std::vector<int> gpu_leaders(const Placement& p) {
  p.check();
  std::vector<int> out;
  out.reserve(p.per_gpu.size());
  for (const auto& g : p.per_gpu) {
    const int width = int(g.size());
    int pick = -1;
    for (int id : g)
      if (id % width == 0 && (pick < 0 || id < pick)) pick = id;
    out.push_back(pick >= 0 ? pick : *std::min_element(g.begin(), g.end()));
  }
  return out;
}

// reduction.hpp:127-139: ring r = r-th GMI of every GPU, starting at GPU r.
std::vector<std::vector<int>> disjoint_rings(const Placement& p) {
  p.check();
  if (!p.same_width()) fail(GMI_ERR_MULTISTREAM, "multiple streams per GPU: layout is not uniform");
  const int g = p.gpus();
  const int t = int(p.per_gpu.front().size());
  if (t > g)
    fail(GMI_ERR_MULTISTREAM, "multiple streams per GPU: " + std::to_string(t) + " rings over " +
                                  std::to_string(g) + " GPUs");
  std::vector<std::vector<int>> rings(t, std::vector<int>(g));
  for (int r = 0; r < t; ++r)
    for (int j = 0; j < g; ++j) rings[r][j] = p.per_gpu[(r + j) % g][r];
  return rings;
}

// Table 3 (reduction.hpp:142-152).
double closed_form_latency(Algo a, int g, int t, double m_p, double b1, double b2) {
  if (g < 1 || t < 1 || m_p <= 0) invalid("need g >= 1, t >= 1, m_p > 0");
  const double n = double(g) * t;
  switch (a) {
    case Algo::MPR: return 2.0 * (n - 1) * m_p / (n * b1);
    case Algo::MRR: return 2.0 * (g - 1) * (t + 1) * m_p / (g * b2);
    case Algo::HAR: return 2.0 * (g - 1) * m_p / (g * b2) + 2.0 * (t - 1) * m_p / (t * b1);
  }
  invalid("unknown strategy");
}

namespace {

// Hops of one bandwidth-optimal ring allreduce: n-1 reduce-scatter rounds then n-1
// all-gather rounds, each member forwarding m_p/n bytes to its successor per round.
// Host-path rounds also record the CPU-side accumulation (zero cost).
int emit_ring(std::vector<Hop>& hops, const std::vector<int>& ring, Link link, int first_step,
              double m_p) {
  const int n = int(ring.size());
  if (n < 2) return 0;
  const double piece = m_p / n;
  for (int phase = 0; phase < 2; ++phase)
    for (int r = 0; r < n - 1; ++r)
      for (int i = 0; i < n; ++i) {
        const int step = first_step + phase * (n - 1) + r;
        const int nxt = ring[(i + 1) % n];
        hops.push_back({step, ring[i], nxt, piece, link});
        if (phase == 0 && link == Link::HostBounce)
          hops.push_back({step, ring[i], nxt, piece, Link::LocalReduce});
      }
  return 2 * (n - 1);
}

}  // namespace

Schedule build_schedule(Algo a, const Placement& p, std::size_t len, double elem_bytes, double b1,
                        double b2) {
  p.check();
  const double m_p = double(len) * elem_bytes;
  const int g = p.gpus();
  Schedule s;
  s.algo = a;
  s.result_holder = p.per_gpu[0][0];
  Link bcast = Link::Ring;
  int step = 0;

  switch (a) {
    case Algo::MPR:
      step += emit_ring(s.hops, p.flat(), Link::HostBounce, step, m_p);
      bcast = Link::HostBounce;
      break;
    case Algo::MRR: {
      const auto rings = disjoint_rings(p);
      for (const auto& ring : rings) step += emit_ring(s.hops, ring, Link::Ring, step, m_p);
      std::vector<int> ends;
      if (rings.size() >= 2)
        for (const auto& ring : rings) ends.push_back(ring.back());
      else
        ends = rings.front();
      if (g >= 2 && ends.size() >= 2) {
        const int ne = int(ends.size());
        for (int r = 0; r < 2 * (g - 1); ++r)
          for (int j = 0; j < ne; ++j) s.hops.push_back({step + r, ends[j], ends[(j + 1) % ne], m_p / g, Link::Ring});
        step += 2 * (g - 1);
      }
      s.result_holder = ends.front();
      break;
    }
    case Algo::HAR: {
      int widest = 0;  // per-GPU host rings share one step window
      for (const auto& local : p.per_gpu) widest = std::max(widest, emit_ring(s.hops, local, Link::HostBounce, step, m_p));
      step += widest;
      const auto leads = gpu_leaders(p);
      step += emit_ring(s.hops, leads, Link::Ring, step, m_p);
      s.result_holder = leads.front();
      break;
    }
  }

  // Ideal link model: hops in one step overlap, steps serialize, CPU folds are free.
  std::map<int, double> per_step;
  for (const Hop& h : s.hops) {
    const double cost = h.link == Link::HostBounce ? h.bytes / b1 : h.link == Link::Ring ? h.bytes / b2 : 0.0;
    double& slot = per_step[h.step];
    slot = std::max(slot, cost);
  }
  for (const auto& kv : per_step) s.latency += kv.second;

  const auto members = p.flat();
  for (int id : members)
    if (id != s.result_holder) s.hops.push_back({step, s.result_holder, id, m_p, bcast});
  if (members.size() > 1) s.broadcast_latency = bcast == Link::HostBounce ? m_p / b1 : m_p / b2;
  return s;
}

}  // namespace gmi::plan
