// Experience-channel accounting for the decoupled mode (config 4): agents emit
// records at the serving cadence, records are grouped k at a time into three channel
// transfer units, routed to a same-GPU trainer or the least-loaded one, batched and
// consumed. Reference behaviour: channels.hpp:93-397. This module is the host-side
// accounting model; the device-side experience hand-off of the decoupled trainer is in
// host/trainer.cpp (serve_rollout / record_iteration).
#include <algorithm>
#include <cmath>
#include <optional>
#include <tuple>

#include "errors.hpp"
#include "planner.hpp"

namespace gmi::plan {

void check_channels(const ChannelConfig& c) {
  if (c.k < 1) invalid("compress_threshold must be >= 1");
  if (c.target < 1) invalid("target_batch must be >= 1");
  if (c.overhead < 0) invalid("per_message_overhead must be >= 0");
}

namespace {

std::optional<int> colocated_trainer(const Assignment& a, int agent) {
  int gpu = -1;
  for (const auto& [g, ids] : a.per_gpu)
    if (std::find(ids.begin(), ids.end(), agent) != ids.end()) {
      gpu = g;
      break;
    }
  if (gpu < 0) fail(GMI_ERR_PIPELINE, "gmi " + std::to_string(agent) + " not in plan");
  std::optional<int> best;
  for (int id : a.per_gpu.at(gpu))
    if ((a.roles.at(id) & kTrainer) && (!best || id < *best)) best = id;
  return best;
}

struct Router {
  std::map<int, long> load;
  int pick() const {
    int best = load.begin()->first;
    for (const auto& [id, l] : load)
      if (l < load.at(best)) best = id;
    return best;
  }
};

struct Group {
  double start = 0, arrive = 0;
  int agent = 0;
  long seq = 0;
  std::optional<int> dst;
  std::vector<RecordKey> recs;
};

// Slice cuts each delivery into <= target batches; stack accumulates until target.
struct Batcher {
  BatchKind mode;
  int target;
  std::vector<RecordKey> pending;
  void feed(int trainer, const std::vector<RecordKey>& recs, double t, std::vector<Batch>& out) {
    if (mode == BatchKind::Slice) {
      for (std::size_t i = 0; i < recs.size();) {
        Batch b{trainer, t, {}};
        for (; i < recs.size() && int(b.recs.size()) < target; ++i) b.recs.push_back(recs[i]);
        out.push_back(std::move(b));
      }
      return;
    }
    pending.insert(pending.end(), recs.begin(), recs.end());
    if (int(pending.size()) >= target) {
      out.push_back({trainer, t, std::move(pending)});
      pending.clear();
    }
  }
};

}  // namespace

FlowStats run_channels(const Workload& w, const Assignment& a, const Machine& m, const ChannelConfig& c,
                       double duration) {
  if (duration <= 0) invalid("duration must be positive");
  check_channels(c);
  std::vector<int> agents, trainers;
  for (const auto& [id, roles] : a.roles) {
    if (roles & kAgent) agents.push_back(id);
    if (roles & kTrainer) trainers.push_back(id);
  }
  if (agents.empty()) fail(GMI_ERR_PIPELINE, "no agent GMIs in plan");
  if (trainers.empty()) fail(GMI_ERR_PIPELINE, "no trainer GMIs in plan");
  Router router;
  for (int t : trainers) router.load[t] = 0;

  const double cadence = w.interaction();
  const double channel_bytes[3] = {w.S, w.A, w.W};
  FlowStats st;
  std::vector<Group> groups;

  for (std::size_t ai = 0; ai < agents.size(); ++ai) {
    const int agent = agents[ai];
    const auto direct = colocated_trainer(a, agent);
    const double bw = direct ? m.b1 : m.b2;
    double phase = 0;
    if (c.seed != 0)
      phase = cadence * double((c.seed * 2654435761u + unsigned(ai) * 40503u) % 1024u) / 1024.0;
    double t = phase;
    const long budget = long(std::floor((duration - phase) / cadence));
    long made = 0, gseq = 0;
    std::vector<RecordKey> staged;
    while (made < budget) {
      t += cadence;
      staged.push_back({agent, made});
      ++made;
      if (int(staged.size()) == c.k || made == budget) {
        Group g;
        g.agent = agent;
        g.seq = gseq++;
        g.dst = direct;
        g.recs = staged;
        g.start = t;
        for (double per_rec : channel_bytes) {
          const double payload = per_rec * double(staged.size());
          const double cost = c.overhead + payload / bw;
          t += cost;
          st.busy += cost;
          st.bytes += payload;
        }
        st.units += 3;
        g.arrive = t;
        groups.push_back(std::move(g));
        staged.clear();
      }
    }
    st.produced += made;
  }

  std::sort(groups.begin(), groups.end(), [](const Group& x, const Group& y) {
    return std::tie(x.start, x.agent, x.seq) < std::tie(y.start, y.agent, y.seq);
  });
  for (auto& g : groups) {
    const int dst = g.dst ? *g.dst : router.pick();
    router.load.at(dst) += long(g.recs.size());
    g.dst = dst;
  }
  st.per_trainer = router.load;

  std::sort(groups.begin(), groups.end(), [](const Group& x, const Group& y) {
    return std::tie(x.arrive, x.agent, x.seq) < std::tie(y.arrive, y.agent, y.seq);
  });
  std::map<int, Batcher> batchers;
  std::map<int, double> last;
  for (const auto& g : groups) {
    const int dst = *g.dst;
    st.delivery_span = std::max(st.delivery_span, g.arrive);
    last[dst] = g.arrive;
    auto it = batchers.try_emplace(dst, Batcher{c.mode, c.target, {}}).first;
    it->second.feed(dst, g.recs, g.arrive, st.out);
  }
  for (auto& [tr, b] : batchers)
    if (!b.pending.empty()) {
      st.out.push_back({tr, last[tr], std::move(b.pending)});
      b.pending.clear();
    }

  const double per_rec = w.trainer.t_iter / double(c.target);
  std::stable_sort(st.out.begin(), st.out.end(), [](const Batch& x, const Batch& y) {
    return std::tie(x.emit, x.trainer) < std::tie(y.emit, y.trainer);
  });
  std::map<int, double> done;
  for (const auto& b : st.out) {
    double& d = done[b.trainer];
    d = std::max(d, b.emit) + double(b.recs.size()) * per_rec;
    st.training_span = std::max(st.training_span, d);
    st.delivered += long(b.recs.size());
  }
  st.batches = long(st.out.size());
  if (st.delivery_span > 0) st.pps = double(st.produced) / st.delivery_span;
  if (st.training_span > 0) st.ttop = double(st.delivered) / st.training_span;
  return st;
}

}  // namespace gmi::plan
