// TEST INFRASTRUCTURE ONLY — times the reference's own execute() (reduction.hpp:225-334,
// single-threaded C++ as shipped) on the BASELINE layouts at the real gradient lengths.
// Compiled in place against /root/reference by oracle/Makefile; bench.py's cpu_baseline leg
// (reduction_vs_reference) times it beside K1 on the same layouts. One JSON object per line.
#include <chrono>
#include <cstdio>
#include <string>
#include <vector>

#include "gmux/reduction.hpp"

using namespace gmux;

int main(int argc, char** argv) {
  struct Case {
    const char* name;
    Strategy s;
    int g, t;
    std::size_t len;
  };
  const std::vector<Case> cases = {
      {"AT-1x4", Strategy::MPR, 1, 4, 114121},       {"AT3x256-1x1", Strategy::MPR, 1, 1, 296713},
      {"HM-1x4", Strategy::MPR, 1, 4, 286822},       {"HM-2x4", Strategy::HAR, 2, 4, 286822},
      {"HM-8x4", Strategy::MRR, 8, 4, 286822},       {"SH-2x7", Strategy::HAR, 2, 7, 1535765},
      {"SH-8x4", Strategy::MRR, 8, 4, 1535765},      {"SH-8x7", Strategy::MRR, 8, 7, 1535765},
  };
  const int reps = argc > 1 ? std::stoi(argv[1]) : 3;
  const Topology topo = default_topology(8);
  for (const auto& c : cases) {
    GmiLayout lay;
    int id = 0;
    for (int i = 0; i < c.g; ++i) {
      lay.mpl.emplace_back();
      for (int j = 0; j < c.t; ++j) lay.mpl.back().push_back(id++);
    }
    std::vector<GradientBuffer> bufs;
    for (int i : lay.all_gmis()) {
      GradientBuffer b{i, std::vector<double>(c.len)};
      for (std::size_t e = 0; e < c.len; ++e) b.values[e] = 1.0 + 0.001 * i + 1e-6 * double(e);
      bufs.push_back(std::move(b));
    }
    double best = 1e30;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      const ReductionRun run = execute(c.s, lay, bufs, topo);
      const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (dt < best) best = dt;
      if (run.result.size() != c.len) return 1;
    }
    const double in_bytes = double(c.len) * 8.0 * c.g * c.t;
    std::printf("{\"case\":\"%s\",\"strategy\":\"%s\",\"g\":%d,\"t\":%d,\"len\":%zu,\"seconds\":%.6f,\"input_GBps\":%.4f}\n",
                c.name, to_string(c.s).c_str(), c.g, c.t, c.len, best, in_bytes / best / 1e9);
  }
  return 0;
}
