// Device experience channels (K9): the reference's channel pipeline
// (channels.hpp:110-391 -- dispense -> compress(k) -> migrate (direct / LeastLoadRouter) ->
// Batcher -> trainers) executed on the GPU over real experience payloads.
//
// Every agent GMI owns three channel buffers in device memory (state S, action A, reward W bytes
// per record, [records][bytes]); its records are produced at the serving cadence T_s + T_a.
//   dispense + compress(k): a group of k consecutive records of an agent forms one transfer
//     unit per channel -- a contiguous k-record slice of that channel buffer (zero-copy: the
//     dispenser's per-channel queues ARE the channel buffers);
//   schedule: one thread per agent replays the reference's timing model (each record advances
//     the agent clock by the cadence, each of the group's three sends costs o + bytes / bw with
//     bw = b1 to a colocated trainer else b2, channels.hpp:299-341) in fp64 with the host's
//     operation order, so send / arrival times are bit-identical to simulate_pipeline;
//   migrate: groups in send order (stable radix sort on the send time over (agent, seq) order)
//     go to the colocated trainer or the least-loaded one (lowest id on ties, :139-156, 345-354);
//   deliver + batch: groups in arrival order land in their trainer's receive buffers (a bulk
//     copy per group and channel, the migrator's data movement) at the trainer's running
//     offset; the Batcher (stack / slice, :196-234) cuts the delivered stream into training
//     batches, each a contiguous range of the receive buffer; tails flush per trainer;
//   training model: batches in (emit, trainer) order are consumed at target_batch records per
//     T_t (:373-385) -> PPS / TTOP exactly as simulate_pipeline computes them.
// The data plane (payload copies) is parallel; the decision chain (clocks, routing, batching)
// is inherently sequential in the reference and runs in single device threads over the sorted
// group arrays.
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "../host/errors.hpp"
#include "../host/planner.hpp"

namespace gmi::plan {

namespace {

struct DevGroup {
  double start, arrive;
  double cost[3];  // per-channel transfer cost (o + bytes / bw)
  int agent;       // agent index (plan order)
  int dst;         // trainer index
  long seq;        // group sequence number of the agent
  long rec0;       // first record (agent-local) of the group
  int count;       // records in the group
  long off;        // delivery offset in the trainer's receive buffers
};

struct DevAgent {
  int direct;  // colocated trainer index, -1 if none
  long budget;
  long groups0;  // first group index of this agent
  double phase;
};

struct DevBatch {
  int trainer;
  double emit;
  long off;
  long count;
};

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// One thread per agent: the agent's record clock and group send / arrival times.
__global__ void schedule_kernel(DevAgent* agents, int nagents, DevGroup* groups, double cadence, int k,
                                double overhead, double b1, double b2, double S, double A, double W) {
  const int ai = blockIdx.x * blockDim.x + threadIdx.x;
  if (ai >= nagents) return;
  const DevAgent ag = agents[ai];
  const double bw = ag.direct >= 0 ? b1 : b2;
  const double bytes[3] = {S, A, W};
  double t = ag.phase;
  long made = 0, g = 0;
  int staged = 0;
  while (made < ag.budget) {
    t = dadd(t, cadence);
    ++staged;
    ++made;
    if (staged == k || made == ag.budget) {
      DevGroup& gr = groups[ag.groups0 + g];
      gr.agent = ai;
      gr.seq = g;
      gr.rec0 = made - staged;
      gr.count = staged;
      gr.start = t;
      gr.dst = ag.direct;
      for (int c = 0; c < 3; ++c) {
        const double payload = __dmul_rn(bytes[c], double(staged));
        const double cost = dadd(overhead, __ddiv_rn(payload, bw));
        t = dadd(t, cost);
        gr.cost[c] = cost;
      }
      gr.arrive = t;
      ++g;
      staged = 0;
    }
  }
}

// Send-order keys / arrival-order keys: non-negative doubles sort as their bit patterns.
__global__ void keys_kernel(const DevGroup* groups, long n, int which, unsigned long long* keys, int* idx) {
  const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = __double_as_longlong(which == 0 ? groups[i].start : groups[i].arrive);
  idx[i] = int(i);
}

// LeastLoadRouter over the groups in send order (single thread: the decision chain is sequential).
__global__ void route_kernel(DevGroup* groups, const int* order, long n, long* load, int ntrainers) {
  for (long j = 0; j < n; ++j) {
    DevGroup& g = groups[order[j]];
    int dst = g.dst;
    if (dst < 0) {
      dst = 0;
      for (int t = 1; t < ntrainers; ++t)
        if (load[t] < load[dst]) dst = t;
    }
    load[dst] += g.count;
    g.dst = dst;
  }
}

// Delivery in arrival order + Batcher; tails flushed per trainer in id order.
__global__ void deliver_kernel(DevGroup* groups, const int* order, long n, int ntrainers, int mode_stack,
                               int target, long* off, long* pending, double* last, DevBatch* batches,
                               long* nbatches, double* delivery_span) {
  long nb = 0;
  double span = 0.0;
  for (long j = 0; j < n; ++j) {
    DevGroup& g = groups[order[j]];
    const int t = g.dst;
    span = fmax(span, g.arrive);
    last[t] = g.arrive;
    g.off = off[t];
    off[t] += g.count;
    if (!mode_stack) {
      for (long i = 0; i < g.count; i += target) {
        const long c = min((long)target, g.count - i);
        batches[nb++] = {t, g.arrive, g.off + i, c};
      }
    } else {
      pending[t] += g.count;
      if (pending[t] >= target) {
        batches[nb++] = {t, g.arrive, off[t] - pending[t], pending[t]};
        pending[t] = 0;
      }
    }
  }
  for (int t = 0; t < ntrainers; ++t)
    if (pending[t] > 0) batches[nb++] = {t, last[t], off[t] - pending[t], pending[t]};
  *nbatches = nb;
  *delivery_span = span;
}

// The migrator's data movement: one CTA per (group, channel) copies the unit's records into the
// destination trainer's receive buffer at the group's delivery offset, and records the keys.
__global__ void __launch_bounds__(256) copy_kernel(const DevGroup* groups, const char* const* agent_buf,
                                                   char* const* trainer_buf, int nagents, int ntrainers,
                                                   int bytes_s, int bytes_a, int bytes_w, int* key_agent,
                                                   long* key_seq, long key_stride) {
  const DevGroup g = groups[blockIdx.x];
  const int c = blockIdx.y;
  const int rb = c == 0 ? bytes_s : c == 1 ? bytes_a : bytes_w;
  const char* src = agent_buf[c * nagents + g.agent] + g.rec0 * rb;
  char* dst = trainer_buf[c * ntrainers + g.dst] + g.off * rb;
  const long n = (long)g.count * rb;
  if (rb % 16 == 0) {  // the unit is one contiguous slice: 16-byte moves
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (long i = threadIdx.x; i < n / 16; i += blockDim.x) d4[i] = __ldg(s4 + i);
  } else if (rb % 4 == 0) {
    const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src);
    uint32_t* d4 = reinterpret_cast<uint32_t*>(dst);
    for (long i = threadIdx.x; i < n / 4; i += blockDim.x) d4[i] = __ldg(s4 + i);
  } else {
    for (long i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  }
  if (c == 0)
    for (int r = threadIdx.x; r < g.count; r += blockDim.x) {
      key_agent[g.dst * key_stride + g.off + r] = g.agent;
      key_seq[g.dst * key_stride + g.off + r] = g.rec0 + r;
    }
}

// Training-time model over batches sorted by (emit, trainer) (stable).
__global__ void train_model_kernel(const DevBatch* batches, const int* order, long nb, int ntrainers,
                                   double per_rec, double* done, double* training_span, long* delivered) {
  double span = 0.0;
  long del = 0;
  for (long j = 0; j < nb; ++j) {
    const DevBatch& b = batches[order[j]];
    double& d = done[b.trainer];
    d = dadd(fmax(d, b.emit), __dmul_rn(double(b.count), per_rec));
    span = fmax(span, d);
    del += b.count;
  }
  *training_span = span;
  *delivered = del;
}

__global__ void batch_keys_kernel(const DevBatch* b, long n, int pass, unsigned long long* keys, int* idx,
                                  const int* prev) {
  const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int src = pass == 0 ? int(i) : prev[i];
  keys[i] = pass == 0 ? (unsigned long long)b[src].trainer : (unsigned long long)__double_as_longlong(b[src].emit);
  idx[i] = src;
}

template <class T>
T* dalloc(std::vector<void*>& owned, size_t n) {
  void* p = nullptr;
  GMI_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  GMI_CUDA_CHECK(cudaMemset(p, 0, std::max<size_t>(n, 1) * sizeof(T)));
  owned.push_back(p);
  return static_cast<T*>(p);
}

// Stable radix sort of (key, index) pairs; returns the sorted index array (device).
int* sort_pairs(std::vector<void*>& owned, unsigned long long* keys, int* idx, long n, cudaStream_t s) {
  unsigned long long* ko = dalloc<unsigned long long>(owned, n);
  int* io = dalloc<int>(owned, n);
  size_t tmp = 0;
  GMI_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, ko, idx, io, int(n), 0, 64, s));
  void* t = dalloc<char>(owned, tmp);
  GMI_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(t, tmp, keys, ko, idx, io, int(n), 0, 64, s));
  return io;
}

}  // namespace

FlowStats run_channels_device(const Workload& w, const Assignment& a, const Machine& m, const ChannelConfig& c,
                              double duration, const std::vector<const void*>& agent_buf,
                              const std::vector<void*>& trainer_buf, long trainer_capacity, void* stream,
                              std::vector<int>* key_agent_out, std::vector<long>* key_seq_out) {
  if (duration <= 0) invalid("duration must be positive");
  check_channels(c);
  std::vector<int> agents, trainers;
  for (const auto& [id, roles] : a.roles) {
    if (roles & kAgent) agents.push_back(id);
    if (roles & kTrainer) trainers.push_back(id);
  }
  if (agents.empty()) fail(GMI_ERR_PIPELINE, "no agent GMIs in plan");
  if (trainers.empty()) fail(GMI_ERR_PIPELINE, "no trainer GMIs in plan");
  const int na = int(agents.size()), nt = int(trainers.size());
  if (int(agent_buf.size()) != 3 * na || int(trainer_buf.size()) != 3 * nt)
    invalid("channel buffers: 3 per agent (state, action, reward) and 3 per trainer");
  const double bytes[3] = {w.S, w.A, w.W};
  for (double b : bytes)
    if (b <= 0 || b != std::floor(b)) invalid("channel record sizes must be whole positive byte counts");
  auto gpu_of = [&](int gmi) {
    for (const auto& [g, ids] : a.per_gpu)
      if (std::find(ids.begin(), ids.end(), gmi) != ids.end()) return g;
    fail(GMI_ERR_PIPELINE, "gmi " + std::to_string(gmi) + " not in plan");
  };
  const double cadence = w.interaction();
  std::vector<DevAgent> ag(na);
  long ngroups = 0, produced = 0;
  for (int i = 0; i < na; ++i) {
    const int gpu = gpu_of(agents[i]);
    int direct = -1;  // colocated trainer, lowest id (channels.hpp:168-176)
    for (int id : a.per_gpu.at(gpu))
      if ((a.roles.at(id) & kTrainer) && (direct < 0 || id < trainers[direct]))
        direct = int(std::find(trainers.begin(), trainers.end(), id) - trainers.begin());
    double phase = 0;
    if (c.seed != 0) phase = cadence * double((c.seed * 2654435761u + unsigned(i) * 40503u) % 1024u) / 1024.0;
    const long budget = long(std::floor((duration - phase) / cadence));
    ag[i] = {direct, std::max(0L, budget), ngroups, phase};
    ngroups += (ag[i].budget + c.k - 1) / c.k;
    produced += ag[i].budget;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<void*> owned;
  FlowStats st;
  try {
    DevAgent* d_ag = dalloc<DevAgent>(owned, na);
    DevGroup* d_gr = dalloc<DevGroup>(owned, ngroups);
    GMI_CUDA_CHECK(cudaMemcpyAsync(d_ag, ag.data(), na * sizeof(DevAgent), cudaMemcpyHostToDevice, s));
    schedule_kernel<<<(na + 127) / 128, 128, 0, s>>>(d_ag, na, d_gr, cadence, c.k, c.overhead, m.b1, m.b2, w.S, w.A,
                                                     w.W);
    GMI_CUDA_CHECK(cudaGetLastError());
    const int blk = int((ngroups + 255) / 256);
    unsigned long long* keys = dalloc<unsigned long long>(owned, ngroups);
    int* idx = dalloc<int>(owned, ngroups);
    long* load = dalloc<long>(owned, nt);
    if (ngroups > 0) {
      keys_kernel<<<blk, 256, 0, s>>>(d_gr, ngroups, 0, keys, idx);
      int* send_order = sort_pairs(owned, keys, idx, ngroups, s);
      route_kernel<<<1, 1, 0, s>>>(d_gr, send_order, ngroups, load, nt);
      keys_kernel<<<blk, 256, 0, s>>>(d_gr, ngroups, 1, keys, idx);
    }
    int* arrive_order = ngroups > 0 ? sort_pairs(owned, keys, idx, ngroups, s) : idx;
    long* off = dalloc<long>(owned, nt);
    long* pending = dalloc<long>(owned, nt);
    double* last = dalloc<double>(owned, nt);
    const long max_batches = ngroups * (c.mode == BatchKind::Slice ? (c.k + c.target - 1) / c.target : 1) + nt;
    DevBatch* d_b = dalloc<DevBatch>(owned, max_batches);
    long* scal = dalloc<long>(owned, 4);
    double* dscal = dalloc<double>(owned, 4);
    deliver_kernel<<<1, 1, 0, s>>>(d_gr, arrive_order, ngroups, nt, c.mode == BatchKind::Stack ? 1 : 0, c.target, off,
                                   pending, last, d_b, scal, dscal);
    // data plane
    std::vector<long> loads(nt);
    GMI_CUDA_CHECK(cudaMemcpyAsync(loads.data(), load, nt * sizeof(long), cudaMemcpyDeviceToHost, s));
    GMI_CUDA_CHECK(cudaStreamSynchronize(s));
    for (long l : loads)
      if (l > trainer_capacity) invalid("trainer receive buffers too small for the routed records");
    const char** d_abuf = dalloc<const char*>(owned, 3 * na);
    char** d_tbuf = dalloc<char*>(owned, 3 * nt);
    GMI_CUDA_CHECK(cudaMemcpyAsync(d_abuf, agent_buf.data(), 3 * na * sizeof(void*), cudaMemcpyHostToDevice, s));
    GMI_CUDA_CHECK(cudaMemcpyAsync(d_tbuf, trainer_buf.data(), 3 * nt * sizeof(void*), cudaMemcpyHostToDevice, s));
    int* kag = dalloc<int>(owned, (size_t)nt * std::max(1L, trainer_capacity));
    long* kseq = dalloc<long>(owned, (size_t)nt * std::max(1L, trainer_capacity));
    if (ngroups > 0)
      copy_kernel<<<dim3(unsigned(ngroups), 3), 256, 0, s>>>(d_gr, d_abuf, d_tbuf, na, nt, int(w.S), int(w.A),
                                                             int(w.W), kag, kseq, trainer_capacity);
    GMI_CUDA_CHECK(cudaGetLastError());
    // training-time model over batches in (emit, trainer) order
    long nb = 0;
    GMI_CUDA_CHECK(cudaMemcpyAsync(&nb, scal, sizeof(long), cudaMemcpyDeviceToHost, s));
    GMI_CUDA_CHECK(cudaStreamSynchronize(s));
    double* done = dalloc<double>(owned, nt);
    const double per_rec = w.trainer.t_iter / double(c.target);
    int* border = nullptr;
    if (nb > 0) {
      unsigned long long* bk = dalloc<unsigned long long>(owned, nb);
      int* bi = dalloc<int>(owned, nb);
      batch_keys_kernel<<<int((nb + 255) / 256), 256, 0, s>>>(d_b, nb, 0, bk, bi, nullptr);
      int* by_trainer = sort_pairs(owned, bk, bi, nb, s);
      batch_keys_kernel<<<int((nb + 255) / 256), 256, 0, s>>>(d_b, nb, 1, bk, bi, by_trainer);
      border = sort_pairs(owned, bk, bi, nb, s);
      train_model_kernel<<<1, 1, 0, s>>>(d_b, border, nb, nt, per_rec, done, dscal + 1, scal + 1);
    }
    // results back to the host (FlowStats, the pipeline-handle format)
    std::vector<DevGroup> hg(ngroups);
    std::vector<DevBatch> hb(nb);
    std::vector<int> ho(nb);
    long hscal[4] = {};
    double hd[4] = {};
    GMI_CUDA_CHECK(cudaMemcpyAsync(hg.data(), d_gr, ngroups * sizeof(DevGroup), cudaMemcpyDeviceToHost, s));
    if (nb > 0) {
      GMI_CUDA_CHECK(cudaMemcpyAsync(hb.data(), d_b, nb * sizeof(DevBatch), cudaMemcpyDeviceToHost, s));
      GMI_CUDA_CHECK(cudaMemcpyAsync(ho.data(), border, nb * sizeof(int), cudaMemcpyDeviceToHost, s));
    }
    GMI_CUDA_CHECK(cudaMemcpyAsync(hscal, scal, sizeof(hscal), cudaMemcpyDeviceToHost, s));
    GMI_CUDA_CHECK(cudaMemcpyAsync(hd, dscal, sizeof(hd), cudaMemcpyDeviceToHost, s));
    std::vector<int> ka((size_t)nt * std::max(1L, trainer_capacity));
    std::vector<long> ks(ka.size());
    GMI_CUDA_CHECK(cudaMemcpyAsync(ka.data(), kag, ka.size() * sizeof(int), cudaMemcpyDeviceToHost, s));
    GMI_CUDA_CHECK(cudaMemcpyAsync(ks.data(), kseq, ks.size() * sizeof(long), cudaMemcpyDeviceToHost, s));
    GMI_CUDA_CHECK(cudaStreamSynchronize(s));
    // accounting sums in the host model's order (agent-major, group, channel)
    for (const auto& g : hg)
      for (int ch = 0; ch < 3; ++ch) {
        st.busy += g.cost[ch];
        st.bytes += bytes[ch] * double(g.count);
      }
    st.produced = produced;
    st.units = 3 * ngroups;
    st.delivery_span = hd[0];
    st.training_span = hd[1];
    st.delivered = hscal[1];
    for (int t = 0; t < nt; ++t) st.per_trainer[trainers[t]] = loads[t];
    for (long j = 0; j < nb; ++j) {
      const DevBatch& b = hb[ho[j]];
      Batch out{trainers[b.trainer], b.emit, {}};
      for (long r = 0; r < b.count; ++r) {
        const size_t k = (size_t)b.trainer * trainer_capacity + b.off + r;
        out.recs.push_back({agents[ka[k]], ks[k]});
      }
      st.out.push_back(std::move(out));
    }
    st.batches = nb;
    if (st.delivery_span > 0) st.pps = double(st.produced) / st.delivery_span;
    if (st.training_span > 0) st.ttop = double(st.delivered) / st.training_span;
    if (key_agent_out) {
      key_agent_out->resize(ka.size());
      for (size_t i = 0; i < ka.size(); ++i) (*key_agent_out)[i] = ka[i] >= 0 ? agents[ka[i]] : -1;
    }
    if (key_seq_out) *key_seq_out = ks;
  } catch (...) {
    for (void* p : owned) cudaFree(p);
    throw;
  }
  for (void* p : owned) cudaFree(p);
  return st;
}

}  // namespace gmi::plan
