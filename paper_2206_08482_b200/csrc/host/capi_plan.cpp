// extern "C" surface of the planner (include/gmi.h): flattening/unflattening of the
// planner types and exception -> error-code translation.
#include <cmath>
#include <cstring>
#include <exception>
#include <fstream>
#include <memory>
#include <sstream>

#include "errors.hpp"
#include "planner.hpp"

using namespace gmi;
using namespace gmi::plan;

namespace {

Placement to_placement(int num_gpus, const int* counts, const int* ids) {
  if (num_gpus < 0) invalid("num_gpus must be >= 0");
  Placement p;
  p.per_gpu.resize(num_gpus);
  int k = 0;
  for (int g = 0; g < num_gpus; ++g) {
    if (counts[g] < 0) invalid("negative GMI count");
    p.per_gpu[g].assign(ids + k, ids + k + counts[g]);
    k += counts[g];
  }
  return p;
}

Algo to_algo(int s) {
  if (s < 0 || s > 2) invalid("unknown strategy");
  return Algo(s);
}

Tpl to_tpl(int t) {
  if (t < 0 || t > 4) invalid("unknown template kind");
  return Tpl(t);
}

Machine to_machine(const gmi_topology_t* t) {
  if (!t) invalid("null topology");
  Machine m;
  m.b1 = t->b1;
  m.b2 = t->b2;
  for (int i = 0; i < t->num_gpus; ++i) {
    const gmi_gpu_t& g = t->gpus[i];
    if (g.arch != 70 && g.arch != 80 && g.arch != 100) invalid("unknown GPU architecture");
    m.gpus.push_back({g.id, Arch(g.arch), g.sm_units, g.mem_gb});
  }
  for (int i = 0; i < t->num_parts; ++i) {
    const gmi_partition_t& p = t->parts[i];
    m.parts.push_back({p.gmi_id, p.gpu_id, p.backend == 1 ? Backend::MIG : Backend::MPS, p.sm_share, p.mem_gb});
  }
  return m;
}

Workload to_workload(const gmi_workload_t* w) {
  if (!w) invalid("null workload");
  Workload o;
  o.name = std::string(w->name, strnlen(w->name, sizeof(w->name)));
  o.S = w->state_bytes;
  o.A = w->action_bytes;
  o.W = w->reward_bytes;
  o.Mp = w->model_bytes;
  o.m = w->steps_per_train;
  o.alpha = w->alpha;
  o.beta = w->beta;
  if (w->num_dims < 0 || w->num_dims > GMI_MAX_DIMS) invalid("num_dims out of range");
  o.dims.assign(w->policy_dims, w->policy_dims + w->num_dims);
  o.sim = {w->simulator.r_sm, w->simulator.r_mem, w->simulator.t_iter};
  o.agent = {w->agent.r_sm, w->agent.r_mem, w->agent.t_iter};
  o.trainer = {w->trainer.r_sm, w->trainer.r_mem, w->trainer.t_iter};
  return o;
}

void from_workload(const Workload& w, gmi_workload_t* o) {
  std::memset(o, 0, sizeof(*o));
  std::strncpy(o->name, w.name.c_str(), sizeof(o->name) - 1);
  o->state_bytes = w.S;
  o->action_bytes = w.A;
  o->reward_bytes = w.W;
  o->model_bytes = w.Mp;
  o->steps_per_train = w.m;
  o->alpha = w.alpha;
  o->beta = w.beta;
  if (w.dims.size() > GMI_MAX_DIMS) invalid("too many policy dims");
  o->num_dims = int(w.dims.size());
  for (std::size_t i = 0; i < w.dims.size(); ++i) o->policy_dims[i] = w.dims[i];
  o->simulator = {w.sim.r_sm, w.sim.r_mem, w.sim.t_iter};
  o->agent = {w.agent.r_sm, w.agent.r_mem, w.agent.t_iter};
  o->trainer = {w.trainer.r_sm, w.trainer.r_mem, w.trainer.t_iter};
}

Projection to_projection(const gmi_estimator_t* e) {
  if (!e) invalid("null estimator");
  return Projection{to_workload(&e->workload), e->b1, e->b2, e->latency_scale};
}

SearchGrid to_grid(const gmi_search_config_t* c) {
  SearchGrid g;
  if (!c) return g;
  g.envs.assign(c->num_env_grid, c->num_env_grid + (c->grid_len > 0 ? c->grid_len : 0));
  g.max_gpg = c->max_gmis_per_gpu;
  g.sat = c->sat_threshold;
  return g;
}

SyntheticProbe to_synth(const gmi_synthetic_model_t* m) {
  SyntheticProbe s;
  if (!m) return s;
  s.peak_top = m->peak_top;
  s.mem_base = m->mem_base;
  s.mem_per_env = m->mem_per_env;
  s.mem_capacity = m->mem_capacity;
  s.min_share = m->min_runnable_share;
  s.knee_base = m->knee_base;
  for (int i = 0; i < m->num_knee; ++i) s.knee_override[m->knee_keys[i]] = m->knee_values[i];
  for (int i = 0; i < m->num_cap; ++i) s.cap_scale[m->cap_keys[i]] = m->cap_values[i];
  return s;
}

ChannelConfig to_channels(const gmi_pipeline_config_t* c) {
  ChannelConfig o;
  if (!c) return o;
  o.k = c->compress_threshold;
  o.mode = c->batch_mode == 0 ? BatchKind::Slice : BatchKind::Stack;
  o.target = c->target_batch;
  o.overhead = c->per_message_overhead;
  o.seed = c->seed;
  return o;
}

void from_channels(const ChannelConfig& c, gmi_pipeline_config_t* o) {
  o->compress_threshold = c.k;
  o->batch_mode = c.mode == BatchKind::Slice ? 0 : 1;
  o->target_batch = c.target;
  o->per_message_overhead = c.overhead;
  o->seed = c.seed;
}

void fill_probe(const Probe& p, int* runnable, double* top, double* mem) {
  *runnable = p.runnable ? 1 : 0;
  *top = p.top;
  *mem = p.mem;
}

}  // namespace

extern "C" {

// ------------------------------------------------------------------ layouts
GMI_API int gmi_select_strategy(int num_gpus, const int* counts, const int* ids, int* strategy) {
  return guarded([&] { *strategy = int(choose_algo(to_placement(num_gpus, counts, ids))); });
}

GMI_API int gmi_leader_gmis(int num_gpus, const int* counts, const int* ids, int* leaders) {
  return guarded([&] {
    const auto l = gpu_leaders(to_placement(num_gpus, counts, ids));
    std::copy(l.begin(), l.end(), leaders);
  });
}

GMI_API int gmi_mrr_rings(int num_gpus, const int* counts, const int* ids, int* rings, int* num_rings) {
  return guarded([&] {
    const auto r = disjoint_rings(to_placement(num_gpus, counts, ids));
    *num_rings = int(r.size());
    int k = 0;
    for (const auto& ring : r)
      for (int id : ring) rings[k++] = id;
  });
}

GMI_API int gmi_predict_latency(int strategy, int g, int t, double m_p, double b1, double b2, double* latency) {
  return guarded([&] { *latency = closed_form_latency(to_algo(strategy), g, t, m_p, b1, b2); });
}

GMI_API int gmi_reduction_schedule(int strategy, int num_gpus, const int* counts, const int* ids, size_t len,
                                   double elem_bytes, double b1, double b2, gmi_trace_event_t* trace,
                                   size_t trace_cap, gmi_reduction_info_t* info) {
  return guarded([&] {
    const Schedule s = build_schedule(to_algo(strategy), to_placement(num_gpus, counts, ids), len,
                                      elem_bytes, b1, b2);
    info->strategy = int(s.algo);
    info->result_holder = s.result_holder;
    info->latency = s.latency;
    info->broadcast_latency = s.broadcast_latency;
    info->trace_len = s.hops.size();
    if (trace) {
      if (trace_cap < s.hops.size()) invalid("trace buffer too small");
      for (std::size_t i = 0; i < s.hops.size(); ++i) {
        const Hop& h = s.hops[i];
        trace[i] = {h.step, h.src, h.dst, int(h.link), h.bytes};
      }
    }
  });
}

// ------------------------------------------------------------------ topology
GMI_API int gmi_validate_layout(const gmi_topology_t* topo, gmi_violation_t* out, int cap, int* count) {
  return guarded([&] {
    const auto v = check_machine(to_machine(topo));
    *count = int(v.size());
    for (int i = 0; i < int(v.size()) && i < cap; ++i) {
      out[i].gpu_id = v[i].first;
      std::strncpy(out[i].rule, v[i].second.c_str(), sizeof(out[i].rule) - 1);
      out[i].rule[sizeof(out[i].rule) - 1] = 0;
    }
  });
}

GMI_API int gmi_select_backend(int arch, int training, int* backend) {
  return guarded([&] {
    if (arch != 70 && arch != 80 && arch != 100) invalid("unsupported GPU architecture");
    *backend = int(backend_for(Arch(arch), training != 0));
  });
}

GMI_API int gmi_path_bandwidth(const gmi_topology_t* topo, int src, int dst, int* kind, double* bw) {
  return guarded([&] { *kind = int(link_between(to_machine(topo), src, dst, bw)); });
}

// ------------------------------------------------------------------ workload
GMI_API int gmi_load_benchmark(const char* name, gmi_workload_t* out) {
  return guarded([&] { from_workload(catalog(name ? name : ""), out); });
}

GMI_API int gmi_green_sms(double share, int sm_units, int* out) {
  return guarded([&] {
    if (!out) invalid("null argument");
    if (!(share > 0 && share <= 1.0)) invalid("share outside (0, 1]");
    plan::Gpu g;
    g.arch = plan::Arch::SM100;
    g.sm_units = sm_units;
    *out = plan::green_sms(share, g);
  });
}

GMI_API int gmi_validate_workload(const gmi_workload_t* w) {
  return guarded([&] { check_workload(to_workload(w)); });
}

GMI_API int gmi_dense_param_count(const int* dims, int n, size_t* out) {
  return guarded([&] { *out = mlp_params(std::vector<int>(dims, dims + (n > 0 ? n : 0))); });
}

GMI_API int gmi_policy_value_param_count(const int* dims, int n, size_t* out) {
  return guarded([&] { *out = actor_critic_params(std::vector<int>(dims, dims + (n > 0 ? n : 0))); });
}

// ------------------------------------------------------------------ placement + costs
GMI_API int gmi_serving_cost(int tpl, const gmi_workload_t* w, double* resource, double* comm) {
  return guarded([&] {
    const Cost c = serving_cost(to_tpl(tpl), to_workload(w));
    *resource = c.resource;
    *comm = c.comm;
  });
}

GMI_API int gmi_training_cost(int tpl, const gmi_workload_t* w, int n, double* resource, double* comm) {
  return guarded([&] {
    const Cost c = training_cost(to_tpl(tpl), to_workload(w), n);
    *resource = c.resource;
    *comm = c.comm;
  });
}

GMI_API int gmi_allreduce_bytes(int n, double model_bytes, double* out) {
  return guarded([&] { *out = allreduce_volume(n, model_bytes); });
}

GMI_API int gmi_throughput(int training, double resource, double comm, const gmi_workload_t* w, double r_all,
                           double bw, double* out) {
  return guarded([&] {
    const Cost c{resource, comm};
    *out = training ? training_rate(c, to_workload(w), r_all, bw) : serving_rate(c, to_workload(w), r_all, bw);
  });
}

GMI_API int gmi_throughput_ratio(int training, const gmi_workload_t* w, double factor, double* out) {
  return guarded([&] { *out = training ? training_gain(to_workload(w), factor) : serving_gain(to_workload(w), factor); });
}

GMI_API int gmi_colocation_penalty(int training, const gmi_workload_t* w, double* out) {
  return guarded([&] { *out = training ? training_penalty(to_workload(w)) : serving_penalty(to_workload(w)); });
}

GMI_API int gmi_build_plan(int tpl, const gmi_topology_t* topo, int gpg, int* gpu_ids, int* gmi_ids,
                           int* role_masks, int* serving) {
  return guarded([&] {
    const Assignment a = assign(to_tpl(tpl), to_machine(topo), gpg);
    int gi = 0, k = 0;
    for (const auto& [gpu, ids] : a.per_gpu) {
      gpu_ids[gi] = gpu;
      const bool srv = std::find(a.serving.begin(), a.serving.end(), gpu) != a.serving.end();
      serving[gi] = a.tpl == Tpl::Async ? (srv ? 1 : 0) : -1;
      ++gi;
      for (int id : ids) gmi_ids[k++] = id;
    }
    for (const auto& [id, mask] : a.roles) role_masks[id] = mask;
  });
}

// ------------------------------------------------------------------ adaptive GMI manager
GMI_API int gmi_saturation(double top, double pre_top, double mem, double pre_mem, double* out) {
  return guarded([&] { *out = saturation_ratio(top, pre_top, mem, pre_mem); });
}

GMI_API int gmi_comm_discount(const gmi_estimator_t* est, int gpg, int num_gpu, double* out) {
  return guarded([&] { *out = to_projection(est).discount(gpg, num_gpu); });
}

GMI_API int gmi_estimate(const gmi_estimator_t* est, int gpg, int num_gpu, double top, double* out) {
  return guarded([&] { *out = to_projection(est).project(gpg, num_gpu, top); });
}

GMI_API int gmi_explore(gmi_probe_fn probe, void* user, const gmi_estimator_t* est, const char* bench,
                        int num_gpu, const gmi_search_config_t* cfg, gmi_search_result_t* out,
                        gmi_visit_t* visits, size_t cap) {
  return guarded([&] {
    if (!probe) invalid("null probe");
    ProbeFn fn = [&](const std::string& b, int gpg, int env) {
      int ok = 0;
      double top = 0, mem = 0;
      const int rc = probe(user, b.c_str(), gpg, env, &ok, &top, &mem);
      if (rc != GMI_OK) fail(rc, "profiler failed at gmis_per_gpu=" + std::to_string(gpg) + " num_env=" + std::to_string(env));
      return Probe{ok != 0, top, mem};
    };
    const SearchOutcome r = search(fn, to_projection(est), bench ? bench : "", num_gpu, to_grid(cfg));
    out->feasible = r.feasible ? 1 : 0;
    std::memset(out->reason, 0, sizeof(out->reason));
    std::strncpy(out->reason, r.reason.c_str(), sizeof(out->reason) - 1);
    out->num_env = r.env;
    out->gmis_per_gpu = r.gpg;
    out->est_throughput = r.est;
    out->num_visited = r.visits.size();
    if (visits) {
      if (cap < r.visits.size()) invalid("visits buffer too small");
      for (std::size_t i = 0; i < r.visits.size(); ++i) {
        const Visit& v = r.visits[i];
        visits[i] = {v.gpg, v.env, v.runnable ? 1 : 0, v.top, v.mem, v.sat ? 1 : 0, v.sat.value_or(0.0),
                     v.acc ? 1 : 0, v.acc.value_or(0.0), v.pruned ? 1 : 0};
      }
    }
  });
}

GMI_API void gmi_synthetic_model_defaults(gmi_synthetic_model_t* m) {
  const SyntheticProbe d;
  std::memset(m, 0, sizeof(*m));
  m->peak_top = d.peak_top;
  m->mem_base = d.mem_base;
  m->mem_per_env = d.mem_per_env;
  m->mem_capacity = d.mem_capacity;
  m->min_runnable_share = d.min_share;
  m->knee_base = d.knee_base;
}

GMI_API int gmi_synthetic_profile(const gmi_synthetic_model_t* m, const char* bench, int gpg, int env,
                                  int* runnable, double* top, double* mem) {
  return guarded([&] { fill_probe(to_synth(m)(bench ? bench : "", gpg, env), runnable, top, mem); });
}

GMI_API int gmi_trace_profiler_load(const char* path, void** handle) {
  return guarded([&] { *handle = new TableProbe(TableProbe::from_file(path ? path : "")); });
}

GMI_API int gmi_trace_profiler_profile(void* h, const char* bench, int gpg, int env, int* runnable, double* top,
                                       double* mem) {
  return guarded([&] {
    if (!h) invalid("null trace profiler");
    fill_probe((*static_cast<TableProbe*>(h))(bench ? bench : "", gpg, env), runnable, top, mem);
  });
}

GMI_API void gmi_trace_profiler_free(void* h) { delete static_cast<TableProbe*>(h); }

// ------------------------------------------------------------------ experience channels
GMI_API void gmi_pipeline_config_defaults(gmi_pipeline_config_t* c) { from_channels(ChannelConfig{}, c); }

GMI_API int gmi_simulate_pipeline(const gmi_workload_t* w, const gmi_plan_t* plan, const gmi_topology_t* topo,
                                  const gmi_pipeline_config_t* cfg, double duration, void** handle,
                                  gmi_pipeline_metrics_t* out) {
  return guarded([&] {
    if (!plan) invalid("null plan");
    Assignment a;
    a.tpl = to_tpl(plan->template_kind);
    int k = 0;
    for (int g = 0; g < plan->num_gpus; ++g) {
      auto& ids = a.per_gpu[plan->gpu_ids[g]];
      for (int j = 0; j < plan->counts[g]; ++j, ++k) {
        ids.push_back(plan->gmi_ids[k]);
        a.roles[plan->gmi_ids[k]] = plan->role_masks[k];
      }
    }
    auto st = std::make_unique<FlowStats>(run_channels(to_workload(w), a, to_machine(topo), to_channels(cfg), duration));
    *out = {st->pps, st->ttop, st->produced, st->delivered, st->units, st->batches, st->bytes, st->busy,
            st->delivery_span, st->training_span, st->per_trainer.size()};
    if (handle) *handle = st.release();
  });
}

GMI_API int gmi_channel_run(const gmi_workload_t* w, const gmi_plan_t* plan, const gmi_topology_t* topo,
                            const gmi_pipeline_config_t* cfg, double duration, const void* const* agent_bufs,
                            int num_agent_bufs, void* const* trainer_bufs, int num_trainer_bufs,
                            long trainer_capacity, void* stream, void** handle, gmi_pipeline_metrics_t* out) {
  return guarded([&] {
    if (!plan || !agent_bufs || !trainer_bufs || !out) invalid("null argument");
    Assignment a;
    a.tpl = to_tpl(plan->template_kind);
    int k = 0;
    for (int g = 0; g < plan->num_gpus; ++g) {
      auto& ids = a.per_gpu[plan->gpu_ids[g]];
      for (int j = 0; j < plan->counts[g]; ++j, ++k) {
        ids.push_back(plan->gmi_ids[k]);
        a.roles[plan->gmi_ids[k]] = plan->role_masks[k];
      }
    }
    std::vector<const void*> ab(agent_bufs, agent_bufs + num_agent_bufs);
    std::vector<void*> tb(trainer_bufs, trainer_bufs + num_trainer_bufs);
    auto st = std::make_unique<FlowStats>(run_channels_device(to_workload(w), a, to_machine(topo), to_channels(cfg),
                                                              duration, ab, tb, trainer_capacity, stream));
    *out = {st->pps, st->ttop, st->produced, st->delivered, st->units, st->batches, st->bytes, st->busy,
            st->delivery_span, st->training_span, st->per_trainer.size()};
    if (handle) *handle = st.release();
  });
}

GMI_API int gmi_pipeline_trainer_records(void* h, int* trainers, long* records) {
  return guarded([&] {
    int i = 0;
    for (const auto& [t, n] : static_cast<FlowStats*>(h)->per_trainer) {
      trainers[i] = t;
      records[i] = n;
      ++i;
    }
  });
}

GMI_API size_t gmi_pipeline_num_batches(void* h) { return h ? static_cast<FlowStats*>(h)->out.size() : 0; }

GMI_API int gmi_pipeline_batch(void* h, size_t i, int* trainer, double* emit, size_t* n) {
  return guarded([&] {
    const auto& b = static_cast<FlowStats*>(h)->out.at(i);
    *trainer = b.trainer;
    *emit = b.emit;
    *n = b.recs.size();
  });
}

GMI_API int gmi_pipeline_batch_records(void* h, size_t i, int* agents, long* seqs) {
  return guarded([&] {
    const auto& b = static_cast<FlowStats*>(h)->out.at(i);
    for (std::size_t j = 0; j < b.recs.size(); ++j) {
      agents[j] = b.recs[j].agent;
      seqs[j] = b.recs[j].seq;
    }
  });
}

GMI_API void gmi_pipeline_free(void* h) { delete static_cast<FlowStats*>(h); }

// ------------------------------------------------------------------ config schema
GMI_API int gmi_config_parse(const char* text, const char* origin, void** handle) {
  return guarded([&] { *handle = new CfgFile(parse_cfg(text ? text : "", origin ? origin : "<config>")); });
}

GMI_API int gmi_config_load(const char* path, void** handle) {
  return guarded([&] {
    const std::string p = path ? path : "";
    std::ifstream in(p);
    if (!in) fail(GMI_ERR_CONFIG, "config not found: " + p);
    std::stringstream ss;
    ss << in.rdbuf();
    *handle = new CfgFile(parse_cfg(ss.str(), p));
  });
}

GMI_API int gmi_config_has(void* h, const char* section, int* out) {
  return guarded([&] { *out = static_cast<CfgFile*>(h)->has(section ? section : "") ? 1 : 0; });
}

GMI_API int gmi_config_topology(void* h, gmi_gpu_t* gpus, int gcap, int* ng, gmi_partition_t* parts, int pcap,
                                int* np, double* b1, double* b2) {
  return guarded([&] {
    const Machine m = cfg_machine(*static_cast<CfgFile*>(h));
    *ng = int(m.gpus.size());
    *np = int(m.parts.size());
    *b1 = m.b1;
    *b2 = m.b2;
    for (int i = 0; i < *ng && i < gcap; ++i)
      gpus[i] = {m.gpus[i].id, int(m.gpus[i].arch), m.gpus[i].sm_units, m.gpus[i].mem_gb};
    for (int i = 0; i < *np && i < pcap; ++i)
      parts[i] = {m.parts[i].gmi_id, m.parts[i].gpu_id, int(m.parts[i].backend), m.parts[i].sm_share, m.parts[i].mem_gb};
  });
}

GMI_API int gmi_config_workload(void* h, const char* fallback, gmi_workload_t* out) {
  return guarded([&] { from_workload(cfg_workload(*static_cast<CfgFile*>(h), fallback ? fallback : "AT"), out); });
}

GMI_API int gmi_config_model(void* h, gmi_model_params_t* out) {
  return guarded([&] {
    const CfgModel m = cfg_model(*static_cast<CfgFile*>(h));
    out->serving_combw_factor = m.serving_factor;
    out->training_combw_factor = m.training_factor;
    out->gmis_per_gpu = m.gmis_per_gpu;
    out->latency_scale = m.latency_scale;
    from_channels(m.channels, &out->pipeline);
  });
}

GMI_API int gmi_config_search(void* h, gmi_search_settings_t* out) {
  return guarded([&] {
    const CfgSearch s = cfg_search(*static_cast<CfgFile*>(h));
    std::memset(out, 0, sizeof(*out));
    if (s.grid.envs.size() > GMI_MAX_GRID) invalid("num_env grid longer than GMI_MAX_GRID");
    out->grid_len = int(s.grid.envs.size());
    std::copy(s.grid.envs.begin(), s.grid.envs.end(), out->grid);
    out->max_gmis_per_gpu = s.grid.max_gpg;
    out->sat_threshold = s.grid.sat;
    out->has_profile_trace = s.trace ? 1 : 0;
    if (s.trace) std::strncpy(out->profile_trace, s.trace->c_str(), sizeof(out->profile_trace) - 1);
  });
}

GMI_API int gmi_config_get(void* h, const char* section, const char* key, char* value, size_t cap, int* found) {
  return guarded([&] {
    const auto v = static_cast<CfgFile*>(h)->get(section ? section : "", key ? key : "");
    *found = v ? 1 : 0;
    if (v && cap > 0) {
      std::strncpy(value, v->c_str(), cap - 1);
      value[cap - 1] = 0;
    }
  });
}

GMI_API void gmi_config_free(void* h) { delete static_cast<CfgFile*>(h); }

}  // extern "C"
