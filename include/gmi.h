/* gmi.h — C-ABI of libgmi, the B200-native data-parallel PPO iteration with
 * GMI (GPU multiplexing instance) placement and layout-aware gradient reduction.
 *
 * Plain C types only: caller-owned host arrays and device pointers, explicit
 * cudaStream_t passed as void*, integer return codes, a thread-local message.
 * The C++ drop-in `namespace gmux` (include/gmux/gmux.hpp) is a header-only
 * wrapper over these entry points that restores the reference's types and
 * exception classes.
 *
 * Reference interfaces replaced (paths relative to the reference tree,
 * proj/include/gmux/):  see each declaration.
 */
#ifndef GMI_H_
#define GMI_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define GMI_API __attribute__((visibility("default")))
#else
#define GMI_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ errors
 * Codes mirror the reference CLI's exit-code split (tools/gmux.cpp:389-411):
 * gmi_exit_code() maps INVALID/CONFIG -> 2, every other failure -> 1. */
enum {
  GMI_OK = 0,
  GMI_ERR_DOMAIN = 1,      /* std::runtime_error                          */
  GMI_ERR_INVALID = 2,     /* std::invalid_argument                       */
  GMI_ERR_MULTISTREAM = 3, /* gmux::MultiStreamError (reduction.hpp:91)   */
  GMI_ERR_PLAN = 4,        /* gmux::PlanError (mapping.hpp:209)           */
  GMI_ERR_PIPELINE = 5,    /* gmux::PipelineError (channels.hpp:105)      */
  GMI_ERR_CONFIG = 6,      /* gmux::ConfigError (config.hpp:39)           */
  GMI_ERR_CUDA = 7,        /* CUDA runtime / driver failure               */
  GMI_ERR_NCCL = 8         /* NCCL failure                                */
};

GMI_API const char* gmi_last_error(void);
GMI_API int gmi_exit_code(int err);
GMI_API int gmi_version(void);

/* ------------------------------------------------------------------ layouts
 * A GMI layout (the reference's mapping list, reduction.hpp:39-68) is passed
 * flattened: num_gpus per-GPU lists, counts[g] ids on GPU g, ids GPU-major. */
enum { GMI_MPR = 0, GMI_MRR = 1, GMI_HAR = 2 };
enum { GMI_LINK_INTRA = 0, GMI_LINK_HOST_BOUNCE = 1, GMI_LINK_RING = 2, GMI_LINK_LOCAL_REDUCE = 3 };

/* select_strategy (reduction.hpp:98-106), Alg. 1. */
GMI_API int gmi_select_strategy(int num_gpus, const int* counts, const int* ids, int* strategy);
/* leader_gmis (reduction.hpp:110-122); leaders[num_gpus]. */
GMI_API int gmi_leader_gmis(int num_gpus, const int* counts, const int* ids, int* leaders);
/* mrr_rings (reduction.hpp:127-139); rings[t*g] row-major, *num_rings = t.
 * GMI_ERR_MULTISTREAM on ragged layouts or t > g. */
GMI_API int gmi_mrr_rings(int num_gpus, const int* counts, const int* ids, int* rings, int* num_rings);
/* predict_latency (reduction.hpp:142-152), Table 3. */
GMI_API int gmi_predict_latency(int strategy, int g, int t, double m_p, double b1, double b2,
                                double* latency);

typedef struct {
  int step, src, dst, kind; /* kind: GMI_LINK_* */
  double bytes;
} gmi_trace_event_t;

typedef struct {
  int strategy;
  int result_holder;
  double latency;           /* reduction phases only (== predict_latency on uniform layouts) */
  double broadcast_latency; /* final flush to every GMI */
  size_t trace_len;
} gmi_reduction_info_t;

/* Communication schedule of execute() (reduction.hpp:225-334) for len elements of
 * elem_bytes (8 = the reference's fp64 buffers): trace + ideal-link latencies.
 * Call with trace == NULL to size, then again with trace_cap >= info->trace_len. */
GMI_API int gmi_reduction_schedule(int strategy, int num_gpus, const int* counts, const int* ids,
                                   size_t len, double elem_bytes, double b1, double b2,
                                   gmi_trace_event_t* trace, size_t trace_cap,
                                   gmi_reduction_info_t* info);

enum { GMI_F32 = 0, GMI_F64 = 1 };
/* Device-backed execute(): elementwise sum of the GMIs' device buffers in exactly the
 * reference's ring fold order (bit-identical for fp64), written to `out` (len elements)
 * and, when broadcast != 0, to every input buffer. bufs[i] belongs to the i-th id of the
 * flattened layout. HBM-bound kernel on `stream` (cudaStream_t). */
GMI_API int gmi_reduce_device(int strategy, int num_gpus, const int* counts, const int* ids,
                              void* const* bufs, void* out, size_t len, int dtype, int broadcast,
                              void* stream);

/* The SURVEY §8b allreduce over one layout's GMIs (replaces execute(), reduction.hpp:225-334,
 * for device-resident gradients): the GMIs' buffers are summed in the reference's fold order for
 * `strategy` (the order of gmi_reduce_device) and the total is written back into EVERY buffer (in
 * place, like a collective). streams: one cudaStream_t per GMI in flattened layout order, or NULL
 * (all on the default stream); the reduction runs on streams[0] once every GMI stream has reached
 * the call, and every GMI stream continues only after it. run (may be NULL): the reference's
 * modelled latency and broadcast latency for len 8-byte elements over b1 / b2 bytes/s (execute()'s
 * accounting, reduction.hpp:304-329; trace_len = its trace length). */
GMI_API int gmi_allreduce(int strategy, int num_gpus, const int* counts, const int* ids, void* const* dev_bufs,
                          size_t len, int dtype, void* const* streams, double b1, double b2,
                          gmi_reduction_info_t* run);

/* execute() with HOST buffers (the reference's calling convention, reduction.hpp:225):
 * bufs[i] (len elements of dtype) belongs to the i-th id of the flattened layout; the call
 * stages them into device memory, runs gmi_reduce_device and copies the result back to
 * `result` (len elements). Synchronous. */
GMI_API int gmi_execute_host(int strategy, int num_gpus, const int* counts, const int* ids,
                             const void* const* bufs, size_t len, int dtype, void* result);

/* B200 extension: SMs of the green context that realises an MPS `share` on an sm100 GPU
 * (whole 8-SM groups of 148 SMs, or of sm_units when > 8). validate_layout flags sm100 shares
 * below one group and checks sm100 MIG partitions against the B200 profile table. */
GMI_API int gmi_green_sms(double share, int sm_units, int* out);

/* ------------------------------------------------------------------ topology
 * topology.hpp:60-252. arch: 70, 80 or 100 (sm100 is a B200 extension).
 * backend: 0 = MPS share (realised as an SM-partitioned green context), 1 = MIG. */
typedef struct {
  int id, arch, sm_units;
  double mem_gb;
} gmi_gpu_t;

typedef struct {
  int gmi_id, gpu_id, backend;
  double sm_share, mem_gb;
} gmi_partition_t;

typedef struct {
  const gmi_gpu_t* gpus;
  int num_gpus;
  const gmi_partition_t* parts;
  int num_parts;
  double b1, b2;
} gmi_topology_t;

typedef struct {
  int gpu_id; /* -1 for topology-wide rules */
  char rule[160];
} gmi_violation_t;

/* validate_layout (topology.hpp:134-212): violations are data, not failures. */
GMI_API int gmi_validate_layout(const gmi_topology_t* topo, gmi_violation_t* out, int cap,
                                int* count);
/* select_backend (topology.hpp:216-222). */
GMI_API int gmi_select_backend(int arch, int training, int* backend);
/* path_bandwidth (topology.hpp:243-252); *bw is +inf for GMI_LINK_INTRA. */
GMI_API int gmi_path_bandwidth(const gmi_topology_t* topo, int src_gmi, int dst_gmi, int* kind,
                               double* bw);

/* ------------------------------------------------------------------ workload
 * workload.hpp:26-134. */
#define GMI_MAX_DIMS 16
typedef struct {
  double r_sm, r_mem, t_iter;
} gmi_role_profile_t;

typedef struct {
  char name[32];
  double state_bytes, action_bytes, reward_bytes, model_bytes;
  int steps_per_train;
  double alpha, beta;
  int num_dims;
  int policy_dims[GMI_MAX_DIMS];
  gmi_role_profile_t simulator, agent, trainer;
} gmi_workload_t;

GMI_API int gmi_load_benchmark(const char* name, gmi_workload_t* out);
GMI_API int gmi_validate_workload(const gmi_workload_t* w);
GMI_API int gmi_dense_param_count(const int* dims, int n, size_t* out);
GMI_API int gmi_policy_value_param_count(const int* dims, int n, size_t* out);

/* ------------------------------------------------------------------ placement + costs
 * mapping.hpp:95-279. template_kind: 0 TDG, 1 TCG, 2 TDG_EX, 3 TCG_EX, 4 async_decoupled.
 * Role masks: 1 simulator, 2 agent, 4 trainer. */
enum { GMI_TDG = 0, GMI_TCG = 1, GMI_TDG_EX = 2, GMI_TCG_EX = 3, GMI_ASYNC = 4 };
enum { GMI_ROLE_SIM = 1, GMI_ROLE_AGENT = 2, GMI_ROLE_TRAINER = 4 };

GMI_API int gmi_serving_cost(int tpl, const gmi_workload_t* w, double* resource, double* comm);
GMI_API int gmi_training_cost(int tpl, const gmi_workload_t* w, int n_gmis, double* resource,
                              double* comm);
GMI_API int gmi_allreduce_bytes(int n_gmis, double model_bytes, double* out);
/* training != 0: training_throughput (Eq. 3), else serving_throughput (Eq. 2). */
GMI_API int gmi_throughput(int training, double resource, double comm, const gmi_workload_t* w,
                           double r_all, double bandwidth, double* out);
GMI_API int gmi_throughput_ratio(int training, const gmi_workload_t* w, double combw_factor,
                                 double* out);
GMI_API int gmi_colocation_penalty(int training, const gmi_workload_t* w, double* out);

/* build_plan (mapping.hpp:216-279). GMI ids are sequential GPU-major, so outputs are:
 * gpu_ids[num_gpus] sorted, gmi_ids[num_gpus * gmis_per_gpu] GPU-major, role_masks
 * indexed by gmi id, serving[num_gpus] = 1 serving / 0 training / -1 not async. */
GMI_API int gmi_build_plan(int tpl, const gmi_topology_t* topo, int gmis_per_gpu, int* gpu_ids,
                           int* gmi_ids, int* role_masks, int* serving);

/* ------------------------------------------------------------------ adaptive GMI manager
 * search.hpp:26-249 (Alg. 2). The probe callback is the reference's Profiler::profile
 * (search.hpp:32-37); it returns 0 or an error code that aborts the search. */
typedef int (*gmi_probe_fn)(void* user, const char* bench, int gmis_per_gpu, int num_env,
                            int* runnable, double* top, double* mem);

/* Measured profiler (B200): the real PPO iteration of `bench`'s catalog MLP on `device` with
 * `gmis_per_gpu` GMIs (backend 0 streams, 1 green contexts) of `num_env` envs each, timed over
 * `iters` graph-replayed iterations. top = per-GMI env-steps/s, mem = per-GMI device GB;
 * shapes that cannot be built report runnable = 0 (search.hpp:32-37 semantics). */
GMI_API int gmi_gpu_profile(const char* bench, int gmis_per_gpu, int num_env, int device, int backend,
                            int iters, int* runnable, double* top, double* mem);
/* gmi_probe_fn adapter over gmi_gpu_profile; user -> int[3] {device, backend, iters}. */
GMI_API int gmi_gpu_probe(void* user, const char* bench, int gmis_per_gpu, int num_env, int* runnable,
                          double* top, double* mem);

typedef struct {
  const int* num_env_grid;
  int grid_len;
  int max_gmis_per_gpu;
  double sat_threshold;
} gmi_search_config_t;

typedef struct {
  gmi_workload_t workload;
  double b1, b2, latency_scale;
} gmi_estimator_t;

typedef struct {
  int gmis_per_gpu, num_env, runnable;
  double top, mem;
  int has_sat;
  double sat;
  int has_acc_top;
  double acc_top;
  int pruned_here;
} gmi_visit_t;

typedef struct {
  int feasible;
  char reason[96];
  int num_env, gmis_per_gpu;
  double est_throughput;
  size_t num_visited;
} gmi_search_result_t;

GMI_API int gmi_saturation(double top, double pre_top, double mem, double pre_mem, double* out);
GMI_API int gmi_comm_discount(const gmi_estimator_t* est, int gmis_per_gpu, int num_gpu, double* out);
GMI_API int gmi_estimate(const gmi_estimator_t* est, int gmis_per_gpu, int num_gpu,
                         double per_gmi_top, double* out);
/* explore(): visits must hold max_gmis_per_gpu * grid_len entries. */
GMI_API int gmi_explore(gmi_probe_fn probe, void* user, const gmi_estimator_t* est,
                        const char* bench, int num_gpu, const gmi_search_config_t* cfg,
                        gmi_search_result_t* out, gmi_visit_t* visits, size_t visits_cap);

/* SyntheticCostModel (search.hpp:100-132); override tables as (key, value) pairs. */
typedef struct {
  double peak_top, mem_base, mem_per_env, mem_capacity, min_runnable_share;
  int knee_base;
  int num_knee;
  const int* knee_keys;
  const int* knee_values;
  int num_cap;
  const int* cap_keys;
  const double* cap_values;
} gmi_synthetic_model_t;
GMI_API void gmi_synthetic_model_defaults(gmi_synthetic_model_t* m);
GMI_API int gmi_synthetic_profile(const gmi_synthetic_model_t* m, const char* bench,
                                  int gmis_per_gpu, int num_env, int* runnable, double* top,
                                  double* mem);
/* RecordedTraceProfiler (search.hpp:136-171). */
GMI_API int gmi_trace_profiler_load(const char* path, void** handle);
GMI_API int gmi_trace_profiler_profile(void* handle, const char* bench, int gmis_per_gpu,
                                       int num_env, int* runnable, double* top, double* mem);
GMI_API void gmi_trace_profiler_free(void* handle);

/* ------------------------------------------------------------------ experience channels
 * channels.hpp:85-397 (decoupled mode accounting). */
typedef struct {
  int compress_threshold;
  int batch_mode; /* 0 slice, 1 stack */
  int target_batch;
  double per_message_overhead;
  unsigned seed;
} gmi_pipeline_config_t;

typedef struct {
  double pps, ttop;
  long records_produced, records_delivered, units_sent, batches_emitted;
  double bytes_moved, transfer_busy_time, delivery_makespan, training_makespan;
  size_t num_trainers;
} gmi_pipeline_metrics_t;

/* An explicit plan: per-GPU lists (gpu_ids[num_gpus], counts, gmi_ids GPU-major) and one
 * role mask per listed gmi id (parallel to gmi_ids). */
typedef struct {
  int template_kind;
  int num_gpus;
  const int* gpu_ids;
  const int* counts;
  const int* gmi_ids;
  const int* role_masks;
} gmi_plan_t;

GMI_API void gmi_pipeline_config_defaults(gmi_pipeline_config_t* c);
GMI_API int gmi_simulate_pipeline(const gmi_workload_t* w, const gmi_plan_t* plan,
                                  const gmi_topology_t* topo, const gmi_pipeline_config_t* cfg,
                                  double duration, void** handle, gmi_pipeline_metrics_t* out);
/* The same pipeline on the GPU over real payloads (cuda/channels.cu, K9): every agent GMI (role
 * mask & AGENT, ascending id) supplies three device channel buffers -- agent_bufs[c * agents + a],
 * c = 0 state (S bytes per record), 1 action (A), 2 reward (W); records in production order --
 * and every trainer GMI three receive buffers of trainer_capacity records
 * (trainer_bufs[c * trainers + t]). compress(k) units, send / arrival clocks, direct vs
 * least-load routing, delivery, stack / slice batching and PPS / TTOP follow
 * gmi_simulate_pipeline bit for bit; the delivered records land in the receive buffers in
 * delivery order (batches are contiguous ranges). The handle answers the gmi_pipeline_*
 * accessors below. */
GMI_API int gmi_channel_run(const gmi_workload_t* w, const gmi_plan_t* plan, const gmi_topology_t* topo,
                            const gmi_pipeline_config_t* cfg, double duration, const void* const* agent_bufs,
                            int num_agent_bufs, void* const* trainer_bufs, int num_trainer_bufs,
                            long trainer_capacity, void* stream, void** handle, gmi_pipeline_metrics_t* out);
GMI_API int gmi_pipeline_trainer_records(void* handle, int* trainers, long* records);
GMI_API size_t gmi_pipeline_num_batches(void* handle);
GMI_API int gmi_pipeline_batch(void* handle, size_t i, int* trainer, double* emit_time,
                               size_t* num_records);
GMI_API int gmi_pipeline_batch_records(void* handle, size_t i, int* agent_gmis, long* seqs);
GMI_API void gmi_pipeline_free(void* handle);

/* ------------------------------------------------------------------ config schema
 * config.hpp:125-301; sections are evaluated lazily like the reference loaders. */
typedef struct {
  double serving_combw_factor, training_combw_factor;
  int gmis_per_gpu;
  double latency_scale;
  gmi_pipeline_config_t pipeline;
} gmi_model_params_t;

#define GMI_MAX_GRID 32
typedef struct {
  int grid[GMI_MAX_GRID];
  int grid_len;
  int max_gmis_per_gpu;
  double sat_threshold;
  int has_profile_trace;
  char profile_trace[512];
} gmi_search_settings_t;

GMI_API int gmi_config_parse(const char* text, const char* origin, void** handle);
GMI_API int gmi_config_load(const char* path, void** handle);
GMI_API int gmi_config_has(void* handle, const char* section, int* out);
/* Sizes first: call with caps of 0 to read *num_gpus / *num_parts. */
GMI_API int gmi_config_topology(void* handle, gmi_gpu_t* gpus, int gpu_cap, int* num_gpus,
                                gmi_partition_t* parts, int part_cap, int* num_parts, double* b1,
                                double* b2);
GMI_API int gmi_config_workload(void* handle, const char* fallback, gmi_workload_t* out);
GMI_API int gmi_config_model(void* handle, gmi_model_params_t* out);
GMI_API int gmi_config_search(void* handle, gmi_search_settings_t* out);
/* Raw value lookup (any section, incl. B200 extensions such as [ppo]); *found = 0/1. */
GMI_API int gmi_config_get(void* handle, const char* section, const char* key, char* value,
                           size_t cap, int* found);
GMI_API void gmi_config_free(void* handle);

/* ------------------------------------------------------------------ PPO iteration (B200)
 * The data-parallel TCG_EX training iteration (holistic GMIs: simulator + agent + trainer,
 * mapping.hpp:246-249) that the reference models only as T_s + T_a + T_t + COM/BW
 * (mapping.hpp:123-128, workload.hpp:43-45). One trainer drives one GPU (`rank` of
 * `num_gpus`) with `gmis_per_gpu` GMIs; envs are split over the job's GMIs by
 * [N*c/n, N*(c+1)/n) (reduction.hpp:164-166). Gradients are reduced per minibatch:
 * K1 fold across the GPU's GMIs, then NCCL across GPUs; Adam runs once per GPU on the
 * shared replica. Semantics: DESIGN.md §PPO (mirrored by oracle/ppo_oracle.c). */
#define GMI_MAX_HIDDEN 8
typedef struct {
  int obs_dim, act_dim;
  int num_hidden;
  int hidden[GMI_MAX_HIDDEN];
  int num_envs; /* whole job */
  int horizon, epochs, minibatches;
  float gamma, lam, clip, lr, beta1, beta2, adam_eps, vf_coef, ent_coef;
  unsigned long long seed;
  int num_gpus, gmis_per_gpu; /* job layout (GPU-major GMI ids) */
  int rank;                   /* GPU index of this trainer within the job */
  int device;                 /* CUDA device ordinal */
  int gmi_backend;            /* 0: one CUDA stream per GMI; 1: SM-partitioned green contexts */
  int sm_per_gmi;             /* green-context SMs per GMI (multiple of 8; 0 = even split) */
  int use_graph;              /* capture the update phase in a CUDA graph */
  int instrument;             /* time GEMM launches with CUDA events (roofline) */
  /* Decoupled (asynchronous) mode, BASELINE config 4 / PAPER.md:378-407: per GPU one serving
   * GMI (simulator + agent, roles of mapping.hpp:243) on `serving_sms` SMs streams experience
   * through a device channel to the trainer GMI on the remaining SMs. Iteration i trains on the
   * experience the serving GMI generated with the weights of iteration i-1 while it generates
   * iteration i+1's experience with the weights of iteration i (one-iteration policy lag; the
   * behaviour log-probs are recorded, so the clipped ratio stays exact). gmis_per_gpu counts
   * trainer GMIs and must be 1.
   * decoupled = 2: AsyncDecoupled across GPUs (mapping.hpp:265-276; reference data path
   * channels.hpp:182-191 migrate): num_gpus even; ranks [0, G/2) are serving GPUs (simulator +
   * agent on the whole GPU), rank G/2 + s is a trainer GPU that trains on serving rank s's envs
   * (the 1:1 pairing LeastLoadRouter produces for equal units). Same one-iteration lag: the
   * trainer pulls rollout i from its partner's link window over NVLink, trains, and pushes the
   * new policy snapshot back; device flags in the windows order the hand-offs. The trainer
   * ranks form a data-parallel job of G/2 ranks (rank s; comm as below, among trainers only).
   * Wire each pair with gmi_ppo_link_attach / gmi_ppo_link_connect before the first iteration;
   * both ranks call gmi_ppo_iteration the same number of times. */
  int decoupled;
  int serving_sms;            /* green-context SMs of the serving GMI (multiple of 8; 0 = 16) */
  /* Cross-GPU gradient exchange (num_gpus > 1; HAR leader step, reduction.hpp:287-299):
   * 0 = ncclAllReduce on the update stream, then Adam on every rank (baseline);
   * 1 = peer exchange: one fused kernel per update over peer memory (NVLink P2P) that sums the
   *     ranks' folded gradients in the reference's leader-ring order, runs Adam on this rank's
   *     shard and writes the new weights into every rank (reduce-scatter -> sharded Adam ->
   *     all-gather, cuda/exchange.cu). The ranks must be wired before the first iteration with
   *     gmi_ppo_comm_attach (one process per GPU, CUDA IPC handles) or gmi_ppo_comm_connect (all
   *     ranks in one process). With num_gpus == 1 the exchange runs over the rank itself. */
  int comm;
} gmi_ppo_config_t;

typedef struct {
  double policy_loss, value_loss, approx_kl, clip_frac; /* last minibatch of GMI 0 */
  double mean_reward;                                   /* rollout mean of GMI 0 */
  long long env_steps;                                  /* this GPU, this iteration */
  double gemm_ms;   /* instrument: summed GEMM time this iteration (GMI 0 stream) */
  double gemm_flop; /* instrument: algorithmic GEMM flops of those launches */
  int gemm_launches;
  int kernel_launches; /* every libgmi kernel launched this iteration (this GPU) */
  double gemm_bytes;   /* instrument: algorithmic GEMM bytes (operands read + outputs written) */
} gmi_ppo_stats_t;

GMI_API void gmi_ppo_config_defaults(gmi_ppo_config_t* cfg);
/* nccl_id: 128-byte ncclUniqueId shared by all ranks (NULL when num_gpus == 1). */
GMI_API int gmi_ppo_create(const gmi_ppo_config_t* cfg, const void* nccl_id, void** trainer);
GMI_API void gmi_ppo_free(void* trainer);
GMI_API int gmi_nccl_unique_id(void* out128);
/* One PPO iteration: rollout (horizon steps), values, GAE, epochs x minibatches of
 * forward / loss / backward / gradient reduction / Adam. Blocks until done; stats may be NULL. */
GMI_API int gmi_ppo_iteration(void* trainer, gmi_ppo_stats_t* stats);
/* Asynchronous variant: enqueue one iteration on the trainer's streams, no host sync. */
GMI_API int gmi_ppo_iteration_async(void* trainer);
GMI_API int gmi_ppo_synchronize(void* trainer, gmi_ppo_stats_t* stats);
/* Adaptive GMI manager (search.hpp:32-37): re-split the green-context SM
 * partitions of a live trainer (gmi_backend = 1). `gpu` is the trainer's rank; sm_counts[t]
 * gives each GMI's SMs (multiples of 8; decoupled: {serving, trainer}, one entry may be 0 =
 * the rest). Buffers, parameters and optimizer state stay; streams, GEMM plans and the
 * iteration graph are rebuilt. t must equal the trainer's GMI count. */
GMI_API int gmi_resize(void* trainer, int gpu, const int* sm_counts, int t);
/* Per-role SM-share retuning from measured throughput: for each candidate split
 * (candidates[c * t .. c * t + t), t = the trainer's GMI count, decoupled: {serving, trainer})
 * resize, run `iters` timed iterations (after one eager and one capture iteration) and record
 * env-steps/s in throughput[c]; the trainer is left at the best split (*best). Training
 * continues through the probe iterations (they are real updates). */
GMI_API int gmi_ppo_tune_shares(void* trainer, const int* candidates, int ncand, int iters, int* best,
                                double* throughput);
/* Peer exchange wiring (cfg.comm = 1). gmi_ppo_comm_handle: the 64-byte CUDA IPC handle of this
 * rank's exchange window (flags, published gradient, fp32 parameters, bf16 shadow); every rank
 * gathers all handles in rank order (e.g. torch.distributed all_gather_object) and passes the
 * num_gpus x 64 bytes to gmi_ppo_comm_attach. gmi_ppo_comm_connect wires n = num_gpus trainers
 * that live in this process (trainers[r] has rank r; same or peer-capable devices). */
GMI_API int gmi_ppo_comm_handle(void* trainer, void* out64);
GMI_API int gmi_ppo_comm_attach(void* trainer, const void* handles);
GMI_API int gmi_ppo_comm_connect(void* const* trainers, int n);
/* Experience link of an AsyncDecoupled pair (cfg.decoupled = 2). gmi_ppo_link_handle: the
 * 64-byte CUDA IPC handle of this rank's link window ([flags | policy snapshot | experience
 * channel]); pass the partner's to gmi_ppo_link_attach (serving rank s <-> trainer rank
 * G/2 + s, one process per GPU). gmi_ppo_link_connect wires a pair living in one process
 * (distinct, peer-capable devices). Iterating an unwired rank fails with GMI_ERR_INVALID. */
GMI_API int gmi_ppo_link_handle(void* trainer, void* out64);
GMI_API int gmi_ppo_link_attach(void* trainer, const void* peer64);
GMI_API int gmi_ppo_link_connect(void* serving, void* trainer);
/* Rollout + values + GAE of the next iteration only (parity checks). The following
 * gmi_ppo_iteration trains on this rollout instead of rolling out again; calling the hook
 * twice without an iteration in between fails with GMI_ERR_INVALID. */
GMI_API int gmi_ppo_rollout(void* trainer);
/* One minibatch gradient of local GMI `gmi` on caller rows (host fp32; B = minibatch size). */
GMI_API int gmi_ppo_minibatch_grad(void* trainer, int gmi, const float* X, const float* act,
                                   const float* oldlp, const float* adv, const float* ret, int B,
                                   float* grad_out);
/* Host copies of device state. what: params adam_m adam_v (shared) | grad x obs act logp rew
 * val adv ret done ep_step ep_len ep_count (per local GMI). Returns the element count via *n
 * when dst is NULL. */
GMI_API int gmi_ppo_get(void* trainer, const char* what, int gmi, void* dst, long long* n);
GMI_API int gmi_ppo_set(void* trainer, const char* what, int gmi, const void* src, long long n);
GMI_API int gmi_ppo_param_count(void* trainer, long long* padded, long long* real);
/* cudaStream_t of local GMI `gmi` (-1: the update / reduction stream; -2: the serving GMI's
 * stream in decoupled mode, the whole rank's work on a decoupled = 2 serving rank). */
GMI_API int gmi_ppo_stream(void* trainer, int gmi, void** stream);

/* Per-phase device time of the last completed iteration when cfg.instrument = 1: CUDA
 * events around every launch on GMI 0's stream and the update stream, plus the
 * algorithmic flops (tensor-core phases) or HBM bytes (memory-bound phases) of those
 * launches, for the per-kernel roofline. */
enum {
  GMI_PH_ROLL_GEMM, /* rollout: policy hidden layers, M = envs per GMI */
  GMI_PH_ROLL_HEAD, /* rollout: policy head GEMM */
  GMI_PH_ACT_ENV,   /* rollout: Gaussian action + env step + reset + next obs */
  GMI_PH_VAL_GEMM,  /* values: value-net hidden layers over (T+1) x envs rows */
  GMI_PH_VAL_HEAD,  /* values: value head GEMM + bias */
  GMI_PH_GAE,       /* GAE scan + advantage statistics */
  GMI_PH_SHUFFLE,   /* epoch permutation gather */
  GMI_PH_FWD_GEMM,  /* update: hidden forward (both nets) */
  GMI_PH_HEAD_FWD,  /* update: head forward GEMMs */
  GMI_PH_HEAD_LOSS, /* update: clipped surrogate / value loss + head output grads */
  GMI_PH_HEAD_DX,   /* update: head input-gradient GEMM */
  GMI_PH_HEAD_DW,   /* update: head weight-gradient GEMM */
  GMI_PH_DW_GEMM,   /* update: hidden weight-gradient GEMMs (split-K slabs) */
  GMI_PH_COLSUM,    /* update: bias-gradient column sums */
  GMI_PH_DX_GEMM,   /* update: hidden input-gradient GEMMs */
  GMI_PH_SEGMENTS,  /* update: fixed-order gradient assembly */
  GMI_PH_REDUCE,    /* K1 intra-GPU GMI gradient fold */
  GMI_PH_ALLREDUCE, /* NCCL cross-GPU gradient all-reduce */
  GMI_PH_ADAM,      /* Adam on the shared replica */
  GMI_PH_OTHER,     /* copies, control block */
  GMI_PPO_PHASES
};
typedef struct {
  double ms;    /* summed event time of the phase's launches */
  double flop;  /* algorithmic flops (GEMM phases) */
  double bytes; /* algorithmic HBM bytes (memory-bound phases) */
  int launches;
} gmi_ppo_phase_t;
GMI_API const char* gmi_ppo_phase_name(int phase);
GMI_API int gmi_ppo_profile(void* trainer, gmi_ppo_phase_t* out /* [GMI_PPO_PHASES] */);
/* Per-GMI busy time of the last instrumented iteration (cfg.instrument = 1): summed CUDA-event
 * time of every launch on each execution unit, with the unit's SM count (its green-context
 * partition, or the whole GPU for plain streams). Units: decoupled -> serving GMI, trainer GMI;
 * otherwise the local GMIs; the last unit is the update / reduction stream. busy_ms / (SMs-
 * weighted) iteration time = the GMI's stream-level SM utilisation. *count = number of units. */
GMI_API int gmi_ppo_unit_busy(void* trainer, double* busy_ms, int* sms, int cap, int* count);
/* Toggle cfg.instrument on a live trainer (re-captures the iteration graph). */
GMI_API int gmi_ppo_set_instrument(void* trainer, int on);

/* ------------------------------------------------------------------ diagnostics
 * Single tcgen05 GEMM launch, D[m][n] = sum_k A(m,k) B(n,k), bf16 in, fp32 accumulate.
 * a_mn/b_mn: 0 = operand stored [rows x K], 1 = stored [K x rows].
 * epi: 0 = bf16 elu(acc + bias), 1 = bf16 acc * elu'(aux), 2 = fp32 (split-K slabs).
 * weight_stationary: 1 = B resident in shared memory (N <= 256, K <= 256, splits == 1). */
GMI_API int gmi_dev_gemm(int a_mn, int b_mn, int epi, int M, int N, int K, const void* A, long long lda,
                 const void* B, long long ldb, void* out, long long ldo, const float* bias,
                 const void* aux, long long ld_aux, int splits, int weight_stationary, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GMI_H_ */
