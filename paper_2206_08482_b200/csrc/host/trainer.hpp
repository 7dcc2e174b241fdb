// B200 PPO trainer: one instance drives one GPU of the data-parallel job (TCG_EX
// holistic GMIs). Owns device memory, GMI execution resources (streams or green
// contexts), the prebuilt GEMM problem descriptors, the NCCL communicator and the CUDA
// graph that replays one whole iteration.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "../cuda/gemm_host.hpp"
#include "../cuda/ppo.cuh"
#include "gmi.h"
#include "planner.hpp"

namespace gmi {

struct Tensor {  // one weight or bias block inside the flat parameter vector
  long long w = 0, b = 0;
  int out = 0, in = 0, out_p = 0, in_p = 0;
};

// Geometry shared bit-for-bit with oracle/ppo_oracle.c and tests/golden_util.param_layout.
struct Geometry {
  int L = 0, S = 0, A = 0;
  std::vector<int> width, wp;  // [0] = obs, 1..L hidden; wp padded to 32
  Tensor net[2][GMI_MAX_HIDDEN + 1];
  long long log_std = 0, P = 0, real_params = 0;
  static Geometry make(const gmi_ppo_config_t& c);
};

class GmiResources;  // streams / green contexts (gmi_exec.cpp)

class Trainer {
 public:
  Trainer(const gmi_ppo_config_t& cfg, const void* nccl_id);
  ~Trainer();

  void enqueue_iteration(bool host_control);
  void enqueue_rollout();
  void synchronize(gmi_ppo_stats_t* stats);
  void minibatch_grad(int gmi, const float* X, const float* act, const float* oldlp, const float* adv,
                      const float* ret, int B, float* grad_out);
  long long get(const std::string& what, int gmi, void* dst);
  void set(const std::string& what, int gmi, const void* src, long long n);
  const Geometry& geometry() const { return geo_; }
  cudaStream_t stream(int gmi) const;

 private:
  struct Gmi;

  void init(const void* nccl_id);
  void release() noexcept;
  void alloc();
  void init_params();
  void build_plans();
  void ensure_bias_table(long long steps);
  void write_control();
  void record_iteration(bool with_rollout);  // one iteration's launches (eager or under capture)
  void serve_rollout(Gmi& g);  // decoupled mode: the serving GMI's rollout into the channel
  void build_serving_plans(Gmi& g);   // decoupled mode, wide nets: per-layer serving plans
  void serve_rollout_layers(Gmi& g);  // ... and their launches
  void rollout(Gmi& g);
  void values(Gmi& g);
  void train_minibatch(Gmi& g, int k, int adam_step = -1);  // adam_step >= 0: fused Adam
  void reduce_and_step(int k);
  void launch_adam_on(cudaStream_t st, const float* grad, int step_in_iter);
  void gemm(Gmi& g, int phase, const GemmParams& P, int bn, int amn, int bmn, int epi, double flop, int ws = 0,
            cudaStream_t stream = nullptr, int ctas = 0);
  // Runs f (which enqueues work on s); with cfg.instrument and s = GMI 0's stream or the
  // update stream, brackets it with CUDA events booked to `phase` (+ algorithmic flop/bytes).
  template <class F>
  void timed(cudaStream_t s, int phase, double flop, double bytes, F&& f);

  gmi_ppo_config_t cfg_;
  Geometry geo_;
  int T_ = 0, K_ = 0, n_local_ = 0, n_total_ = 0;
  std::unique_ptr<GmiResources> exec_;
  std::vector<std::unique_ptr<Gmi>> gmis_;
  std::vector<void*> allocs_;
  std::vector<void*> plan_allocs_;  // GEMM-plan scratch (rebuilt by resize)

  // shared per GPU
  float *params_ = nullptr, *m_ = nullptr, *v_ = nullptr, *grad_sum_ = nullptr, *bc_ = nullptr;
  __nv_bfloat16* shadow_ = nullptr;
  long long bc_cap_ = 0;
  ppo::Control* ctl_dev_ = nullptr;
  ppo::Control* ctl_host_ = nullptr;  // pinned
  float* stats_dev_ = nullptr;        // [8]
  float* stats_host_ = nullptr;       // pinned
  cudaStream_t upd_ = nullptr;        // update / reduction stream
  cudaEvent_t ev_adam_ = nullptr;
  cudaEvent_t ev_start_ = nullptr;
  void* nccl_ = nullptr;
  // decoupled mode (cfg.decoupled): serving GMI stream, experience-channel events, the policy
  // snapshot the serving GMI acts with, and its own control block (rollout index)
  bool decoupled_ = false;
  bool upd_in_gmi_ = false;  // update stream owned by the trainer GMI's green context
  cudaStream_t serve_s_ = nullptr;
  cudaEvent_t ev_copied_ = nullptr, ev_rolled_ = nullptr;
  float* params_roll_ = nullptr;
  __nv_bfloat16* shadow_roll_ = nullptr;
  ppo::Control* ctl_roll_ = nullptr;
  long long rollouts_ = 0;  // serving-GMI rollouts enqueued so far
  // AsyncDecoupled across GPUs (cfg.decoupled = 2, mapping.hpp:265-276): ranks [0, G/2) serve,
  // rank G/2 + s trains on serving rank s's experience. cfg_ holds the pair's data-parallel
  // sub-job view (rank s of G/2); link_rank_ / link_gpus_ the job's. Both ranks lay out the same
  // link window [flags | policy snapshot | experience channel] (IPC-exported): the trainer pulls
  // the channel from its partner's window and pushes the snapshot back; device flags order it.
  bool split_ = false, serving_ = false, linked_ = false;
  int link_rank_ = 0, link_gpus_ = 0;
  char* lwin_ = nullptr;                  // this rank's link window
  char* lpeer_ = nullptr;                 // the partner's (mapped)
  unsigned long long* lctr_ = nullptr;    // device counters of the link's wait / signal sites
  size_t loff_params_ = 0, loff_shadow_ = 0, loff_X_ = 0, loff_act_ = 0, loff_logp_ = 0, loff_adv_ = 0,
         loff_ret_ = 0, loff_stats_ = 0, lwin_bytes_ = 0;
  void serve_iteration();  // serving rank: one rollout per gmi_ppo_iteration
  unsigned long long* link_flag(bool peer, size_t off) const;
  // peer exchange (cfg.comm = 1, cuda/exchange.cu): this rank's window [flags | pub | params |
  // shadow] (IPC-exportable cudaMalloc), the peer-pointer table, and IPC mappings opened
  bool xchg_ = false;
  bool connected_ = false;
  char* win_ = nullptr;
  size_t win_off_gmi_ = 0, win_off_params_ = 0, win_off_shadow_ = 0;
  plan::Algo strategy_ = plan::Algo::MPR;  // Alg. 1 on the job layout (cross-GPU fold order)
  ppo::ExchangeArgs xa_{};
  std::vector<void*> ipc_opened_;
  void* gemm_trace_ = nullptr;  // GMI_GEMM_TRACE development aid
  void* head_trace_ = nullptr;  // GMI_HEAD_TRACE development aid
  bool bwd_par_ = false;   // dx chain || dW GEMMs on two streams of the GMI
  int bwd_dx_share_ = 50;  // percent of the GMI's SMs given to the dx branch
  int iteration_ = 0;      // iterations enqueued so far
  bool rollout_pending_ = false;  // gmi_ppo_rollout produced the next iteration's rollout
  bool adam_in_gmi_stream_ = false;  // GMI_ADAM_FUSED: Adam runs in the GMI stream (no B preload)
  // One GMI on one GPU (GMI_ADAM_INLINE=0 disables): Adam launched in the GMI stream right after the gradient
  // assembly (no cross-stream event hops per minibatch); only the first weight-stationary launch
  // after it (the next minibatch's forward) gives up its early weight load
  bool adam_inline_ = false;
  bool no_b_preload_once_ = false;
  long long adam_steps_ = 0;
  int launches_ = 0;       // kernels in one iteration
  bool capturing_ = false;
  cudaGraphExec_t graph_ = nullptr;
  // instrumentation: one event pair per launch of GMI 0 / the update stream
  struct Mark {
    cudaEvent_t a = nullptr, b = nullptr;
    int phase = 0;
    int unit = 0;         // execution unit (busy_units order) the launch ran on
    bool in_phases = false;  // GMI 0 / update stream: booked to phases_
    double flop = 0, bytes = 0;
  };
  std::vector<Mark> marks_;
  int marks_used_ = 0;
  gmi_ppo_phase_t phases_[GMI_PPO_PHASES] = {};
  std::vector<double> unit_busy_ms_;  // per execution unit, last instrumented iteration
  int unit_of(cudaStream_t s) const;  // -1: not instrumented

 public:
  const gmi_ppo_phase_t* phases() const { return phases_; }
  void resize(const int* sms, int n);  // gmi_resize
  int rank() const { return split_ ? link_rank_ : cfg_.rank; }
  int units() const { return decoupled_ ? 2 : n_local_; }  // GMIs with an SM partition
  // peer exchange wiring (gmi_ppo_comm_*)
  void comm_handle(void* out64) const;
  void comm_attach(const void* handles);
  static void comm_connect(Trainer* const* trainers, int n);
  // cross-GPU experience link (decoupled = 2): IPC handle of the link window, map the partner's
  void link_handle(void* out64) const;
  void link_attach(const void* peer64);
  static void link_connect(Trainer* serving, Trainer* trainer);  // one process, two devices
  bool serving() const { return split_ && serving_; }
  // Execution units in report order: decoupled -> [serving GMI, trainer GMI], else the local
  // GMIs; then the update stream. busy = summed kernel time of the unit's instrumented launches.
  int busy_units(double* busy_ms, int* sms, int cap) const;
  void set_instrument(int on);
};

}  // namespace gmi
