// B200 PPO trainer (host side): memory layout, GMI scheduling and the launch sequence
// of one data-parallel PPO iteration. The arithmetic contract is DESIGN.md §PPO, restated
// on the CPU by oracle/ppo_oracle.c (test infrastructure only, never linked here).
//
// Per iteration and GMI (own stream / green context):
//   rollout   T x [L tcgen05 GEMMs (policy, M = N envs) + act/env kernel]
//   values    ceil((T+1)N / M) x [L GEMMs (value net) + value head]
//   GAE       warp-shuffle scan + advantage statistics
//   update    E epochs x [shuffle + K minibatches x (L fwd GEMMs (both nets grouped),
//             head/loss, head weight-grad GEMM, L weight-grad GEMMs + L-1 input-grad GEMMs,
//             bias sums, gradient assembly)]; after each minibatch the update stream folds
//             the GMIs' gradients (K1, reference fold order), all-reduces across GPUs (NCCL)
//             and runs Adam once on the GPU's shared replica.
// From the second iteration on, the whole sequence (all GMI streams, events, NCCL) is
// replayed from one captured CUDA graph; a device-side control block carries the
// iteration counter so the graph is iteration-agnostic.
#include "trainer.hpp"

#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "../cuda/rng.cuh"
#include "../cuda/head_fused.cuh"
#include "../cuda/train_fwd.cuh"
#include "../cuda/rollout.cuh"
#include "errors.hpp"
#include "gmi_exec.hpp"
#include "planner.hpp"

namespace gmi {

void reduce_device(plan::Algo algo, const plan::Placement& p, void* const* bufs, void* out, size_t len, int dtype,
                   bool broadcast, cudaStream_t stream);
namespace ppo {
void launch_control_advance(Control* c, int dsteps, cudaStream_t s);
}

namespace {

int pad32(int x) { return (x + 31) / 32 * 32; }
long long align64(long long x) { return (x + 63) / 64 * 64; }

uint16_t bf16_bits(float f) {  // round-to-nearest-even, like __float2bfloat16_rn
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return uint16_t((u >> 16) | ((u & 0x007fffffu) ? 0x40u : 0u));
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}

float bf16_float(uint16_t b) {
  const uint32_t u = uint32_t(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

#define NCCL_CHECK(expr)                                                                                  \
  do {                                                                                                    \
    ncclResult_t _r = (expr);                                                                             \
    if (_r != ncclSuccess) ::gmi::fail(GMI_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
  } while (0)

// Wide weight-stationary families on by default (bit mask, see build_plans). Measured on B200
// (profiles/r2/SUMMARY.md, r2h): input gradients with K <= 256 resident per 128-column part win
// (HM 8192 envs 35.0 -> 37.3 M env-steps/s, dx 2.03 -> 1.58 ms; SH 14.1 -> 14.3 M); the K <= 512
// variants (4 operand stages next to 128 KB of weights, N = 128 MMAs) lose to the streaming
// kernel (SH forward 2.37 -> 2.83 ms, dx 2.27 -> 2.72 ms), and forward parts at K <= 256 are
// neutral (HM -1 %, SH +1 %), so only bit 2 is on.
constexpr int kWideDefault = 0x4;

// Splits of the weight-gradient GEMM: enough k-slabs to give ~one tile per SM.
void pick_splits(int M, int N, int bn, int problems, int rows, int sms, int* splits, int* kbps) {
  const int base = gemm_tiles(M, N, bn, problems, 1);
  const int nkb = (rows + kGemmBlockK - 1) / kGemmBlockK;
  const int s = std::max(1, std::min(nkb, sms / std::max(1, base)));
  const int per = (nkb + s - 1) / s;
  *kbps = per;
  *splits = (nkb + per - 1) / per;
}

}  // namespace

// ------------------------------------------------------------------ geometry
Geometry Geometry::make(const gmi_ppo_config_t& c) {
  Geometry g;
  if (c.num_hidden < 1 || c.num_hidden > GMI_MAX_HIDDEN) invalid("num_hidden must be in [1, 8]");
  if (c.obs_dim < 1 || c.act_dim < 1) invalid("obs_dim and act_dim must be positive");
  g.L = c.num_hidden;
  g.S = c.obs_dim;
  g.A = c.act_dim;
  g.width.push_back(c.obs_dim);
  for (int l = 0; l < g.L; ++l) {
    if (c.hidden[l] < 1) invalid("hidden widths must be positive");
    g.width.push_back(c.hidden[l]);
  }
  for (int w : g.width) g.wp.push_back(pad32(w));
  long long off = 0;
  for (int n = 0; n < 2; ++n)
    for (int l = 0; l <= g.L; ++l) {
      Tensor& t = g.net[n][l];
      t.in = g.width[l];
      t.in_p = g.wp[l];
      t.out = l < g.L ? g.width[l + 1] : (n == 0 ? c.act_dim : 1);
      t.out_p = l < g.L ? g.wp[l + 1] : t.out;
      t.w = off;
      off = align64(off + (long long)t.out_p * t.in_p);
      t.b = off;
      off = align64(off + t.out_p);
      g.real_params += (long long)t.out * t.in + t.out;
    }
  g.log_std = off;
  g.P = align64(off + c.act_dim);
  return g;
}

// ------------------------------------------------------------------ per-GMI state
struct Trainer::Gmi {
  int local = 0, gid = 0, env0 = 0, N = 0, B = 0, Bm = 0, Mrows = 0, ctas = 0;
  cudaStream_t s = nullptr;
  cudaEvent_t ev_done = nullptr;
  cudaStream_t s2 = nullptr;  // second stream of the GMI (backward branch parallelism)
  cudaEvent_t ev_fork = nullptr, ev_d[GMI_MAX_HIDDEN] = {};
  float* x = nullptr;
  int *ep_step = nullptr, *ep_len = nullptr, *ep_count = nullptr;
  __nv_bfloat16* X_roll = nullptr;
  float *act = nullptr, *logp = nullptr, *rew = nullptr, *V = nullptr, *adv = nullptr, *ret = nullptr;
  uint8_t* done = nullptr;
  // decoupled mode: the experience channel the serving GMI writes (same layouts as X_roll,
  // act, logp, rew, done); the trainer migrates it into the buffers above at slot start
  __nv_bfloat16* ch_X = nullptr;
  float *ch_act = nullptr, *ch_logp = nullptr, *ch_rew = nullptr;
  uint8_t* ch_done = nullptr;
  float *ch_V = nullptr, *ch_adv = nullptr, *ch_ret = nullptr, *ch_adv_stats = nullptr;
  double* ch_gae_part = nullptr;
  ppo::ValueArgs ch_val_args{};  // value pass of the serving GMI (snapshot weights, channel obs)
  double* gae_part = nullptr;
  float* adv_stats = nullptr;  // mean, std, mean reward
  __nv_bfloat16* X_sh = nullptr;
  float *act_sh = nullptr, *oldlp_sh = nullptr, *adv_sh = nullptr, *ret_sh = nullptr;
  __nv_bfloat16* H[2][GMI_MAX_HIDDEN] = {};
  __nv_bfloat16* D[2][GMI_MAX_HIDDEN] = {};  // dPre_l per layer (bf16 [Bm][w_p])
  __nv_bfloat16 *Gpi = nullptr, *Gv = nullptr;
  float* outh[2] = {};  // [Mrows][64] fp32 head outputs: mu (policy), v in column 0 (value)
  float* slab[2][GMI_MAX_HIDDEN] = {};
  float* colsum[2][GMI_MAX_HIDDEN] = {};
  float* head_slab[2] = {};
  int head_slab_parts[2] = {};  // fused head: per-net CTA count (value net in [1])
  float* head_part = nullptr;
  float* grad = nullptr;
  GemmParams fwd_roll[GMI_MAX_HIDDEN], fwd_val[GMI_MAX_HIDDEN], fwd_train[GMI_MAX_HIDDEN];
  GemmParams dw[GMI_MAX_HIDDEN], dx[GMI_MAX_HIDDEN], dhead;
  GemmParams head_roll, head_val, head_train, head_dx;  // head forward / input-grad GEMMs
  int bn_roll[GMI_MAX_HIDDEN] = {}, bn_val[GMI_MAX_HIDDEN] = {}, bn_fwd[GMI_MAX_HIDDEN] = {};
  int bn_dx[GMI_MAX_HIDDEN] = {}, bn_dw[GMI_MAX_HIDDEN] = {}, bn_head = 0, bn_hdx = 0;
  int ws_val[GMI_MAX_HIDDEN] = {}, ws_fwd[GMI_MAX_HIDDEN] = {}, ws_dx[GMI_MAX_HIDDEN] = {}, ws_hdx = 0;
  double flop_roll[GMI_MAX_HIDDEN] = {}, flop_fwd[GMI_MAX_HIDDEN] = {}, flop_dw[GMI_MAX_HIDDEN] = {},
         flop_dx[GMI_MAX_HIDDEN] = {}, flop_head = 0;
  std::vector<ppo::Segment> segs;
  bool fused_roll = false;
  int roll_cluster = 0;  // > 0: cluster rollout with this many CTAs per 128-env tile
  bool fused_val = false;
  ppo::ValueArgs val_args{};
  ppo::RolloutArgs roll_args{};
  bool fused_bias[GMI_MAX_HIDDEN] = {};  // bias gradient summed inside the layer's dW GEMM
  bool dw_pair[GMI_MAX_HIDDEN] = {};     // weight gradient on SM pairs (cuda/gemm_pair.cu)
  bool dx_halves[GMI_MAX_HIDDEN] = {};   // input gradient as 4 weight-stationary problems (N-halves)
  bool dw_grouped = false;               // dW of layers L-1 and L-2 in one launch (dw[L-1], 4 problems)
  bool dw_all = false;                   // dW of every layer in one launch (dw[L-1], 2L problems)
  bool fused_head = false;
  int head_grid = 0;
  ppo::HeadFusedArgs head_args{};
  bool fused_fwd = false;  // hidden forward + head step in one launch (train_fwd.cu)
  GemmParams fwd_chain{};  // all hidden forward layers (both nets) chained in one launch
  bool chain_fwd = false;
  // decoupled mode, nets too wide for the fused rollout / value kernels: the serving GMI's own
  // per-layer plans (channel observations, snapshot weights, its own activation buffers)
  bool srv_layers = false;
  int srv_ctas = 0;
  __nv_bfloat16* srv_H[2][GMI_MAX_HIDDEN] = {};
  float* srv_outh[2] = {};
  GemmParams srv_fwd_roll[GMI_MAX_HIDDEN], srv_fwd_val[GMI_MAX_HIDDEN], srv_head_roll, srv_head_val;
  int srv_bn_roll[GMI_MAX_HIDDEN] = {}, srv_bn_val[GMI_MAX_HIDDEN] = {}, srv_ws_val[GMI_MAX_HIDDEN] = {};
  ppo::TrainFwdArgs fwd_args{};
};

// ------------------------------------------------------------------ construction
// Everything the constructor acquires is released by release(), which is idempotent over
// partially built state, so a constructor that throws midway (OOM, infeasible green-context
// split, NCCL failure) leaks nothing (a GpuProfiler probe sweep keeps creating trainers).
Trainer::Trainer(const gmi_ppo_config_t& cfg, const void* nccl_id) : cfg_(cfg) {
  try {
    init(nccl_id);
  } catch (...) {
    release();
    throw;
  }
}

void Trainer::init(const void* nccl_id) {
  const gmi_ppo_config_t& cfg = cfg_;
  geo_ = Geometry::make(cfg);
  if (cfg.horizon < 1 || cfg.horizon > 32) invalid("horizon must be in [1, 32]");
  if (cfg.epochs < 1 || cfg.minibatches < 1) invalid("epochs and minibatches must be >= 1");
  if (cfg.num_gpus < 1 || cfg.gmis_per_gpu < 1) invalid("num_gpus and gmis_per_gpu must be >= 1");
  if (cfg.rank < 0 || cfg.rank >= cfg.num_gpus) invalid("rank out of range");
  if (cfg.decoupled < 0 || cfg.decoupled > 2) invalid("decoupled must be 0, 1 (per GPU) or 2 (across GPUs)");
  split_ = cfg.decoupled == 2;
  if (split_) {
    // AsyncDecoupled (mapping.hpp:265-276): serving GPUs first; 1:1 serving -> trainer pairs
    if (cfg.num_gpus < 2 || cfg.num_gpus % 2 != 0)
      invalid("decoupled = 2 (AsyncDecoupled across GPUs) needs an even num_gpus >= 2: ranks [0, G/2) serve, "
              "rank G/2 + s trains on serving rank s's experience");
    link_rank_ = cfg.rank;
    link_gpus_ = cfg.num_gpus;
    serving_ = cfg.rank < cfg.num_gpus / 2;
    cfg_.rank = cfg.rank % (cfg.num_gpus / 2);  // the pair's rank in the trainers' data-parallel job
    cfg_.num_gpus = cfg.num_gpus / 2;
  }
  if (geo_.A > ppo::kMaxAct) invalid("act_dim > 31 unsupported");
  if (geo_.S > 256) invalid("obs_dim > 256 unsupported");
  if (geo_.wp[geo_.L] > ppo::kMaxHeadIn) invalid("last hidden width > 512 unsupported");
  T_ = cfg.horizon;
  {
    // backward branch parallelism (GMI_BWD_PAR=1): measured neutral on B200 (the branches share
    // the same L2/HBM bandwidth), so it is opt-in
    const char* par = std::getenv("GMI_BWD_PAR");
    bwd_par_ = par && par[0] == '1';
    const char* share = std::getenv("GMI_BWD_DX_SHARE");  // percent of the GMI's SMs for dx
    if (share) bwd_dx_share_ = std::max(10, std::min(90, std::atoi(share)));
  }
  K_ = cfg.minibatches;
  n_local_ = cfg.gmis_per_gpu;
  n_total_ = cfg.num_gpus * cfg.gmis_per_gpu;
  if (cfg.num_envs < n_total_) invalid("fewer environments than GMIs");
  GMI_CUDA_CHECK(cudaSetDevice(cfg.device));
  decoupled_ = cfg.decoupled != 0;
  if (decoupled_) {
    // GMI 2r: simulator + agent (serving), GMI 2r+1: trainer (mapping.hpp:243-249 roles)
    if (n_local_ != 1) invalid("decoupled mode runs one trainer GMI per GPU (gmis_per_gpu = 1)");
    const int serving = cfg.serving_sms > 0 ? cfg.serving_sms : 16;
    // across GPUs the serving and trainer roles each own a whole GPU (plain streams)
    exec_ = std::make_unique<GmiResources>(cfg.device, std::vector<int>{serving, 0}, split_ ? 0 : cfg.gmi_backend);
    serve_s_ = exec_->stream(0);
    GMI_CUDA_CHECK(cudaEventCreateWithFlags(&ev_copied_, cudaEventDisableTiming));
    GMI_CUDA_CHECK(cudaEventCreateWithFlags(&ev_rolled_, cudaEventDisableTiming));
  } else {
    exec_ = std::make_unique<GmiResources>(cfg.device, n_local_, cfg.gmi_backend, cfg.sm_per_gmi);
  }
  const int tix = decoupled_ ? 1 : 0;  // execution-resource index of the first trainer GMI
  // decoupled, one GPU: the trainer's update stream (Adam, snapshot) stays inside its partition;
  // with NCCL in the update chain it stays in the primary context the communicator was made in
  // GMI_FORCE_NCCL=1 (tests): a one-rank communicator on a single GPU, so the NCCL all-reduce
  // in the captured iteration graph is exercised on one-GPU boxes (identity sum, bit-exact)
  const char* force = std::getenv("GMI_FORCE_NCCL");
  xchg_ = cfg.comm == 1 && !(split_ && serving_);  // serving ranks take no part in the update
  if (cfg.comm != 0 && cfg.comm != 1) invalid("comm must be 0 (NCCL) or 1 (peer exchange)");
  if (xchg_ && cfg.num_gpus > ppo::kMaxRanks) invalid("peer exchange supports up to 8 GPUs per job");
  const bool force_nccl = !xchg_ && cfg.num_gpus == 1 && force && force[0] == '1' && !split_;
  upd_in_gmi_ = decoupled_ && !split_ && cfg.num_gpus == 1 && !force_nccl;
  if (upd_in_gmi_)
    upd_ = exec_->extra_stream(1);
  else
    GMI_CUDA_CHECK(cudaStreamCreateWithFlags(&upd_, cudaStreamNonBlocking));
  GMI_CUDA_CHECK(cudaEventCreateWithFlags(&ev_adam_, cudaEventDisableTiming));
  GMI_CUDA_CHECK(cudaEventCreateWithFlags(&ev_start_, cudaEventDisableTiming));
  const int sms = device_sm_count();
  for (int i = 0; i < n_local_; ++i) {
    auto g = std::make_unique<Gmi>();
    g->local = i;
    g->gid = cfg.rank * n_local_ + i;
    g->env0 = int((long long)cfg.num_envs * g->gid / n_total_);
    g->N = int((long long)cfg.num_envs * (g->gid + 1) / n_total_) - g->env0;
    g->B = T_ * g->N;
    if (g->B % K_ != 0) invalid("horizon * envs per GMI must be divisible by minibatches");
    g->Bm = g->B / K_;
    if (g->Bm % 64 != 0) invalid("minibatch rows per GMI must be a multiple of 64 (use envs per GMI % 8 == 0)");
    g->Mrows = std::max(g->Bm, g->N);
    g->s = exec_->stream(tix + i);
    g->s2 = exec_->aux_stream(tix + i);
    g->ctas = exec_->sm_count(tix + i) > 0 ? exec_->sm_count(tix + i) : sms;
    gmis_.push_back(std::move(g));  // owned before its events exist (release() on failure)
    Gmi& gm = *gmis_.back();
    GMI_CUDA_CHECK(cudaEventCreateWithFlags(&gm.ev_done, cudaEventDisableTiming));
    GMI_CUDA_CHECK(cudaEventCreateWithFlags(&gm.ev_fork, cudaEventDisableTiming));
    for (auto& e : gm.ev_d) GMI_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  alloc();
  init_params();
  build_plans();
  ensure_bias_table(1 << 20);
  if (xchg_) {
    // Alg. 1 on the job layout (GPU-major ids, t per GPU) decides the cross-GPU fold order
    plan::Placement job;
    job.per_gpu.resize(cfg.num_gpus);
    for (int q = 0, id = 0; q < cfg.num_gpus; ++q)
      for (int j = 0; j < n_local_; ++j) job.per_gpu[q].push_back(id++);
    strategy_ = plan::choose_algo(job);
    if (n_local_ > ppo::kMaxLocalGmis) invalid("peer exchange supports up to 16 GMIs per GPU");
    xa_.mrr = strategy_ == plan::Algo::MRR ? 1 : 0;
    xa_.t = n_local_;
    xa_.G = cfg.num_gpus;
    xa_.rank = cfg.rank;
    xa_.P = geo_.P;
    for (int c = 0; c < cfg.num_gpus; ++c) xa_.chunk0[c] = geo_.P * c / cfg.num_gpus;
    for (int c = 0; c < n_local_; ++c) xa_.chunk0_t[c] = geo_.P * c / n_local_;
    xa_.lo = geo_.P * cfg.rank / cfg.num_gpus;
    xa_.hi = geo_.P * (cfg.rank + 1) / cfg.num_gpus;
    // one element per thread while the shard fits 1184 x 256 threads (latency-bound step: the
    // widest grid wins); same on every rank (the wait counts G x C flags)
    xa_.ctas = int(std::max<long long>(1, std::min<long long>(ppo::kMaxXchgCtas, (geo_.P / cfg.num_gpus + 255) / 256)));
    if (cfg.num_gpus == 1) {  // one rank: the exchange runs over the rank itself
      Trainer* self = this;
      comm_connect(&self, 1);
    }
  } else if ((cfg.num_gpus > 1 || force_nccl) && !(split_ && serving_)) {
    ncclUniqueId id;  // decoupled = 2: an id of the trainer ranks' communicator
    if (force_nccl) {
      NCCL_CHECK(ncclGetUniqueId(&id));
    } else {
      if (!nccl_id) invalid("nccl_id required when num_gpus > 1");
      std::memcpy(&id, nccl_id, sizeof(id));
    }
    ncclComm_t comm;
    NCCL_CHECK(ncclCommInitRank(&comm, cfg.num_gpus, id, cfg.rank));
    nccl_ = comm;
  }
  for (auto& g : gmis_) {
    ppo::EnvParams ep{g->N, geo_.S, geo_.A, geo_.wp[0], g->env0, T_, cfg_.seed};
    ppo::launch_env_init(ep, g->x, g->ep_step, g->ep_len, g->ep_count, decoupled_ ? g->ch_X : g->X_roll, g->s);
  }
  GMI_CUDA_CHECK(cudaEventRecord(ev_adam_, upd_));
  GMI_CUDA_CHECK(cudaDeviceSynchronize());
}

Trainer::~Trainer() { release(); }

void Trainer::release() noexcept {
  cudaDeviceSynchronize();
  if (graph_) cudaGraphExecDestroy(graph_);
  graph_ = nullptr;
  if (nccl_) ncclCommDestroy(static_cast<ncclComm_t>(nccl_));
  nccl_ = nullptr;
  for (void* p : ipc_opened_) cudaIpcCloseMemHandle(p);
  ipc_opened_.clear();
  for (auto& m : marks_) {
    cudaEventDestroy(m.a);
    cudaEventDestroy(m.b);
  }
  marks_.clear();
  for (auto& g : gmis_) {
    if (g->ev_done) cudaEventDestroy(g->ev_done);
    if (g->ev_fork) cudaEventDestroy(g->ev_fork);
    for (auto e : g->ev_d)
      if (e) cudaEventDestroy(e);
  }
  gmis_.clear();
  if (ev_copied_) cudaEventDestroy(ev_copied_);
  if (ev_rolled_) cudaEventDestroy(ev_rolled_);
  if (ev_adam_) cudaEventDestroy(ev_adam_);
  if (ev_start_) cudaEventDestroy(ev_start_);
  ev_copied_ = ev_rolled_ = ev_adam_ = ev_start_ = nullptr;
  if (upd_ && !upd_in_gmi_) cudaStreamDestroy(upd_);
  upd_ = nullptr;
  for (void* p : allocs_) cudaFree(p);
  allocs_.clear();
  for (void* p : plan_allocs_) cudaFree(p);
  plan_allocs_.clear();
  if (ctl_host_) cudaFreeHost(ctl_host_);
  if (stats_host_) cudaFreeHost(stats_host_);
  ctl_host_ = nullptr;
  stats_host_ = nullptr;
  exec_.reset();
}

// -1: the update stream; -2: the serving GMI's stream (decoupled); else GMI gmi's stream
cudaStream_t Trainer::stream(int gmi) const {
  if (gmi == -2) return serve_s_;
  return gmi < 0 ? upd_ : gmis_.at(gmi)->s;
}

void Trainer::alloc() {
  auto dev = [&](size_t bytes) {
    void* p = nullptr;
    GMI_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
    GMI_CUDA_CHECK(cudaMemset(p, 0, std::max<size_t>(bytes, 256)));
    allocs_.push_back(p);
    return p;
  };
  const long long P = geo_.P;
  if (xchg_) {
    // exchange window: [flags 16 KB | fold P fp32 | t GMI gradients P fp32 | params P fp32 |
    // shadow P bf16]; peers read the fold (HAR) or the GMI gradients (MRR)
    win_off_gmi_ = ppo::kXchgHeader + (size_t)P * 4;
    win_off_params_ = win_off_gmi_ + (size_t)n_local_ * P * 4;
    win_off_shadow_ = win_off_params_ + (size_t)P * 4;
    win_ = static_cast<char*>(dev(win_off_shadow_ + (size_t)P * 2));
    grad_sum_ = reinterpret_cast<float*>(win_ + ppo::kXchgHeader);
    params_ = reinterpret_cast<float*>(win_ + win_off_params_);
    shadow_ = reinterpret_cast<__nv_bfloat16*>(win_ + win_off_shadow_);
  } else {
    params_ = static_cast<float*>(dev(P * 4));
    grad_sum_ = static_cast<float*>(dev(P * 4));
    shadow_ = static_cast<__nv_bfloat16*>(dev(P * 2));
  }
  m_ = static_cast<float*>(dev(P * 4));
  v_ = static_cast<float*>(dev(P * 4));
  ctl_dev_ = static_cast<ppo::Control*>(dev(sizeof(ppo::Control)));
  stats_dev_ = static_cast<float*>(dev(8 * 4));
  GMI_CUDA_CHECK(cudaMallocHost(&ctl_host_, sizeof(ppo::Control)));
  GMI_CUDA_CHECK(cudaMallocHost(&stats_host_, 8 * 4));
  std::memset(ctl_host_, 0, sizeof(ppo::Control));
  std::memset(stats_host_, 0, 8 * 4);
  if (split_) {
    // link window, same layout on both ranks: [flags 4 KB: R @0 (trainer's), C @128, S @256
    // (serving's) | snapshot params P fp32 | shadow P bf16 | channel X | act | logp | adv | ret |
    // adv_stats] -- the part of the channel the trainer migrates
    const long long N = gmis_[0]->N, T = T_;
    size_t off = 4096;
    auto take = [&](size_t bytes) {
      const size_t o = off;
      off = (off + bytes + 255) / 256 * 256;
      return o;
    };
    loff_params_ = take(P * 4);
    loff_shadow_ = take(P * 2);
    loff_X_ = take((T + 1) * N * geo_.wp[0] * 2);
    loff_act_ = take(T * N * geo_.A * 4);
    loff_logp_ = take(T * N * 4);
    loff_adv_ = take(T * N * 4);
    loff_ret_ = take(T * N * 4);
    loff_stats_ = take(16);
    lwin_bytes_ = off;
    lwin_ = static_cast<char*>(dev(lwin_bytes_));
    lctr_ = static_cast<unsigned long long*>(dev(16 * 8));
  }
  if (decoupled_) {
    params_roll_ = split_ ? reinterpret_cast<float*>(lwin_ + loff_params_) : static_cast<float*>(dev(P * 4));
    shadow_roll_ = split_ ? reinterpret_cast<__nv_bfloat16*>(lwin_ + loff_shadow_)
                          : static_cast<__nv_bfloat16*>(dev(P * 2));
    ctl_roll_ = static_cast<ppo::Control*>(dev(sizeof(ppo::Control)));
  }

  const int S_p = geo_.wp[0], A = geo_.A, L = geo_.L;
  int maxw = 0;
  for (int l = 1; l <= L; ++l) maxw = std::max(maxw, geo_.wp[l]);
  for (auto& gp : gmis_) {
    Gmi& g = *gp;
    const long long N = g.N, T = T_, B = g.B;
    g.x = static_cast<float*>(dev(N * geo_.S * 4));
    g.ep_step = static_cast<int*>(dev(N * 4));
    g.ep_len = static_cast<int*>(dev(N * 4));
    g.ep_count = static_cast<int*>(dev(N * 4));
    g.X_roll = static_cast<__nv_bfloat16*>(dev((T + 1) * N * S_p * 2));
    g.act = static_cast<float*>(dev(T * N * A * 4));
    g.logp = static_cast<float*>(dev(T * N * 4));
    g.rew = static_cast<float*>(dev(T * N * 4));
    g.done = static_cast<uint8_t*>(dev(T * N));
    if (decoupled_ && split_) {
      g.ch_X = reinterpret_cast<__nv_bfloat16*>(lwin_ + loff_X_);
      g.ch_act = reinterpret_cast<float*>(lwin_ + loff_act_);
      g.ch_logp = reinterpret_cast<float*>(lwin_ + loff_logp_);
      g.ch_adv = reinterpret_cast<float*>(lwin_ + loff_adv_);
      g.ch_ret = reinterpret_cast<float*>(lwin_ + loff_ret_);
      g.ch_adv_stats = reinterpret_cast<float*>(lwin_ + loff_stats_);
    } else if (decoupled_) {
      g.ch_X = static_cast<__nv_bfloat16*>(dev((T + 1) * N * S_p * 2));
      g.ch_act = static_cast<float*>(dev(T * N * A * 4));
      g.ch_logp = static_cast<float*>(dev(T * N * 4));
      g.ch_adv = static_cast<float*>(dev(T * N * 4));
      g.ch_ret = static_cast<float*>(dev(T * N * 4));
      g.ch_adv_stats = static_cast<float*>(dev(4 * 4));
    }
    if (decoupled_) {
      g.ch_rew = static_cast<float*>(dev(T * N * 4));
      g.ch_done = static_cast<uint8_t*>(dev(T * N));
      g.ch_V = static_cast<float*>(dev((T + 1) * N * 4));
      g.ch_gae_part = static_cast<double*>(dev(ppo::gae_blocks(g.N) * 3 * 8));
    }
    g.V = static_cast<float*>(dev((T + 1) * N * 4));
    g.adv = static_cast<float*>(dev(T * N * 4));
    g.ret = static_cast<float*>(dev(T * N * 4));
    g.gae_part = static_cast<double*>(dev(ppo::gae_blocks(g.N) * 3 * 8));
    g.adv_stats = static_cast<float*>(dev(4 * 4));
    g.X_sh = static_cast<__nv_bfloat16*>(dev(B * S_p * 2));
    g.act_sh = static_cast<float*>(dev(B * A * 4));
    g.oldlp_sh = static_cast<float*>(dev(B * 4));
    g.adv_sh = static_cast<float*>(dev(B * 4));
    g.ret_sh = static_cast<float*>(dev(B * 4));
    for (int n = 0; n < 2; ++n) {
      for (int l = 0; l < L; ++l) g.H[n][l] = static_cast<__nv_bfloat16*>(dev((long long)g.Mrows * geo_.wp[l + 1] * 2));
      for (int l = 0; l < L; ++l) g.D[n][l] = static_cast<__nv_bfloat16*>(dev((long long)g.Bm * maxw * 2));
    }
    g.Gpi = static_cast<__nv_bfloat16*>(dev((long long)g.Bm * ppo::kHeadG * 2));
    g.Gv = static_cast<__nv_bfloat16*>(dev((long long)g.Bm * ppo::kHeadG * 2));
    for (int n = 0; n < 2; ++n) g.outh[n] = static_cast<float*>(dev((long long)g.Mrows * ppo::kHeadG * 4));
    // peer exchange: GMI gradients live in the exchange window (MRR reads them remotely)
    g.grad = xchg_ ? reinterpret_cast<float*>(win_ + win_off_gmi_ + (size_t)g.local * P * 4)
                   : static_cast<float*>(dev(P * 4));
    g.head_part = static_cast<float*>(dev((long long)ppo::head_loss_blocks(g.Bm) * ppo::head_partial_stride(A) * 4));
  }
}

void Trainer::init_params() {
  const long long P = geo_.P;
  std::vector<float> p(P, 0.f);
  for (int n = 0; n < 2; ++n)
    for (int l = 0; l <= geo_.L; ++l) {
      const Tensor& t = geo_.net[n][l];
      const float bound = 1.0f / std::sqrt(float(t.in));
      const uint32_t wid = uint32_t((n * 16 + l) * 2), bid = wid + 1;
      for (int r = 0; r < t.out; ++r) {
        for (int k = 0; k < t.in; ++k) {
          uint32_t o[4];
          rng::draw(cfg_.seed, wid, uint32_t(r * t.in + k), 0, rng::kInit, o);
          const float u2 = rng::u01(o[0]) * 2.0f;
          p[t.w + (long long)r * t.in_p + k] = (u2 - 1.0f) * bound;
        }
        uint32_t o[4];
        rng::draw(cfg_.seed, bid, uint32_t(r), 0, rng::kInit, o);
        const float u2 = rng::u01(o[0]) * 2.0f;
        p[t.b + r] = (u2 - 1.0f) * bound;
      }
    }
  set("params", -1, p.data(), P);
}

// ------------------------------------------------------------------ GEMM descriptors
void Trainer::build_plans() {
  const int L = geo_.L, S_p = geo_.wp[0], A = geo_.A, hp = geo_.wp[L];
  // Kernel-written scratch (slabs, partial rows). GMI_POISON=1 fills it with NaN bytes so a
  // read-before-write shows up in the parity tests instead of depending on allocator history.
  const char* poison = std::getenv("GMI_POISON");
  // plan scratch depends on the GMIs' SM counts: a rebuild (gmi_resize) frees the previous set
  for (void* p : plan_allocs_) cudaFree(p);
  plan_allocs_.clear();
  auto dev = [&](size_t bytes) {
    void* p = nullptr;
    GMI_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
    if (poison && poison[0] == '1') GMI_CUDA_CHECK(cudaMemset(p, 0xFF, std::max<size_t>(bytes, 256)));
    plan_allocs_.push_back(p);
    return static_cast<float*>(p);
  };
  for (auto& gp : gmis_) {
    Gmi& g = *gp;
    g.segs.clear();
    // wide weight-stationary layers (128-column parts), per GEMM family and resident K:
    // bit 0 forward K <= 256, bit 1 forward K <= 512, bit 2 input gradient K <= 256, bit 3 input
    // gradient K <= 512 (GMI_WS_WIDE overrides, for measurements)
    int wide_mask = kWideDefault;
    if (const char* e = std::getenv("GMI_WS_WIDE")) wide_mask = std::atoi(e);
    const long long rollrows = (long long)(T_ + 1) * g.N;
    for (int l = 0; l < L; ++l) {
      const int in_p = geo_.wp[l], out_p = geo_.wp[l + 1];
      const double real = 2.0 * geo_.net[0][l].out * geo_.net[0][l].in;
      auto fwd_problem = [&](int n, const CUtensorMap& amap, int M, int bn) {
        GemmProblem p{};
        p.map_a = amap;
        p.map_b = tma_kmajor(shadow_ + geo_.net[n][l].w, in_p, out_p, in_p, bn);
        p.map_out = make_tma_out_bf16(g.H[n][l], out_p, g.Mrows, out_p);
        p.bias = params_ + geo_.net[n][l].b;
        p.M = M;
        p.N = out_p;
        p.K = in_p;
        p.kb_per_split = (in_p + kGemmBlockK - 1) / kGemmBlockK;
        return p;
      };
      // rollout (policy, M = N envs) and value forward (value net, chunks of Mrows rows)
      // read observation slots of X_roll through a row offset per launch.
      // per-step rollout GEMMs (M = envs, latency-bound chains of 3-5 launches per env step):
      // 128-wide tiles measured best on B200 (HM 8192 envs: rollout GEMMs 1.17 -> 1.06 ms per
      // iteration vs 64; SH 4096 envs: 1.63 -> 1.49 ms; 256 is slower than both)
      g.bn_roll[l] = out_p >= 128 ? 128 : gemm_choose_bn(g.N, out_p, 1, 1, g.ctas);
      const CUtensorMap a_roll = l == 0 ? tma_kmajor(g.X_roll, S_p, rollrows, S_p, kGemmBlockM)
                                        : tma_kmajor(g.H[0][l - 1], in_p, g.Mrows, in_p, kGemmBlockM);
      g.fwd_roll[l] = GemmParams{};
      g.fwd_roll[l].prob[0] = fwd_problem(0, a_roll, g.N, g.bn_roll[l]);
      g.fwd_roll[l].num_problems = 1;
      g.fwd_roll[l].splits = 1;
      // weight-stationary where every CTA gets a tile (weights loaded once per CTA)
      const int ws_val = gemm_ws_bn(g.Mrows, out_p, in_p, 1, g.ctas);
      g.ws_val[l] = ws_val > 0;
      g.bn_val[l] = ws_val > 0 ? ws_val : gemm_choose_bn(g.Mrows, out_p, 1, 1, g.ctas);
      const CUtensorMap a_val = l == 0 ? tma_kmajor(g.X_roll, S_p, rollrows, S_p, kGemmBlockM)
                                       : tma_kmajor(g.H[1][l - 1], in_p, g.Mrows, in_p, kGemmBlockM);
      g.fwd_val[l] = GemmParams{};
      g.fwd_val[l].prob[0] = fwd_problem(1, a_val, g.Mrows, g.bn_val[l]);
      g.fwd_val[l].num_problems = 1;
      g.fwd_val[l].splits = 1;
      // training forward: both nets grouped over the minibatch rows of the epoch copy
      const int ws_fwd = gemm_ws_bn(g.Bm, out_p, in_p, 2, g.ctas);
      // layers too wide for that (HM 400 / SH 512 widths): weight-stationary over 128-column
      // parts of the output, one problem per (net, part), the part's weights resident (K <= 512)
      int fparts = 1;
      int ws_fwide = ws_fwd > 0 ? 0 : gemm_ws_wide(g.Bm, out_p, in_p, 2, g.ctas, &fparts);
      if (ws_fwide && !(wide_mask >> (ws_fwide - 1) & 1)) ws_fwide = 0, fparts = 1;
      g.ws_fwd[l] = ws_fwd > 0 ? 1 : ws_fwide;
      g.bn_fwd[l] = ws_fwd > 0 ? ws_fwd : ws_fwide ? 128 : gemm_choose_bn(g.Bm, out_p, 2, 1, g.ctas);
      g.fwd_train[l] = GemmParams{};
      for (int n = 0; n < 2; ++n) {
        const CUtensorMap a = l == 0 ? tma_kmajor(g.X_sh, S_p, g.B, S_p, kGemmBlockM)
                                     : tma_kmajor(g.H[n][l - 1], in_p, g.Mrows, in_p, kGemmBlockM);
        if (!ws_fwide) {
          g.fwd_train[l].prob[n] = fwd_problem(n, a, g.Bm, g.bn_fwd[l]);
          continue;
        }
        for (int j = 0; j < fparts; ++j) {
          const int c0 = 128 * j, nc = std::min(128, out_p - c0);
          GemmProblem p{};
          p.map_a = a;
          p.map_b = tma_kmajor(shadow_ + geo_.net[n][l].w + (long long)c0 * in_p, in_p, nc, in_p, 128);
          p.map_out = make_tma_out_bf16(g.H[n][l] + c0, nc, g.Mrows, out_p);
          p.bias = params_ + geo_.net[n][l].b + c0;
          p.M = g.Bm;
          p.N = nc;
          p.K = in_p;
          p.kb_per_split = (in_p + kGemmBlockK - 1) / kGemmBlockK;
          g.fwd_train[l].prob[n * fparts + j] = p;
        }
      }
      g.fwd_train[l].num_problems = 2 * fparts;
      g.fwd_train[l].splits = 1;
      g.flop_roll[l] = real * g.N;
      g.flop_fwd[l] = 2.0 * real * g.Bm;

      // weight gradient dW_l[out_p][in_p] = sum_rows dPre_l^T in_l (both operands MN-major)
      const int bnw = in_p <= 64 ? 64 : in_p <= 128 ? 128 : 256;  // instantiated block widths
      g.bn_dw[l] = bnw;
      int splits = 1, kbps = 1;
      // backward branch parallelism: the dW launches get the SMs the dx branch leaves
      const int dw_sms = bwd_par_ ? std::max(1, g.ctas - std::max(1, g.ctas * bwd_dx_share_ / 100)) : g.ctas;
      pick_splits(out_p, in_p, bnw, 2, g.Bm, dw_sms, &splits, &kbps);
      g.dw[l] = GemmParams{};
      for (int n = 0; n < 2; ++n) {
        g.slab[n][l] = dev((size_t)splits * out_p * in_p * 4);
        g.colsum[n][l] = dev((size_t)std::max(ppo::colsum_blocks(g.Bm), splits) * out_p * 4);
        GemmProblem p{};
        p.map_a = tma_mnmajor(g.D[n][l], out_p, g.Bm, out_p);
        p.map_b = l == 0 ? tma_mnmajor(g.X_sh, S_p, g.B, S_p) : tma_mnmajor(g.H[n][l - 1], in_p, g.Bm, in_p);
        p.map_out = make_tma_out_f32(g.slab[n][l], in_p, out_p, splits, in_p, (uint64_t)out_p * in_p);
        p.colsum = g.colsum[n][l];  // bias gradient of layer l: column sums of dPre_l per split
        p.M = out_p;
        p.N = in_p;
        p.K = g.Bm;
        p.kb_per_split = kbps;
        g.dw[l].prob[n] = p;
      }
      g.dw[l].num_problems = 2;
      g.dw[l].splits = splits;
      g.fused_bias[l] = true;
      // 256 x 256 layers, opt-in (GMI_DW_PAIR=1): SM-pair kernel (tcgen05 cta_group::2,
      // cuda/gemm_pair.cu), same slabs. It cuts L2->SM traffic by a third (ncu: 67 vs 100 MB per
      // launch) but measured slower on B200 (25.9 vs 20.3 us per launch), so it is off by default.
      const char* pair_on = std::getenv("GMI_DW_PAIR");
      g.dw_pair[l] = gemm_pair_applicable(out_p, in_p, 1, 1, EPI_F32) && pair_on && pair_on[0] == '1';
      if (g.dw_pair[l]) {  // one (problem, split) tile per co-resident SM pair: a single wave
        const int pairs = std::max(2, std::min(gemm_pair_max_clusters(), g.ctas / 2));
        const int nkb = (g.Bm + kGemmBlockK - 1) / kGemmBlockK;
        const int per = (nkb + pairs / 2 - 1) / (pairs / 2);
        for (int n = 0; n < 2; ++n) g.dw[l].prob[n].kb_per_split = per;
        g.dw[l].splits = (nkb + per - 1) / per;
      }
      g.flop_dw[l] = 2.0 * real * g.Bm;

      // input gradient dPre_{l-1} = (dPre_l W_l) * elu'(H_{l-1}); W_l read MN-major
      if (l > 0) {
        // input gradients stream W with the dPre tiles: measured faster than weight-stationary here
        // (the elu' operand already doubles the activation traffic; WS has one staging buffer)
        // Default for 256-wide inputs: weight-stationary over four problems (2 nets x 2 N-halves
        // of 128 columns): each CTA keeps one 256 x 128 weight half resident and streams only the
        // dPre tiles, with one 32-column chunk per epilogue warp per tile.
        const char* dx4_off = std::getenv("GMI_DX_WS4_OFF");
        g.dx_halves[l] = in_p == 256 && out_p <= 256 && !(dx4_off && dx4_off[0] == '1') &&
                         gemm_ws_bn(g.Bm, 128, out_p, 4, g.ctas) == 128;
        int ws_dx = g.dx_halves[l] ? 128 : std::getenv("GMI_DX_WS") ? gemm_ws_bn(g.Bm, in_p, out_p, 2, g.ctas) : 0;
        // wide layers (in_p or out_p > 256): weight-stationary over 128-column parts of dPre_{l-1}
        int halves = g.dx_halves[l] ? 2 : 1;
        int ws_dxwide = ws_dx > 0 || (in_p <= 256 && out_p <= 256) ? 0 : gemm_ws_wide(g.Bm, in_p, out_p, 2, g.ctas, &halves);
        if (ws_dxwide && !(wide_mask >> (ws_dxwide + 1) & 1)) ws_dxwide = 0, halves = 1;
        if (ws_dxwide) ws_dx = 128;
        g.ws_dx[l] = ws_dxwide ? ws_dxwide : ws_dx > 0 ? 1 : 0;
        g.bn_dx[l] = ws_dx > 0 ? ws_dx : gemm_choose_bn(g.Bm, in_p, 2, 1, g.ctas);
        if (const char* bn = std::getenv("GMI_DX_BN"); bn && ws_dx == 0) g.bn_dx[l] = std::atoi(bn);  // experiments
        g.dx[l] = GemmParams{};
        const int ncols_full = ws_dxwide ? 128 : in_p / halves;
        for (int n = 0; n < 2; ++n)
          for (int hh = 0; hh < halves; ++hh) {
            const int c0 = hh * ncols_full, ncols = std::min(ncols_full, in_p - c0);
            GemmProblem p{};
            p.map_a = tma_kmajor(g.D[n][l], out_p, g.Bm, out_p, kGemmBlockM);
            p.map_b = tma_mnmajor(shadow_ + geo_.net[n][l].w + c0, ncols, out_p, in_p);
            p.map_out = make_tma_out_bf16(g.D[n][l - 1] + c0, ncols, g.Bm, in_p);
            p.aux = g.H[n][l - 1] + c0;
            p.ld_aux = in_p;
            p.map_aux = tma_aux(p.aux, ncols, g.Bm, in_p);
            p.M = g.Bm;
            p.N = ncols;
            p.K = out_p;
            p.kb_per_split = (out_p + kGemmBlockK - 1) / kGemmBlockK;
            g.dx[l].prob[n * halves + hh] = p;
          }
        g.dx[l].num_problems = 2 * halves;
        g.dx[l].splits = 1;
        g.flop_dx[l] = 2.0 * real * g.Bm;
      }
    }
    // heads on the tensor cores. Forward: mu = H_L W_mu^T (N padded to 64, rows >= A read as
    // zero by TMA), v = H^v_L w_v^T; fp32 outputs, bias added by the consumer kernels.
    const int head_rows[2] = {A, 1};
    auto head_fwd = [&](int n, int M, const CUtensorMap& amap) {
      GemmProblem p{};
      p.map_a = amap;
      p.map_b = tma_kmajor(shadow_ + geo_.net[n][L].w, hp, head_rows[n], hp, 64);
      p.map_out = make_tma_out_f32(g.outh[n], ppo::kHeadG, g.Mrows, 1, ppo::kHeadG, (uint64_t)g.Mrows * ppo::kHeadG);
      p.M = M;
      p.N = ppo::kHeadG;
      p.K = hp;
      p.kb_per_split = (hp + kGemmBlockK - 1) / kGemmBlockK;
      return p;
    };
    g.head_roll = GemmParams{};
    g.head_roll.prob[0] = head_fwd(0, g.N, tma_kmajor(g.H[0][L - 1], hp, g.Mrows, hp, kGemmBlockM));
    g.head_roll.num_problems = 1;
    g.head_roll.splits = 1;
    g.head_val = GemmParams{};
    g.head_val.prob[0] = head_fwd(1, g.Mrows, tma_kmajor(g.H[1][L - 1], hp, g.Mrows, hp, kGemmBlockM));
    g.head_val.num_problems = 1;
    g.head_val.splits = 1;
    g.head_train = GemmParams{};
    for (int n = 0; n < 2; ++n)
      g.head_train.prob[n] = head_fwd(n, g.Bm, tma_kmajor(g.H[n][L - 1], hp, g.Mrows, hp, kGemmBlockM));
    g.head_train.num_problems = 2;
    g.head_train.splits = 1;
    // Head input gradient: dPre_{L-1} = (G W_head) * elu'(H_L), K = 64 (zero-padded G).
    const int ws_hdx = gemm_ws_bn(g.Bm, hp, ppo::kHeadG, 2, g.ctas);
    g.ws_hdx = ws_hdx > 0;
    g.bn_hdx = ws_hdx > 0 ? ws_hdx : gemm_choose_bn(g.Bm, hp, 2, 1, g.ctas);
    g.head_dx = GemmParams{};
    {
      const __nv_bfloat16* G[2] = {g.Gpi, g.Gv};
      for (int n = 0; n < 2; ++n) {
        GemmProblem p{};
        p.map_a = tma_kmajor(G[n], ppo::kHeadG, g.Bm, ppo::kHeadG, kGemmBlockM);
        p.map_b = tma_mnmajor(shadow_ + geo_.net[n][L].w, hp, head_rows[n], hp);
        p.map_out = make_tma_out_bf16(g.D[n][L - 1], hp, g.Bm, hp);
        p.aux = g.H[n][L - 1];
        p.ld_aux = hp;
        p.map_aux = tma_aux(p.aux, hp, g.Bm, hp);
        p.M = g.Bm;
        p.N = hp;
        p.K = ppo::kHeadG;
        p.kb_per_split = 1;
        g.head_dx.prob[n] = p;
      }
      g.head_dx.num_problems = 2;
      g.head_dx.splits = 1;
    }
    // head weight gradients on the tensor cores: dW_mu = G_pi^T H_L, dw_v = G_v^T H^v_L
    const int bnh = hp <= 64 ? 64 : hp <= 128 ? 128 : 256;
    g.bn_head = bnh;
    int hsplits = 1, hkbps = 1;
    pick_splits(A, hp, bnh, 2, g.Bm, g.ctas, &hsplits, &hkbps);
    g.head_slab[0] = dev((size_t)hsplits * A * hp * 4);
    g.head_slab[1] = dev((size_t)hsplits * hp * 4);
    g.dhead = GemmParams{};
    const __nv_bfloat16* G[2] = {g.Gpi, g.Gv};
    for (int n = 0; n < 2; ++n) {
      GemmProblem p{};
      p.map_a = tma_mnmajor(G[n], ppo::kHeadG, g.Bm, ppo::kHeadG);
      p.map_b = tma_mnmajor(g.H[n][L - 1], hp, g.Bm, hp);
      const int rows = n == 0 ? A : 1;
      p.map_out = make_tma_out_f32(g.head_slab[n], hp, rows, hsplits, hp, (uint64_t)rows * hp);
      p.M = A;  // both problems share the tile grid; the value map clips to one row
      p.N = hp;
      p.K = g.Bm;
      p.kb_per_split = hkbps;
      g.dhead.prob[n] = p;
    }
    g.dhead.num_problems = 2;
    g.dhead.splits = hsplits;
    g.flop_head = 2.0 * (A + 1) * double(geo_.width[L]) * g.Bm;

    // fused head (forward + loss + head input / weight gradients + bias sums of layer L-1)
    const char* head_unfused = std::getenv("GMI_HEAD_UNFUSED");
    g.fused_head = ppo::head_fusable(hp, A) && !(head_unfused && head_unfused[0] == '1');
    int head_parts = ppo::head_loss_blocks(g.Bm), hslab_parts = hsplits;
    if (g.fused_head) {
      g.head_grid = ppo::head_fused_grid(g.Bm, g.ctas);
      ppo::HeadFusedArgs& h = g.head_args;
      // the opt-in fused training forward maps nets as CTA b -> net b % 2: even split there
      const char* tf = std::getenv("GMI_TRAIN_FWD");
      h.npol = tf && tf[0] == '1' ? g.head_grid / 2 : ppo::head_fused_npol(g.head_grid, A);
      const int net_ctas[2] = {h.npol, g.head_grid - h.npol};
      const int per_net = std::max(net_ctas[0], net_ctas[1]);
      for (int n = 0; n < 2; ++n) {
        ppo::HeadNet& hn = h.net[n];
        hn.n_out = head_rows[n];
        hn.nh = hn.n_out <= 16 ? 16 : 32;
        hn.map_h = tma_kmajor(g.H[n][L - 1], hp, g.Bm, hp, kGemmBlockM);
        hn.map_wk = tma_kmajor(shadow_ + geo_.net[n][L].w, hp, hn.n_out, hp, hn.nh);
        hn.map_wm = make_tma_2d_bf16(shadow_ + geo_.net[n][L].w, hp, hn.n_out, hp, 64, 32);  // [32 K][64 N]
        hn.map_d = make_tma_out_bf16(g.D[n][L - 1], hp, g.Bm, hp);
        hn.bias = params_ + geo_.net[n][L].b;
        g.head_slab[n] = dev((size_t)per_net * hn.n_out * hp * 4);
        hn.dw_slab = g.head_slab[n];
      }
      h.log_std = params_ + geo_.log_std;
      h.act = g.act_sh;
      h.oldlp = g.oldlp_sh;
      h.adv = g.adv_sh;
      h.ret = g.ret_sh;
      g.head_part = dev((size_t)g.head_grid * ppo::head_partial_stride(A) * 4);  // one record per CTA
      h.part = g.head_part;
      h.Bm = g.Bm;
      h.A = A;
      h.hp = hp;
      h.clip = cfg_.clip;
      h.vf_coef = cfg_.vf_coef;
      h.ent_coef = cfg_.ent_coef;
      head_parts = g.head_grid;
      hslab_parts = net_ctas[0];
      g.head_slab_parts[1] = net_ctas[1];
      const char* htr = std::getenv("GMI_HEAD_TRACE");
      if (htr && htr[0] == '1' && !head_trace_) {
        head_trace_ = dev(64 * 8);
        ppo::head_fused_set_trace(static_cast<unsigned long long*>(head_trace_));
      }
      // whole training forward + head step on chip (same per-CTA records as the head kernel).
      // Opt-in (GMI_TRAIN_FWD=1): bit-identical, but with one tile in flight per CTA its MMA ->
      // epilogue chain is serial and it measured slower on B200 than the per-layer GEMMs plus
      // the fused head kernel, which overlap through PDL (3.65 vs 3.37 ms per iteration).
      // chained training forward (gemm.cuh, GemmParams::chain): every hidden layer weight-stationary
      // with the same full-width block N, so each CTA carries its row tiles through all layers
      const char* nochain = std::getenv("GMI_FWD_CHAIN");
      g.chain_fwd = !(nochain && nochain[0] == '0') && 2 * L <= kGemmMaxProblems;
      for (int l = 0; l < L; ++l)
        g.chain_fwd = g.chain_fwd && g.ws_fwd[l] == 1 && g.bn_fwd[l] == g.bn_fwd[0] && geo_.wp[l + 1] == g.bn_fwd[0];
      if (g.chain_fwd) {
        g.fwd_chain = GemmParams{};
        for (int l = 0; l < L; ++l)
          for (int n = 0; n < 2; ++n) g.fwd_chain.prob[2 * l + n] = g.fwd_train[l].prob[n];
        g.fwd_chain.num_problems = 2;
        g.fwd_chain.splits = 1;
        g.fwd_chain.chain = L;
      }
      const char* fwd_on = std::getenv("GMI_TRAIN_FWD");
      g.fused_fwd = ppo::train_fwd_fusable(L, geo_.wp.data(), S_p, A) && fwd_on && fwd_on[0] == '1';
      if (g.fused_fwd) {
        ppo::TrainFwdArgs& f = g.fwd_args;
        f.map_x = tma_kmajor(g.X_sh, S_p, (long long)g.B, S_p, kGemmBlockM);
        for (int n = 0; n < 2; ++n) {
          ppo::TrainFwdNet& fn = f.net[n];
          for (int l = 0; l < L; ++l) {
            const Tensor& t = geo_.net[n][l];
            fn.map_w[l] = tma_kmajor(shadow_ + t.w, t.in_p, t.out_p, t.in_p, t.out_p);
            fn.bias[l] = params_ + t.b;
            fn.in_p[l] = t.in_p;
            fn.out_n[l] = t.out_p;
            if (l < L - 1) fn.map_h[l] = tma_kmajor(g.H[n][l], t.out_p, g.Bm, t.out_p, 32);
          }
          const ppo::HeadNet& hn = h.net[n];
          fn.n_out = hn.n_out;
          fn.nh = hn.nh;
          fn.map_w[L] = tma_kmajor(shadow_ + geo_.net[n][L].w, hp, hn.n_out, hp, hn.nh);
          fn.map_wm = make_tma_2d_bf16(shadow_ + geo_.net[n][L].w, hp, hn.n_out, hp, 64, 32);
          fn.map_d = tma_kmajor(g.D[n][L - 1], hp, g.Bm, hp, 32);
          fn.bias[L] = params_ + geo_.net[n][L].b;
          fn.in_p[L] = hp;
          fn.out_n[L] = hn.nh;
          fn.dw_slab = hn.dw_slab;
        }
        f.log_std = h.log_std;
        f.act = h.act;
        f.oldlp = h.oldlp;
        f.adv = h.adv;
        f.ret = h.ret;
        f.part = h.part;
        f.Bm = g.Bm;
        f.A = A;
        f.L = L;
        f.hp = hp;
        f.S_p = S_p;
        f.clip = cfg_.clip;
        f.vf_coef = cfg_.vf_coef;
        f.ent_coef = cfg_.ent_coef;
        const char* trace = std::getenv("GMI_TRAIN_FWD_TRACE");
        if (trace && trace[0] == '1') f.trace = reinterpret_cast<unsigned long long*>(dev(64 * 8));
      }
    }

    // Weight gradients of the last two hidden layers in one grouped launch (4 problems: 2 nets x
    // 2 layers) once dPre of both exist (after dx(L-1)): half the split-K slabs for the same
    // grid (splits 37 -> 18 at 256 x 256), so half the slab writes and gradient-assembly reads,
    // and one launch ramp/tail less per minibatch. GMI_DW_GROUP=0 keeps one launch per layer.
    {
      const char* grp = std::getenv("GMI_DW_GROUP");
      const int a = L - 1, b = L - 2;
      g.dw_grouped = L >= 3 && !(grp && grp[0] == '0') && !bwd_par_ && !g.dw_pair[a] && !g.dw_pair[b] &&
                     geo_.wp[a + 1] == geo_.wp[a] && geo_.wp[a] == geo_.wp[b];
      if (g.dw_grouped) {
        const int out_p = geo_.wp[a + 1], in_p = geo_.wp[a];
        int splits = 1, kbps = 1;
        pick_splits(out_p, in_p, g.bn_dw[a], 4, g.Bm, g.ctas, &splits, &kbps);
        GemmParams P{};
        for (int j = 0; j < 4; ++j) {
          const int l = j < 2 ? a : b, n = j & 1;
          GemmProblem p = g.dw[l].prob[n];
          p.map_out = make_tma_out_f32(g.slab[n][l], in_p, out_p, splits, in_p, (uint64_t)out_p * in_p);
          p.kb_per_split = kbps;
          P.prob[j] = p;
        }
        P.num_problems = 4;
        P.splits = splits;
        g.dw[a] = P;
        g.dw[b].splits = splits;
        g.flop_dw[a] += g.flop_dw[b];
      }
      // Every layer in one launch (GMI_DW_ALL=0 keeps the pair above + a layer-0 launch): when
      // all hidden widths are equal (same M) and every input fits one block N, the first layer's
      // problems (N = S_p, narrower) join the group after the last input gradient; their B tiles
      // are zero-filled past S_p by TMA. One launch ramp / tail and one split-K slab set less per
      // minibatch (AT: splits 18 + 37 -> 12 for 2 x 3 problems).
      const char* all_env = std::getenv("GMI_DW_ALL");
      bool all = g.dw_grouped && L >= 2 && 2 * L <= kGemmMaxProblems && !(all_env && all_env[0] == '0');
      for (int l = 0; l < L && all; ++l)
        all = geo_.wp[l + 1] == geo_.wp[L] && geo_.wp[l] <= g.bn_dw[a] && !g.dw_pair[l] && g.fused_bias[l];
      g.dw_all = all;
      if (all) {
        const int out_p = geo_.wp[L];
        int splits = 1, kbps = 1;
        pick_splits(out_p, g.bn_dw[a], g.bn_dw[a], 2 * L, g.Bm, g.ctas, &splits, &kbps);
        GemmParams P{};
        for (int l = L - 1, j = 0; l >= 0; --l)
          for (int n = 0; n < 2; ++n, ++j) {
            const int in_p = geo_.wp[l];
            // the per-layer problem as planned above (grouped layers: from the pair launch)
            GemmProblem p = g.dw_grouped && (l == a || l == b) ? g.dw[a].prob[(l == a ? 0 : 2) + n] : g.dw[l].prob[n];
            p.map_out = make_tma_out_f32(g.slab[n][l], in_p, out_p, splits, in_p, (uint64_t)out_p * in_p);
            p.kb_per_split = kbps;
            P.prob[j] = p;
          }
        P.num_problems = 2 * L;
        P.splits = splits;
        double flop = 0;
        for (int l = 0; l < L; ++l) {
          if (!(g.dw_grouped && l == b)) flop += g.flop_dw[l];
          g.dw[l].splits = splits;
        }
        g.dw[a] = P;
        g.flop_dw[a] = flop;
      }
    }
    // Layers of different widths (HM 200-400-100, SH 512-512-512-256): every layer's weight
    // gradient still in one launch after the last input gradient, as a heterogeneous split-K
    // group (each problem its own M x N tiles of block N 256, one split count for all), instead
    // of one launch per layer (GMI_DW_HETERO=0 keeps those).
    if (!g.dw_all && L >= 2 && 2 * L <= kGemmMaxProblems && !bwd_par_) {
      const char* he = std::getenv("GMI_DW_HETERO");
      bool het = !(he && he[0] == '0');
      for (int l = 0; l < L && het; ++l) het = !g.dw_pair[l] && g.fused_bias[l];
      if (het) {
        constexpr int bn = 256;
        int base = 0;
        for (int l = 0; l < L; ++l) base += 2 * gemm_tiles(geo_.wp[l + 1], geo_.wp[l], bn, 1, 1);
        const int nkb = (g.Bm + kGemmBlockK - 1) / kGemmBlockK;
        const int s0 = std::max(1, std::min(nkb, g.ctas / std::max(1, base)));
        const int kbps = (nkb + s0 - 1) / s0, splits = (nkb + kbps - 1) / kbps;
        GemmParams P{};
        double flop = 0;
        for (int l = L - 1, j = 0; l >= 0; --l) {
          const int in_p = geo_.wp[l], out_p = geo_.wp[l + 1];
          for (int n = 0; n < 2; ++n, ++j) {
            GemmProblem p = g.dw[l].prob[n];
            p.map_out = make_tma_out_f32(g.slab[n][l], in_p, out_p, splits, in_p, (uint64_t)out_p * in_p);
            p.kb_per_split = kbps;
            P.prob[j] = p;
          }
          flop += g.flop_dw[l];
          g.dw[l].splits = splits;
        }
        P.num_problems = 2 * L;
        P.splits = splits;
        P.hetero = 1;
        g.dw[L - 1] = P;
        g.flop_dw[L - 1] = flop;
        g.bn_dw[L - 1] = bn;
        g.dw_all = true;  // same schedule: every dx first, then this launch
      }
    }

    // gradient assembly segments (fixed-order sums of slabs / partials into the flat grad)
    const int cb = ppo::colsum_blocks(g.Bm);
    const int hs = ppo::head_partial_stride(A);
    for (int n = 0; n < 2; ++n)
      for (int l = 0; l < L; ++l) {
        const Tensor& t = geo_.net[n][l];
        g.segs.push_back({g.grad + t.w, g.slab[n][l], (long long)t.out_p * t.in_p, t.out_p * t.in_p, g.dw[l].splits});
        const int parts = g.fused_bias[l] ? g.dw[l].splits : cb;
        g.segs.push_back({g.grad + t.b, g.colsum[n][l], t.out_p, t.out_p, parts});
      }
    g.segs.push_back({g.grad + geo_.net[0][L].w, g.head_slab[0], (long long)A * hp, A * hp, hslab_parts});
    g.segs.push_back({g.grad + geo_.net[1][L].w, g.head_slab[1], hp, hp,
                      g.fused_head ? g.head_slab_parts[1] : hslab_parts});
    g.segs.push_back({g.grad + geo_.net[0][L].b, g.head_part, hs, A, head_parts});
    g.segs.push_back({g.grad + geo_.net[1][L].b, g.head_part + A, hs, 1, head_parts});
    g.segs.push_back({g.grad + geo_.log_std, g.head_part + A + 1, hs, A, head_parts});
    if (g.local == 0) g.segs.push_back({stats_dev_, g.head_part + 2 * A + 1, hs, 4, head_parts});
    for (auto& sg : g.segs)  // parameter segments may carry the fused Adam update
      sg.param_off = (sg.dst >= g.grad && sg.dst < g.grad + geo_.P) ? (long long)(sg.dst - g.grad) : -1;

    // fused value pass (value MLP on chip over all (T+1) x N observations)
    // (hidden widths <= 256: value_mlp_kernel<false>; up to 512 when the tiles fit: <true>)
    const char* vunf = std::getenv("GMI_VALUE_UNFUSED");
    const char* nowide = std::getenv("GMI_NO_WIDE_FUSED");
    const bool wide_ok = !(nowide && nowide[0] == '1');
    ppo::WidePlan vplan{};
    const bool val_narrow = ppo::rollout_fusable(L, geo_.wp.data(), S_p, A);
    const bool val_wide = !val_narrow && wide_ok && ppo::value_wide_fusable(L, geo_.wp.data(), &vplan);
    g.fused_val = (val_narrow || val_wide) && !(vunf && vunf[0] == '1');
    if (g.fused_val) {
      ppo::ValueArgs& v = g.val_args;
      v.wide = val_wide;
      v.plan = vplan;
      v.map_obs = tma_kmajor(g.X_roll, S_p, (long long)(T_ + 1) * g.N, S_p, kGemmBlockM);
      for (int l = 0; l < L; ++l) {
        const Tensor& t = geo_.net[1][l];
        v.map_w[l] = tma_kmajor(shadow_ + t.w, t.in_p, t.out_p, t.in_p, val_wide ? vplan.wrows[l] : t.out_p);
        v.bias[l] = params_ + t.b;
        v.in_p[l] = t.in_p;
        v.out_n[l] = t.out_p;
      }
      v.map_w[L] = tma_kmajor(shadow_ + geo_.net[1][L].w, hp, 1, hp, 16);
      v.bias[L] = params_ + geo_.net[1][L].b;
      v.in_p[L] = hp;
      v.out_n[L] = 16;
      v.L = L;
      v.rows = (long long)(T_ + 1) * g.N;
      v.V = g.V;
      if (decoupled_) {  // the serving GMI's copy: snapshot weights over the channel's observations
        ppo::ValueArgs& c = g.ch_val_args;
        c = v;
        c.map_obs = tma_kmajor(g.ch_X, S_p, (long long)(T_ + 1) * g.N, S_p, kGemmBlockM);
        for (int l = 0; l < L; ++l) {
          const Tensor& t = geo_.net[1][l];
          c.map_w[l] = tma_kmajor(shadow_roll_ + t.w, t.in_p, t.out_p, t.in_p, val_wide ? vplan.wrows[l] : t.out_p);
          c.bias[l] = params_roll_ + t.b;
        }
        c.map_w[L] = tma_kmajor(shadow_roll_ + geo_.net[1][L].w, hp, 1, hp, 16);
        c.bias[L] = params_roll_ + geo_.net[1][L].b;
        c.V = g.ch_V;
      }
    }

    // fused rollout (one persistent kernel per rollout) when the policy MLP fits on chip
    // (hidden widths <= 256: rollout_kernel / the cluster variant; up to 512: rollout_kernel<8, true>)
    const char* unfused = std::getenv("GMI_ROLLOUT_UNFUSED");
    ppo::WidePlan rplan{};
    const bool roll_narrow = ppo::rollout_fusable(L, geo_.wp.data(), S_p, A);
    const bool roll_wide = !roll_narrow && wide_ok && ppo::rollout_wide_fusable(L, geo_.wp.data(), S_p, A, &rplan);
    g.fused_roll = (roll_narrow || roll_wide) && !(unfused && unfused[0] == '1');
    if (g.fused_roll) {
      ppo::RolloutArgs& r = g.roll_args;
      r.wide = roll_wide;
      r.plan = rplan;
      // decoupled mode: the serving GMI acts with the policy snapshot and writes the channel
      __nv_bfloat16* wsrc = decoupled_ ? shadow_roll_ : shadow_;
      float* psrc = decoupled_ ? params_roll_ : params_;
      __nv_bfloat16* Xr = decoupled_ ? g.ch_X : g.X_roll;
      r.map_obs = tma_kmajor(Xr, S_p, g.N, S_p, kGemmBlockM);
      for (int l = 0; l < L; ++l) {
        const Tensor& t = geo_.net[0][l];
        r.map_w[l] = tma_kmajor(wsrc + t.w, t.in_p, t.out_p, t.in_p, roll_wide ? rplan.wrows[l] : t.out_p);
        r.bias[l] = psrc + t.b;
        r.in_p[l] = t.in_p;
        r.out_n[l] = t.out_p;
      }
      const int head_n = A <= 16 ? 16 : 32;
      r.map_w[L] = tma_kmajor(wsrc + geo_.net[0][L].w, hp, A, hp, head_n);
      // cluster variant: 64-row weight slices per CTA, 16-row head (rollout_cluster.cu)
      const char* nocl = std::getenv("GMI_ROLLOUT_NOCLUSTER");
      g.roll_cluster = (nocl && nocl[0] == '1') || roll_wide ? 0 : ppo::rollout_cluster_size(L, geo_.wp.data(), S_p, A, g.N);
      // a small serving partition runs the rollout in waves: one CTA per env tile then beats
      // 4-CTA clusters (measured on B200: 1.9 vs 4.3 ms for 4096 envs on 16 SMs)
      if (decoupled_ && exec_->sm_count(0) > 0 && g.roll_cluster * (g.N / kGemmBlockM) > exec_->sm_count(0))
        g.roll_cluster = 0;
      if (g.roll_cluster) {
        for (int l = 0; l < L; ++l) {
          const Tensor& t = geo_.net[0][l];
          r.map_w[l] = tma_kmajor(wsrc + t.w, t.in_p, t.out_p, t.in_p, 64);
        }
        r.map_w[L] = tma_kmajor(wsrc + geo_.net[0][L].w, hp, A, hp, 16);
      }
      r.bias[L] = psrc + geo_.net[0][L].b;
      r.in_p[L] = hp;
      r.out_n[L] = head_n;
      r.log_std = psrc + geo_.log_std;
      r.L = L;
      r.A = A;
      r.S = geo_.S;
      r.S_p = S_p;
      r.N = g.N;
      r.T = T_;
      r.env0 = g.env0;
      r.seed = cfg_.seed;
      r.x = g.x;
      r.ep_step = g.ep_step;
      r.ep_len = g.ep_len;
      r.ep_count = g.ep_count;
      r.X_roll = Xr;
      r.act = decoupled_ ? g.ch_act : g.act;
      r.logp = decoupled_ ? g.ch_logp : g.logp;
      r.rew = decoupled_ ? g.ch_rew : g.rew;
      r.done = decoupled_ ? g.ch_done : g.done;
      r.ctl = decoupled_ ? ctl_roll_ : ctl_dev_;
      const char* trace = std::getenv("GMI_ROLLOUT_TRACE");
      if (trace && trace[0] == '1') r.trace = reinterpret_cast<unsigned long long*>(dev((size_t)T_ * 16 * 8));
    }
    if (decoupled_ && !(g.fused_roll && g.fused_val)) build_serving_plans(g);
  }
}

// Decoupled mode with nets the fused rollout / value kernels cannot hold (widths > 256): the
// serving GMI runs the per-layer path on its own partition -- the same GEMMs as the synchronous
// rollout, but reading the experience channel's observations and the policy snapshot, and
// writing its own activation buffers (the trainer GMI's are busy training concurrently).
void Trainer::build_serving_plans(Gmi& g) {
  const int L = geo_.L, S_p = geo_.wp[0], A = geo_.A, hp = geo_.wp[L];
  auto dev = [&](size_t bytes) {
    void* p = nullptr;
    GMI_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
    GMI_CUDA_CHECK(cudaMemset(p, 0, std::max<size_t>(bytes, 256)));
    plan_allocs_.push_back(p);
    return p;
  };
  g.srv_layers = true;
  g.srv_ctas = exec_->sm_count(0) > 0 ? exec_->sm_count(0) : device_sm_count();
  const long long rollrows = (long long)(T_ + 1) * g.N;
  for (int n = 0; n < 2; ++n) {
    for (int l = 0; l < L; ++l)
      g.srv_H[n][l] = static_cast<__nv_bfloat16*>(dev((size_t)g.Mrows * geo_.wp[l + 1] * 2));
    g.srv_outh[n] = static_cast<float*>(dev((size_t)g.Mrows * ppo::kHeadG * 4));
  }
  for (int l = 0; l < L; ++l) {
    const int in_p = geo_.wp[l], out_p = geo_.wp[l + 1];
    auto problem = [&](int n, const CUtensorMap& amap, int M, int bn) {
      GemmProblem p{};
      p.map_a = amap;
      p.map_b = tma_kmajor(shadow_roll_ + geo_.net[n][l].w, in_p, out_p, in_p, bn);
      p.map_out = make_tma_out_bf16(g.srv_H[n][l], out_p, g.Mrows, out_p);
      p.bias = params_roll_ + geo_.net[n][l].b;
      p.M = M;
      p.N = out_p;
      p.K = in_p;
      p.kb_per_split = (in_p + kGemmBlockK - 1) / kGemmBlockK;
      return p;
    };
    g.srv_bn_roll[l] = gemm_choose_bn(g.N, out_p, 1, 1, g.srv_ctas);
    const CUtensorMap a_roll = l == 0 ? tma_kmajor(g.ch_X, S_p, rollrows, S_p, kGemmBlockM)
                                      : tma_kmajor(g.srv_H[0][l - 1], in_p, g.Mrows, in_p, kGemmBlockM);
    g.srv_fwd_roll[l] = GemmParams{};
    g.srv_fwd_roll[l].prob[0] = problem(0, a_roll, g.N, g.srv_bn_roll[l]);
    g.srv_fwd_roll[l].num_problems = 1;
    g.srv_fwd_roll[l].splits = 1;
    const int ws_val = gemm_ws_bn(g.Mrows, out_p, in_p, 1, g.srv_ctas);
    g.srv_ws_val[l] = ws_val > 0;
    g.srv_bn_val[l] = ws_val > 0 ? ws_val : gemm_choose_bn(g.Mrows, out_p, 1, 1, g.srv_ctas);
    const CUtensorMap a_val = l == 0 ? tma_kmajor(g.ch_X, S_p, rollrows, S_p, kGemmBlockM)
                                     : tma_kmajor(g.srv_H[1][l - 1], in_p, g.Mrows, in_p, kGemmBlockM);
    g.srv_fwd_val[l] = GemmParams{};
    g.srv_fwd_val[l].prob[0] = problem(1, a_val, g.Mrows, g.srv_bn_val[l]);
    g.srv_fwd_val[l].num_problems = 1;
    g.srv_fwd_val[l].splits = 1;
  }
  const int head_rows[2] = {A, 1};
  for (int n = 0; n < 2; ++n) {
    GemmProblem p{};
    p.map_a = tma_kmajor(g.srv_H[n][L - 1], hp, g.Mrows, hp, kGemmBlockM);
    p.map_b = tma_kmajor(shadow_roll_ + geo_.net[n][L].w, hp, head_rows[n], hp, 64);
    p.map_out = make_tma_out_f32(g.srv_outh[n], ppo::kHeadG, g.Mrows, 1, ppo::kHeadG, (uint64_t)g.Mrows * ppo::kHeadG);
    p.M = n == 0 ? g.N : g.Mrows;
    p.N = ppo::kHeadG;
    p.K = hp;
    p.kb_per_split = (hp + kGemmBlockK - 1) / kGemmBlockK;
    GemmParams& P = n == 0 ? g.srv_head_roll : g.srv_head_val;
    P = GemmParams{};
    P.prob[0] = p;
    P.num_problems = 1;
    P.splits = 1;
  }
}

// The serving GMI's rollout + values with the per-layer plans above (decoupled, wide nets).
void Trainer::serve_rollout_layers(Gmi& g) {
  const int L = geo_.L, S_p = geo_.wp[0], A = geo_.A;
  const Tensor& phead = geo_.net[0][L];
  const Tensor& vhead = geo_.net[1][L];
  const double env_bytes = double(g.N) * (8.0 * A + 8.0 * geo_.S + 2.0 * S_p + 29.0);
  for (int t = 0; t < T_; ++t) {
    for (int l = 0; l < L; ++l) {
      GemmParams P = g.srv_fwd_roll[l];
      if (l == 0) P.prob[0].a_row0 = t * g.N;
      gemm(g, GMI_PH_ROLL_GEMM, P, g.srv_bn_roll[l], 0, 0, EPI_BIAS_ELU, g.flop_roll[l], 0, serve_s_, g.srv_ctas);
    }
    gemm(g, GMI_PH_ROLL_HEAD, g.srv_head_roll, 64, 0, 0, EPI_F32, 2.0 * A * geo_.width[L] * g.N, 0, serve_s_,
         g.srv_ctas);
    ppo::ActEnvArgs a{};
    a.ep = {g.N, geo_.S, A, S_p, g.env0, T_, cfg_.seed};
    a.mu = g.srv_outh[0];
    a.b_mu = params_roll_ + phead.b;
    a.log_std = params_roll_ + geo_.log_std;
    a.x = g.x;
    a.ep_step = g.ep_step;
    a.ep_len = g.ep_len;
    a.ep_count = g.ep_count;
    a.X_next = g.ch_X + (long long)(t + 1) * g.N * S_p;
    a.act = g.ch_act + (long long)t * g.N * A;
    a.logp = g.ch_logp + (long long)t * g.N;
    a.rew = g.ch_rew + (long long)t * g.N;
    a.done = g.ch_done + (long long)t * g.N;
    a.t = t;
    a.ctl = ctl_roll_;
    timed(serve_s_, GMI_PH_ACT_ENV, 0.0, env_bytes, [&] { ppo::launch_act_env(a, serve_s_); });
    ++launches_;
  }
  const long long rows = (long long)(T_ + 1) * g.N;
  for (long long c0 = 0; c0 < rows; c0 += g.Mrows) {
    const int m = int(std::min<long long>(g.Mrows, rows - c0));
    for (int l = 0; l < L; ++l) {
      GemmParams P = g.srv_fwd_val[l];
      P.prob[0].M = m;
      if (l == 0) P.prob[0].a_row0 = int(c0);
      gemm(g, GMI_PH_VAL_GEMM, P, g.srv_bn_val[l], 0, 0, EPI_BIAS_ELU, g.flop_roll[l] * double(m) / g.N,
           g.srv_ws_val[l], serve_s_, g.srv_ctas);
    }
    GemmParams Ph = g.srv_head_val;
    Ph.prob[0].M = m;
    gemm(g, GMI_PH_VAL_HEAD, Ph, 64, 0, 0, EPI_F32, 2.0 * geo_.width[L] * m, 0, serve_s_, g.srv_ctas);
    timed(serve_s_, GMI_PH_VAL_HEAD, 0.0, 8.0 * m,
          [&] { ppo::launch_value_head(g.srv_outh[1], params_roll_ + vhead.b, g.ch_V + c0, m, serve_s_); });
    ++launches_;
  }
}

// ------------------------------------------------------------------ launch helpers
int Trainer::unit_of(cudaStream_t s) const {
  if (s == upd_) return decoupled_ ? 2 : n_local_;
  if (decoupled_ && s == serve_s_) return 0;
  for (const auto& g : gmis_)
    if (s == g->s || s == g->s2) return decoupled_ ? 1 : g->local;
  return -1;
}

int Trainer::busy_units(double* busy_ms, int* sms, int cap) const {
  const int n = decoupled_ ? 3 : n_local_ + 1;
  for (int i = 0; i < n && i < cap; ++i) {
    if (busy_ms) busy_ms[i] = i < int(unit_busy_ms_.size()) ? unit_busy_ms_[i] : 0.0;
    if (sms) {
      const bool upd = i == n - 1;
      // GMI i is execution resource i (decoupled: 0 serving, 1 trainer)
      sms[i] = upd ? (upd_in_gmi_ ? exec_->sm_count(1) : 0) : exec_->sm_count(i);
      if (sms[i] <= 0) sms[i] = device_sm_count();
    }
  }
  return n;
}

template <class F>
void Trainer::timed(cudaStream_t s, int phase, double flop, double bytes, F&& f) {
  const int unit = cfg_.instrument ? unit_of(s) : -1;
  if (unit < 0) {
    f();
    return;
  }
  if (marks_used_ >= int(marks_.size())) {
    Mark m;
    GMI_CUDA_CHECK(cudaEventCreate(&m.a));
    GMI_CUDA_CHECK(cudaEventCreate(&m.b));
    marks_.push_back(m);
  }
  Mark& m = marks_[marks_used_++];
  // under stream capture a plain record only forms a dependency; the external flag makes it
  // a real event-record node of the graph, so the replay timestamps it
  const unsigned flags = capturing_ ? cudaEventRecordExternal : cudaEventRecordDefault;
  GMI_CUDA_CHECK(cudaEventRecordWithFlags(m.a, s, flags));
  f();
  GMI_CUDA_CHECK(cudaEventRecordWithFlags(m.b, s, flags));
  m.phase = phase;
  m.unit = unit;
  m.in_phases = s == upd_ || s == gmis_[0]->s || s == gmis_[0]->s2;
  m.flop = flop;
  m.bytes = bytes;
}

// Algorithmic bytes of one grouped GEMM launch: each operand read once, each output written
// once (bf16 activations / dPre, or fp32 split-K slabs), plus the elu' operand of EPI_DACT.
// Problems that share an operand (the N-halves of one input-gradient GEMM read the same dPre
// rows) count it once.
static double gemm_bytes(const GemmParams& P, int epi) {
  double b = 0;
  for (int i = 0; i < P.num_problems * std::max(1, P.chain); ++i) {
    const GemmProblem& p = P.prob[i];
    bool a_seen = false;
    for (int j = 0; j < i; ++j) a_seen |= std::memcmp(&P.prob[j].map_a, &p.map_a, sizeof(CUtensorMap)) == 0;
    b += 2.0 * p.K * ((a_seen ? 0.0 : double(p.M)) + p.N);
    b += double(p.M) * p.N * (epi == EPI_F32 ? 4.0 * P.splits : epi == EPI_DACT ? 4.0 : 2.0);
  }
  return b;
}

void Trainer::gemm(Gmi& g, int phase, const GemmParams& P0, int bn, int amn, int bmn, int epi, double flop, int ws,
                   cudaStream_t stream, int ctas) {
  cudaStream_t st = stream ? stream : g.s;
  // weight-stationary B = the layer's weights: only Adam writes them, on the update stream
  // (ordered by an event) -- unless Adam is fused into this GMI's gradient assembly
  GemmParams P = P0;
  static const char* no_bs = std::getenv("GMI_NO_BSTABLE");  // experiment: no early weight loads
  P.b_stable = ws && !adam_in_gmi_stream_ && !(no_bs && no_bs[0] == '1') && !no_b_preload_once_ ? 1 : 0;
  if (ws) no_b_preload_once_ = false;
  // GMI_GEMM_TRACE=<phase id>: globaltimer stamps of CTA 0 for every launch of that phase
  // (the last one of the iteration wins; read with get("gemm_trace")). Development aid.
  // GMI_GEMM_TRACE_NTH=<k>: only the k-th recorded launch of the phase (e.g. 0 = the first
  // minibatch's last layer for the backward phases).
  static const char* tr_env = std::getenv("GMI_GEMM_TRACE");
  static const char* tr_nth = std::getenv("GMI_GEMM_TRACE_NTH");
  static int tr_calls = 0;
  if (tr_env && std::atoi(tr_env) == phase && (!tr_nth || tr_calls++ == std::atoi(tr_nth))) {
    if (!gemm_trace_) {
      GMI_CUDA_CHECK(cudaMalloc(&gemm_trace_, 128 * 8));
      GMI_CUDA_CHECK(cudaMemset(gemm_trace_, 0, 128 * 8));
      allocs_.push_back(gemm_trace_);
    }
    GemmParams Pt = P;
    Pt.trace = static_cast<unsigned long long*>(gemm_trace_);
    timed(st, phase, flop, gemm_bytes(P, epi), [&] { gemm_launch(Pt, bn, amn, bmn, epi, st, ctas > 0 ? ctas : g.ctas, ws); });
    ++launches_;
    return;
  }
  timed(st, phase, flop, gemm_bytes(P, epi), [&] { gemm_launch(P, bn, amn, bmn, epi, st, ctas > 0 ? ctas : g.ctas, ws); });
  ++launches_;
}

void Trainer::set_instrument(int on) {
  GMI_CUDA_CHECK(cudaDeviceSynchronize());
  cfg_.instrument = on ? 1 : 0;
  if (graph_) {  // the captured sequence has (or lacks) the event records
    GMI_CUDA_CHECK(cudaGraphExecDestroy(graph_));
    graph_ = nullptr;
  }
}

void Trainer::ensure_bias_table(long long steps) {
  if (steps <= bc_cap_) return;
  // Adam bias corrections 1-b^s for s = 1..cap in double, rounded to fp32 (as the oracle)
  GMI_CUDA_CHECK(cudaDeviceSynchronize());
  const long long cap = std::max<long long>(steps, 2 * bc_cap_);
  std::vector<float> tab(2 * cap);
  for (long long s = 0; s < cap; ++s) {
    tab[2 * s] = float(1.0 - std::pow(double(cfg_.beta1), double(s + 1)));
    tab[2 * s + 1] = float(1.0 - std::pow(double(cfg_.beta2), double(s + 1)));
  }
  void* p = nullptr;
  GMI_CUDA_CHECK(cudaMalloc(&p, tab.size() * 4));
  GMI_CUDA_CHECK(cudaMemcpy(p, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice));
  allocs_.push_back(p);
  bc_ = static_cast<float*>(p);
  bc_cap_ = cap;
  if (graph_) {  // the captured Adam launches point at the old table
    GMI_CUDA_CHECK(cudaGraphExecDestroy(graph_));
    graph_ = nullptr;
  }
}

// Host -> device control block (the iteration's only host input): used on the first
// iteration, by the rollout parity hook, and on the synchronous public path.
void Trainer::write_control() {
  GMI_CUDA_CHECK(cudaStreamSynchronize(upd_));
  ctl_host_->iteration = iteration_;
  ctl_host_->adam_step0 = adam_steps_;
  GMI_CUDA_CHECK(cudaMemcpyAsync(ctl_dev_, ctl_host_, sizeof(ppo::Control), cudaMemcpyHostToDevice, upd_));
}

// ------------------------------------------------------------------ phases
void Trainer::rollout(Gmi& g) {
  const int L = geo_.L, S_p = geo_.wp[0], S = geo_.S, A = geo_.A;
  if (iteration_ > 0)  // the last observation of the previous rollout seeds this one
    timed(g.s, GMI_PH_OTHER, 0.0, 4.0 * g.N * S_p, [&] {
      GMI_CUDA_CHECK(cudaMemcpyAsync(g.X_roll, g.X_roll + (long long)T_ * g.N * S_p, (size_t)g.N * S_p * 2,
                                     cudaMemcpyDeviceToDevice, g.s));
    });
  const Tensor& head = geo_.net[0][L];
  const double env_bytes = double(g.N) * (8.0 * A + 8.0 * S + 2.0 * S_p + 29.0);
  if (g.fused_roll) {  // whole rollout in one persistent kernel (cuda/rollout.cu)
    double flop = 2.0 * geo_.A * geo_.width[L] * g.N;
    for (int l = 0; l < L; ++l) flop += g.flop_roll[l];
    timed(g.s, GMI_PH_ROLL_GEMM, flop * T_, 0.0, [&] {
      if (g.roll_cluster)
        ppo::launch_rollout_cluster(g.roll_args, g.roll_cluster, g.s);
      else
        ppo::launch_rollout(g.roll_args, g.s);
    });
    ++launches_;
    return;
  }
  for (int t = 0; t < T_; ++t) {
    for (int l = 0; l < L; ++l) {
      GemmParams P = g.fwd_roll[l];
      if (l == 0) P.prob[0].a_row0 = t * g.N;
      gemm(g, GMI_PH_ROLL_GEMM, P, g.bn_roll[l], 0, 0, EPI_BIAS_ELU, g.flop_roll[l]);
    }
    gemm(g, GMI_PH_ROLL_HEAD, g.head_roll, 64, 0, 0, EPI_F32, 2.0 * geo_.A * geo_.width[L] * g.N);
    ppo::ActEnvArgs a{};
    a.ep = {g.N, geo_.S, geo_.A, S_p, g.env0, T_, cfg_.seed};
    a.mu = g.outh[0];
    a.b_mu = params_ + head.b;
    a.log_std = params_ + geo_.log_std;
    a.x = g.x;
    a.ep_step = g.ep_step;
    a.ep_len = g.ep_len;
    a.ep_count = g.ep_count;
    a.X_next = g.X_roll + (long long)(t + 1) * g.N * S_p;
    a.act = g.act + (long long)t * g.N * geo_.A;
    a.logp = g.logp + (long long)t * g.N;
    a.rew = g.rew + (long long)t * g.N;
    a.done = g.done + (long long)t * g.N;
    a.t = t;
    a.ctl = ctl_dev_;
    timed(g.s, GMI_PH_ACT_ENV, 0.0, env_bytes, [&] { ppo::launch_act_env(a, g.s); });
    ++launches_;
  }
}

void Trainer::values(Gmi& g) {
  const int L = geo_.L;
  const long long rows = (long long)(T_ + 1) * g.N;
  const Tensor& head = geo_.net[1][L];
  if (g.fused_val) {  // the whole value MLP on chip, one persistent launch (cuda/value_mlp.cu)
    double flop = 2.0 * geo_.width[L] * rows;
    for (int l = 0; l < L; ++l) flop += g.flop_roll[l] * double(rows) / g.N;
    timed(g.s, GMI_PH_VAL_GEMM, flop, 0.0, [&] { ppo::launch_value_mlp(g.val_args, g.ctas, g.s); });
    ++launches_;
  }
  for (long long c0 = 0; c0 < rows && !g.fused_val; c0 += g.Mrows) {
    const int m = int(std::min<long long>(g.Mrows, rows - c0));
    for (int l = 0; l < L; ++l) {
      GemmParams P = g.fwd_val[l];
      P.prob[0].M = m;
      if (l == 0) P.prob[0].a_row0 = int(c0);
      gemm(g, GMI_PH_VAL_GEMM, P, g.bn_val[l], 0, 0, EPI_BIAS_ELU, g.flop_roll[l] * double(m) / g.N, g.ws_val[l]);
    }
    GemmParams Ph = g.head_val;
    Ph.prob[0].M = m;
    gemm(g, GMI_PH_VAL_HEAD, Ph, 64, 0, 0, EPI_F32, 2.0 * geo_.width[L] * m);
    timed(g.s, GMI_PH_VAL_HEAD, 0.0, 8.0 * m,
          [&] { ppo::launch_value_head(g.outh[1], params_ + head.b, g.V + c0, m, g.s); });
    ++launches_;
  }
  const double TN = double(T_) * g.N;
  timed(g.s, GMI_PH_GAE, 0.0, 17.0 * TN + 4.0 * g.N, [&] {
    ppo::launch_gae(g.rew, g.done, g.V, g.adv, g.ret, g.gae_part, g.N, T_, cfg_.gamma, cfg_.lam, g.s);
    ppo::launch_adv_stats(g.gae_part, ppo::gae_blocks(g.N), (long long)T_ * g.N, g.adv_stats, g.s);
  });
  launches_ += 2;
}

void Trainer::train_minibatch(Gmi& g, int k, int adam_step) {
  const int L = geo_.L, A = geo_.A;
  if (g.fused_fwd) {  // hidden forward (both nets) + head step, one launch
    ppo::TrainFwdArgs f = g.fwd_args;
    f.row0 = (long long)k * g.Bm;
    double flop = 3.0 * 2.0 * (A + 1) * geo_.width[L] * g.Bm;
    for (int l = 0; l < L; ++l) flop += g.flop_fwd[l];
    timed(g.s, GMI_PH_FWD_GEMM, flop, 0.0, [&] { ppo::launch_train_fwd(f, g.head_grid, g.s); });
    ++launches_;
  }
  if (g.chain_fwd && !g.fused_fwd) {  // all hidden layers of both nets in one launch
    GemmParams P = g.fwd_chain;
    P.prob[0].a_row0 = P.prob[1].a_row0 = k * g.Bm;
    double flop = 0;
    for (int l = 0; l < L; ++l) flop += g.flop_fwd[l];
    gemm(g, GMI_PH_FWD_GEMM, P, g.bn_fwd[0], 0, 0, EPI_BIAS_ELU, flop, 1);
  }
  for (int l = 0; l < L && !g.fused_fwd && !g.chain_fwd; ++l) {
    GemmParams P = g.fwd_train[l];
    if (l == 0)
      for (int i = 0; i < P.num_problems; ++i) P.prob[i].a_row0 = k * g.Bm;
    gemm(g, GMI_PH_FWD_GEMM, P, g.bn_fwd[l], 0, 0, EPI_BIAS_ELU, g.flop_fwd[l], g.ws_fwd[l]);
  }
  const double hflop = 2.0 * (A + 1) * geo_.width[L] * g.Bm;
  if (g.fused_fwd) {
  } else if (g.fused_head) {  // head forward + loss + head input/weight grads + bias sums, one launch
    ppo::HeadFusedArgs h = g.head_args;
    h.row0 = (long long)k * g.Bm;
    timed(g.s, GMI_PH_HEAD_LOSS, 3.0 * hflop, 0.0, [&] { ppo::launch_head_fused(h, g.head_grid, g.s); });
    ++launches_;
  } else {
    gemm(g, GMI_PH_HEAD_FWD, g.head_train, 64, 0, 0, EPI_F32, hflop);
    ppo::HeadLossArgs h{};
  h.mu = g.outh[0];
  h.v = g.outh[1];
  h.b_mu = params_ + geo_.net[0][L].b;
  h.b_v = params_ + geo_.net[1][L].b;
  h.log_std = params_ + geo_.log_std;
  const long long r0 = (long long)k * g.Bm;
  h.act = g.act_sh + r0 * A;
  h.oldlp = g.oldlp_sh + r0;
  h.adv = g.adv_sh + r0;
  h.ret = g.ret_sh + r0;
  h.Gpi = g.Gpi;
  h.Gv = g.Gv;
  h.partial = g.head_part;
  h.B = g.Bm;
  h.A = A;
  h.clip = cfg_.clip;
  h.vf_coef = cfg_.vf_coef;
  h.ent_coef = cfg_.ent_coef;
    timed(g.s, GMI_PH_HEAD_LOSS, 0.0, double(g.Bm) * (10.0 * A + 18.0), [&] { ppo::launch_head_loss(h, g.s); });
    ++launches_;
    gemm(g, GMI_PH_HEAD_DX, g.head_dx, g.bn_hdx, 0, 1, EPI_DACT, hflop, g.ws_hdx);
    gemm(g, GMI_PH_HEAD_DW, g.dhead, g.bn_head, 1, 1, EPI_F32, g.flop_head);
  }
  // Backward branch parallelism: the input-gradient chain dx(L-1) -> ... -> dx(1) runs on the
  // GMI's second stream while the weight-gradient GEMMs dW(l) follow on the main stream as soon
  // as their dPre_l is ready (per-layer dPre buffers, so there is no write-after-read hazard).
  // Each branch gets its own share of the GMI's SMs (GMI_BWD_SPLIT=dx_ctas,dw_ctas to tune).
  bool par = bwd_par_;
  for (int l = 0; l < L; ++l) par = par && g.fused_bias[l];
  if (par && L > 1) {
    const int dx_ctas = std::max(1, g.ctas * bwd_dx_share_ / 100), dw_ctas = std::max(1, g.ctas - dx_ctas);
    GMI_CUDA_CHECK(cudaEventRecord(g.ev_fork, g.s));
    GMI_CUDA_CHECK(cudaStreamWaitEvent(g.s2, g.ev_fork, 0));
    for (int l = L - 1; l >= 1; --l) {
      gemm(g, GMI_PH_DX_GEMM, g.dx[l], g.bn_dx[l], 0, 1, EPI_DACT, g.flop_dx[l], g.ws_dx[l], g.s2, dx_ctas);
      GMI_CUDA_CHECK(cudaEventRecord(g.ev_d[l - 1], g.s2));
    }
    for (int l = L - 1; l >= 0; --l) {
      if (l < L - 1) GMI_CUDA_CHECK(cudaStreamWaitEvent(g.s, g.ev_d[l], 0));
      GemmParams P = g.dw[l];
      if (l == 0) P.prob[0].b_row0 = P.prob[1].b_row0 = k * g.Bm;
      if (g.dw_pair[l]) {
        timed(g.s, GMI_PH_DW_GEMM, g.flop_dw[l], 0.0, [&] { gemm_pair_launch(P, dw_ctas, g.s); });
        ++launches_;
      } else {
        gemm(g, GMI_PH_DW_GEMM, P, g.bn_dw[l], 1, 1, EPI_F32, g.flop_dw[l], 0, g.s, dw_ctas);
      }
    }
  }
  if (g.dw_all && !(par && L > 1)) {  // every input gradient, then every layer's dW in one launch
    for (int l = L - 1; l >= 1; --l)
      gemm(g, GMI_PH_DX_GEMM, g.dx[l], g.bn_dx[l], 0, 1, EPI_DACT, g.flop_dx[l], g.ws_dx[l]);
    GemmParams P = g.dw[L - 1];
    P.prob[2 * L - 2].b_row0 = P.prob[2 * L - 1].b_row0 = k * g.Bm;  // layer 0 reads X of this minibatch
    gemm(g, GMI_PH_DW_GEMM, P, g.bn_dw[L - 1], 1, 1, EPI_F32, g.flop_dw[L - 1]);
  }
  for (int l = L - 1; l >= 0 && !(par && L > 1) && !g.dw_all; --l) {
    // grouped: dW(L-1) waits for dPre(L-2) and runs with dW(L-2) as one launch (plan above)
    const int lw = g.dw_grouped && l == L - 2 ? L - 1 : l;
    GemmParams P = g.dw[lw];
    if (l == 0) P.prob[0].b_row0 = P.prob[1].b_row0 = k * g.Bm;
    if (g.dw_grouped && l == L - 1) {
      // deferred
    } else if (g.dw_pair[l]) {
      timed(g.s, GMI_PH_DW_GEMM, g.flop_dw[l], 0.0, [&] { gemm_pair_launch(P, g.ctas, g.s); });
      ++launches_;
    } else {
      gemm(g, GMI_PH_DW_GEMM, P, g.bn_dw[lw], 1, 1, EPI_F32, g.flop_dw[lw]);
    }
    if (!g.fused_bias[l]) {  // else summed by the DACT GEMM that produced dPre_l
      const __nv_bfloat16* Ds[2] = {g.D[0][l], g.D[1][l]};
      const int widths[2] = {geo_.wp[l + 1], geo_.wp[l + 1]};
      float* outs[2] = {g.colsum[0][l], g.colsum[1][l]};
      timed(g.s, GMI_PH_COLSUM, 0.0, 2.0 * 2.0 * g.Bm * geo_.wp[l + 1],
            [&] { ppo::launch_colsum(Ds, widths, outs, 2, g.Bm, g.s); });
      ++launches_;
    }
    if (l > 0) gemm(g, GMI_PH_DX_GEMM, g.dx[l], g.bn_dx[l], 0, 1, EPI_DACT, g.flop_dx[l], g.ws_dx[l]);
  }
  double seg_bytes = 0;
  for (const auto& sg : g.segs) seg_bytes += 4.0 * sg.len * (sg.nparts + 1.0);
  if (adam_step >= 0) {  // single GMI, single GPU: Adam fused into the gradient assembly
    ppo::SegAdam ad{params_, m_, v_, shadow_, bc_, ctl_dev_, adam_step,
                    cfg_.lr, cfg_.beta1, cfg_.beta2, cfg_.adam_eps, 1.0f / float(n_total_)};
    seg_bytes += 30.0 * geo_.P;
    timed(g.s, GMI_PH_SEGMENTS, 0.0, seg_bytes,
          [&] { ppo::launch_segments(g.segs.data(), int(g.segs.size()), g.s, &ad); });
  } else {
    timed(g.s, GMI_PH_SEGMENTS, 0.0, seg_bytes,
          [&] { ppo::launch_segments(g.segs.data(), int(g.segs.size()), g.s); });
  }
  launches_ += (int(g.segs.size()) + 63) / 64;
}

void Trainer::reduce_and_step(int step_in_iter) {
  for (auto& g : gmis_) GMI_CUDA_CHECK(cudaStreamWaitEvent(upd_, g->ev_done, 0));
  float* src = gmis_[0]->grad;
  // K1: fold the GPU's GMIs in ring order (MPR / HAR step 1) -- inside the exchange kernel for one
  // rank, read remotely per GMI for MRR
  if (n_local_ > 1 && !(xchg_ && (xa_.mrr || cfg_.num_gpus == 1))) {
    plan::Placement p;
    p.per_gpu.resize(1);
    std::vector<void*> bufs;
    for (auto& g : gmis_) {
      p.per_gpu[0].push_back(g->local);
      bufs.push_back(g->grad);
    }
    timed(upd_, GMI_PH_REDUCE, 0.0, 4.0 * geo_.P * (n_local_ + 1), [&] {
      reduce_device(plan::Algo::MPR, p, bufs.data(), grad_sum_, size_t(geo_.P), GMI_F32, false, upd_);
    });
    ++launches_;
    src = grad_sum_;
  }
  if (xchg_) {  // fused reduce-scatter -> sharded Adam -> all-gather over peer memory
    ppo::ExchangeArgs a = xa_;
    a.m = m_;
    a.v = v_;
    a.bc = bc_;
    a.ctl = ctl_dev_;
    a.step_in_iter = step_in_iter;
    a.lr = cfg_.lr;
    a.b1 = cfg_.beta1;
    a.b2 = cfg_.beta2;
    a.eps = cfg_.adam_eps;
    a.inv_n = 1.0f / float(n_total_);
    // per rank and update and shard element: G (HAR) or G x t (MRR) 4-byte reads, Adam's m / v /
    // p (16 B), 6 B written per replica
    const double shard = double(xa_.hi - xa_.lo), reads = cfg_.num_gpus * (xa_.mrr ? n_local_ : 1);
    timed(upd_, cfg_.num_gpus == 1 ? GMI_PH_ADAM : GMI_PH_ALLREDUCE, 0.0,
          shard * (4.0 * (cfg_.num_gpus == 1 ? n_local_ : reads) + 16.0 + 6.0 * cfg_.num_gpus),
          [&] { ppo::launch_exchange_adam(a, upd_); });
    launches_ += cfg_.num_gpus == 1 ? 1 : 3;
    GMI_CUDA_CHECK(cudaEventRecord(ev_adam_, upd_));
    return;
  }
  if (nccl_) {
    const double bus = 2.0 * (cfg_.num_gpus - 1) / cfg_.num_gpus * 4.0 * geo_.P;
    timed(upd_, GMI_PH_ALLREDUCE, 0.0, bus, [&] {
      NCCL_CHECK(ncclAllReduce(src, grad_sum_, size_t(geo_.P), ncclFloat32, ncclSum,
                               static_cast<ncclComm_t>(nccl_), upd_));
    });
    src = grad_sum_;
  }
  launch_adam_on(upd_, src, step_in_iter);
  GMI_CUDA_CHECK(cudaEventRecord(ev_adam_, upd_));
}

void Trainer::launch_adam_on(cudaStream_t st, const float* grad, int step_in_iter) {
  ppo::AdamArgs a{};
  a.p = params_;
  a.m = m_;
  a.v = v_;
  a.shadow = shadow_;
  a.g = grad;
  a.bc = bc_;
  a.ctl = ctl_dev_;
  a.step_in_iter = step_in_iter;
  a.n = geo_.P;
  a.lr = cfg_.lr;
  a.b1 = cfg_.beta1;
  a.b2 = cfg_.beta2;
  a.eps = cfg_.adam_eps;
  a.inv_n = 1.0f / float(n_total_);
  timed(st, GMI_PH_ADAM, 0.0, 30.0 * geo_.P, [&] { ppo::launch_adam(a, st); });
  ++launches_;
}

// Decoupled mode: the serving GMI (its own SM partition) steps every env T times with the
// policy snapshot, evaluates the critic on the T+1 observation slots and runs GAE, writing the
// experience channel; rollouts after the first continue from the last observation of the
// previous one. Its control block counts rollouts (noise keys).
void Trainer::serve_rollout(Gmi& g) {
  const int S_p = geo_.wp[0];
  if (rollouts_ > 0)
    timed(serve_s_, GMI_PH_OTHER, 0.0, 4.0 * g.N * S_p, [&] {
      GMI_CUDA_CHECK(cudaMemcpyAsync(g.ch_X, g.ch_X + (long long)T_ * g.N * S_p, (size_t)g.N * S_p * 2,
                                     cudaMemcpyDeviceToDevice, serve_s_));
    });
  if (g.srv_layers) {  // wide nets: the per-layer path on the serving partition
    serve_rollout_layers(g);
  } else {
    timed(serve_s_, GMI_PH_ROLL_GEMM, 0.0, 0.0, [&] {
      if (g.roll_cluster)
        ppo::launch_rollout_cluster(g.roll_args, g.roll_cluster, serve_s_);
      else
        ppo::launch_rollout(g.roll_args, serve_s_);
    });
    // values of all T+1 observation slots with the same snapshot, then GAE: the channel carries
    // ready advantages / returns, so the trainer starts straight at the epoch shuffle
    const int sms = exec_->sm_count(0) > 0 ? exec_->sm_count(0) : device_sm_count();
    timed(serve_s_, GMI_PH_VAL_GEMM, 0.0, 0.0, [&] { ppo::launch_value_mlp(g.ch_val_args, sms, serve_s_); });
  }
  timed(serve_s_, GMI_PH_GAE, 0.0, 0.0, [&] {
    ppo::launch_gae(g.ch_rew, g.ch_done, g.ch_V, g.ch_adv, g.ch_ret, g.ch_gae_part, g.N, T_, cfg_.gamma, cfg_.lam,
                    serve_s_);
    ppo::launch_adv_stats(g.ch_gae_part, ppo::gae_blocks(g.N), (long long)T_ * g.N, g.ch_adv_stats, serve_s_);
    ppo::launch_control_advance(ctl_roll_, 0, serve_s_);
  });
  GMI_CUDA_CHECK(cudaEventRecord(ev_rolled_, serve_s_));
  launches_ += 5;
  ++rollouts_;
}

// Parity hook: the next iteration's rollout + values + GAE only. The following iteration trains
// on this rollout instead of rolling out again (so the env never steps twice from one
// observation slot and noise keys are never reused); a second hook before it is rejected.
void Trainer::enqueue_rollout() {
  if (decoupled_) invalid("gmi_ppo_rollout: the serving GMI rolls out inside each decoupled iteration");
  if (rollout_pending_) invalid("gmi_ppo_rollout: a rollout is already pending; run gmi_ppo_iteration to train on it");
  GMI_CUDA_CHECK(cudaSetDevice(cfg_.device));
  rollout_pending_ = true;
  write_control();
  GMI_CUDA_CHECK(cudaEventRecord(ev_start_, upd_));
  for (auto& g : gmis_) {
    GMI_CUDA_CHECK(cudaStreamWaitEvent(g->s, ev_start_, 0));
    rollout(*g);
    values(*g);
    GMI_CUDA_CHECK(cudaEventRecord(g->ev_done, g->s));
    GMI_CUDA_CHECK(cudaStreamWaitEvent(upd_, g->ev_done, 0));
  }
}

// Every kernel / copy / collective of one iteration, on the GMI streams and upd_.
void Trainer::record_iteration(bool with_rollout) {
  launches_ = 0;
  marks_used_ = 0;
  {
    const char* af = std::getenv("GMI_ADAM_FUSED");  // see the fused_adam note below
    adam_in_gmi_stream_ = n_local_ == 1 && !nccl_ && !xchg_ && af && af[0] == '1';
    const char* ai = std::getenv("GMI_ADAM_INLINE");
    // measured on B200: 48.3 -> 49.2 M env-steps/s at the bench shape (two cross-stream event hops
    // per minibatch gone; the forward chain after Adam loads its weights after griddepcontrol.wait);
    // decoupled trainer: 52.7 -> 53.7 M (three paired runs on one box, r3k).
    adam_inline_ = n_local_ == 1 && !nccl_ && !xchg_ && !adam_in_gmi_stream_ && !(ai && ai[0] == '0');
  }
  GMI_CUDA_CHECK(cudaEventRecord(ev_start_, upd_));
  if (!with_rollout) {  // trains on the rollout a gmi_ppo_rollout hook produced
    for (auto& g : gmis_) GMI_CUDA_CHECK(cudaStreamWaitEvent(g->s, ev_start_, 0));
  } else if (decoupled_) {
    // migrate the channel's experience (rollout i) into the trainer's buffers, then let the
    // serving GMI produce rollout i+1 with the snapshot theta_i while this slot trains
    Gmi& g = *gmis_[0];
    const long long TN = (long long)T_ * g.N;
    const int S_p = geo_.wp[0], A = geo_.A;
    GMI_CUDA_CHECK(cudaStreamWaitEvent(g.s, ev_start_, 0));
    // across GPUs (decoupled = 2): wait until the partner published rollout i (R >= i + 1), then
    // pull it over NVLink from the partner's link window
    if (split_) ppo::launch_link_wait(link_flag(false, 0), nullptr, lctr_ + 2, 0, g.s);
    auto ch = [&](const void* local, size_t off) -> const void* { return split_ ? lpeer_ + off : local; };
    timed(g.s, GMI_PH_OTHER, 0.0, 2.0 * ((TN + g.N) * S_p * 2 + TN * (4.0 * A + 12.0) + 16.0), [&] {
      auto mig = [&](void* dst, const void* src, size_t bytes) {
        GMI_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, g.s));
      };
      mig(g.X_roll, ch(g.ch_X, loff_X_), (size_t)(TN + g.N) * S_p * 2);
      mig(g.act, ch(g.ch_act, loff_act_), (size_t)TN * A * 4);
      mig(g.logp, ch(g.ch_logp, loff_logp_), (size_t)TN * 4);
      mig(g.adv, ch(g.ch_adv, loff_adv_), (size_t)TN * 4);
      mig(g.ret, ch(g.ch_ret, loff_ret_), (size_t)TN * 4);
      mig(g.adv_stats, ch(g.ch_adv_stats, loff_stats_), 16);
    });
    if (split_) {  // the channel is free again: C = i + 1
      ppo::launch_link_signal(link_flag(true, 128), lctr_ + 3, 0, g.s);
      launches_ += 2;
    } else {
      GMI_CUDA_CHECK(cudaEventRecord(ev_copied_, g.s));
      GMI_CUDA_CHECK(cudaStreamWaitEvent(serve_s_, ev_copied_, 0));
      serve_rollout(g);
    }
  } else {
    for (auto& g : gmis_) {
      GMI_CUDA_CHECK(cudaStreamWaitEvent(g->s, ev_start_, 0));
      rollout(*g);
      values(*g);
    }
  }
  int step = 0;
  // One GMI on one GPU: Adam can run inside the gradient-assembly kernel (GMI_ADAM_FUSED=1).
  // Measured slightly slower than the separate Adam launch on B200 (3.62 vs 3.60 ms per
  // iteration), so the separate kernel stays the default.
  const char* adam_fused = std::getenv("GMI_ADAM_FUSED");
  const bool fused_adam = n_local_ == 1 && !nccl_ && !xchg_ && adam_fused && adam_fused[0] == '1';
  for (int e = 0; e < cfg_.epochs; ++e) {
    for (auto& g : gmis_) {
      if (step > 0 && !fused_adam && !adam_inline_) GMI_CUDA_CHECK(cudaStreamWaitEvent(g->s, ev_adam_, 0));
      timed(g->s, GMI_PH_SHUFFLE, 0.0, 2.0 * g->B * (2.0 * geo_.wp[0] + 4.0 * geo_.A + 12.0), [&] {
        ppo::launch_shuffle(g->X_roll, g->act, g->logp, g->adv, g->ret, g->adv_stats, g->X_sh, g->act_sh,
                            g->oldlp_sh, g->adv_sh, g->ret_sh, g->N, T_, geo_.wp[0], geo_.A, cfg_.seed, g->gid, e,
                            ctl_dev_, g->s);
      });
      ++launches_;
    }
    for (int k = 0; k < K_; ++k, ++step) {
      for (auto& g : gmis_) {
        if (fused_adam) {
          train_minibatch(*g, k, step);
          GMI_CUDA_CHECK(cudaEventRecord(g->ev_done, g->s));
          continue;
        }
        if (adam_inline_) {  // Adam of the previous step is the in-stream predecessor; this
          // step's Adam runs inside the gradient assembly (each element updated as it is summed)
          no_b_preload_once_ = step > 0;
          train_minibatch(*g, k, step);
          GMI_CUDA_CHECK(cudaEventRecord(g->ev_done, g->s));
          continue;
        }
        if (step > 0) GMI_CUDA_CHECK(cudaStreamWaitEvent(g->s, ev_adam_, 0));
        train_minibatch(*g, k);
        GMI_CUDA_CHECK(cudaEventRecord(g->ev_done, g->s));
      }
      if (!fused_adam && !adam_inline_) reduce_and_step(step);
    }
  }
  for (auto& g : gmis_) GMI_CUDA_CHECK(cudaStreamWaitEvent(upd_, g->ev_done, 0));
  if (split_) {
    // the partner's rollout i+1 is done with the snapshot (R >= i + 2): push theta_{i+1} into its
    // link window over NVLink, then S = i + 2
    ppo::launch_link_wait(link_flag(false, 0), nullptr, lctr_ + 4, 1, upd_);
    GMI_CUDA_CHECK(cudaMemcpyAsync(lpeer_ + loff_params_, params_, (size_t)geo_.P * 4, cudaMemcpyDeviceToDevice, upd_));
    GMI_CUDA_CHECK(cudaMemcpyAsync(lpeer_ + loff_shadow_, shadow_, (size_t)geo_.P * 2, cudaMemcpyDeviceToDevice, upd_));
    ppo::launch_link_signal(link_flag(true, 256), lctr_ + 5, 1, upd_);
    launches_ += 2;
  } else if (decoupled_) {  // rollout i+1 is done with the snapshot: refresh it to theta_{i+1}
    GMI_CUDA_CHECK(cudaStreamWaitEvent(upd_, ev_rolled_, 0));
    GMI_CUDA_CHECK(cudaMemcpyAsync(params_roll_, params_, (size_t)geo_.P * 4, cudaMemcpyDeviceToDevice, upd_));
    GMI_CUDA_CHECK(cudaMemcpyAsync(shadow_roll_, shadow_, (size_t)geo_.P * 2, cudaMemcpyDeviceToDevice, upd_));
  }
  timed(upd_, GMI_PH_OTHER, 0.0, 0.0, [&] {
    GMI_CUDA_CHECK(cudaMemcpyAsync(stats_dev_ + 4, gmis_[0]->adv_stats, 3 * 4, cudaMemcpyDeviceToDevice, upd_));
    GMI_CUDA_CHECK(cudaMemcpyAsync(stats_host_, stats_dev_, 8 * 4, cudaMemcpyDeviceToHost, upd_));
    ppo::launch_control_advance(ctl_dev_, cfg_.epochs * K_, upd_);
  });
  ++launches_;
}

// gmi_resize: re-split this GPU's green-context partitions on a live trainer. Env state,
// experience, parameters, optimizer state and the exchange window stay where they are; the
// streams move to the new partitions and the GEMM plans (split-K / tile choices depend on each
// GMI's SM count) and the iteration graph are rebuilt. The GMI count is fixed (changing it
// re-partitions the envs over GMIs, which is a new trainer).
void Trainer::resize(const int* sms, int n) {
  if (!exec_ || exec_->backend() != 1)
    invalid("gmi_resize: SM shares exist only for green-context GMIs (gmi_backend = 1)");
  const int units = decoupled_ ? 2 : n_local_;
  if (n != units)
    invalid("gmi_resize: t = " + std::to_string(n) + " but this GPU runs " + std::to_string(units) +
            " GMIs (changing the count re-partitions the envs; create a new trainer)");
  GMI_CUDA_CHECK(cudaSetDevice(cfg_.device));
  GMI_CUDA_CHECK(cudaDeviceSynchronize());
  auto fresh = std::make_unique<GmiResources>(cfg_.device, std::vector<int>(sms, sms + n), 1);  // validates
  if (graph_) GMI_CUDA_CHECK(cudaGraphExecDestroy(graph_));
  graph_ = nullptr;
  exec_ = std::move(fresh);  // the old partitions (and their streams) are released here
  const int tix = decoupled_ ? 1 : 0;
  if (decoupled_) serve_s_ = exec_->stream(0);
  if (upd_in_gmi_) upd_ = exec_->extra_stream(1);
  for (auto& g : gmis_) {
    g->s = exec_->stream(tix + g->local);
    g->s2 = exec_->aux_stream(tix + g->local);
    g->ctas = exec_->sm_count(tix + g->local);
  }
  build_plans();
  GMI_CUDA_CHECK(cudaDeviceSynchronize());
}

// AsyncDecoupled across GPUs, serving rank: rollout i+1 once the trainer has pulled rollout i
// (C >= i + 1) and pushed the snapshot theta_i (S >= i + 1); the first call first rolls out
// rollout 0 with theta_0 (initialised here from the same seed as the trainer's). Eager launches
// on the serving stream; every rollout ends with R = rollouts.
void Trainer::serve_iteration() {
  Gmi& g = *gmis_[0];
  launches_ = 0;
  marks_used_ = 0;
  if (rollouts_ == 0) {
    GMI_CUDA_CHECK(cudaMemcpyAsync(params_roll_, params_, (size_t)geo_.P * 4, cudaMemcpyDeviceToDevice, serve_s_));
    GMI_CUDA_CHECK(cudaMemcpyAsync(shadow_roll_, shadow_, (size_t)geo_.P * 2, cudaMemcpyDeviceToDevice, serve_s_));
    GMI_CUDA_CHECK(cudaMemsetAsync(ctl_roll_, 0, sizeof(ppo::Control), serve_s_));
    ppo::launch_link_signal(link_flag(false, 256), lctr_ + 6, 0, serve_s_);  // own S = 1: theta_0 present
    serve_rollout(g);
    ppo::launch_link_signal(link_flag(true, 0), lctr_ + 0, 0, serve_s_);
  }
  ppo::launch_link_wait(link_flag(false, 128), link_flag(false, 256), lctr_ + 1, 0, serve_s_);
  serve_rollout(g);
  ppo::launch_link_signal(link_flag(true, 0), lctr_ + 0, 0, serve_s_);
  launches_ += 2;
}

unsigned long long* Trainer::link_flag(bool peer, size_t off) const {
  return reinterpret_cast<unsigned long long*>((peer ? lpeer_ : lwin_) + off);
}

void Trainer::link_handle(void* out64) const {
  if (!split_) invalid("gmi_ppo_link_handle: the trainer was not created with decoupled = 2");
  cudaIpcMemHandle_t h;
  GMI_CUDA_CHECK(cudaIpcGetMemHandle(&h, lwin_));
  std::memcpy(out64, &h, sizeof(h));
}

void Trainer::link_attach(const void* peer64) {
  if (!split_) invalid("gmi_ppo_link_attach: the trainer was not created with decoupled = 2");
  if (linked_) invalid("gmi_ppo_link_attach: already wired");
  GMI_CUDA_CHECK(cudaSetDevice(cfg_.device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, peer64, sizeof(h));
  void* p = nullptr;
  GMI_CUDA_CHECK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  ipc_opened_.push_back(p);
  lpeer_ = static_cast<char*>(p);
  linked_ = true;
}

void Trainer::link_connect(Trainer* sv, Trainer* tr) {
  if (!sv || !tr || !sv->split_ || !tr->split_ || !sv->serving_ || tr->serving_)
    invalid("gmi_ppo_link_connect: (serving rank, trainer rank) of one decoupled = 2 job");
  if (sv->link_gpus_ != tr->link_gpus_ || tr->link_rank_ != sv->link_rank_ + sv->link_gpus_ / 2 ||
      sv->lwin_bytes_ != tr->lwin_bytes_)
    invalid("gmi_ppo_link_connect: the trainer rank must be serving rank + num_gpus / 2 of the same job");
  if (sv->linked_ || tr->linked_) invalid("gmi_ppo_link_connect: already wired");
  if (sv->cfg_.device == tr->cfg_.device)
    invalid("gmi_ppo_link_connect: ranks on one GPU need one process each (gmi_ppo_link_attach)");
  for (auto [a, b] : {std::pair<Trainer*, Trainer*>{sv, tr}, {tr, sv}}) {
    GMI_CUDA_CHECK(cudaSetDevice(a->cfg_.device));
    const cudaError_t e = cudaDeviceEnablePeerAccess(b->cfg_.device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else GMI_CUDA_CHECK(e);
    a->lpeer_ = b->lwin_;
    a->linked_ = true;
  }
}

void Trainer::comm_handle(void* out64) const {
  if (!xchg_) invalid("gmi_ppo_comm_handle: the trainer was not created with comm = 1");
  cudaIpcMemHandle_t h;
  GMI_CUDA_CHECK(cudaIpcGetMemHandle(&h, win_));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(out64, &h, sizeof(h));
}

void Trainer::comm_attach(const void* handles) {
  if (!xchg_) invalid("gmi_ppo_comm_attach: the trainer was not created with comm = 1");
  if (connected_) invalid("gmi_ppo_comm_attach: already wired");
  GMI_CUDA_CHECK(cudaSetDevice(cfg_.device));
  const char* hb = static_cast<const char*>(handles);
  for (int q = 0; q < cfg_.num_gpus; ++q) {
    char* base = win_;
    if (q != cfg_.rank) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, hb + 64 * q, 64);
      void* p = nullptr;
      GMI_CUDA_CHECK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      ipc_opened_.push_back(p);
      base = static_cast<char*>(p);
    }
    xa_.ready[q] = reinterpret_cast<unsigned long long*>(base);
    xa_.done[q] = reinterpret_cast<unsigned long long*>(base + ppo::kXchgDoneOff);
    xa_.pub[q] = reinterpret_cast<const float*>(n_local_ == 1 ? base + win_off_gmi_ : base + ppo::kXchgHeader);
    for (int j = 0; j < n_local_; ++j)
      xa_.gpub[q][j] = reinterpret_cast<const float*>(base + win_off_gmi_ + (size_t)j * geo_.P * 4);
    xa_.params[q] = reinterpret_cast<float*>(base + win_off_params_);
    xa_.shadow[q] = reinterpret_cast<__nv_bfloat16*>(base + win_off_shadow_);
  }
  connected_ = true;
}

void Trainer::comm_connect(Trainer* const* t, int n) {
  if (n < 1 || n > ppo::kMaxRanks) invalid("gmi_ppo_comm_connect: 1..8 trainers");
  for (int r = 0; r < n; ++r) {
    if (!t[r] || !t[r]->xchg_) invalid("gmi_ppo_comm_connect: every trainer needs comm = 1");
    if (t[r]->cfg_.rank != r || t[r]->cfg_.num_gpus != n || t[r]->geo_.P != t[0]->geo_.P ||
        t[r]->n_local_ != t[0]->n_local_)
      invalid("gmi_ppo_comm_connect: trainers[r] must be rank r of one num_gpus = n job");
    if (t[r]->connected_) invalid("gmi_ppo_comm_connect: already wired");
    // Ranks of one process must sit on distinct devices: two ranks sharing a device in one
    // context can have their streams multiplexed onto one hardware queue, where a rank's wait for
    // its peer would block the peer's own work (ranks sharing a GPU: one process each + IPC).
    for (int q = 0; q < r && n > 1; ++q)
      if (t[q]->cfg_.device == t[r]->cfg_.device)
        invalid("gmi_ppo_comm_connect: ranks " + std::to_string(q) + " and " + std::to_string(r) +
                " share device " + std::to_string(t[r]->cfg_.device) +
                "; ranks on one GPU need one process each (gmi_ppo_comm_attach)");
  }
  for (int r = 0; r < n; ++r) {
    Trainer& me = *t[r];
    GMI_CUDA_CHECK(cudaSetDevice(me.cfg_.device));
    for (int q = 0; q < n; ++q) {
      const Trainer& peer = *t[q];
      if (peer.cfg_.device != me.cfg_.device) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(peer.cfg_.device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else GMI_CUDA_CHECK(e);
      }
      me.xa_.ready[q] = reinterpret_cast<unsigned long long*>(peer.win_);
      me.xa_.done[q] = reinterpret_cast<unsigned long long*>(peer.win_ + ppo::kXchgDoneOff);
      me.xa_.pub[q] = peer.n_local_ == 1 ? peer.gmis_[0]->grad : peer.grad_sum_;
      for (int j = 0; j < peer.n_local_; ++j) me.xa_.gpub[q][j] = peer.gmis_[j]->grad;
      me.xa_.params[q] = peer.params_;
      me.xa_.shadow[q] = peer.shadow_;
    }
    me.connected_ = true;
  }
  GMI_CUDA_CHECK(cudaSetDevice(t[n - 1]->cfg_.device));
}

void Trainer::enqueue_iteration(bool host_control) {
  if (xchg_ && !connected_)
    invalid("peer exchange not wired: call gmi_ppo_comm_attach / gmi_ppo_comm_connect before iterating");
  if (split_ && !linked_)
    invalid("experience link not wired: call gmi_ppo_link_attach / gmi_ppo_link_connect before iterating");
  GMI_CUDA_CHECK(cudaSetDevice(cfg_.device));
  if (split_ && serving_) {
    serve_iteration();
    iteration_ += 1;
    return;
  }
  ensure_bias_table(adam_steps_ + (long long)cfg_.epochs * K_ + 1);
  if (host_control || iteration_ == 0) write_control();
  if (decoupled_ && !split_ && rollouts_ == 0) {  // prologue: rollout 0 with theta_0 (not overlapped)
    GMI_CUDA_CHECK(cudaMemcpyAsync(params_roll_, params_, (size_t)geo_.P * 4, cudaMemcpyDeviceToDevice, upd_));
    GMI_CUDA_CHECK(cudaMemcpyAsync(shadow_roll_, shadow_, (size_t)geo_.P * 2, cudaMemcpyDeviceToDevice, upd_));
    GMI_CUDA_CHECK(cudaMemsetAsync(ctl_roll_, 0, sizeof(ppo::Control), upd_));
    GMI_CUDA_CHECK(cudaEventRecord(ev_start_, upd_));
    GMI_CUDA_CHECK(cudaStreamWaitEvent(serve_s_, ev_start_, 0));
    serve_rollout(*gmis_[0]);
    GMI_CUDA_CHECK(cudaStreamWaitEvent(upd_, ev_rolled_, 0));
  }
  if (rollout_pending_) {  // after the rollout hook: the update phases only, eagerly
    rollout_pending_ = false;
    record_iteration(false);
  } else if (cfg_.use_graph && iteration_ > 0) {
    if (!graph_) {
      GMI_CUDA_CHECK(cudaStreamSynchronize(upd_));
      cudaGraph_t gr;
      GMI_CUDA_CHECK(cudaStreamBeginCapture(upd_, cudaStreamCaptureModeThreadLocal));
      capturing_ = true;
      try {
        record_iteration(true);
      } catch (...) {
        cudaStreamEndCapture(upd_, &gr);
        capturing_ = false;
        throw;
      }
      capturing_ = false;
      GMI_CUDA_CHECK(cudaStreamEndCapture(upd_, &gr));
      GMI_CUDA_CHECK(cudaGraphInstantiate(&graph_, gr, 0));
      GMI_CUDA_CHECK(cudaGraphDestroy(gr));
    }
    GMI_CUDA_CHECK(cudaGraphLaunch(graph_, upd_));
  } else {
    record_iteration(true);
  }
  iteration_ += 1;
  adam_steps_ += (long long)cfg_.epochs * K_;
}

void Trainer::synchronize(gmi_ppo_stats_t* st) {
  GMI_CUDA_CHECK(cudaStreamSynchronize(upd_));
  for (auto& g : gmis_) GMI_CUDA_CHECK(cudaStreamSynchronize(g->s));
  if (serve_s_) GMI_CUDA_CHECK(cudaStreamSynchronize(serve_s_));
  gmi_ppo_phase_t gemm{};
  if (cfg_.instrument) {
    std::memset(phases_, 0, sizeof(phases_));
    unit_busy_ms_.assign(decoupled_ ? 3 : n_local_ + 1, 0.0);
    for (int i = 0; i < marks_used_; ++i) {
      float ms = 0;
      GMI_CUDA_CHECK(cudaEventElapsedTime(&ms, marks_[i].a, marks_[i].b));
      unit_busy_ms_.at(marks_[i].unit) += ms;
      if (!marks_[i].in_phases) continue;
      gmi_ppo_phase_t& ph = phases_[marks_[i].phase];
      ph.ms += ms;
      ph.flop += marks_[i].flop;
      ph.bytes += marks_[i].bytes;
      ph.launches += 1;
      if (marks_[i].flop > 0) {
        gemm.ms += ms;
        gemm.flop += marks_[i].flop;
        gemm.bytes += marks_[i].bytes;
        gemm.launches += 1;
      }
    }
  }
  if (!st) return;
  std::memset(st, 0, sizeof(*st));
  const double Bm = gmis_[0]->Bm;
  st->policy_loss = stats_host_[0] / Bm;
  st->value_loss = stats_host_[1] / Bm;
  st->approx_kl = stats_host_[2] / Bm;
  st->clip_frac = stats_host_[3] / Bm;
  st->mean_reward = stats_host_[6];
  long long steps = 0;  // decoupled = 2: counted by the serving ranks only (a job-wide sum stays right)
  for (auto& g : gmis_) steps += split_ && !serving_ ? 0 : (long long)T_ * g->N;
  st->env_steps = steps;
  st->kernel_launches = launches_;
  st->gemm_ms = gemm.ms;
  st->gemm_flop = gemm.flop;
  st->gemm_launches = gemm.launches;
  st->gemm_bytes = gemm.bytes;
}

// ------------------------------------------------------------------ parity hooks
void Trainer::minibatch_grad(int gi, const float* X, const float* act, const float* oldlp, const float* adv,
                             const float* ret, int B, float* grad_out) {
  Gmi& g = *gmis_.at(gi);
  if (B != g.Bm) invalid("minibatch rows must equal the trainer's minibatch size");
  const int S = geo_.S, S_p = geo_.wp[0], A = geo_.A;
  std::vector<uint16_t> xb((size_t)B * S_p, 0);
  for (int r = 0; r < B; ++r)
    for (int i = 0; i < S; ++i) xb[(size_t)r * S_p + i] = bf16_bits(X[(size_t)r * S + i]);
  GMI_CUDA_CHECK(cudaDeviceSynchronize());
  GMI_CUDA_CHECK(cudaMemcpy(g.X_sh, xb.data(), xb.size() * 2, cudaMemcpyHostToDevice));
  GMI_CUDA_CHECK(cudaMemcpy(g.act_sh, act, (size_t)B * A * 4, cudaMemcpyHostToDevice));
  GMI_CUDA_CHECK(cudaMemcpy(g.oldlp_sh, oldlp, (size_t)B * 4, cudaMemcpyHostToDevice));
  GMI_CUDA_CHECK(cudaMemcpy(g.adv_sh, adv, (size_t)B * 4, cudaMemcpyHostToDevice));
  GMI_CUDA_CHECK(cudaMemcpy(g.ret_sh, ret, (size_t)B * 4, cudaMemcpyHostToDevice));
  train_minibatch(g, 0);
  GMI_CUDA_CHECK(cudaStreamSynchronize(g.s));
  GMI_CUDA_CHECK(cudaMemcpy(grad_out, g.grad, (size_t)geo_.P * 4, cudaMemcpyDeviceToHost));
}

long long Trainer::get(const std::string& what, int gi, void* dst) {
  GMI_CUDA_CHECK(cudaDeviceSynchronize());
  auto copy = [&](const void* src, long long n, int esz) {
    if (dst) GMI_CUDA_CHECK(cudaMemcpy(dst, src, (size_t)n * esz, cudaMemcpyDeviceToHost));
    return n;
  };
  const long long P = geo_.P;
  if (what == "params") return copy(split_ && serving_ ? params_roll_ : params_, P, 4);
  if (what == "adam_m") return copy(m_, P, 4);
  if (what == "adam_v") return copy(v_, P, 4);
  Gmi& g = *gmis_.at(gi);
  const long long N = g.N, T = T_, S = geo_.S, A = geo_.A;
  if (split_ && !serving_ && (what == "rew" || what == "val" || what == "done" || what == "x" || what == "ep_step" ||
                              what == "ep_len" || what == "ep_count"))
    invalid("decoupled = 2: '" + what + "' lives on the serving rank");
  if (what == "grad") return copy(g.grad, P, 4);
  if (what == "x") return copy(g.x, N * S, 4);
  // epoch copy of the last shuffle (rows permuted by the epoch's bijection)
  if (what == "oldlp_sh") return copy(g.oldlp_sh, T * N, 4);
  if (what == "act_sh") return copy(g.act_sh, T * N * A, 4);
  if (what == "trained_logp") return copy(g.logp, T * N, 4);  // the trainer's rollout copy
  // decoupled mode: rollout fields (act/logp/rew/done/obs/val/adv/ret) are the latest rollout
  // in the experience channel, one rollout ahead of the trainer
  const bool ch = decoupled_ && !(split_ && !serving_);
  if (what == "act") return copy(ch ? g.ch_act : g.act, T * N * A, 4);
  if (what == "logp") return copy(ch ? g.ch_logp : g.logp, T * N, 4);
  if (what == "rew") return copy(ch ? g.ch_rew : g.rew, T * N, 4);
  if (what == "val") return copy(ch ? g.ch_V : g.V, (T + 1) * N, 4);
  if (what == "adv") return copy(ch ? g.ch_adv : g.adv, T * N, 4);
  if (what == "ret") return copy(ch ? g.ch_ret : g.ret, T * N, 4);
  if (what == "done") return copy(ch ? g.ch_done : g.done, T * N, 1);
  if (what == "ep_step") return copy(g.ep_step, N, 4);
  if (what == "ep_len") return copy(g.ep_len, N, 4);
  if (what == "ep_count") return copy(g.ep_count, N, 4);
  if (what.size() == 3 && (what[0] == 'H' || what[0] == 'D')) {  // debug: H<net><layer> / D<net><layer>
    const int n = what[1] - '0', l = what[2] - '0';
    if (n < 0 || n > 1 || l < 0 || l >= geo_.L) invalid("bad activation name");
    const long long w = geo_.wp[l + 1], rows = g.Bm;
    if (dst) {
      std::vector<uint16_t> raw((size_t)(rows * w));
      const void* src = what[0] == 'H' ? (const void*)g.H[n][l] : (const void*)g.D[n][l];
      GMI_CUDA_CHECK(cudaMemcpy(raw.data(), src, raw.size() * 2, cudaMemcpyDeviceToHost));
      float* o = static_cast<float*>(dst);
      for (size_t i = 0; i < raw.size(); ++i) o[i] = bf16_float(raw[i]);
    }
    return rows * w;
  }
  if (what == "head_part") {  // per-block head-gradient / loss partial records (debug)
    const int parts = g.fused_head ? g.head_grid : ppo::head_loss_blocks(g.Bm);
    return copy(g.head_part, (long long)parts * ppo::head_partial_stride(geo_.A), 4);
  }
  if (what == "head_trace") {  // GMI_HEAD_TRACE=1 with a TRACE=1 build
    if (!head_trace_) invalid("head trace not enabled (GMI_HEAD_TRACE=1)");
    return copy(head_trace_, 64, 8);
  }
  if (what == "gemm_trace") {
    if (!gemm_trace_) invalid("GEMM trace not enabled (GMI_GEMM_TRACE=<phase>)");
    return copy(gemm_trace_, 128, 8);
  }
  if (what == "train_fwd_trace") {  // GMI_TRAIN_FWD_TRACE=1: stamps of CTA 0, last minibatch
    if (!g.fwd_args.trace) invalid("train-forward trace not enabled (GMI_TRAIN_FWD_TRACE=1)");
    return copy(g.fwd_args.trace, 64, 8);
  }
  if (what == "rollout_trace") {  // GMI_ROLLOUT_TRACE=1: globaltimer stamps of CTA 0 (int64)
    if (!g.roll_args.trace) invalid("rollout trace not enabled (GMI_ROLLOUT_TRACE=1)");
    return copy(g.roll_args.trace, T * 16, 8);
  }
  if (what == "obs") {  // bf16 X_roll -> fp32 [(T+1)][N][S]
    const long long n = (T + 1) * N * S;
    if (dst) {
      const int S_p = geo_.wp[0];
      std::vector<uint16_t> raw((size_t)(T + 1) * N * S_p);
      GMI_CUDA_CHECK(cudaMemcpy(raw.data(), ch ? g.ch_X : g.X_roll, raw.size() * 2, cudaMemcpyDeviceToHost));
      float* o = static_cast<float*>(dst);
      for (long long r = 0; r < (T + 1) * N; ++r)
        for (long long i = 0; i < S; ++i) o[r * S + i] = bf16_float(raw[(size_t)(r * S_p + i)]);
    }
    return n;
  }
  invalid("unknown state field: " + what);
}

void Trainer::set(const std::string& what, int gi, const void* src, long long n) {
  GMI_CUDA_CHECK(cudaDeviceSynchronize());
  auto put = [&](void* d, long long want, int esz) {
    if (n != want) invalid("size mismatch for " + what);
    GMI_CUDA_CHECK(cudaMemcpy(d, src, (size_t)n * esz, cudaMemcpyHostToDevice));
  };
  const long long P = geo_.P;
  if (what == "params") {
    put(params_, P, 4);
    std::vector<uint16_t> sh(P);
    const float* f = static_cast<const float*>(src);
    for (long long i = 0; i < P; ++i) sh[i] = bf16_bits(f[i]);
    GMI_CUDA_CHECK(cudaMemcpy(shadow_, sh.data(), P * 2, cudaMemcpyHostToDevice));
    return;
  }
  if (what == "adam_m") return put(m_, P, 4);
  if (what == "adam_v") return put(v_, P, 4);
  Gmi& g = *gmis_.at(gi);
  if (what == "x") return put(g.x, (long long)g.N * geo_.S, 4);
  if (what == "ep_step") return put(g.ep_step, g.N, 4);
  if (what == "ep_count") return put(g.ep_count, g.N, 4);
  invalid("field not settable: " + what);
}

}  // namespace gmi

// ------------------------------------------------------------------ C-ABI
extern "C" {

GMI_API void gmi_ppo_config_defaults(gmi_ppo_config_t* c) {
  std::memset(c, 0, sizeof(*c));
  c->obs_dim = 60;
  c->act_dim = 8;
  c->num_hidden = 3;
  c->hidden[0] = c->hidden[1] = c->hidden[2] = 256;
  c->num_envs = 4096;
  c->horizon = 32;
  c->epochs = 4;
  c->minibatches = 4;
  c->gamma = 0.99f;
  c->lam = 0.95f;
  c->clip = 0.2f;
  c->lr = 3e-4f;
  c->beta1 = 0.9f;
  c->beta2 = 0.999f;
  c->adam_eps = 1e-8f;
  c->vf_coef = 1.0f;
  c->ent_coef = 0.0f;
  c->seed = 20240811ull;
  c->num_gpus = 1;
  c->gmis_per_gpu = 1;
  c->use_graph = 1;
}

GMI_API int gmi_ppo_create(const gmi_ppo_config_t* cfg, const void* nccl_id, void** trainer) {
  return gmi::guarded([&] {
    if (!cfg || !trainer) gmi::invalid("null argument");
    *trainer = new gmi::Trainer(*cfg, nccl_id);
  });
}

GMI_API void gmi_ppo_free(void* t) { delete static_cast<gmi::Trainer*>(t); }

GMI_API int gmi_nccl_unique_id(void* out) {
  return gmi::guarded([&] {
    ncclUniqueId id;
    NCCL_CHECK(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
  });
}

GMI_API int gmi_ppo_iteration(void* t, gmi_ppo_stats_t* st) {
  return gmi::guarded([&] {
    auto* tr = static_cast<gmi::Trainer*>(t);
    tr->enqueue_iteration(true);
    tr->synchronize(st);
  });
}

GMI_API int gmi_ppo_iteration_async(void* t) {
  return gmi::guarded([&] { static_cast<gmi::Trainer*>(t)->enqueue_iteration(false); });
}

GMI_API int gmi_ppo_synchronize(void* t, gmi_ppo_stats_t* st) {
  return gmi::guarded([&] { static_cast<gmi::Trainer*>(t)->synchronize(st); });
}

GMI_API int gmi_resize(void* t, int gpu, const int* sm_counts, int n) {
  return gmi::guarded([&] {
    if (!t || !sm_counts) gmi::invalid("null argument");
    auto* tr = static_cast<gmi::Trainer*>(t);
    if (gpu != tr->rank()) gmi::invalid("gmi_resize: this trainer drives GPU (rank) " + std::to_string(tr->rank()));
    tr->resize(sm_counts, n);
  });
}

GMI_API int gmi_ppo_tune_shares(void* t, const int* candidates, int ncand, int iters, int* best,
                                double* throughput) {
  return gmi::guarded([&] {
    if (!t || !candidates || ncand < 1 || iters < 1) gmi::invalid("gmi_ppo_tune_shares: bad arguments");
    auto* tr = static_cast<gmi::Trainer*>(t);
    const int n = tr->units();
    cudaEvent_t a, b;
    GMI_CUDA_CHECK(cudaEventCreate(&a));
    GMI_CUDA_CHECK(cudaEventCreate(&b));
    int bi = 0;
    double bv = -1.0;
    try {
      for (int c = 0; c < ncand; ++c) {
        tr->resize(candidates + (size_t)c * n, n);
        tr->enqueue_iteration(false);  // eager after a resize (rebuilds the graph on the next call)
        tr->enqueue_iteration(false);  // capture
        tr->synchronize(nullptr);
        GMI_CUDA_CHECK(cudaEventRecord(a, tr->stream(-1)));
        for (int i = 0; i < iters; ++i) tr->enqueue_iteration(false);
        GMI_CUDA_CHECK(cudaEventRecord(b, tr->stream(-1)));
        gmi_ppo_stats_t st;
        tr->synchronize(&st);
        float ms = 0.f;
        GMI_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
        const double v = double(st.env_steps) * iters / (double(ms) / 1e3);
        if (throughput) throughput[c] = v;
        if (v > bv) bv = v, bi = c;
      }
      tr->resize(candidates + (size_t)bi * n, n);
    } catch (...) {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      throw;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (best) *best = bi;
  });
}

GMI_API int gmi_ppo_comm_handle(void* t, void* out64) {
  return gmi::guarded([&] {
    if (!t || !out64) gmi::invalid("null argument");
    static_cast<gmi::Trainer*>(t)->comm_handle(out64);
  });
}

GMI_API int gmi_ppo_comm_attach(void* t, const void* handles) {
  return gmi::guarded([&] {
    if (!t || !handles) gmi::invalid("null argument");
    static_cast<gmi::Trainer*>(t)->comm_attach(handles);
  });
}

GMI_API int gmi_ppo_comm_connect(void* const* trainers, int n) {
  return gmi::guarded([&] {
    if (!trainers) gmi::invalid("null argument");
    std::vector<gmi::Trainer*> v(n > 0 ? n : 0);
    for (int i = 0; i < n; ++i) v[i] = static_cast<gmi::Trainer*>(trainers[i]);
    gmi::Trainer::comm_connect(v.data(), n);
  });
}

GMI_API int gmi_ppo_link_handle(void* t, void* out64) {
  return gmi::guarded([&] {
    if (!t || !out64) gmi::invalid("null argument");
    static_cast<gmi::Trainer*>(t)->link_handle(out64);
  });
}

GMI_API int gmi_ppo_link_attach(void* t, const void* peer64) {
  return gmi::guarded([&] {
    if (!t || !peer64) gmi::invalid("null argument");
    static_cast<gmi::Trainer*>(t)->link_attach(peer64);
  });
}

GMI_API int gmi_ppo_link_connect(void* serving, void* trainer) {
  return gmi::guarded([&] {
    gmi::Trainer::link_connect(static_cast<gmi::Trainer*>(serving), static_cast<gmi::Trainer*>(trainer));
  });
}

GMI_API int gmi_ppo_rollout(void* t) {
  return gmi::guarded([&] {
    auto* tr = static_cast<gmi::Trainer*>(t);
    tr->enqueue_rollout();
    tr->synchronize(nullptr);
  });
}

GMI_API int gmi_ppo_minibatch_grad(void* t, int gmi, const float* X, const float* act, const float* oldlp,
                                   const float* adv, const float* ret, int B, float* grad_out) {
  return gmi::guarded([&] { static_cast<gmi::Trainer*>(t)->minibatch_grad(gmi, X, act, oldlp, adv, ret, B, grad_out); });
}

GMI_API int gmi_ppo_get(void* t, const char* what, int gmi, void* dst, long long* n) {
  return gmi::guarded([&] {
    const long long c = static_cast<gmi::Trainer*>(t)->get(what ? what : "", gmi, dst);
    if (n) *n = c;
  });
}

GMI_API int gmi_ppo_set(void* t, const char* what, int gmi, const void* src, long long n) {
  return gmi::guarded([&] { static_cast<gmi::Trainer*>(t)->set(what ? what : "", gmi, src, n); });
}

GMI_API int gmi_ppo_param_count(void* t, long long* padded, long long* real) {
  return gmi::guarded([&] {
    const auto& g = static_cast<gmi::Trainer*>(t)->geometry();
    if (padded) *padded = g.P;
    if (real) *real = g.real_params;
  });
}

GMI_API int gmi_ppo_stream(void* t, int gmi, void** stream) {
  return gmi::guarded([&] { *stream = static_cast<gmi::Trainer*>(t)->stream(gmi); });
}

GMI_API const char* gmi_ppo_phase_name(int phase) {
  static const char* const names[GMI_PPO_PHASES] = {
      "roll_gemm", "roll_head", "act_env", "val_gemm", "val_head", "gae",      "shuffle",
      "fwd_gemm",  "head_fwd",  "head_loss", "head_dx", "head_dw", "dw_gemm", "colsum",
      "dx_gemm",   "segments",  "reduce",  "allreduce", "adam",   "other"};
  return phase >= 0 && phase < GMI_PPO_PHASES ? names[phase] : nullptr;
}

GMI_API int gmi_ppo_profile(void* t, gmi_ppo_phase_t* out) {
  return gmi::guarded([&] {
    if (!out) gmi::invalid("null output");
    std::memcpy(out, static_cast<gmi::Trainer*>(t)->phases(), sizeof(gmi_ppo_phase_t) * GMI_PPO_PHASES);
  });
}

GMI_API int gmi_ppo_unit_busy(void* t, double* busy_ms, int* sms, int cap, int* count) {
  return gmi::guarded([&] {
    const int n = static_cast<gmi::Trainer*>(t)->busy_units(busy_ms, sms, cap);
    if (count) *count = n;
  });
}

GMI_API int gmi_ppo_set_instrument(void* t, int on) {
  return gmi::guarded([&] { static_cast<gmi::Trainer*>(t)->set_instrument(on); });
}

}  // extern "C"
