// Device-side interface of the PPO iteration kernels (K3-K8 of SURVEY §2.2) and their
// host launch wrappers. Layouts (per GMI, N envs, horizon T, padded obs width S_p):
//   env state   x[N][S] fp32, ep_step/ep_len/ep_count[N] int32
//   rollout     X_roll[(T+1)][N][S_p] bf16 (GEMM-ready observations, pads stay 0),
//               act[T][N][A], logp/rew[T][N] fp32, done[T][N] u8, V[(T+1)][N] fp32
//   advantages  adv/ret[T][N] fp32, normalised in the epoch shuffle
//   epoch copy  X_sh[B][S_p] bf16, act_sh[B][A], oldlp/adv/ret_sh[B]  (B = T*N, permuted)
//   head grads  G_pi[Bm][64] / G_v[Bm][64] bf16 (dL/dmu, dL/dv; zero pads) for the
//               tensor-core head weight-gradient GEMM
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "rng.cuh"  // GMI_HD

namespace gmi::ppo {

constexpr int kMaxAct = 31;  // lane 31 carries the value head in the head kernel
constexpr int kMaxHeadIn = 512;
constexpr int kHeadG = 64;  // padded width of the G_pi / G_v buffers

// Device-resident control block, refreshed by the host (H2D) once per iteration.
struct Control {
  int iteration;
  int pad_;
  long long adam_step0;  // Adam steps completed before this iteration
};

struct EnvParams {
  int N, S, A, S_p;
  int env0;  // global id of env 0 of this GMI
  int T;
  uint64_t seed;
};

struct ActEnvArgs {
  EnvParams ep;
  const float* mu;    // [N][64] policy-head GEMM output (bias not yet added)
  const float* b_mu;  // [A]
  const float* log_std;
  float* x;
  int* ep_step;
  const int* ep_len;
  int* ep_count;
  __nv_bfloat16* X_next;  // X_roll + (t+1)*N*S_p
  float* act;             // act + t*N*A
  float* logp;            // + t*N
  float* rew;
  uint8_t* done;
  int t;
  const Control* ctl;
};

struct HeadLossArgs {
  const float* mu;  // [B][64] policy-head GEMM output (no bias)
  const float* v;   // [B][64] value-head GEMM output, column 0 (no bias)
  const float* b_mu;
  const float* b_v;
  const float* log_std;
  const float* act;  // [B][A]
  const float* oldlp;
  const float* adv;
  const float* ret;
  __nv_bfloat16* Gpi;  // [B][64] dL/dmu (bf16), input of the head input/weight-gradient GEMMs
  __nv_bfloat16* Gv;   // [B][64] dL/dv in column 0
  float* partial;      // [blocks][head_partial_stride(A)]
  int B, A;
  float clip, vf_coef, ent_coef;
};

// One head-loss partial record: db_mu[A], db_v, dlog_std[A], 4 loss statistics.
GMI_HD constexpr int head_partial_stride(int A) { return 2 * A + 5; }
constexpr int kHeadRowsPerBlock = 64;

struct Segment {  // dst[i] = sum_{p < nparts} src[p * stride + i]  (fixed order)
  float* dst;
  const float* src;
  long long stride;
  int len;
  int nparts;
  long long param_off = -1;  // >= 0: dst[i] is the gradient of parameter param_off + i (fused Adam)
};

// Adam applied by the gradient-assembly kernel right after an element's gradient is summed
// (single GMI, single GPU: no cross-GMI fold or all-reduce sits in between).
struct SegAdam {
  float* p;
  float* m;
  float* v;
  __nv_bfloat16* shadow;
  const float* bc;  // [2*steps] bias corrections
  const Control* ctl;
  int step_in_iter;
  float lr, b1, b2, eps, inv_n;
};

// Cross-GPU exchange + sharded Adam over peer memory (cuda/exchange.cu).
constexpr int kMaxRanks = 8;
constexpr int kMaxLocalGmis = 16;
constexpr int kMaxXchgCtas = 1184;      // exchange grid (8 CTAs per SM at most)
constexpr int kXchgDoneOff = 1024;      // window: done flags [kMaxRanks][kMaxXchgCtas] u64 from here
constexpr int kXchgHeader = 1024 + kMaxRanks * kMaxXchgCtas * 8;  // ready flag + done flags (~75 KB)
struct ExchangeArgs {
  int mrr;                               // 0: leader ring over pub (HAR / one rank), 1: MRR over gpub
  int t;                                 // GMIs per rank (MRR)
  const float* pub[kMaxRanks];           // each rank's published (K1-folded) gradient
  const float* gpub[kMaxRanks][kMaxLocalGmis];  // MRR: each rank's per-GMI gradients
  float* params[kMaxRanks];              // each rank's fp32 master parameters
  __nv_bfloat16* shadow[kMaxRanks];      // each rank's bf16 shadow
  unsigned long long* ready[kMaxRanks];  // each rank's "gradient of step s published" flag
  unsigned long long* done[kMaxRanks];   // each rank's done flags [source rank][CTA] ("step s written into me")
  int G, rank, ctas;
  long long P, lo, hi;  // flat length; this rank's shard [lo, hi)
  long long chunk0[kMaxRanks];  // ring chunk starts P c / G
  long long chunk0_t[kMaxLocalGmis];  // local ring chunk starts P c / t (fused K1 fold, one rank)
  float* m;             // Adam moments (only the shard is used)
  float* v;
  const float* bc;
  const Control* ctl;
  int step_in_iter;
  float lr, b1, b2, eps, inv_n;
};
void launch_exchange_adam(const ExchangeArgs& a, cudaStream_t s);
// Cross-GPU experience link (AsyncDecoupled, cfg.decoupled = 2; exchange.cu): wait until
// f1 (and f2 if given) >= ++*ctr + add; signal *flag = ++*ctr + add (system-scope release).
void launch_link_wait(const unsigned long long* f1, const unsigned long long* f2, unsigned long long* ctr,
                      unsigned long long add, cudaStream_t s);
void launch_link_signal(unsigned long long* flag, unsigned long long* ctr, unsigned long long add, cudaStream_t s);

struct AdamArgs {
  float* p;
  float* m;
  float* v;
  __nv_bfloat16* shadow;
  const float* g;
  const float* bc;  // [2*steps] bias-correction table: 1-b1^s, 1-b2^s for s = 1..
  const Control* ctl;
  int step_in_iter;  // 0-based minibatch update index inside the iteration
  long long n;
  float lr, b1, b2, eps, inv_n;
};

void launch_env_init(const EnvParams& ep, float* x, int* ep_step, int* ep_len, int* ep_count,
                     __nv_bfloat16* X0, cudaStream_t s);
void launch_act_env(const ActEnvArgs& a, cudaStream_t s);
void launch_value_head(const float* vraw, const float* b, float* out, int rows, cudaStream_t s);
void launch_gae(const float* rew, const uint8_t* done, const float* V, float* adv, float* ret,
                double* partials, int N, int T, float gamma, float lam, cudaStream_t s);
int gae_blocks(int N);
void launch_adv_stats(const double* partials, int nparts, long long count, float* stats,
                      cudaStream_t s);
void launch_shuffle(const __nv_bfloat16* X_roll, const float* act, const float* logp,
                    const float* adv, const float* ret, const float* adv_stats, __nv_bfloat16* X_sh,
                    float* act_sh, float* oldlp_sh, float* adv_sh, float* ret_sh, int N, int T,
                    int S_p, int A, uint64_t seed, int gmi_gid, int epoch, const Control* ctl,
                    cudaStream_t s);
void launch_head_loss(const HeadLossArgs& a, cudaStream_t s);
int head_loss_blocks(int B);
void launch_colsum(const __nv_bfloat16* const* D, const int* widths, float* const* partial,
                   int nproblems, int rows, cudaStream_t s);
int colsum_blocks(int rows);
void launch_segments(const Segment* segs, int nsegs, cudaStream_t s, const SegAdam* adam = nullptr);
void launch_adam(const AdamArgs& a, cudaStream_t s);

}  // namespace gmi::ppo
