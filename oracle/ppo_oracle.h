/* TEST INFRASTRUCTURE ONLY — CPU restatement of the B200 PPO iteration.
 *
 * PARITY STATUS: the reference (arXiv 2206.08482 gmux) contains no PPO arithmetic
 * ("actual PPO/A3C learning math ... out of scope"; only the abstract
 * T_s/T_a/T_t of workload.hpp:26-45 and the MLP shapes of workload.hpp:104-134).
 * This restatement is therefore pinned by (1) the reference's shape contracts (param
 * counts, workload.hpp:95-100), (2) the reference's partition rule for env -> GMI
 * ([N*c/n, N*(c+1)/n), reduction.hpp:164-166) and fold order for the gradient sum
 * (reduction.hpp:170-212), and (3) torch-CPU autograd / torch.optim.Adam / bf16 rounding
 * checks of the MLP / loss / Adam pieces, run live in tests/test_ppo_oracle.py. Env
 * dynamics, seeds and PPO hyper-parameters are builder-pinned.
 */
#ifndef PPO_ORACLE_H_
#define PPO_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PPO_MAX_HIDDEN 8

typedef struct {
  int obs_dim, act_dim;
  int num_hidden;
  int hidden[PPO_MAX_HIDDEN];
  int num_envs; /* whole job */
  int horizon, epochs, minibatches;
  float gamma, lam, clip, lr, beta1, beta2, adam_eps, vf_coef, ent_coef;
  unsigned long long seed;
  int num_gpus, gmis_per_gpu; /* data-parallel layout of the job (GPU-major GMIs) */
  int threads;                /* OpenMP threads, <= 0: all */
  int exact_fp32;             /* 1: skip the bf16 operand rounding (torch-fp32 pinning mode) */
} ppo_cfg_t;

typedef struct {
  double policy_loss, value_loss, entropy, approx_kl, clip_frac; /* last minibatch, GMI 0 */
  double mean_reward;                                            /* rollout mean, all envs */
  long long env_steps;
} ppo_stats_t;

void* ppo_oracle_create(const ppo_cfg_t* cfg);
void ppo_oracle_free(void* h);
int ppo_oracle_iteration(void* h, ppo_stats_t* out);
/* Decoupled (asynchronous serving/trainer) iteration, one-iteration policy lag; see
 * ppo_oracle.c. Do not mix with ppo_oracle_iteration on one handle. */
int ppo_oracle_iteration_decoupled(void* h, ppo_stats_t* out);
/* Runs only the rollout + GAE part of the next iteration (no update); the following
 * ppo_oracle_iteration trains on it instead of rolling out again. Returns -2 (and does
 * nothing) when such a rollout is already pending. */
int ppo_oracle_rollout(void* h);

/* One minibatch gradient of GMI `gmi` on caller rows with the current parameters:
 * X[B][obs_dim] (used as given), act[B][A], oldlp/adv/ret[B]; grad[P]; stats[4] =
 * policy loss, value loss, approx kl, clip fraction. */
int ppo_oracle_minibatch(void* h, int gmi, const float* X, const float* act, const float* oldlp,
                         const float* adv, const float* ret, int B, float* grad, double* stats);
/* One Adam step on the flat vectors with the given summed gradient (sum over n GMIs). */
int ppo_oracle_adam(void* h, const float* grad_sum);

/* Padded geometry and flat parameter vector (identical layout to the device trainer). */
long long ppo_oracle_param_count(void* h);  /* padded length of the flat vector */
int ppo_oracle_width(void* h, int layer);   /* padded width of layer (0 = obs) */
int ppo_oracle_get(void* h, const char* what, int gmi, void* dst, long long n);
int ppo_oracle_set(void* h, const char* what, int gmi, const void* src, long long n);

/* Deterministic primitives shared (by restatement) with the device code. */
void ppo_philox(uint32_t k0, uint32_t k1, const uint32_t ctr[4], uint32_t out[4]);
uint32_t ppo_perm_index(uint32_t j, uint32_t n, const uint32_t keys[4]);
int ppo_oracle_perm(unsigned long long seed, int gmi, int iteration, int epoch, uint32_t n, uint32_t* out);
float ppo_bf16_round(float x);

#ifdef __cplusplus
}
#endif

#endif
