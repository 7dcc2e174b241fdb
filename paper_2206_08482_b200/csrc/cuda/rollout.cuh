// Host/device interface of the fused rollout kernel (rollout.cu).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ppo.cuh"

namespace gmi::ppo {

constexpr int kRollMaxL = 4;  // hidden layers supported by the fused rollout

struct RolloutArgs {
  CUtensorMap map_obs;                 // X_roll slot 0: bf16 {S_p, N}, box {64, 128}, SW128
  CUtensorMap map_w[kRollMaxL + 1];    // bf16 shadow weights {in_p, rows}, box {64, out_n}; [L] = policy head
  const float* bias[kRollMaxL + 1];    // [L] = policy-head bias (b_mu)
  const float* log_std;
  int in_p[kRollMaxL + 1];             // K per layer (obs width, hidden widths; padded to 32)
  int out_n[kRollMaxL + 1];            // MMA N per layer (hidden out_p; head 16 or 32)
  int L, A, S, S_p, N, T, env0;
  uint64_t seed;
  float* x;
  int* ep_step;
  const int* ep_len;
  int* ep_count;
  __nv_bfloat16* X_roll;  // [(T+1)][N][S_p]
  float* act;             // [T][N][A]
  float* logp;            // [T][N]
  float* rew;
  uint8_t* done;
  const Control* ctl;
  unsigned long long* trace;  // optional [T][16] globaltimer stamps of CTA 0 (development aid)
};

// Fused value pass (value_mlp.cu): V[r] = value_net(X_roll row r) for rows [0, rows).
struct ValueArgs {
  CUtensorMap map_obs;               // X_roll {S_p, rows}, box {64, 128}
  CUtensorMap map_w[kRollMaxL + 1];  // value-net weights, box {64, out_n}; [L] = value head (16 rows)
  const float* bias[kRollMaxL + 1];
  int in_p[kRollMaxL + 1];
  int out_n[kRollMaxL + 1];  // hidden out_p; head 16
  int L;
  long long rows;
  float* V;
};
void launch_value_mlp(const ValueArgs& a, int max_ctas, cudaStream_t s);

// Whether the fused rollout supports this MLP (hidden widths <= 256, <= 4 layers, S_p <= 256, A <= 31).
bool rollout_fusable(int L, const int* widths_p, int S_p, int A);
void launch_rollout(const RolloutArgs& a, cudaStream_t s);
// Cluster variant (rollout_cluster.cu): returns the CTAs per 128-env tile (0 = not applicable).
// map_w[l] must then be built with 64-row boxes (hidden slices) and map_w[L] with 16-row boxes.
int rollout_cluster_size(int L, const int* widths_p, int S_p, int A, int N);
void launch_rollout_cluster(const RolloutArgs& a, int C, cudaStream_t s);

}  // namespace gmi::ppo
