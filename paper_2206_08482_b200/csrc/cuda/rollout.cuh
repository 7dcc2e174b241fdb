// Host/device interface of the fused rollout kernel (rollout.cu).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ppo.cuh"

namespace gmi::ppo {

constexpr int kRollMaxL = 4;  // hidden layers supported by the fused rollout

// Shared-memory / TMEM plan of the wide on-chip MLP (hidden widths up to 512, e.g. HM
// 108:200:400:100). Activations live in ONE region, updated in place: layer l's epilogue runs
// only after all of layer l's MMAs completed, so its input tile is dead and the output (layer
// l+1's input, SW128 K-chunks of 64 columns) overwrites it; the next layer's MMAs start per
// K-chunk pair as the epilogue writes them. Freed space goes to a deeper weight ring (up to 8
// stages of [<=128 rows x 64 K], one per (K-chunk, 128-column N part)), which is what the
// per-step weight stream from L2 is bound by. Layer l accumulates at TMEM columns
// [tmem[l], tmem[l] + out); where that overlaps layer l-1's accumulator (out_{l-1} + out_l >
// 512) it waits for the previous layer's epilogue to drain completely (drain[l]).
struct WidePlan {
  uint32_t in_off[kRollMaxL + 1];  // smem byte offset of layer l's input tile
  uint32_t ring_off, bar_off, smem;
  int nstages;               // weight ring depth
  int obs_sep;               // value pass: observation tile in its own buffer (in_off[0])
  int wrows[kRollMaxL + 1];  // weight rows per ring stage (box rows of map_w[l]): min(128, out)
  int tmem[kRollMaxL + 1];
  int drain[kRollMaxL + 1];
  int wrap;  // value pass: the next tile's layer 0 overlaps this tile's head accumulator
};
constexpr uint32_t kWideStage = 128 * 128;  // 128 weight rows x 64 K bf16

// Builds the plan for widths_p[0] = S_p, widths_p[1..L] = hidden widths (padded to 32) and a
// head of head_n columns; rollout = true reserves the fp32 mu / tanh(u) staging in the region
// and keeps the observation tile in it. false when the tiles do not fit in shared memory.
bool plan_wide(int L, const int* widths_p, int head_n, bool rollout, WidePlan* out);

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
  int wide;                   // 1: wide kernel with `plan` (map_w boxes of plan.wrows rows)
  WidePlan plan;
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
  int wide;  // 1: wide kernel with `plan`
  WidePlan plan;
};
void launch_value_mlp(const ValueArgs& a, int max_ctas, cudaStream_t s);

// Whether the fused rollout supports this MLP (hidden widths <= 256, <= 4 layers, S_p <= 128, A <= 31).
bool rollout_fusable(int L, const int* widths_p, int S_p, int A);
// Whether the wide variant (rollout_kernel<.., WIDE>, hidden widths <= 512) holds it; fills *plan.
bool rollout_wide_fusable(int L, const int* widths_p, int S_p, int A, WidePlan* plan);
// Whether the wide value pass holds the value MLP (head of 16 columns); fills *plan.
bool value_wide_fusable(int L, const int* widths_p, WidePlan* plan);
void launch_rollout(const RolloutArgs& a, cudaStream_t s);
// Cluster variant (rollout_cluster.cu): returns the CTAs per 128-env tile (0 = not applicable).
// map_w[l] must then be built with 64-row boxes (hidden slices) and map_w[L] with 16-row boxes.
int rollout_cluster_size(int L, const int* widths_p, int S_p, int A, int N);
void launch_rollout_cluster(const RolloutArgs& a, int C, cudaStream_t s);

}  // namespace gmi::ppo
