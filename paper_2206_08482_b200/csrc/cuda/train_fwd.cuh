// Host/device interface of the fused training-forward kernel (train_fwd.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "ppo.cuh"
#include "rollout.cuh"  // kRollMaxL

namespace gmi::ppo {

struct TrainFwdNet {
  CUtensorMap map_w[kRollMaxL + 1];  // hidden layers: K-major {in_p, out_p} box {64, out_p}; [L] head box {64, nh}
  CUtensorMap map_wm;                // head weights viewed [K = n_out rows][N = hp], box {64, 32}
  CUtensorMap map_h[kRollMaxL];      // H_l (l < L-1) out [Bm][w_p] bf16, box {64, 32}, SW128
  CUtensorMap map_d;                 // dPre of the last hidden layer, [Bm][hp] bf16, box {64, 32}, SW128
  const float* bias[kRollMaxL + 1];  // [L] = head bias
  float* dw_slab;                    // [ctas per net][n_out][hp] head weight gradient
  int in_p[kRollMaxL + 1];
  int out_n[kRollMaxL + 1];          // hidden out_p; [L] = nh
  int n_out;                         // A (policy) or 1 (value)
  int nh;                            // head MMA N: 16 or 32
};

struct alignas(64) TrainFwdArgs {
  CUtensorMap map_x;  // epoch copy X_sh [B][S_p] bf16, box {64, 128}
  TrainFwdNet net[2]; // [0] policy, [1] value
  const float* log_std;
  const float* act;   // epoch copy rows (row0 + r)
  const float* oldlp;
  const float* adv;
  const float* ret;
  float* part;        // [grid][head_partial_stride(A)], same records as the fused head kernel
  long long row0;     // first epoch-copy row of this minibatch
  int Bm, A, L, hp, S_p;
  float clip, vf_coef, ent_coef;
  unsigned long long* trace;  // optional [4 tiles][16] globaltimer stamps of CTA 0 (development aid)
};

// Whole forward of one minibatch (hidden layers on chip, H_1..H_{L-1} stored for the backward)
// plus the PPO head step of head_fused.cu. L must be 1 or 3, widths <= 256, S_p <= 192.
bool train_fwd_fusable(int L, const int* widths_p, int S_p, int A);
// Grid and per-CTA outputs follow head_fused_grid / the fused head's records.
void launch_train_fwd(const TrainFwdArgs& a, int grid, cudaStream_t s);

}  // namespace gmi::ppo
