// Host/device interface of the fused PPO head kernel (head_fused.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "ppo.cuh"

namespace gmi::ppo {

struct HeadNet {
  CUtensorMap map_h;   // H_L [Bm][hp] bf16, box {64, 128}, SW128
  CUtensorMap map_wk;  // head weights [n_out][hp] K-major, box {64, nh}, SW128 (rows >= n_out zero)
  CUtensorMap map_wm;  // same weights viewed [K = n_out rows][N = hp], box {64, 32}, SW128
  CUtensorMap map_d;   // dPre_{L-1} out [Bm][hp] bf16, box {32, 32}, SW64
  const float* bias;   // head bias [n_out]
  float* dw_slab;      // [ctas per net][n_out][hp]  head weight gradient
  int n_out;           // A (policy) or 1 (value)
  int nh;              // MMA N of the head: 16 or 32
};

struct alignas(64) HeadFusedArgs {
  HeadNet net[2];      // [0] policy, [1] value
  const float* log_std;
  const float* act;    // epoch copy rows (row0 + r)
  const float* oldlp;
  const float* adv;
  const float* ret;
  float* part;         // [grid][head_partial_stride(A)]: db_mu, db_v, dlog_std, 4 loss statistics
  long long row0;      // first epoch-copy row of this minibatch
  int Bm, A, hp;
  int npol;            // CTAs [0, npol) serve the policy net, [npol, grid) the value net
  float clip, vf_coef, ent_coef;
};

bool head_fusable(int hp, int A);
int head_fused_grid(int Bm, int sms);
// Policy CTAs of a head grid, in proportion to the per-tile loss cost (GMI_HEAD_NPOL overrides).
int head_fused_npol(int grid, int A);
void launch_head_fused(const HeadFusedArgs& a, int grid, cudaStream_t s);
void head_fused_set_trace(unsigned long long* buf);  // development trace (TRACE=1 builds)

}  // namespace gmi::ppo
