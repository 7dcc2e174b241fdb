// PPO iteration kernels for sm_100a (non-GEMM parts; the hidden-layer GEMMs are the
// tcgen05 kernels in gemm.cuh). All of these are HBM- or latency-bound elementwise /
// reduction kernels; the dominant traffic per kernel is noted beside it.
//
// Numerics follow oracle/ppo_oracle.c: every fp32 expression that the oracle evaluates
// with -ffp-contract=off is evaluated here with explicit _rn intrinsics (no FMA
// contraction) wherever bit-equality is attainable (env resets, Adam); transcendentals
// (tanhf/sinf/expf/logf) and reduction orders differ by ulps.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "../host/errors.hpp"
#include "launch.cuh"
#include "ppo.cuh"
#include "ppo_common.cuh"
#include "rng.cuh"

namespace gmi::ppo {

namespace {

constexpr float kDt = 0.05f, kDamp = 1.0f, kCouple = 0.1f, kCtrl = 0.1f, kStateC = 0.1f;
constexpr float kTwoPi = 6.28318530717958648f;
constexpr int kMaxObsPerLane = 8;  // S <= 256


// Reset state x[0..S) of env `gid` for episode `count`: U(-0.1, 0.1), bit-exact vs oracle.
__device__ __forceinline__ float reset_value(uint64_t seed, int gid, int count, int i) {
  uint32_t r[4];
  rng::draw(seed, uint32_t(gid), uint32_t(count), uint32_t(i / 4), rng::kReset, r);
  return __fsub_rn(__fmul_rn(rng::u01(r[i & 3]), 0.2f), 0.1f);
}

// ------------------------------------------------------------------ env init
__global__ void env_init_kernel(EnvParams ep, float* x, int* ep_step, int* ep_len, int* ep_count,
                                __nv_bfloat16* X0) {
  pdl_trigger();
  pdl_wait();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ep.N) return;
  const int gid = ep.env0 + e;
  uint32_t r[4];
  rng::draw(ep.seed, uint32_t(gid), 0u, 0u, rng::kEpisode, r);
  const int len = 16 + int(r[0] % 48u);
  ep_len[e] = len;
  ep_step[e] = int(r[1] % uint32_t(len));
  ep_count[e] = 0;
  for (int i = 0; i < ep.S; ++i) {
    const float v = reset_value(ep.seed, gid, 0, i);
    x[(long long)e * ep.S + i] = v;
    X0[(long long)e * ep.S_p + i] = __float2bfloat16_rn(v);
  }
}

// ------------------------------------------------------------------ K3+K4 head: act + env step
// One warp per env: policy head (mu = H_L W_mu^T + b), Gaussian sample, log-prob, clipped
// actions, synthetic Ant-like dynamics, reward, integer episode clock / reset, and the
// next GEMM-ready observation row. Traffic/env: H_L row (2*hp B) + 2*S*4 (state) + 2*S_p
// (obs) + (A+3)*4 B.
__global__ void __launch_bounds__(256, 8) act_env_kernel(const ActEnvArgs a) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const EnvParams& ep = a.ep;
  const int A = ep.A, S = ep.S;
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (e >= ep.N) return;
  const int gid = ep.env0 + e;

  // mu: policy-head GEMM output (tensor cores) + bias
  const float mu_mine = lane < A ? a.mu[(long long)e * kHeadG + lane] + a.b_mu[lane] : 0.f;

  // N(0,1) noise: lane q draws Philox block q -> 4 normals for actions 4q..4q+3
  const uint32_t step = uint32_t(a.ctl->iteration * ep.T + a.t);
  float nrm[4] = {0.f, 0.f, 0.f, 0.f};
  if (lane * 4 < A) {
    uint32_t r[4];
    rng::draw(ep.seed, uint32_t(gid), step, uint32_t(lane), rng::kNoise, r);
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const float rad = sqrtf(-2.0f * logf(rng::u01_open0(r[2 * p])));
      const float th = kTwoPi * rng::u01(r[2 * p + 1]);
      float sn, cs;
      sincosf(th, &sn, &cs);  // same values as cosf / sinf, one range reduction (as rollout.cu)
      nrm[2 * p] = rad * cs;
      nrm[2 * p + 1] = rad * sn;
    }
  }
  float got[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) got[j] = __shfl_sync(0xffffffffu, nrm[j], (lane >> 2) & 31);
  const float eps = (lane & 3) == 0 ? got[0] : (lane & 3) == 1 ? got[1] : (lane & 3) == 2 ? got[2] : got[3];

  float act = 0.f, lp_term = 0.f, u = 0.f;
  if (lane < A) {
    const float ls = a.log_std[lane];
    const float sig = expf(ls);
    act = mu_mine + sig * eps;
    const float z = (act - mu_mine) / sig;
    lp_term = -0.5f * z * z - ls - kLog2PiHalf;
    u = fminf(fmaxf(act, -1.f), 1.f);
    a.act[(long long)e * A + lane] = act;
  }
  const float logp = warp_sum(lp_term);
  const float usq = warp_sum(u * u);
  const float tu = tanhf(u);  // drive of action lane: tanh(clip(a)), once per action

  // dynamics: lane owns dims i = lane + 32 j, driven by action i mod A (kept incrementally:
  // (i + 32) mod A = i mod A + 32 mod A, minus A on wrap)
  float* xe = a.x + (long long)e * S;
  float xn[kMaxObsPerLane];
  float xsq_part = 0.f;
  const int step32 = 32 % A;
  int src = lane % A;
#pragma unroll
  for (int j = 0; j < kMaxObsPerLane; ++j) {
    const int i = lane + 32 * j;
    const float drive = __shfl_sync(0xffffffffu, tu, i < S ? src : 0);
    src += step32;
    src -= src >= A ? A : 0;
    if (i < S) {
      const float xi = xe[i];
      const float nb = xe[i + 1 < S ? i + 1 : 0];
      const float inner = __fadd_rn(__fsub_rn(drive, __fmul_rn(kDamp, xi)), __fmul_rn(kCouple, env_sin(nb)));
      xn[j] = __fadd_rn(xi, __fmul_rn(kDt, inner));
      xsq_part = __fadd_rn(xsq_part, __fmul_rn(xn[j], xn[j]));
    } else {
      xn[j] = 0.f;
    }
  }
  const float xsq = warp_sum(xsq_part);
  const float xn0 = __shfl_sync(0xffffffffu, xn[0], 0);
  const int st = a.ep_step[e];
  const bool done = st + 1 >= a.ep_len[e];
  const int count = a.ep_count[e] + (done ? 1 : 0);
  __syncwarp();
  __nv_bfloat16* xo = a.X_next + (long long)e * ep.S_p;
#pragma unroll
  for (int j = 0; j < kMaxObsPerLane; ++j) {
    const int i = lane + 32 * j;
    if (i < S) {
      const float v = done ? reset_value(ep.seed, gid, count, i) : xn[j];
      xe[i] = v;
      xo[i] = __float2bfloat16_rn(v);
    }
  }
  if (lane == 0) {
    const float r0 = __fsub_rn(__fadd_rn(1.0f, xn0), __fdiv_rn(__fmul_rn(kCtrl, usq), float(A)));
    a.rew[e] = __fsub_rn(r0, __fdiv_rn(__fmul_rn(kStateC, xsq), float(S)));
    a.logp[e] = logp;
    a.done[e] = done ? 1 : 0;
    a.ep_step[e] = done ? 0 : st + 1;
    a.ep_count[e] = count;
  }
}

// ------------------------------------------------------------------ value head
// V[r] = value-head GEMM output (column 0) + bias.
__global__ void __launch_bounds__(256) value_head_kernel(const float* vraw, const float* b, float* out, int rows) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) out[r] = vraw[(long long)r * kHeadG] + b[0];
}

// ------------------------------------------------------------------ K5 GAE
// Block = 32 envs x 32 steps. Tiles are staged through shared memory so HBM access is
// coalesced along envs; each warp then owns one env with lane = time step and runs the
// reverse affine recurrence A_t = d_t + c_t A_{t+1} as a 5-step shuffle scan.
__global__ void __launch_bounds__(1024) gae_kernel(const float* rew, const uint8_t* done, const float* V,
                                                   float* adv, float* ret, double* partials, int N, int T,
                                                   float gamma, float gl) {
  __shared__ float r_s[32][33], v_s[33][33], a_s[32][33], q_s[32][33];
  __shared__ unsigned char d_s[32][33];
  __shared__ double red[3][32];
  pdl_trigger();
  pdl_wait();
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int e0 = blockIdx.x * 32;
  const int e = e0 + tx;
  const bool ok = e < N;
  if (ty < T) {
    r_s[ty][tx] = ok ? rew[(long long)ty * N + e] : 0.f;
    d_s[ty][tx] = ok ? done[(long long)ty * N + e] : 1;
  }
  if (ty <= T) v_s[ty][tx] = ok ? V[(long long)ty * N + e] : 0.f;
  if (ty == 0 && T == 32) v_s[32][tx] = ok ? V[(long long)32 * N + e] : 0.f;
  __syncthreads();

  // warp ty -> env column ty, lane tx -> time step
  const int t = tx;
  float delta = 0.f, c = 0.f;
  if (t < T) {
    const float nonterm = d_s[t][ty] ? 0.f : 1.f;
    delta = __fsub_rn(__fadd_rn(r_s[t][ty], __fmul_rn(__fmul_rn(gamma, v_s[t + 1][ty]), nonterm)), v_s[t][ty]);
    c = __fmul_rn(gl, nonterm);
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float d2 = __shfl_down_sync(0xffffffffu, delta, o);
    const float c2 = __shfl_down_sync(0xffffffffu, c, o);
    if (t + o < 32) {
      delta = __fadd_rn(delta, __fmul_rn(c, d2));
      c = __fmul_rn(c, c2);
    }
  }
  if (t < T) {
    a_s[t][ty] = delta;
    q_s[t][ty] = __fadd_rn(delta, v_s[t][ty]);
  }
  __syncthreads();
  double s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (ty < T && ok) {
    const float av = a_s[ty][tx];
    adv[(long long)ty * N + e] = av;
    ret[(long long)ty * N + e] = q_s[ty][tx];
    s1 = av;
    s2 = double(av) * double(av);
    s3 = r_s[ty][tx];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    s3 += __shfl_xor_sync(0xffffffffu, s3, o);
  }
  if (tx == 0) {
    red[0][ty] = s1;
    red[1][ty] = s2;
    red[2][ty] = s3;
  }
  __syncthreads();
  if (ty == 0) {
    double a1 = red[0][tx], a2 = red[1][tx], a3 = red[2][tx];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
      a3 += __shfl_xor_sync(0xffffffffu, a3, o);
    }
    if (tx == 0) {
      partials[3 * blockIdx.x] = a1;
      partials[3 * blockIdx.x + 1] = a2;
      partials[3 * blockIdx.x + 2] = a3;
    }
  }
}

__global__ void adv_stats_kernel(const double* partials, int nparts, long long count, float* stats) {
  __shared__ double sh[3][256];
  pdl_trigger();
  pdl_wait();
  double s1 = 0.0, s2 = 0.0, s3 = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
    s1 += partials[3 * i];
    s2 += partials[3 * i + 1];
    s3 += partials[3 * i + 2];
  }
  sh[0][threadIdx.x] = s1;
  sh[1][threadIdx.x] = s2;
  sh[2][threadIdx.x] = s3;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o)
      for (int q = 0; q < 3; ++q) sh[q][threadIdx.x] += sh[q][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double mean = sh[0][0] / double(count);
    double var = count > 1 ? (sh[1][0] - sh[0][0] * mean) / double(count - 1) : 0.0;
    if (var < 0) var = 0;
    stats[0] = float(mean);
    stats[1] = float(sqrt(var) + 1e-8);
    stats[2] = float(sh[2][0] / double(count));
  }
}

// ------------------------------------------------------------------ epoch shuffle
// Row j of the epoch copy is sample perm(j); 16-byte chunks of the bf16 obs row per thread.
__global__ void __launch_bounds__(256) shuffle_kernel(const __nv_bfloat16* X_roll, const float* act,
                                                      const float* logp, const float* adv, const float* ret,
                                                      const float* stats, __nv_bfloat16* X_sh, float* act_sh,
                                                      float* oldlp_sh, float* adv_sh, float* ret_sh, int N, int T,
                                                      int S_p, int A, uint64_t seed, int gmi_gid, int epoch,
                                                      const Control* ctl) {
  pdl_trigger();
  pdl_wait();
  // Block = 256 rows of the epoch copy: the Feistel permutation index is computed once per row
  // (shared memory), then the block's threads copy the rows' 16-byte observation chunks (S_p / 8
  // consecutive threads per row) and the per-row scalars, so no lane does serial work.
  __shared__ long long src_s[256];
  const int cpr = S_p / 8;  // 16-byte chunks per row
  const long long B = (long long)T * N;
  const long long r0 = (long long)blockIdx.x * 256;
  const int rows = int(B - r0 < 256 ? B - r0 : 256);
  if (threadIdx.x < rows) {
    uint32_t keys[4];
    rng::draw(seed, uint32_t(gmi_gid), uint32_t(ctl->iteration), uint32_t(epoch), rng::kPerm, keys);
    src_s[threadIdx.x] = rng::perm_index(uint32_t(r0 + threadIdx.x), uint32_t(B), keys);
  }
  __syncthreads();
  // 8 gathered loads in flight per thread before their stores (the stores could alias the loads
  // as far as the compiler knows, so a load -> store loop would run one round trip per chunk)
  for (int k0 = threadIdx.x; k0 < rows * cpr; k0 += 8 * 256) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = k0 + u * 256;
      if (k < rows * cpr) {
        const int r = k / cpr, c = k - r * cpr;
        v[u] = reinterpret_cast<const uint4*>(X_roll + src_s[r] * S_p)[c];
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = k0 + u * 256;
      if (k < rows * cpr) {
        const int r = k / cpr, c = k - r * cpr;
        reinterpret_cast<uint4*>(X_sh + (r0 + r) * S_p)[c] = v[u];
      }
    }
  }
  for (int k0 = threadIdx.x; k0 < rows * A; k0 += 8 * 256) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = k0 + u * 256;
      if (k < rows * A) {
        const int r = k / A, i = k - r * A;
        v[u] = act[src_s[r] * A + i];
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = k0 + u * 256;
      if (k < rows * A) {
        const int r = k / A, i = k - r * A;
        act_sh[(r0 + r) * A + i] = v[u];
      }
    }
  }
  if (threadIdx.x < rows) {
    const long long j = r0 + threadIdx.x, src = src_s[threadIdx.x];
    oldlp_sh[j] = logp[src];
    adv_sh[j] = __fdiv_rn(__fsub_rn(adv[src], stats[0]), stats[1]);
    ret_sh[j] = ret[src];
  }
}

// ------------------------------------------------------------------ K8 Adam (fp32 master + bf16 shadow)
// 28 B/param of algorithmic traffic: read p, m, v, g; write p, m, v, shadow(2 B).
__global__ void __launch_bounds__(256) adam_kernel(const AdamArgs a) {
  pdl_trigger();
  pdl_wait();
  const long long s = a.ctl->adam_step0 + a.step_in_iter;  // completed steps before this one
  const float bc1 = a.bc[2 * s], bc2 = a.bc[2 * s + 1];
  const float ob1 = __fsub_rn(1.0f, a.b1), ob2 = __fsub_rn(1.0f, a.b2);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
    const float g = __fmul_rn(a.g[i], a.inv_n);
    const float m = __fadd_rn(__fmul_rn(a.b1, a.m[i]), __fmul_rn(ob1, g));
    const float v = __fadd_rn(__fmul_rn(a.b2, a.v[i]), __fmul_rn(__fmul_rn(ob2, g), g));
    a.m[i] = m;
    a.v[i] = v;
    const float mh = __fdiv_rn(m, bc1), vh = __fdiv_rn(v, bc2);
    const float p = __fsub_rn(a.p[i], __fmul_rn(a.lr, __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), a.eps))));
    a.p[i] = p;
    a.shadow[i] = __float2bfloat16_rn(p);
  }
}

}  // namespace

void launch_env_init(const EnvParams& ep, float* x, int* ep_step, int* ep_len, int* ep_count, __nv_bfloat16* X0,
                     cudaStream_t s) {
  launch_pdl(env_init_kernel, dim3((ep.N + 127) / 128), dim3(128), 0, s, ep, x, ep_step, ep_len, ep_count, X0);
}

void launch_act_env(const ActEnvArgs& a, cudaStream_t s) {
  if (a.ep.A > kMaxAct) invalid("act_dim > 31 unsupported by the act/env kernel");
  if (a.ep.S > 32 * kMaxObsPerLane) invalid("obs_dim > 256 unsupported by the act/env kernel");
  const int blocks = (a.ep.N * 32 + 255) / 256;
  launch_pdl(act_env_kernel, dim3(blocks), dim3(256), 0, s, a);
}

void launch_value_head(const float* vraw, const float* b, float* out, int rows, cudaStream_t s) {
  launch_pdl(value_head_kernel, dim3((rows + 255) / 256), dim3(256), 0, s, vraw, b, out, rows);
}

int gae_blocks(int N) { return (N + 31) / 32; }

void launch_gae(const float* rew, const uint8_t* done, const float* V, float* adv, float* ret, double* partials,
                int N, int T, float gamma, float lam, cudaStream_t s) {
  if (T > 32) invalid("horizon > 32 unsupported by the GAE scan");
  launch_pdl(gae_kernel, dim3(gae_blocks(N)), dim3(1024), 0, s, rew, done, V, adv, ret, partials, N, T, gamma,
             gamma * lam);
}

void launch_adv_stats(const double* partials, int nparts, long long count, float* stats, cudaStream_t s) {
  launch_pdl(adv_stats_kernel, dim3(1), dim3(256), 0, s, partials, nparts, count, stats);
}

void launch_shuffle(const __nv_bfloat16* X_roll, const float* act, const float* logp, const float* adv,
                    const float* ret, const float* adv_stats, __nv_bfloat16* X_sh, float* act_sh, float* oldlp_sh,
                    float* adv_sh, float* ret_sh, int N, int T, int S_p, int A, uint64_t seed, int gmi_gid, int epoch,
                    const Control* ctl, cudaStream_t s) {
  const long long rows = (long long)T * N;
  launch_pdl(shuffle_kernel, dim3(unsigned((rows + 255) / 256)), dim3(256), 0, s, X_roll, act, logp, adv, ret,
             adv_stats, X_sh, act_sh, oldlp_sh, adv_sh, ret_sh, N, T, S_p, A, seed, gmi_gid, epoch, ctl);
}

namespace {
__global__ void control_advance_kernel(Control* c, int dsteps) {
  pdl_trigger();
  pdl_wait();
  c->iteration += 1;
  c->adam_step0 += dsteps;
}
}  // namespace

// Device-side end-of-iteration bookkeeping, so a captured iteration graph can be replayed.
void launch_control_advance(Control* c, int dsteps, cudaStream_t s) {
  launch_pdl(control_advance_kernel, dim3(1), dim3(1), 0, s, c, dsteps);
}

void launch_adam(const AdamArgs& a, cudaStream_t s) {
  launch_pdl(adam_kernel, dim3(grid_for(a.n, 256, 148 * 8)), dim3(256), 0, s, a);
}

}  // namespace gmi::ppo
