/* TEST INFRASTRUCTURE ONLY — CPU restatement of the B200 data-parallel PPO iteration.
 * Never linked into libgmi.so. Used by tests/ (parity checker) and bench.py's
 * cpu_baseline / --impl reference leg. See ppo_oracle.h for the parity status.
 *
 * The numeric policy mirrors the device path: fp32 state and master weights; the
 * hidden-layer GEMM operands (observations, hidden weights, hidden activations and their
 * pre-activation gradients) are rounded to bf16 at exactly the points where the device
 * stores bf16; dot products accumulate in double here (fp32 in TMEM on the device), so
 * device-vs-oracle differences are accumulation-order-sized. Compiled with
 * -ffp-contract=off.
 *
 * Reference anchors: env -> GMI partition [N*c/n, N*(c+1)/n) (reduction.hpp:164-166);
 * cross-GMI gradient sum in the ring fold order of the strategy Alg. 1 picks
 * (reduction.hpp:98-212); MLP shapes / parameter counts (workload.hpp:86-134);
 * horizon m = steps_per_train = 32 (workload.hpp:113).
 */
#include "ppo_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TAG_NOISE 1u
#define TAG_RESET 2u
#define TAG_EPLEN 3u
#define TAG_INIT 4u
#define TAG_PERM 5u

#define ENV_DT 0.05f
#define ENV_DAMP 1.0f
#define ENV_COUPLE 0.1f
#define ENV_CTRL 0.1f
#define ENV_STATEC 0.1f
#define LOG_2PI_HALF 0.91893853320467274f /* 0.5 * log(2*pi) */
#define TWO_PI 6.28318530717958648f

/* ---------------------------------------------------------------- primitives */
void ppo_philox(uint32_t k0, uint32_t k1, const uint32_t ctr[4], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

static void philox_tag(unsigned long long seed, uint32_t a, uint32_t b, uint32_t c, uint32_t tag,
                       uint32_t out[4]) {
  const uint32_t ctr[4] = {a, b, c, tag};
  ppo_philox((uint32_t)seed, (uint32_t)(seed >> 32), ctr, out);
}

static float u01(uint32_t x) { return (float)(x >> 8) * 5.9604644775390625e-8f; }
static float u01_open0(uint32_t x) { return (float)((x >> 8) + 1u) * 5.9604644775390625e-8f; }

float ppo_bf16_round(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) { /* inf / nan: truncate, keep nan quiet */
    if (u & 0x007fffffu) u |= 0x00400000u;
    u &= 0xffff0000u;
  } else {
    u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
  }
  memcpy(&x, &u, 4);
  return x;
}

/* Epoch permutation of GMI `gmi` (global id) at (iteration, epoch): out[j] = sample of row j. */
int ppo_oracle_perm(unsigned long long seed, int gmi, int iteration, int epoch, uint32_t n, uint32_t* out) {
  uint32_t keys[4];
  philox_tag(seed, (uint32_t)gmi, (uint32_t)iteration, (uint32_t)epoch, TAG_PERM, keys);
  for (uint32_t j = 0; j < n; ++j) out[j] = ppo_perm_index(j, n, keys);
  return 0;
}

uint32_t ppo_perm_index(uint32_t j, uint32_t n, const uint32_t keys[4]) {
  if (n <= 1) return 0;
  uint32_t bits = 0;
  while ((1ull << bits) < n) ++bits;
  const uint32_t mask = bits >= 32 ? 0xffffffffu : ((1u << bits) - 1u);
  const uint32_t half = (bits + 1) / 2;
  uint32_t x = j;
  do {
    for (int r = 0; r < 4; ++r) {
      x ^= x >> half;
      x = (x * 0x9E3779B1u + keys[r]) & mask;
    }
  } while (x >= n);
  return x;
}

static int g_exact = 0; /* set per call from the config */
static float R(float x) { return g_exact ? x : ppo_bf16_round(x); }

static float elu(float x) { return x > 0.f ? x : expm1f(x); }
static float elu_grad_from_out(float h) { return h > 0.f ? 1.f : h + 1.f; }

/* ---------------------------------------------------------------- geometry */
typedef struct {
  long long w, b; /* offsets into the flat parameter vector */
  int out, in;    /* real (unpadded) shape */
  int out_p, in_p;
} tensor_t;

typedef struct {
  ppo_cfg_t c;
  int L;                     /* hidden layers */
  int width[PPO_MAX_HIDDEN + 2];   /* real widths: 0 = obs, 1..L hidden */
  int width_p[PPO_MAX_HIDDEN + 2]; /* padded to 32 */
  tensor_t net[2][PPO_MAX_HIDDEN + 1]; /* [pi|v][layer 0..L] (layer L = head) */
  long long log_std;
  long long P; /* padded flat length */
  int n_gmi;
  int iteration;
  int primed; /* decoupled mode: rollout 0 done */
  int pending; /* ppo_oracle_rollout ran the next iteration's rollout; the iteration trains on it */
  long long adam_step;
  float *params, *adam_m, *adam_v, *grad_sum;
  /* per GMI */
  struct gmi {
    int env0, nenv;
    float* x;               /* [nenv][S] env state */
    int *ep_step, *ep_len, *ep_count;
    float* obs;             /* [(T+1)][nenv][S] bf16-rounded observations */
    float *act, *logp, *rew, *val, *adv, *ret;
    unsigned char* done;
    float* grad;            /* [P] */
  } * g;
  ppo_stats_t last;
} oracle_t;

static int pad32(int x) { return (x + 31) / 32 * 32; }

static long long align64(long long x) { return (x + 63) / 64 * 64; }

static void build_geometry(oracle_t* o) {
  const ppo_cfg_t* c = &o->c;
  o->L = c->num_hidden;
  o->width[0] = c->obs_dim;
  for (int l = 0; l < o->L; ++l) o->width[l + 1] = c->hidden[l];
  for (int l = 0; l <= o->L; ++l) o->width_p[l] = pad32(o->width[l]);
  long long off = 0;
  for (int n = 0; n < 2; ++n) {
    for (int l = 0; l <= o->L; ++l) {
      tensor_t* t = &o->net[n][l];
      t->in = o->width[l];
      t->in_p = o->width_p[l];
      if (l < o->L) {
        t->out = o->width[l + 1];
        t->out_p = o->width_p[l + 1];
      } else {
        t->out = n == 0 ? c->act_dim : 1;
        t->out_p = t->out;
      }
      t->w = off;
      off = align64(off + (long long)t->out_p * t->in_p);
      t->b = off;
      off = align64(off + t->out_p);
    }
  }
  o->log_std = off;
  off = align64(off + c->act_dim);
  o->P = off;
}

static void init_params(oracle_t* o) {
  memset(o->params, 0, sizeof(float) * o->P);
  for (int n = 0; n < 2; ++n)
    for (int l = 0; l <= o->L; ++l) {
      const tensor_t* t = &o->net[n][l];
      const float bound = 1.0f / sqrtf((float)t->in);
      const uint32_t wid = (uint32_t)((n * 16 + l) * 2), bid = wid + 1;
      for (int r = 0; r < t->out; ++r) {
        for (int k = 0; k < t->in; ++k) {
          uint32_t out[4];
          philox_tag(o->c.seed, wid, (uint32_t)(r * t->in + k), 0, TAG_INIT, out);
          o->params[t->w + (long long)r * t->in_p + k] = (u01(out[0]) * 2.0f - 1.0f) * bound;
        }
        uint32_t out[4];
        philox_tag(o->c.seed, bid, (uint32_t)r, 0, TAG_INIT, out);
        o->params[t->b + r] = (u01(out[0]) * 2.0f - 1.0f) * bound;
      }
    }
}

static void env_reset_state(const oracle_t* o, int gid, int ep_count, float* x) {
  for (int i = 0; i < o->c.obs_dim; i += 4) {
    uint32_t out[4];
    philox_tag(o->c.seed, (uint32_t)gid, (uint32_t)ep_count, (uint32_t)(i / 4), TAG_RESET, out);
    for (int q = 0; q < 4 && i + q < o->c.obs_dim; ++q) x[i + q] = u01(out[q]) * 0.2f - 0.1f;
  }
}

/* ---------------------------------------------------------------- MLP */
/* bf16 hidden forward of one row for net n; h[l] receives layer-l outputs (bf16-rounded).
 * x: bf16-rounded input [S]. Returns pointer to last hidden. */
static void mlp_hidden(const oracle_t* o, const float* wbf, int n, const float* x, float** h) {
  /* wbf + P holds every hidden weight block transposed ([in_p][out_p], make_bf16_weights):
   * the k loop is outermost so the out-neuron accumulators vectorise; each accumulator still
   * sums its products in ascending k, so the result is the row-major dot product's. */
  const float* in = x;
  double acc[1024];
  for (int l = 0; l < o->L; ++l) {
    const tensor_t* t = &o->net[n][l];
    const int nout = t->out;
    for (int r = 0; r < nout; ++r) acc[r] = 0.0;
    for (int k = 0; k < t->in; ++k) {
      const double xk = (double)in[k];
      const float* wk = wbf + o->P + t->w + (long long)k * t->out_p;
      for (int r = 0; r < nout; ++r) acc[r] += xk * (double)wk[r];
    }
    for (int r = 0; r < nout; ++r) {
      const float pre = (float)acc[r] + o->params[t->b + r];
      h[l][r] = R(elu(pre));
    }
    in = h[l];
  }
}

static float head_out(const oracle_t* o, const float* wbf, int n, int a, const float* hl) {
  const tensor_t* t = &o->net[n][o->L];
  double acc = 0.0;
  /* heads run on the tensor cores: bf16 head weights, fp32 bias added after the GEMM */
  const float* wr = wbf + t->w + (long long)a * t->in_p;
  for (int k = 0; k < t->in; ++k) acc += (double)hl[k] * (double)wr[k];
  return (float)acc + o->params[t->b + a];
}

static float gauss_logp(const oracle_t* o, const float* act, const float* mu) {
  float lp = 0.f;
  for (int a = 0; a < o->c.act_dim; ++a) {
    const float ls = o->params[o->log_std + a];
    const float z = (act[a] - mu[a]) / expf(ls);
    lp += -0.5f * z * z - ls - LOG_2PI_HALF;
  }
  return lp;
}

/* ---------------------------------------------------------------- rollout + GAE */
/* wbf[0, P): bf16-rounded parameters; wbf[P, 2P): the hidden weight blocks again, transposed
 * to [in_p][out_p] at the same offsets (mlp_hidden's k-outer loop). */
static float* make_bf16_weights(const oracle_t* o) {
  float* wbf = (float*)calloc((size_t)(2 * o->P), sizeof(float));
  for (long long i = 0; i < o->P; ++i) wbf[i] = R(o->params[i]);
  for (int n = 0; n < 2; ++n)
    for (int l = 0; l < o->L; ++l) {
      const tensor_t* t = &o->net[n][l];
      for (int r = 0; r < t->out_p; ++r)
        for (int k = 0; k < t->in_p; ++k)
          wbf[o->P + t->w + (long long)k * t->out_p + r] = wbf[t->w + (long long)r * t->in_p + k];
    }
  return wbf;
}

static void alloc_rows(const oracle_t* o, float** h) {
  for (int l = 0; l < o->L; ++l) h[l] = (float*)calloc((size_t)o->width_p[l + 1], sizeof(float));
}

static void free_rows(const oracle_t* o, float** h) {
  for (int l = 0; l < o->L; ++l) free(h[l]);
}

static void rollout_gmi(oracle_t* o, int gi, const float* wbf) {
  struct gmi* g = &o->g[gi];
  const int S = o->c.obs_dim, A = o->c.act_dim, T = o->c.horizon, N = g->nenv;
#pragma omp parallel
  {
    float* h[PPO_MAX_HIDDEN];
    alloc_rows(o, h);
    float mu[64], act[64], u[64], xn[1024];
#pragma omp for schedule(static)
    for (int e = 0; e < N; ++e) {
      const int gid = g->env0 + e;
      float* x = g->x + (long long)e * S;
      for (int t = 0; t < T; ++t) {
        const float* ob = g->obs + ((long long)t * N + e) * S;
        mlp_hidden(o, wbf, 0, ob, h);
        for (int a = 0; a < A; ++a) mu[a] = head_out(o, wbf, 0, a, h[o->L - 1]);
        const uint32_t step = (uint32_t)(o->iteration * T + t);
        for (int q = 0; q < A; q += 4) {
          uint32_t r[4];
          philox_tag(o->c.seed, (uint32_t)gid, step, (uint32_t)(q / 4), TAG_NOISE, r);
          for (int p = 0; p < 2; ++p) {
            const float rad = sqrtf(-2.0f * logf(u01_open0(r[2 * p])));
            const float th = TWO_PI * u01(r[2 * p + 1]);
            const int a0 = q + 2 * p;
            if (a0 < A) act[a0] = mu[a0] + expf(o->params[o->log_std + a0]) * (rad * cosf(th));
            if (a0 + 1 < A) act[a0 + 1] = mu[a0 + 1] + expf(o->params[o->log_std + a0 + 1]) * (rad * sinf(th));
          }
        }
        const long long ti = (long long)t * N + e;
        memcpy(g->act + ti * A, act, sizeof(float) * A);
        g->logp[ti] = gauss_logp(o, act, mu);
        /* env dynamics */
        float usq = 0.f;
        for (int a = 0; a < A; ++a) {
          u[a] = fminf(fmaxf(act[a], -1.f), 1.f);
          usq += u[a] * u[a];
        }
        float xsq = 0.f;
        for (int i = 0; i < S; ++i) {
          const float drive = tanhf(u[i % A]);
          xn[i] = x[i] + ENV_DT * (drive - ENV_DAMP * x[i] + ENV_COUPLE * sinf(x[(i + 1) % S]));
        }
        for (int i = 0; i < S; ++i) xsq += xn[i] * xn[i];
        g->rew[ti] = 1.0f + xn[0] - ENV_CTRL * usq / (float)A - ENV_STATEC * xsq / (float)S;
        const int done = g->ep_step[e] + 1 >= g->ep_len[e];
        g->done[ti] = (unsigned char)done;
        if (done) {
          g->ep_count[e] += 1;
          g->ep_step[e] = 0;
          env_reset_state(o, gid, g->ep_count[e], x);
        } else {
          g->ep_step[e] += 1;
          memcpy(x, xn, sizeof(float) * S);
        }
        float* nob = g->obs + ((long long)(t + 1) * N + e) * S;
        for (int i = 0; i < S; ++i) nob[i] = R(x[i]);
      }
    }
    free_rows(o, h);
  }
}

static void values_gmi(oracle_t* o, int gi, const float* wbf) {
  struct gmi* g = &o->g[gi];
  const int S = o->c.obs_dim, T = o->c.horizon, N = g->nenv;
#pragma omp parallel
  {
    float* h[PPO_MAX_HIDDEN];
    alloc_rows(o, h);
#pragma omp for schedule(static)
    for (long long r = 0; r < (long long)(T + 1) * N; ++r) {
      mlp_hidden(o, wbf, 1, g->obs + r * S, h);
      g->val[r] = head_out(o, wbf, 1, 0, h[o->L - 1]);
    }
    free_rows(o, h);
  }
}

static void gae_gmi(oracle_t* o, int gi, float* mean_out, float* std_out) {
  struct gmi* g = &o->g[gi];
  const int T = o->c.horizon, N = g->nenv;
  const float gamma = o->c.gamma, gl = o->c.gamma * o->c.lam;
  for (int e = 0; e < N; ++e) {
    float next = 0.f;
    for (int t = T - 1; t >= 0; --t) {
      const long long i = (long long)t * N + e;
      const float nonterm = g->done[i] ? 0.f : 1.f;
      const float delta = g->rew[i] + gamma * g->val[i + N] * nonterm - g->val[i];
      next = delta + gl * nonterm * next;
      g->adv[i] = next;
      g->ret[i] = next + g->val[i];
    }
  }
  double s1 = 0.0, s2 = 0.0;
  const long long B = (long long)T * N;
  for (long long i = 0; i < B; ++i) {
    s1 += g->adv[i];
    s2 += (double)g->adv[i] * (double)g->adv[i];
  }
  const double mean = s1 / (double)B;
  const double var = B > 1 ? (s2 - s1 * mean) / (double)(B - 1) : 0.0;
  *mean_out = (float)mean;
  *std_out = (float)(sqrt(var > 0 ? var : 0) + 1e-8);
}

/* ---------------------------------------------------------------- update */
typedef struct {
  float* X;       /* [Bm][S] */
  float* act;     /* [Bm][A] */
  float *oldlp, *adv, *ret;
  float* H[2][PPO_MAX_HIDDEN]; /* [Bm][w_l] */
  float* D[2][PPO_MAX_HIDDEN]; /* pre-activation grads (bf16-rounded) */
  float* gmu;     /* [Bm][A] */
  float* gls;     /* [Bm][A] */
  float* gv;      /* [Bm] */
  double loss_pi, loss_v, kl, clipped;
} mb_t;

static void mb_alloc(const oracle_t* o, mb_t* m, int Bm);
static void mb_free(const oracle_t* o, mb_t* m);

static void minibatch_grad(oracle_t* o, int gi, mb_t* mb, int Bm, const float* wbf, float* grad) {
  const int A = o->c.act_dim, L = o->L;
  const float clip = o->c.clip;
  const float invB = 1.0f / (float)Bm;
  double lpi = 0, lv = 0, kl = 0, cl = 0;
#pragma omp parallel for schedule(static) reduction(+ : lpi, lv, kl, cl)
  for (int r = 0; r < Bm; ++r) {
    float* hp[PPO_MAX_HIDDEN];
    float* hv[PPO_MAX_HIDDEN];
    for (int l = 0; l < L; ++l) {
      hp[l] = mb->H[0][l] + (long long)r * o->width[l + 1];
      hv[l] = mb->H[1][l] + (long long)r * o->width[l + 1];
    }
    const float* x = mb->X + (long long)r * o->c.obs_dim;
    mlp_hidden(o, wbf, 0, x, hp);
    mlp_hidden(o, wbf, 1, x, hv);
    float mu[64];
    for (int a = 0; a < A; ++a) mu[a] = head_out(o, wbf, 0, a, hp[L - 1]);
    const float v = head_out(o, wbf, 1, 0, hv[L - 1]);
    const float* act = mb->act + (long long)r * A;
    const float lp = gauss_logp(o, act, mu);
    const float ratio = expf(lp - mb->oldlp[r]);
    const float adv = mb->adv[r];
    const float s1 = ratio * adv;
    const float rc = fminf(fmaxf(ratio, 1.f - clip), 1.f + clip);
    const float s2 = rc * adv;
    const int take1 = s1 <= s2;
    lpi += -(double)(take1 ? s1 : s2);
    const float verr = v - mb->ret[r];
    lv += 0.5 * (double)o->c.vf_coef * (double)verr * (double)verr;
    kl += (double)(mb->oldlp[r] - lp);
    cl += (ratio < 1.f - clip || ratio > 1.f + clip) ? 1.0 : 0.0;
    const float glp = take1 ? -s1 * invB : 0.f;
    for (int a = 0; a < A; ++a) {
      const float ls = o->params[o->log_std + a];
      const float sig = expf(ls);
      const float z = (act[a] - mu[a]) / sig;
      mb->gmu[(long long)r * A + a] = glp * z / sig;
      mb->gls[(long long)r * A + a] = glp * (z * z - 1.f) - o->c.ent_coef * invB;
    }
    mb->gv[r] = o->c.vf_coef * verr * invB;
    /* head backward -> dPre of the last hidden layer (bf16) */
    for (int n = 0; n < 2; ++n) {
      const tensor_t* th = &o->net[n][L];
      float* hl = n == 0 ? hp[L - 1] : hv[L - 1];
      float* d = mb->D[n][L - 1] + (long long)r * o->width[L];
      for (int k = 0; k < th->in; ++k) {
        double acc = 0.0;
        if (n == 0)
          for (int a = 0; a < A; ++a)
            acc += (double)R(mb->gmu[(long long)r * A + a]) * (double)wbf[th->w + (long long)a * th->in_p + k];
        else
          acc = (double)R(mb->gv[r]) * (double)wbf[th->w + k];
        d[k] = R((float)acc * elu_grad_from_out(hl[k]));
      }
      /* hidden backward: dPre_{l-1} = (dPre_l W_l) * elu'(H_{l-1}) */
      for (int l = L - 1; l >= 1; --l) {
        const tensor_t* t = &o->net[n][l];
        const float* dl = mb->D[n][l] + (long long)r * o->width[l + 1];
        const float* hprev = (n == 0 ? hp : hv)[l - 1];
        float* dp = mb->D[n][l - 1] + (long long)r * o->width[l];
        double acc[1024];
        for (int k = 0; k < t->in; ++k) acc[k] = 0.0;
        for (int j = 0; j < t->out; ++j) {  /* per k: ascending j, as the column dot product */
          const double dj = (double)dl[j];
          const float* wj = wbf + t->w + (long long)j * t->in_p;
          for (int k = 0; k < t->in; ++k) acc[k] += dj * (double)wj[k];
        }
        for (int k = 0; k < t->in; ++k) dp[k] = R((float)acc[k] * elu_grad_from_out(hprev[k]));
      }
    }
  }
  mb->loss_pi = lpi / Bm;
  mb->loss_v = lv / Bm;
  mb->kl = kl / Bm;
  mb->clipped = cl / Bm;

  /* weight gradients: reductions over the minibatch rows */
  memset(grad, 0, sizeof(float) * o->P);
  for (int n = 0; n < 2; ++n) {
    for (int l = 0; l < L; ++l) {
      const tensor_t* t = &o->net[n][l];
      const float* in = l == 0 ? mb->X : mb->H[n][l - 1];
      const int in_w = l == 0 ? o->c.obs_dim : o->width[l];
      const float* d = mb->D[n][l];
#pragma omp parallel for schedule(dynamic, 1)
      for (int j0 = 0; j0 < t->out; j0 += 16) {
        /* 16 output rows per task share each input row; every (j, k) sums over ascending r */
        const int nj = t->out - j0 < 16 ? t->out - j0 : 16;
        double db[16] = {0};
        double* acc = (double*)calloc((size_t)16 * t->in, sizeof(double));
        for (int r = 0; r < Bm; ++r) {
          const float* row = in + (long long)r * in_w;
          for (int jj = 0; jj < nj; ++jj) {
            const double dj = d[(long long)r * t->out + j0 + jj];
            double* aj = acc + (long long)jj * t->in;
            db[jj] += dj;
            for (int k = 0; k < t->in; ++k) aj[k] += dj * (double)row[k];
          }
        }
        for (int jj = 0; jj < nj; ++jj) {
          const int j = j0 + jj;
          grad[t->b + j] = (float)db[jj];
          for (int k = 0; k < t->in; ++k) grad[t->w + (long long)j * t->in_p + k] = (float)acc[(long long)jj * t->in + k];
        }
        free(acc);
      }
    }
    /* heads */
    const tensor_t* th = &o->net[n][L];
    const float* hl = mb->H[n][L - 1];
    const int hw = o->width[L];
#pragma omp parallel for schedule(static)
    for (int a = 0; a < th->out; ++a) {
      double db = 0.0;
      for (int r = 0; r < Bm; ++r) db += n == 0 ? mb->gmu[(long long)r * A + a] : mb->gv[r];
      grad[th->b + a] = (float)db;
      double* acc = (double*)calloc((size_t)th->in, sizeof(double));
      for (int r = 0; r < Bm; ++r) {
        /* head weight gradients run on the tensor cores with bf16 dL/dmu, dL/dv operands */
        const double ga = (double)R(n == 0 ? mb->gmu[(long long)r * A + a] : mb->gv[r]);
        const float* hr = hl + (long long)r * hw;
        for (int k = 0; k < th->in; ++k) acc[k] += ga * (double)hr[k];
      }
      for (int k = 0; k < th->in; ++k) grad[th->w + (long long)a * th->in_p + k] = (float)acc[k];
      free(acc);
    }
  }
  for (int a = 0; a < A; ++a) {
    double acc = 0.0;
    for (int r = 0; r < Bm; ++r) acc += mb->gls[(long long)r * A + a];
    grad[o->log_std + a] = (float)acc;
  }
  (void)gi;
}

/* Sum of per-GMI gradients in the fold order of the strategy Alg. 1 selects for the uniform
 * G x t layout (reduction.hpp:98-106): G <= 1 MPR (one ring over every GMI), t > G HAR
 * (per-GPU rings, then the leaders' ring, :287-299), else MRR (t rings of one GMI per GPU,
 * ring r = GMI r of GPUs r, r+1, ... (:127-139), then the ring results summed into a zero
 * total in ring order, :255-283). Ring folds start at the owner of the element's chunk
 * (:164-212). */
static int chunk_of(long long e, long long len, int n) { return (int)(((e + 1) * n + len - 1) / len) - 1; }

static void fold_gradients(oracle_t* o) {
  const int n = o->n_gmi, t = o->c.gmis_per_gpu, G = o->c.num_gpus;
  const long long len = o->P;
  for (long long e = 0; e < len; ++e) {
    if (G <= 1) {
      const int c = chunk_of(e, len, n);
      float acc = o->g[c].grad[e];
      for (int j = 1; j < n; ++j) acc = o->g[(c + j) % n].grad[e] + acc;
      o->grad_sum[e] = acc;
    } else if (t > G) {
      const int cl = chunk_of(e, len, t);
      const int cg = chunk_of(e, len, G);
      float acc = 0.f;
      for (int jg = 0; jg < G; ++jg) {
        const int gpu = (cg + jg) % G;
        float loc = o->g[gpu * t + cl].grad[e];
        for (int j = 1; j < t; ++j) loc = o->g[gpu * t + (cl + j) % t].grad[e] + loc;
        acc = jg == 0 ? loc : loc + acc;
      }
      o->grad_sum[e] = acc;
    } else {
      const int c = chunk_of(e, len, G);
      float total = 0.f;
      for (int r = 0; r < t; ++r) {
        /* ring r member j = GMI r of GPU (r + j) % G */
        float acc = o->g[((r + c) % G) * t + r].grad[e];
        for (int j = 1; j < G; ++j) acc = o->g[((r + (c + j) % G) % G) * t + r].grad[e] + acc;
        total = total + acc;
      }
      o->grad_sum[e] = total;
    }
  }
}

static void adam(oracle_t* o) {
  o->adam_step += 1;
  const float b1 = o->c.beta1, b2 = o->c.beta2;
  const float bc1 = (float)(1.0 - pow((double)b1, (double)o->adam_step));
  const float bc2 = (float)(1.0 - pow((double)b2, (double)o->adam_step));
  const float inv_n = 1.0f / (float)o->n_gmi;
  const float ob1 = 1.0f - b1, ob2 = 1.0f - b2;
  for (long long i = 0; i < o->P; ++i) {
    const float gr = o->grad_sum[i] * inv_n;
    const float m = b1 * o->adam_m[i] + ob1 * gr;
    const float v = b2 * o->adam_v[i] + ob2 * gr * gr;
    o->adam_m[i] = m;
    o->adam_v[i] = v;
    const float mh = m / bc1;
    const float vh = v / bc2;
    o->params[i] = o->params[i] - o->c.lr * (mh / (sqrtf(vh) + o->c.adam_eps));
  }
}

/* ---------------------------------------------------------------- API */
void* ppo_oracle_create(const ppo_cfg_t* cfg) {
  if (cfg->num_hidden < 1 || cfg->num_hidden > PPO_MAX_HIDDEN || cfg->act_dim > 64 || cfg->obs_dim > 1024)
    return NULL;
  oracle_t* o = (oracle_t*)calloc(1, sizeof(oracle_t));
  o->c = *cfg;
  g_exact = cfg->exact_fp32;
#ifdef _OPENMP
  if (cfg->threads > 0) omp_set_num_threads(cfg->threads);
#endif
  build_geometry(o);
  o->n_gmi = cfg->num_gpus * cfg->gmis_per_gpu;
  o->params = (float*)calloc((size_t)o->P, sizeof(float));
  o->adam_m = (float*)calloc((size_t)o->P, sizeof(float));
  o->adam_v = (float*)calloc((size_t)o->P, sizeof(float));
  o->grad_sum = (float*)calloc((size_t)o->P, sizeof(float));
  init_params(o);
  o->g = calloc((size_t)o->n_gmi, sizeof(*o->g));
  const int S = cfg->obs_dim, A = cfg->act_dim, T = cfg->horizon;
  for (int c = 0; c < o->n_gmi; ++c) {
    struct gmi* g = &o->g[c];
    g->env0 = (int)((long long)cfg->num_envs * c / o->n_gmi);
    g->nenv = (int)((long long)cfg->num_envs * (c + 1) / o->n_gmi) - g->env0;
    const long long N = g->nenv;
    g->x = (float*)calloc((size_t)(N * S), sizeof(float));
    g->ep_step = (int*)calloc((size_t)N, sizeof(int));
    g->ep_len = (int*)calloc((size_t)N, sizeof(int));
    g->ep_count = (int*)calloc((size_t)N, sizeof(int));
    g->obs = (float*)calloc((size_t)((T + 1) * N * S), sizeof(float));
    g->act = (float*)calloc((size_t)(T * N * A), sizeof(float));
    g->logp = (float*)calloc((size_t)(T * N), sizeof(float));
    g->rew = (float*)calloc((size_t)(T * N), sizeof(float));
    g->val = (float*)calloc((size_t)((T + 1) * N), sizeof(float));
    g->adv = (float*)calloc((size_t)(T * N), sizeof(float));
    g->ret = (float*)calloc((size_t)(T * N), sizeof(float));
    g->done = (unsigned char*)calloc((size_t)(T * N), 1);
    g->grad = (float*)calloc((size_t)o->P, sizeof(float));
    for (int e = 0; e < g->nenv; ++e) {
      const int gid = g->env0 + e;
      uint32_t out[4];
      philox_tag(cfg->seed, (uint32_t)gid, 0, 0, TAG_EPLEN, out);
      g->ep_len[e] = 16 + (int)(out[0] % 48u);
      g->ep_step[e] = (int)(out[1] % (uint32_t)g->ep_len[e]);
      env_reset_state(o, gid, 0, g->x + (long long)e * S);
      for (int i = 0; i < S; ++i) g->obs[(long long)e * S + i] = R(g->x[(long long)e * S + i]);
    }
  }
  return o;
}

void ppo_oracle_free(void* h) {
  oracle_t* o = (oracle_t*)h;
  if (!o) return;
  for (int c = 0; c < o->n_gmi; ++c) {
    struct gmi* g = &o->g[c];
    free(g->x); free(g->ep_step); free(g->ep_len); free(g->ep_count); free(g->obs); free(g->act);
    free(g->logp); free(g->rew); free(g->val); free(g->adv); free(g->ret); free(g->done); free(g->grad);
  }
  free(o->g);
  free(o->params); free(o->adam_m); free(o->adam_v); free(o->grad_sum);
  free(o);
}

static float* g_mean_std; /* scratch for rollout -> update hand-off */

/* Env stepping of every GMI with the current parameters (obs slot 0 carries the last
 * observation of the previous rollout after the first one). */
static void rollout_all(oracle_t* o) {
  float* wbf = make_bf16_weights(o);
  for (int c = 0; c < o->n_gmi; ++c) {
    struct gmi* g = &o->g[c];
    const long long N = g->nenv, S = o->c.obs_dim, T = o->c.horizon;
    if (o->iteration > 0) memmove(g->obs, g->obs + T * N * S, sizeof(float) * N * S);
    rollout_gmi(o, c, wbf);
  }
  free(wbf);
}

/* Values of all T+1 observation slots with the current parameters, GAE, advantage moments. */
static void values_gae_all(oracle_t* o) {
  float* wbf = make_bf16_weights(o);
  double rsum = 0;
  long long rn = 0;
  free(g_mean_std);
  g_mean_std = (float*)calloc((size_t)(2 * o->n_gmi), sizeof(float));
  for (int c = 0; c < o->n_gmi; ++c) {
    struct gmi* g = &o->g[c];
    const long long N = g->nenv, T = o->c.horizon;
    values_gmi(o, c, wbf);
    gae_gmi(o, c, &g_mean_std[2 * c], &g_mean_std[2 * c + 1]);
    for (long long i = 0; i < T * N; ++i) rsum += g->rew[i];
    rn += T * N;
  }
  o->last.mean_reward = rsum / (double)(rn ? rn : 1);
  o->last.env_steps = rn;
  free(wbf);
}

int ppo_oracle_rollout(void* h) {
  oracle_t* o = (oracle_t*)h;
  if (o->pending) return -2; /* the next iteration's rollout already ran */
  g_exact = o->c.exact_fp32;
  rollout_all(o);
  values_gae_all(o);
  o->pending = 1;
  return 0;
}

/* E epochs x K minibatch updates on the GMIs' current experience; iteration += 1. */
static void train_all(oracle_t* o) {
  const int S = o->c.obs_dim, A = o->c.act_dim, T = o->c.horizon, L = o->L;
  float* wbf = NULL;
  mb_t* mbs = (mb_t*)calloc((size_t)o->n_gmi, sizeof(mb_t));
  int* Bm = (int*)calloc((size_t)o->n_gmi, sizeof(int));
  for (int c = 0; c < o->n_gmi; ++c) {
    const int B = T * o->g[c].nenv;
    Bm[c] = B / o->c.minibatches;
    mb_alloc(o, &mbs[c], Bm[c]);
  }
  for (int ep = 0; ep < o->c.epochs; ++ep) {
    uint32_t(*keys)[4] = (uint32_t(*)[4])malloc(sizeof(uint32_t) * 4 * (size_t)o->n_gmi);
    for (int c = 0; c < o->n_gmi; ++c)
      philox_tag(o->c.seed, (uint32_t)c, (uint32_t)o->iteration, (uint32_t)ep, TAG_PERM, keys[c]);
    for (int k = 0; k < o->c.minibatches; ++k) {
      free(wbf);
      wbf = make_bf16_weights(o);
      for (int c = 0; c < o->n_gmi; ++c) {
        struct gmi* g = &o->g[c];
        mb_t* m = &mbs[c];
        const int N = g->nenv, B = T * N;
        const float mean = g_mean_std[2 * c], sd = g_mean_std[2 * c + 1];
        for (int r = 0; r < Bm[c]; ++r) {
          const uint32_t j = ppo_perm_index((uint32_t)(k * Bm[c] + r), (uint32_t)B, keys[c]);
          memcpy(m->X + (long long)r * S, g->obs + (long long)j * S, sizeof(float) * S);
          memcpy(m->act + (long long)r * A, g->act + (long long)j * A, sizeof(float) * A);
          m->oldlp[r] = g->logp[j];
          m->adv[r] = (g->adv[j] - mean) / sd;
          m->ret[r] = g->ret[j];
        }
        minibatch_grad(o, c, m, Bm[c], wbf, g->grad);
      }
      fold_gradients(o);
      adam(o);
    }
    free(keys);
  }
  double ent = 0;
  for (int a = 0; a < A; ++a) ent += 0.5 + (double)LOG_2PI_HALF + (double)o->params[o->log_std + a];
  o->last.policy_loss = mbs[0].loss_pi;
  o->last.value_loss = mbs[0].loss_v;
  o->last.approx_kl = mbs[0].kl;
  o->last.clip_frac = mbs[0].clipped;
  o->last.entropy = ent;
  for (int c = 0; c < o->n_gmi; ++c) mb_free(o, &mbs[c]);
  free(mbs);
  free(Bm);
  free(wbf);
  o->iteration += 1;
}

int ppo_oracle_iteration(void* h, ppo_stats_t* out) {
  oracle_t* o = (oracle_t*)h;
  if (!o->pending) ppo_oracle_rollout(h);
  g_exact = o->c.exact_fp32;
  o->pending = 0;
  train_all(o);
  if (out) *out = o->last;
  return 0;
}

/* Decoupled mode (device: gmi_ppo_config_t.decoupled): the serving GMI produces rollout i+1
 * -- env steps, critic values of its T+1 observation slots and GAE -- with a snapshot of
 * theta_i, while the trainer runs the epochs of iteration i on rollout i (produced with
 * theta_{i-1}; rollout 0 with theta_0). Rollout r keys its action noise with r (= the
 * iteration counter when it runs here). Reported stats: losses of iteration i's update and
 * the mean reward of rollout i. */
int ppo_oracle_iteration_decoupled(void* h, ppo_stats_t* out) {
  oracle_t* o = (oracle_t*)h;
  g_exact = o->c.exact_fp32;
  if (!o->primed) {
    rollout_all(o);
    values_gae_all(o);
    o->primed = 1;
  }
  float* snap = (float*)malloc(sizeof(float) * o->P);
  memcpy(snap, o->params, sizeof(float) * o->P);
  train_all(o);
  const ppo_stats_t trained = o->last;
  float* cur = o->params;
  o->params = snap;
  rollout_all(o);
  values_gae_all(o);
  o->params = cur;
  free(snap);
  if (out) *out = trained;
  /* o->last keeps rollout i+1's reward statistics for the next call's report */
  const double next_reward = o->last.mean_reward;
  o->last = trained;
  o->last.mean_reward = next_reward;
  return 0;
}

static void mb_alloc(const oracle_t* o, mb_t* m, int Bm) {
  const int S = o->c.obs_dim, A = o->c.act_dim;
  m->X = (float*)malloc(sizeof(float) * (size_t)Bm * S);
  m->act = (float*)malloc(sizeof(float) * (size_t)Bm * A);
  m->oldlp = (float*)malloc(sizeof(float) * (size_t)Bm);
  m->adv = (float*)malloc(sizeof(float) * (size_t)Bm);
  m->ret = (float*)malloc(sizeof(float) * (size_t)Bm);
  m->gmu = (float*)malloc(sizeof(float) * (size_t)Bm * A);
  m->gls = (float*)malloc(sizeof(float) * (size_t)Bm * A);
  m->gv = (float*)malloc(sizeof(float) * (size_t)Bm);
  for (int n = 0; n < 2; ++n)
    for (int l = 0; l < o->L; ++l) {
      m->H[n][l] = (float*)malloc(sizeof(float) * (size_t)Bm * o->width[l + 1]);
      m->D[n][l] = (float*)malloc(sizeof(float) * (size_t)Bm * o->width[l + 1]);
    }
}

static void mb_free(const oracle_t* o, mb_t* m) {
  free(m->X); free(m->act); free(m->oldlp); free(m->adv); free(m->ret); free(m->gmu); free(m->gls); free(m->gv);
  for (int n = 0; n < 2; ++n)
    for (int l = 0; l < o->L; ++l) {
      free(m->H[n][l]);
      free(m->D[n][l]);
    }
}

int ppo_oracle_minibatch(void* h, int gmi, const float* X, const float* act, const float* oldlp,
                         const float* adv, const float* ret, int B, float* grad, double* stats) {
  oracle_t* o = (oracle_t*)h;
  g_exact = o->c.exact_fp32;
  mb_t m;
  memset(&m, 0, sizeof(m));
  mb_alloc(o, &m, B);
  memcpy(m.X, X, sizeof(float) * (size_t)B * o->c.obs_dim);
  memcpy(m.act, act, sizeof(float) * (size_t)B * o->c.act_dim);
  memcpy(m.oldlp, oldlp, sizeof(float) * (size_t)B);
  memcpy(m.adv, adv, sizeof(float) * (size_t)B);
  memcpy(m.ret, ret, sizeof(float) * (size_t)B);
  float* wbf = make_bf16_weights(o);
  minibatch_grad(o, gmi, &m, B, wbf, grad);
  if (stats) {
    stats[0] = m.loss_pi;
    stats[1] = m.loss_v;
    stats[2] = m.kl;
    stats[3] = m.clipped;
  }
  free(wbf);
  mb_free(o, &m);
  return 0;
}

int ppo_oracle_adam(void* h, const float* grad_sum) {
  oracle_t* o = (oracle_t*)h;
  memcpy(o->grad_sum, grad_sum, sizeof(float) * o->P);
  adam(o);
  return 0;
}

long long ppo_oracle_param_count(void* h) { return ((oracle_t*)h)->P; }

int ppo_oracle_width(void* h, int layer) {
  oracle_t* o = (oracle_t*)h;
  return layer < 0 || layer > o->L ? -1 : o->width_p[layer];
}

/* what: "params" "adam_m" "adam_v" (gmi ignored) | "grad" "x" "obs" "act" "logp" "rew"
 * "val" "adv" "ret" "done" "ep_step" "ep_len" "ep_count" (per gmi). Sizes in elements. */
static void* field_ptr(oracle_t* o, const char* what, int gmi, long long* n, int* esz) {
  *esz = 4;
  if (!strcmp(what, "params")) { *n = o->P; return o->params; }
  if (!strcmp(what, "adam_m")) { *n = o->P; return o->adam_m; }
  if (!strcmp(what, "adam_v")) { *n = o->P; return o->adam_v; }
  if (gmi < 0 || gmi >= o->n_gmi) return NULL;
  struct gmi* g = &o->g[gmi];
  const long long N = g->nenv, S = o->c.obs_dim, A = o->c.act_dim, T = o->c.horizon;
  if (!strcmp(what, "grad")) { *n = o->P; return g->grad; }
  if (!strcmp(what, "x")) { *n = N * S; return g->x; }
  if (!strcmp(what, "obs")) { *n = (T + 1) * N * S; return g->obs; }
  if (!strcmp(what, "act")) { *n = T * N * A; return g->act; }
  if (!strcmp(what, "logp")) { *n = T * N; return g->logp; }
  if (!strcmp(what, "rew")) { *n = T * N; return g->rew; }
  if (!strcmp(what, "val")) { *n = (T + 1) * N; return g->val; }
  if (!strcmp(what, "adv")) { *n = T * N; return g->adv; }
  if (!strcmp(what, "ret")) { *n = T * N; return g->ret; }
  if (!strcmp(what, "ep_step")) { *n = N; return g->ep_step; }
  if (!strcmp(what, "ep_len")) { *n = N; return g->ep_len; }
  if (!strcmp(what, "ep_count")) { *n = N; return g->ep_count; }
  if (!strcmp(what, "done")) { *n = T * N; *esz = 1; return g->done; }
  return NULL;
}

int ppo_oracle_get(void* h, const char* what, int gmi, void* dst, long long n) {
  long long have;
  int esz;
  void* p = field_ptr((oracle_t*)h, what, gmi, &have, &esz);
  if (!p) return -1;
  if (n > have) n = have;
  memcpy(dst, p, (size_t)(n * esz));
  return (int)(have > 0x7fffffff ? 0x7fffffff : have);
}

int ppo_oracle_set(void* h, const char* what, int gmi, const void* src, long long n) {
  long long have;
  int esz;
  void* p = field_ptr((oracle_t*)h, what, gmi, &have, &esz);
  if (!p || n != have) return -1;
  memcpy(p, src, (size_t)(n * esz));
  return 0;
}
