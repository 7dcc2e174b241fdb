/* TEST INFRASTRUCTURE ONLY — the checker for the device reduction (cuda/reduce.cu).
 * Never linked into libgmi.so; loaded by tests/ and bench.py's cpu_baseline leg only.
 *
 * Literal CPU restatement of the reference's execute() data movement
 * (proj/include/gmux/reduction.hpp:170-212 chunked_ring_allreduce, :249-299 strategies):
 * every ring step copies the outgoing chunks ("sent") before accumulating them into the
 * successor, exactly as the reference does, so the accumulation order is the reference's
 * by construction (not the fold shortcut the GPU kernel uses). Parity of this file with
 * the reference itself is pinned for fp64 by tests/golden/ref_execute.json
 * (tests/test_oracle.py); the fp32 instantiation is the oracle for the PPO gradient path.
 *
 * Layout: num_gpus lists, counts[g] GMIs each, ids GPU-major; bufs[i] is the i-th id's
 * buffer (flattened order) and is NOT modified; result written to out[len].
 */
#include <stdlib.h>
#include <string.h>

#define DEFINE_RING(T, NAME)                                                                     \
  static void NAME(T** v, const int* members, int n, size_t len) {                              \
    if (n < 2) return;                                                                           \
    T** sent = (T**)malloc(sizeof(T*) * (size_t)n);                                              \
    for (int i = 0; i < n; ++i) sent[i] = (T*)malloc(sizeof(T) * (len / (size_t)n + 2));         \
    for (int phase = 0; phase < 2; ++phase)                                                      \
      for (int s = 0; s < n - 1; ++s) {                                                          \
        size_t lo[256], hi[256];                                                                 \
        for (int i = 0; i < n; ++i) { /* reduce-scatter: (i-s); allgather: (i+1-s) mod n */      \
          int c = phase == 0 ? i - s : i + 1 - s;                                                \
          c = ((c % n) + n) % n;                                                                 \
          lo[i] = len * (size_t)c / (size_t)n;                                                   \
          hi[i] = len * (size_t)(c + 1) / (size_t)n;                                             \
          memcpy(sent[i], v[members[i]] + lo[i], sizeof(T) * (hi[i] - lo[i]));                  \
        }                                                                                        \
        for (int i = 0; i < n; ++i) {                                                            \
          T* dst = v[members[(i + 1) % n]];                                                      \
          for (size_t e = 0; e < hi[i] - lo[i]; ++e) {                                           \
            if (phase == 0) dst[lo[i] + e] += sent[i][e];                                        \
            else dst[lo[i] + e] = sent[i][e];                                                    \
          }                                                                                      \
        }                                                                                        \
      }                                                                                          \
    for (int i = 0; i < n; ++i) free(sent[i]);                                                   \
    free(sent);                                                                                  \
  }

DEFINE_RING(float, ring_f32)
DEFINE_RING(double, ring_f64)

/* index of gmi id in the flattened layout */
static int pos_of(const int* ids, int n, int id) {
  for (int i = 0; i < n; ++i)
    if (ids[i] == id) return i;
  return -1;
}

#define DEFINE_EXECUTE(T, NAME, RING)                                                             \
  int NAME(int algo, int g, const int* counts, const int* ids, const T* const* bufs, size_t len, \
           T* out) {                                                                              \
    int n = 0;                                                                                    \
    for (int i = 0; i < g; ++i) n += counts[i];                                                   \
    if (n > 256 || g > 256) return -1;                                                            \
    T** v = (T**)malloc(sizeof(T*) * (size_t)n);                                                  \
    for (int i = 0; i < n; ++i) {                                                                 \
      v[i] = (T*)malloc(sizeof(T) * (len ? len : 1));                                             \
      memcpy(v[i], bufs[i], sizeof(T) * len);                                                     \
    }                                                                                             \
    int members[256], holder = 0, off[257];                                                       \
    off[0] = 0;                                                                                   \
    for (int i = 0; i < g; ++i) off[i + 1] = off[i] + counts[i];                                  \
    if (algo == 0) { /* MPR */                                                                    \
      for (int i = 0; i < n; ++i) members[i] = i;                                                 \
      RING(v, members, n, len);                                                                   \
      holder = 0;                                                                                 \
    } else if (algo == 1) { /* MRR: requires uniform t <= g */                                    \
      const int t = counts[0];                                                                    \
      for (int i = 0; i < g; ++i)                                                                 \
        if (counts[i] != t) return -2;                                                            \
      if (t > g) return -2;                                                                       \
      int ends[256];                                                                              \
      for (int r = 0; r < t; ++r) {                                                               \
        for (int j = 0; j < g; ++j) members[j] = off[(r + j) % g] + r;                            \
        RING(v, members, g, len);                                                                 \
        ends[r] = members[g - 1];                                                                 \
      }                                                                                           \
      int ne = t >= 2 ? t : g;                                                                    \
      if (t < 2)                                                                                  \
        for (int j = 0; j < g; ++j) ends[j] = off[j % g] + 0; /* ring 0 members, rotation r=0 */  \
      if (g >= 2 && ne >= 2) {                                                                    \
        T* total = (T*)calloc(len ? len : 1, sizeof(T));                                          \
        for (int r = 0; r < t; ++r) {                                                             \
          const T* part = v[off[(r + g - 1) % g] + r]; /* ring r's last member */                 \
          for (size_t e = 0; e < len; ++e) total[e] += part[e];                                   \
        }                                                                                         \
        for (int j = 0; j < ne; ++j) memcpy(v[ends[j]], total, sizeof(T) * len);                  \
        free(total);                                                                              \
      }                                                                                           \
      holder = ends[0];                                                                           \
    } else { /* HAR */                                                                            \
      for (int i = 0; i < g; ++i) {                                                               \
        for (int j = 0; j < counts[i]; ++j) members[j] = off[i] + j;                              \
        RING(v, members, counts[i], len);                                                         \
      }                                                                                           \
      int leaders[256];                                                                           \
      for (int i = 0; i < g; ++i) { /* smallest id with id % t_i == 0, else smallest id */        \
        int best = -1, mn = ids[off[i]];                                                          \
        for (int j = off[i]; j < off[i + 1]; ++j) {                                               \
          if (ids[j] % counts[i] == 0 && (best < 0 || ids[j] < best)) best = ids[j];              \
          if (ids[j] < mn) mn = ids[j];                                                           \
        }                                                                                         \
        leaders[i] = pos_of(ids, n, best >= 0 ? best : mn);                                       \
      }                                                                                           \
      RING(v, leaders, g, len);                                                                   \
      holder = leaders[0];                                                                        \
    }                                                                                             \
    memcpy(out, v[holder], sizeof(T) * len);                                                      \
    for (int i = 0; i < n; ++i) free(v[i]);                                                       \
    free(v);                                                                                      \
    return 0;                                                                                     \
  }

DEFINE_EXECUTE(float, oracle_execute_f32, ring_f32)
DEFINE_EXECUTE(double, oracle_execute_f64, ring_f64)
