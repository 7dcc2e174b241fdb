/* gmi.h — C-ABI of libgmi, the B200-native data-parallel PPO iteration with
 * GMI (GPU multiplexing instance) placement and layout-aware gradient reduction.
 *
 * Plain C types only: caller-owned host arrays and device pointers, explicit
 * cudaStream_t passed as void*, integer return codes, a thread-local message.
 * The C++ drop-in `namespace gmux` (include/gmux/gmux.hpp) is a header-only
 * wrapper over these entry points that restores the reference's types and
 * exception classes.
 *
 * Reference interfaces replaced (paths relative to the reference tree,
 * proj/include/gmux/):  see each declaration.
 */
#ifndef GMI_H_
#define GMI_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define GMI_API __attribute__((visibility("default")))
#else
#define GMI_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ errors
 * Codes mirror the reference CLI's exit-code split (tools/gmux.cpp:389-411):
 * gmi_exit_code() maps INVALID/CONFIG -> 2, every other failure -> 1. */
enum {
  GMI_OK = 0,
  GMI_ERR_DOMAIN = 1,      /* std::runtime_error                          */
  GMI_ERR_INVALID = 2,     /* std::invalid_argument                       */
  GMI_ERR_MULTISTREAM = 3, /* gmux::MultiStreamError (reduction.hpp:91)   */
  GMI_ERR_PLAN = 4,        /* gmux::PlanError (mapping.hpp:209)           */
  GMI_ERR_PIPELINE = 5,    /* gmux::PipelineError (channels.hpp:105)      */
  GMI_ERR_CONFIG = 6,      /* gmux::ConfigError (config.hpp:39)           */
  GMI_ERR_CUDA = 7,        /* CUDA runtime / driver failure               */
  GMI_ERR_NCCL = 8         /* NCCL failure                                */
};

GMI_API const char* gmi_last_error(void);
GMI_API int gmi_exit_code(int err);
GMI_API int gmi_version(void);

/* ------------------------------------------------------------------ diagnostics
 * Single tcgen05 GEMM launch, D[m][n] = sum_k A(m,k) B(n,k), bf16 in, fp32 accumulate.
 * a_mn/b_mn: 0 = operand stored [rows x K], 1 = stored [K x rows].
 * epi: 0 = bf16 elu(acc + bias), 1 = bf16 acc * elu'(aux), 2 = fp32 (split-K slabs). */
GMI_API int gmi_dev_gemm(int a_mn, int b_mn, int epi, int M, int N, int K, const void* A, long long lda,
                 const void* B, long long ldb, void* out, long long ldo, const float* bias,
                 const void* aux, long long ld_aux, int splits, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GMI_H_ */
