// Host-visible GEMM descriptor types (see gemm.cuh for the kernel).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdint>

namespace gmi {

enum GemmEpi : int { EPI_BIAS_ELU = 0, EPI_DACT = 1, EPI_F32 = 2 };

constexpr int kGemmBlockM = 128;
constexpr int kGemmBlockK = 64;  // one 128-byte swizzle atom of bf16

struct alignas(64) GemmProblem {
  CUtensorMap map_a;
  CUtensorMap map_b;
  void* out;
  const float* bias;
  const __nv_bfloat16* aux;
  int64_t ld_out;
  int64_t ld_aux;
  int64_t split_stride;  // elements between split-K output slabs (EPI_F32)
  int M, N, K;
  int kb_per_split;
  int a_row0;  // offset added to A's stored-row coordinate (M for K-major, K for MN-major)
  int b_row0;  // offset added to B's stored-row coordinate (N for K-major, K for MN-major)
};

struct alignas(64) GemmParams {
  GemmProblem prob[2];
  int num_problems;
  int splits;
};

}  // namespace gmi
