// Host API of the tcgen05 GEMM (see gemm.cuh).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gemm_types.hpp"

namespace gmi {

struct GemmOperandDesc {
  const void* ptr;
  long long ld;   // elements between consecutive rows of the stored matrix
  bool mn_major;  // false: stored [rows x K]; true: stored [K x rows]
};

CUtensorMap make_tma_2d_bf16(const void* base, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                             uint32_t box_inner, uint32_t box_outer);

// Fills the tensor maps and shape of one problem (kb_per_split = all k-blocks).
void gemm_set_problem(GemmProblem& p, const GemmOperandDesc& a, const GemmOperandDesc& b, int M,
                      int N, int K, int block_n);

void gemm_launch(const GemmParams& P, int block_n, int a_mn, int b_mn, int epi, cudaStream_t s);

int gemm_pick_block_n(int N);

}  // namespace gmi
