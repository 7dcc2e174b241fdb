// Host API of the tcgen05 GEMM (see gemm.cuh).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gemm_types.hpp"

namespace gmi {

// Operand map: bf16 [outer rows x inner cols] with row pitch ld (elements), 128B swizzle.
CUtensorMap make_tma_2d_bf16(const void* base, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                             uint32_t box_inner, uint32_t box_outer);
// bf16 output map [rows x cols], box 32 x 32, 64B swizzle (epilogue staging layout).
CUtensorMap make_tma_out_bf16(const void* base, uint64_t cols, uint64_t rows, uint64_t ld_elems);
// fp32 split-K output map [splits][M][N] (split stride in elements), box 32 x 32 x 1, 128B swizzle.
CUtensorMap make_tma_out_f32(const void* base, uint64_t cols, uint64_t rows, uint64_t splits, uint64_t ld_elems,
                             uint64_t split_stride);

// K-major operand map for A (box rows = 128) or B (box rows = bn); MN-major map (box 64 x 64).
CUtensorMap tma_kmajor(const void* p, int cols, long long rows, long long ld, int box_rows);
CUtensorMap tma_mnmajor(const void* p, int cols, long long rows, long long ld);
// elu' operand of a weight-stationary input-gradient GEMM: bf16 [rows x cols], box 64 x 128, SW128.
CUtensorMap tma_aux(const void* p, int cols, long long rows, long long ld);

// Launches the persistent kernel with min(tiles, max_ctas) CTAs (max_ctas 0 = SM count).
// ws = 1 / 2: weight-stationary mode (requires N <= bn, K <= 256 / 512 (bn <= 128), splits == 1).
void gemm_launch(const GemmParams& P, int bn, int a_mn, int b_mn, int epi, cudaStream_t s, int max_ctas = 0,
                 int ws = 0);
// Weight-stationary choice for a launch: returns the block N (N padded to 64) when every
// CTA gets at least one tile and the weights fit, else 0 (use the streaming kernel).
int gemm_ws_bn(int M, int N, int K, int problems, int sms);
// Wide weight-stationary plan for a layer too wide for gemm_ws_bn (N > 256 or K > 256): N split
// into 128-column parts, one problem per (net, part), block N = 128. Returns the ws mode (1: K <=
// 256, 2: K <= 512) and the part count, or 0 when the weights do not fit, the problems exceed a
// launch, or some CTA would get no tile.
int gemm_ws_wide(int M, int N, int K, int nets, int sms, int* parts);
// Weight-gradient GEMM on SM pairs (gemm_pair.cu): M = N = 256, MN-major operands, fp32 slabs.
bool gemm_pair_applicable(int M, int N, int a_mn, int b_mn, int epi);
void gemm_pair_launch(const GemmParams& P, int max_ctas, cudaStream_t s);
int gemm_pair_max_clusters();
// Grid of a weight-stationary launch (a multiple of `problems`); the fused column-sum
// output has grid / problems rows per problem.
int gemm_ws_grid(int M, int problems, int max_ctas);

// Block N for a launch: the largest of {256,128,64} (<= padded N) that still gives at
// least 4 tiles per SM, else the smallest.
int gemm_choose_bn(int M, int N, int problems, int splits, int sms);
int gemm_tiles(int M, int N, int bn, int problems, int splits);
int device_sm_count();

}  // namespace gmi
