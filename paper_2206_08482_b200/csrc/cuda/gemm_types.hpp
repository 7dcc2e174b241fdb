// Host-visible GEMM descriptor types (see gemm.cuh for the kernel).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdint>

namespace gmi {

enum GemmEpi : int { EPI_BIAS_ELU = 0, EPI_DACT = 1, EPI_F32 = 2 };

constexpr int kGemmBlockM = 128;
constexpr int kGemmBlockK = 64;  // one 128-byte swizzle atom of bf16
constexpr int kGemmMaxKbWS = 4;  // weight-stationary mode: K <= 256
// Resident k-blocks of B per weight-stationary mode: ws = 1 keeps K <= 256 (every block N);
// ws = 2 keeps K <= 512 for block N <= 128 (the wide HM / SH layers, split into 128-column
// problems): 8 x 16 KB of resident weights at N = 128.
constexpr int gemm_ws_kb(int ws) { return ws == 2 ? 8 : kGemmMaxKbWS; }
// Epilogue warps: 16 for the bf16 (elementwise-heavy) epilogues, 8 for fp32 slabs.
constexpr int gemm_epi_warps(int epi) { return epi == 2 ? 8 : 16; }
constexpr int gemm_threads(int epi) { return 64 + 32 * gemm_epi_warps(epi); }  // TMA, MMA, epilogue

struct alignas(64) GemmProblem {
  CUtensorMap map_a;
  CUtensorMap map_b;
  CUtensorMap map_out;  // bf16 2-D {N, rows} box {32,32} SW64, or fp32 3-D {N, M, splits} box {32,32,1} SW128
  CUtensorMap map_aux;  // weight-stationary EPI_DACT: the elu' operand (aux) {N, rows}, box {64, 128} SW128
  const float* bias;
  const __nv_bfloat16* aux;
  int64_t ld_aux;
  // Split-K weight gradient (EPI_F32, MN-major A = dPre): column sums of A over this split's
  // K range (the layer's bias gradient), fp32 [splits][M], or null.
  float* colsum;
  int M, N, K;
  int kb_per_split;
  int a_row0;    // offset added to A's stored-row coordinate (M for K-major, K for MN-major)
  int b_row0;    // offset added to B's stored-row coordinate (N for K-major, K for MN-major)
  int out_row0;  // offset added to the output row coordinate (bf16 outputs)
};

// All problems of one launch share M, N, K and the split count (grouped GEMM).
constexpr int kGemmMaxProblems = 8;

struct alignas(64) GemmParams {
  // grouped problems (e.g. policy / value nets, or their N-halves); chained launches hold
  // layer c's problems at prob[c * num_problems + i]
  GemmProblem prob[kGemmMaxProblems];
  int num_problems;
  int splits;
  // Weight-stationary launches: B (the layer's weights) is not written by the preceding
  // kernel in the stream, so the CTA loads its resident B before griddepcontrol.wait and the
  // load overlaps the previous kernel's tail (set by the host when no in-stream kernel updates
  // the weights right before this launch).
  int b_stable;
  // Chained weight-stationary forward (EPI_BIAS_ELU): `chain` consecutive hidden layers in one
  // launch. Every CTA keeps its row tiles for all layers (layer c+1's tile m reads the H tile m
  // this CTA stored for layer c), so there is no cross-CTA dependency between the layers: a CTA
  // swaps in the next layer's resident weights as soon as its MMAs of the layer are done and
  // goes on, instead of a kernel boundary (launch, prologue, pipeline fill, wave tail) per layer.
  int chain;
  // Heterogeneous split-K group (non-weight-stationary only): problems with their own M and N
  // (sharing K and the split count); problem p owns tiles [tile0[p], tile0[p+1]) of the launch,
  // laid out split-major inside it. Set by gemm_launch when `hetero` is 1.
  int hetero;
  int tile0[kGemmMaxProblems + 1];
  unsigned long long* trace;  // optional [8 tiles][16] globaltimer stamps of CTA 0 (development aid)
};

}  // namespace gmi
