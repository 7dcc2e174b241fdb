// Host side of the tcgen05 GEMM: TMA tensor-map encoding, template dispatch and a
// C-ABI diagnostic entry point used by the GPU parity tests.
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>
#include <string>

#include "../host/errors.hpp"
#include "gemm.cuh"
#include "gemm_host.hpp"

namespace gmi {

namespace {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) fail(GMI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  return fn;
}

}  // namespace

CUtensorMap make_tma_2d_bf16(const void* base, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                             uint32_t box_inner, uint32_t box_outer) {
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0) invalid("TMA base address must be 16-byte aligned");
  if ((ld_elems * 2) % 16 != 0) invalid("TMA row pitch must be a multiple of 16 bytes");
  CUtensorMap map;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld_elems * 2};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estride[2] = {1, 1};
  CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                           strides, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(GMI_ERR_CUDA, "cuTensorMapEncodeTiled failed with code " + std::to_string(int(r)));
  return map;
}

void gemm_set_problem(GemmProblem& p, const GemmOperandDesc& a, const GemmOperandDesc& b, int M,
                      int N, int K, int block_n) {
  // A(m,k): K-major -> row-major [M x K]; MN-major -> row-major [K x M].
  if (a.mn_major)
    p.map_a = make_tma_2d_bf16(a.ptr, M, K, a.ld, 64, kGemmBlockK);
  else
    p.map_a = make_tma_2d_bf16(a.ptr, K, M, a.ld, kGemmBlockK, kGemmBlockM);
  if (b.mn_major)
    p.map_b = make_tma_2d_bf16(b.ptr, N, K, b.ld, 64, kGemmBlockK);
  else
    p.map_b = make_tma_2d_bf16(b.ptr, K, N, b.ld, kGemmBlockK, block_n);
  p.M = M;
  p.N = N;
  p.K = K;
  p.kb_per_split = (K + kGemmBlockK - 1) / kGemmBlockK;
}

namespace {

template <int BN, int ST, int AMN, int BMN, int EPI>
void launch_t(const GemmParams& P, dim3 grid, cudaStream_t s) {
  constexpr int smem = gemm_smem_bytes<BN, ST>();
  auto kern = gemm_tcgen05_kernel<BN, ST, AMN, BMN, EPI>;
  static bool configured = false;  // per instantiation
  if (!configured) {
    GMI_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  kern<<<grid, 128, smem, s>>>(P);
  GMI_CUDA_CHECK(cudaGetLastError());
}

template <int BN, int ST>
void launch_bn(const GemmParams& P, int a_mn, int b_mn, int epi, dim3 grid, cudaStream_t s) {
  const int key = a_mn * 100 + b_mn * 10 + epi;
  switch (key) {
    case 0 * 100 + 0 * 10 + EPI_BIAS_ELU: return launch_t<BN, ST, 0, 0, EPI_BIAS_ELU>(P, grid, s);
    case 0 * 100 + 0 * 10 + EPI_F32: return launch_t<BN, ST, 0, 0, EPI_F32>(P, grid, s);
    case 0 * 100 + 0 * 10 + EPI_DACT: return launch_t<BN, ST, 0, 0, EPI_DACT>(P, grid, s);
    case 0 * 100 + 1 * 10 + EPI_DACT: return launch_t<BN, ST, 0, 1, EPI_DACT>(P, grid, s);
    case 0 * 100 + 1 * 10 + EPI_F32: return launch_t<BN, ST, 0, 1, EPI_F32>(P, grid, s);
    case 1 * 100 + 1 * 10 + EPI_F32: return launch_t<BN, ST, 1, 1, EPI_F32>(P, grid, s);
    case 1 * 100 + 0 * 10 + EPI_F32: return launch_t<BN, ST, 1, 0, EPI_F32>(P, grid, s);
    default: invalid("unsupported GEMM operand-major / epilogue combination");
  }
}

}  // namespace

void gemm_launch(const GemmParams& P, int block_n, int a_mn, int b_mn, int epi, cudaStream_t s) {
  int max_m = 0, max_n = 0;
  for (int i = 0; i < P.num_problems; ++i) {
    max_m = P.prob[i].M > max_m ? P.prob[i].M : max_m;
    max_n = P.prob[i].N > max_n ? P.prob[i].N : max_n;
  }
  dim3 grid((max_m + kGemmBlockM - 1) / kGemmBlockM, (max_n + block_n - 1) / block_n,
            P.num_problems * P.splits);
  switch (block_n) {
    case 64: return launch_bn<64, 4>(P, a_mn, b_mn, epi, grid, s);
    case 128: return launch_bn<128, 4>(P, a_mn, b_mn, epi, grid, s);
    case 256: return launch_bn<256, 4>(P, a_mn, b_mn, epi, grid, s);
    default: invalid("GEMM block_n must be 64, 128 or 256");
  }
}

int gemm_pick_block_n(int N) {
  if (N <= 64) return 64;
  if (N <= 128) return 128;
  return 256;
}

}  // namespace gmi

extern "C" int gmi_dev_gemm(int a_mn, int b_mn, int epi, int M, int N, int K, const void* A,
                            long long lda, const void* B, long long ldb, void* out, long long ldo,
                            const float* bias, const void* aux, long long ld_aux, int splits,
                            void* stream) {
  return gmi::guarded([&] {
    if (M <= 0 || N <= 0 || K <= 0) gmi::invalid("gemm dims must be positive");
    if (N % 32 != 0) gmi::invalid("gemm N must be a multiple of 32");
    if (splits < 1) gmi::invalid("splits must be >= 1");
    gmi::GemmParams P{};
    const int bn = gmi::gemm_pick_block_n(N);
    gmi::gemm_set_problem(P.prob[0], {A, lda, a_mn != 0}, {B, ldb, b_mn != 0}, M, N, K, bn);
    const int nkb = (K + gmi::kGemmBlockK - 1) / gmi::kGemmBlockK;
    P.prob[0].kb_per_split = (nkb + splits - 1) / splits;
    P.prob[0].out = out;
    P.prob[0].ld_out = ldo;
    P.prob[0].bias = bias;
    P.prob[0].aux = static_cast<const __nv_bfloat16*>(aux);
    P.prob[0].ld_aux = ld_aux;
    P.prob[0].split_stride = static_cast<int64_t>(M) * ldo;
    P.num_problems = 1;
    P.splits = splits;
    gmi::gemm_launch(P, bn, a_mn, b_mn, epi, static_cast<cudaStream_t>(stream));
  });
}
