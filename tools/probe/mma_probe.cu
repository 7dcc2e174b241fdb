// Micro-probe (development aid): time of a chain of tcgen05.mma (M=128, K=16 per instruction,
// bf16, SS operands) issued by one thread into one accumulator vs the same work split into two
// N-halves with separate (interleaved) accumulators. nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../../paper_2206_08482_b200/csrc/cuda/ptx.cuh"
using namespace gmi;

__global__ void probe(int n, int split, int nmma, int bmn, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc(&slot, 512);
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(smem), b = a + 16384;
    const int nn = split ? n / 2 : n;
    const uint32_t idesc = ptx::umma_idesc_bf16(128, nn, 0, bmn);
    long long t0 = clock64();
    for (int rep = 0; rep < 4; ++rep) {
      for (int i = 0; i < nmma; ++i) {
        const int k = i % 4;
        if (split) {
          for (int h = 0; h < 2; ++h)
            ptx::mma_bf16(tmem + h * nn, ptx::umma_desc_sw128(a + k * 32, 16, 1024),
                          ptx::umma_desc_sw128(b + h * nn * 128 + k * 32, 16, 1024), idesc, i > 0 ? 1u : 0u);
        } else {
          const uint64_t bd = bmn ? ptx::umma_desc_sw128(b + k * 2048, 8192, 1024) : ptx::umma_desc_sw128(b + k * 32, 16, 1024);
          ptx::mma_bf16(tmem, ptx::umma_desc_sw128(a + k * 32, 16, 1024), bd, idesc, i > 0 ? 1u : 0u);
        }
      }
      ptx::mma_commit(&bar);
      ptx::mbar_wait(&bar, rep & 1);
    }
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0) / 4;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc(tmem, 512);
}

int main(int argc, char** argv) {
  const int nm = argc > 1 ? atoi(argv[1]) : 16;
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int ns[] = {16, 32, 64, 128, 256};
  for (int blocks : {1, 148})
    for (int bmn = 0; bmn < 2; ++bmn)
    for (int n : ns)
      for (int split = 0; split < 2 - bmn; ++split) {
        if (split && n < 32) continue;
        probe<<<blocks, 128, 65536>>>(n, split, nm, bmn, d);
        cudaDeviceSynchronize();
        probe<<<blocks, 128, 65536>>>(n, split, nm, bmn, d);
        unsigned long long h[148];
        cudaMemcpy(h, d, blocks * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < blocks; ++i) avg += h[i];
        avg /= blocks;
        printf("B %s  blocks %3d  N %3d  %s  %d k-steps: %7.0f cycles (%5.1f per k-step)  err=%s\n", bmn ? "MN" : "K ", blocks, n,
               split ? "2 chains (N/2 each)" : "1 chain            ", nm, avg, avg / nm, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
