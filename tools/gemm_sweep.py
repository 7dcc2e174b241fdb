#!/usr/bin/env python3
"""Micro-benchmark of the tcgen05 GEMM (gmi_dev_gemm) on the MLP layer shapes: CUDA-event
time per launch and achieved TFLOP/s, streaming vs weight-stationary mode. Development aid
for DESIGN.md §6; prints one line per configuration."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2206_08482_b200 import _lib  # noqa: E402


def run(a_mn, b_mn, epi, M, N, K, ws, iters=50, splits=1):
    dev = torch.device("cuda")
    if epi == 1:  # dX: A = dPre [M][K] K-major, B = W [K][N] MN-major, aux = H [M][N]
        A = torch.randn(M, K, device=dev).bfloat16()
        B = (torch.randn(K, N, device=dev) / 16).bfloat16()
        aux = torch.randn(M, N, device=dev).bfloat16()
        out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        ldb = N
    elif epi == 0:
        A = torch.randn(M, K, device=dev).bfloat16()
        B = (torch.randn(N, K, device=dev) / 16).bfloat16()
        aux = None
        out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        ldb = K
    else:
        A = torch.randn(M, K, device=dev).bfloat16()
        B = (torch.randn(N, K, device=dev) / 16).bfloat16()
        aux = None
        out = torch.empty(splits, M, N, device=dev, dtype=torch.float32)
        ldb = K
    bias = torch.zeros(N, device=dev)
    side = torch.cuda.Stream()
    args = lambda s: (a_mn, b_mn, epi, M, N, K, C.c_void_p(A.data_ptr()), A.stride(0), C.c_void_p(B.data_ptr()),  # noqa
                      ldb, C.c_void_p(out.data_ptr()), N, C.c_void_p(bias.data_ptr()),
                      C.c_void_p(aux.data_ptr() if aux is not None else 0), N, splits, ws, C.c_void_p(s.cuda_stream))
    with torch.cuda.stream(side):
        for _ in range(3):
            _lib.call("gmi_dev_gemm", *args(side))
    torch.cuda.synchronize()
    # replay from a CUDA graph so host-side tensor-map encoding is not in the timed region
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for _ in range(iters):
            _lib.call("gmi_dev_gemm", *args(side))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    tf = 2.0 * M * N * K / (us * 1e-6) / 1e12
    print(f"epi={epi} M={M} N={N} K={K} ws={ws} splits={splits}: {us:8.2f} us  {tf:7.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    for M in (32768, 65536):
        for K in (64, 256):
            for ws in (0, 1):
                run(0, 0, 0, M, 256, K, ws)
        for ws in (0, 1):
            run(0, 1, 1, M, 256, 256, ws)
        run(0, 0, 2, M, 256, 256, 0)
    run(0, 0, 0, 4096, 256, 256, 0)
