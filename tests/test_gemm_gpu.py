"""tcgen05 GEMM parity against a plain PyTorch fp32 reference of the same op.

Operands are bf16 (the values the kernel sees exactly), so an fp32 torch matmul of the
upcast operands differs from the kernel only by accumulation order (fp32 outputs) plus
the final bf16 rounding (bf16 outputs).
"""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


def _gemm(a_mn, b_mn, epi, M, N, K, A, B, out, bias=None, aux=None, splits=1, ws=0):
    import torch
    from paper_2206_08482_b200 import _lib

    stream = torch.cuda.current_stream().cuda_stream
    _lib.call("gmi_dev_gemm", a_mn, b_mn, epi, M, N, K,
              C.c_void_p(A.data_ptr()), A.stride(0), C.c_void_p(B.data_ptr()), B.stride(0),
              C.c_void_p(out.data_ptr()), out.stride(0) if out.dim() == 2 else out.stride(1),
              C.c_void_p(bias.data_ptr() if bias is not None else 0),
              C.c_void_p(aux.data_ptr() if aux is not None else 0),
              aux.stride(0) if aux is not None else 0, splits, ws, C.c_void_p(stream))
    torch.cuda.synchronize()


def _elu(x):
    import torch
    return torch.where(x > 0, x, torch.expm1(x))


@pytest.mark.parametrize("M,N,K,ldk,ws", [(128, 64, 64, 64, 0), (300, 256, 60, 64, 0), (1024, 128, 256, 256, 0),
                                          (4096, 256, 192, 192, 0), (384, 512, 128, 128, 0),
                                          (40000, 256, 256, 256, 1), (20000, 224, 64, 64, 1), (300, 128, 192, 192, 1),
                                          # ws = 2: K <= 512 resident (one 128-column part of a wide layer)
                                          (20000, 128, 448, 448, 2), (5000, 96, 512, 512, 2), (300, 64, 320, 320, 2)])
def test_forward_bias_elu(cuda, M, N, K, ldk, ws):
    import torch
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N)
    A = torch.zeros(M, ldk, dtype=torch.bfloat16)
    A[:, :K] = (torch.rand(M, K, generator=g) * 2 - 1).bfloat16()
    W = torch.zeros(N, ldk, dtype=torch.bfloat16)
    W[:, :K] = ((torch.rand(N, K, generator=g) * 2 - 1) / K ** 0.5).bfloat16()
    bias = (torch.rand(N, generator=g) - 0.5).float()
    A, W, bias = A.to(cuda), W.to(cuda), bias.to(cuda)
    out = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device=cuda)
    _gemm(0, 0, 0, M, N, K, A, W, out, bias=bias, ws=ws)
    ref = _elu(A[:, :K].float() @ W[:, :K].float().T + bias)
    err = (out.float() - ref).abs().max().item()
    assert err <= 1e-2 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("splits", [1, 3])
def test_f32_split_k(cuda, splits):
    import torch
    M, N, K = 256, 128, 320
    g = torch.Generator(device="cpu").manual_seed(5 + splits)
    A = (torch.rand(M, K, generator=g) - 0.5).bfloat16().to(cuda)
    W = (torch.rand(N, K, generator=g) - 0.5).bfloat16().to(cuda)
    out = torch.zeros(splits, M, N, dtype=torch.float32, device=cuda)
    _gemm(0, 0, 2, M, N, K, A, W, out, splits=splits)
    ref = A.float() @ W.float().T
    got = out.sum(0)
    assert torch.allclose(got, ref, rtol=1e-4, atol=1e-4), (got - ref).abs().max().item()


@pytest.mark.parametrize("M,Nl,Kl,ws", [(512, 256, 192, 0), (33000, 256, 256, 1), (20000, 64, 224, 1),
                                        (20000, 416, 128, 2), (9000, 512, 96, 2)])
def test_dgrad_mn_major_weights(cuda, M, Nl, Kl, ws):
    """dH = (dPre @ W) * elu'(H): B operand is the [N_l x K_l] weight read MN-major."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(11)
    dpre = (torch.rand(M, Nl, generator=g) - 0.5).bfloat16().to(cuda)
    W = ((torch.rand(Nl, Kl, generator=g) - 0.5) / 8).bfloat16().to(cuda)
    H = _elu(torch.randn(M, Kl, generator=g)).bfloat16().to(cuda)
    out = torch.zeros(M, Kl, dtype=torch.bfloat16, device=cuda)
    # D[m][n] = sum_k dpre[m][k] * W[k][n]  -> B(n,k) = W[k][n], stored [K x rows]
    _gemm(0, 1, 1, M, Kl, Nl, dpre, W, out, aux=H, ws=ws)
    Hf = H.float()
    ref = (dpre.float() @ W.float()) * torch.where(Hf > 0, torch.ones_like(Hf), Hf + 1)
    err = (out.float() - ref).abs().max().item()
    assert err <= 1e-2 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("rows,splits", [(4096, 1), (4096, 4), (1000, 3)])
def test_wgrad_both_mn_major(cuda, rows, splits):
    """dW = dPre^T @ H with reduction over the minibatch rows (both operands MN-major)."""
    import torch
    Nl, Kl = 256, 128
    g = torch.Generator(device="cpu").manual_seed(rows + splits)
    dpre = (torch.rand(rows, Nl, generator=g) - 0.5).bfloat16().to(cuda)
    H = (torch.rand(rows, Kl, generator=g) - 0.5).bfloat16().to(cuda)
    out = torch.zeros(splits, Nl, Kl, dtype=torch.float32, device=cuda)
    # D[n][k] = sum_r dpre[r][n] * H[r][k]: A(m=n, k=r) = dpre[r][n], B(n=k, k=r) = H[r][k]
    _gemm(1, 1, 2, Nl, Kl, rows, dpre, H, out, splits=splits)
    ref = dpre.float().T @ H.float()
    got = out.sum(0)
    assert torch.allclose(got, ref, rtol=1e-4, atol=1e-3), (got - ref).abs().max().item()
