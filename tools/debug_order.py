#!/usr/bin/env python3
"""Development check: does a preceding gmi_dev_gemm call change the trainer's (or the
oracle's) minibatch gradient? Prints the policy-head bias gradient from both."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from golden_util import PpoOracle, make_cfg, param_layout  # noqa: E402
from paper_2206_08482_b200 import _lib  # noqa: E402
from paper_2206_08482_b200.ppo import PpoConfig, Trainer  # noqa: E402


def gemm_first():
    M, N, K = 256, 128, 320
    A = (torch.rand(M, K) - 0.5).bfloat16().cuda()
    W = (torch.rand(N, K) - 0.5).bfloat16().cuda()
    out = torch.zeros(3, M, N, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _lib.call("gmi_dev_gemm", 0, 0, 2, M, N, K, C.c_void_p(A.data_ptr()), A.stride(0), C.c_void_p(W.data_ptr()),
              W.stride(0), C.c_void_p(out.data_ptr()), out.stride(1), C.c_void_p(0), C.c_void_p(0), 0, 3, 0,
              C.c_void_p(s))
    torch.cuda.synchronize()


def run():
    S, A, hidden = 60, 8, [256, 256, 256]
    dev = Trainer(PpoConfig(obs_dim=S, act_dim=A, hidden=hidden, num_envs=64))
    orc = PpoOracle(make_cfg(S, A, hidden, 64))
    B = 64 * 32 // 4
    rng = np.random.default_rng(S)
    X = rng.uniform(-1, 1, (B, S)).astype(np.float32)
    act = rng.standard_normal((B, A)).astype(np.float32)
    oldlp = (rng.standard_normal(B) - 3).astype(np.float32)
    adv = rng.standard_normal(B).astype(np.float32)
    ret = rng.standard_normal(B).astype(np.float32)
    g_dev = dev.minibatch_grad(X, act, oldlp, adv, ret)
    g_orc, _ = orc.minibatch(X, act, oldlp, adv, ret)
    t = param_layout(S, A, hidden)[(0, 3)]
    print("dev", np.array2string(g_dev[t["b"]:t["b"] + A], precision=3))
    print("orc", np.array2string(g_orc[t["b"]:t["b"] + A], precision=3), flush=True)
    part = dev.get("head_part").reshape(-1, 2 * A + 5)
    np.set_printoptions(linewidth=200, precision=3)
    print("records (db_mu cols)\n", part[:, :A])


if __name__ == "__main__":
    if sys.argv[1:] == ["gemm"]:
        gemm_first()
    if sys.argv[1:] == ["gemmtests"]:
        import test_gemm_gpu as tg
        for M, N, K, ldk, ws in [(128, 64, 64, 64, 0), (300, 256, 60, 64, 0), (1024, 128, 256, 256, 0),
                                 (4096, 256, 192, 192, 0), (384, 512, 128, 128, 0), (40000, 256, 256, 256, 1),
                                 (20000, 224, 64, 64, 1), (300, 128, 192, 192, 1)]:
            tg.test_forward_bias_elu(torch.device("cuda"), M, N, K, ldk, ws)
    run()
