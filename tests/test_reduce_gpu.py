"""K1 device reduction (libgmi gmi_reduce_device) parity.

fp64: bit-identical to the reference's execute() result on every golden layout, including
the BASELINE layouts at full gradient length (SHA-256 of the reference's result vector).
fp32: bit-identical to the literal ring restatement oracle/reduce_oracle.c.
"""
import ctypes as C

import numpy as np
import pytest

from golden_util import buffer_values, cases, f64_digest, layout_arrays, oracle_execute

pytestmark = pytest.mark.gpu
ALGO = {"MPR": 0, "MRR": 1, "HAR": 2}


def _device_reduce(algo, mpl, host_bufs, broadcast=False):
    import torch
    from paper_2206_08482_b200 import _lib

    dtype = 1 if host_bufs[0].dtype == np.float64 else 0
    dev = [torch.from_numpy(np.ascontiguousarray(b)).cuda() for b in host_bufs]
    out = torch.empty_like(dev[0])
    counts, ids = layout_arrays(mpl)
    ptrs = (C.c_void_p * len(dev))(*[t.data_ptr() for t in dev])
    stream = torch.cuda.current_stream().cuda_stream
    _lib.call("gmi_reduce_device", algo, len(mpl), (C.c_int * len(counts))(*counts),
              (C.c_int * len(ids))(*ids), ptrs, C.c_void_p(out.data_ptr()), out.numel(), dtype,
              1 if broadcast else 0, C.c_void_p(stream))
    torch.cuda.synchronize()
    return out.cpu().numpy(), [d.cpu().numpy() for d in dev]


def test_fp64_bit_identical_to_reference(cuda):
    n = 0
    for c in cases("execute"):
        rq, rs = c["request"], c["response"]
        if "error" in rs:
            continue
        ids = [i for l in rq["mpl"] for i in l]
        bufs = [buffer_values(rq.get("gen", "hash"), rq.get("seed", 0), i, rq["len"]) for i in ids]
        out, _ = _device_reduce(ALGO[rq["strategy"]], rq["mpl"], bufs)
        assert f64_digest(out) == rs["result_sha256"], rq
        n += 1
    assert n > 500


@pytest.mark.parametrize("mpl,algo", [([[0, 1, 2, 3]], 0), ([[0, 1], [2, 3], [4, 5]], 1),
                                      ([[0, 1, 2], [3, 4, 5]], 2), ([[0], [1, 2, 3], [4, 5]], 2),
                                      ([[i] for i in range(8)], 1), ([[0, 1, 2, 3, 4, 5, 6]], 0)])
@pytest.mark.parametrize("length", [1, 7, 1000, 296713])
def test_fp32_bit_identical_to_ring_oracle(cuda, mpl, algo, length):
    ids = [i for l in mpl for i in l]
    bufs = [(buffer_values("hash", 17, i, length) - 0.55).astype(np.float32) for i in ids]
    out, _ = _device_reduce(algo, mpl, bufs)
    ref = oracle_execute(algo, mpl, bufs)
    assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))


def test_broadcast_writes_every_gmi_buffer(cuda):
    mpl = [[0, 1], [2, 3]]
    bufs = [buffer_values("hash", 5, i, 777) for i in range(4)]
    out, after = _device_reduce(1, mpl, bufs, broadcast=True)
    for a in after:
        assert np.array_equal(a, out)


def test_mrr_rejects_oversubscribed_layout(cuda):
    from paper_2206_08482_b200 import gmux
    bufs = [buffer_values("hash", 5, i, 8) for i in range(6)]
    with pytest.raises(gmux.MultiStreamError, match="multiple streams per GPU: 3 rings over 2 GPUs"):
        _device_reduce(1, [[0, 1, 2], [3, 4, 5]], bufs)


def test_execute_dropin_matches_reference_cli_example(cuda):
    """gmux.execute (host buffers -> device -> host) on the README example."""
    from paper_2206_08482_b200 import gmux as G
    lay = G.GmiLayout([[0, 1], [2, 3]])
    bufs = [G.GradientBuffer(i, buffer_values("cli", 0, i, 30).tolist()) for i in lay.all_gmis()]
    ref = {c["request"]["strategy"]: c["response"] for c in cases("execute")[:3]}
    for s in G.Strategy:
        run = G.execute(s, lay, bufs, G.default_topology(2))
        assert run.result == ref[s.name]["result"]
        assert run.latency == ref[s.name]["latency"]


@pytest.mark.parametrize("mpl,algo", [([[0, 1, 2, 3, 4, 5, 6]], 0), ([[0, 1, 2, 3], [4, 5, 6, 7]], 2)])
def test_fp32_bit_identical_at_shadowhand_size(cuda, mpl, algo):
    """Largest BASELINE payload: ShadowHand-like 211:512:512:512:256:20 actor-critic, P = 1,535,765
    parameters (workload.hpp:95-100), folded over 7 GMIs of one GPU (cfg 5, MPR) and a 2 x 4
    layout (HAR); bit-identical to the ring oracle."""
    length = 1535765
    ids = [i for l in mpl for i in l]
    bufs = [(buffer_values("hash", 23, i, length) - 0.55).astype(np.float32) for i in ids]
    out, _ = _device_reduce(algo, mpl, bufs)
    ref = oracle_execute(algo, mpl, bufs)
    assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("mpl,algo", [([[0, 1, 2], [3, 4, 5]], 2), ([[0, 1], [2, 3], [4, 5]], 1),
                                      ([[0, 1, 2, 3]], 0)])
def test_allreduce_in_place_on_gmi_streams(cuda, mpl, algo):
    """gmi_allreduce: every GMI buffer ends with the total, bit-identical to the
    reference's execute() fold (fp64), with one CUDA stream per GMI ordered around the call
    (each GMI stream writes its buffer just before the call; the next kernel on every stream
    sees the total), and the run info equals the reference's modelled latencies."""
    import torch
    from paper_2206_08482_b200 import _lib

    ids = [i for l in mpl for i in l]
    n = 50_000
    host = [buffer_values("hash", 29, i, n) for i in ids]
    ref = oracle_execute(algo, mpl, host)
    streams = [torch.cuda.Stream() for _ in ids]
    dev = []
    for h, st in zip(host, streams):
        with torch.cuda.stream(st):  # the producer of each GMI's gradient runs on its own stream
            t = torch.empty(n, dtype=torch.float64, device="cuda")
            t.copy_(torch.from_numpy(h), non_blocking=False)
            dev.append(t)
    counts, cids = layout_arrays(mpl)
    ptrs = (C.c_void_p * len(dev))(*[t.data_ptr() for t in dev])
    sp = (C.c_void_p * len(streams))(*[st.cuda_stream for st in streams])
    run = _lib.ReductionInfo()
    _lib.call("gmi_allreduce", algo, len(mpl), (C.c_int * len(counts))(*counts), (C.c_int * len(cids))(*cids),
              ptrs, n, 1, sp, 25e9, 12.5e9, C.byref(run))
    outs = []
    for t, st in zip(dev, streams):
        with torch.cuda.stream(st):  # consumers on the GMI streams (no device-wide sync first)
            outs.append((t * 1.0).cpu().numpy())
    for o in outs:
        assert np.array_equal(o.view(np.uint64), ref.view(np.uint64))
    info = _lib.ReductionInfo()
    _lib.call("gmi_reduction_schedule", algo, len(mpl), (C.c_int * len(counts))(*counts),
              (C.c_int * len(cids))(*cids), n, 8.0, 25e9, 12.5e9, None, 0, C.byref(info))
    assert (run.latency, run.broadcast_latency, run.trace_len) == (info.latency, info.broadcast_latency, info.trace_len)
