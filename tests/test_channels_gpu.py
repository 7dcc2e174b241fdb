"""Device experience channels (cuda/channels.cu, gmi_channel_run) against the reference's own
simulate_pipeline (channels.hpp:272-391): every golden pipeline case the reference produced
(tests/golden/ref_pipeline.json: AsyncDecoupled and colocated plans, k = 1 (UCC) and k > 1
(MCC), stack / slice batching, staggered agent phases) runs on the GPU over real payloads.

Checked exactly (fp64 bit-equal, integer-exact): PPS, TTOP, records produced / delivered, units
sent, batches emitted, bytes moved, transfer busy time, delivery / training makespans, records
per trainer, and every training batch (trainer, emit time, record ids). The payloads are
checked byte for byte: each trainer's receive buffers hold, in delivery order, exactly the
state / action / reward records of the ids its batches name."""
import numpy as np
import pytest

from golden_util import cases
from test_planner_golden import TPL, _plan_from, _topology, run

pytestmark = pytest.mark.gpu


def _pattern(torch, agent, n, nbytes, channel):
    # record r of agent a, channel c: bytes (a * 131 + r * 7 + c * 29 + j) mod 251
    r = torch.arange(n, dtype=torch.int64, device="cuda").unsqueeze(1)
    j = torch.arange(nbytes, dtype=torch.int64, device="cuda").unsqueeze(0)
    return ((agent * 131 + r * 7 + channel * 29 + j) % 251).to(torch.uint8)


def test_device_channels_match_reference_pipeline(cuda):
    import torch
    from paper_2206_08482_b200 import gmux as G
    n = 0
    for c in cases("pipeline"):
        rq, rs = c["request"], c["response"]
        wj = rq.get("workload", {})
        w = G.load_benchmark(wj.get("bench", "AT"))
        for k in ("state_bytes", "action_bytes", "reward_bytes"):
            if k in wj:
                setattr(w, k, wj[k])
        sizes = [w.state_bytes, w.action_bytes, w.reward_bytes]
        if any(b != int(b) or b <= 0 for b in sizes):
            continue  # the model allows fractional record sizes; payloads need whole bytes
        sizes = [int(b) for b in sizes]
        cj = rq.get("config", {})
        cfg = G.PipelineConfig(cj.get("compress_threshold", 8),
                               G.BatchMode.Slice if cj.get("batch_mode") == "slice" else G.BatchMode.Stack,
                               cj.get("target_batch", 32), cj.get("per_message_overhead", 1.0), cj.get("seed", 0))
        topo = _topology(rq.get("topology", {"default_gpus": 2}))
        try:
            plan = _plan_from(rq["plan"])
        except Exception:  # noqa: BLE001 -- plan construction errors are covered by the host tests
            continue
        agents = plan.gmis_with_role(G.Role.Agent)
        trainers = plan.gmis_with_role(G.Role.Trainer)
        cap = int(rq["duration"] // max(w.interaction_time(), 1e-12)) + 2
        total = cap * max(1, len(agents))
        abufs = [[_pattern(torch, a, cap, sizes[ch], ch) for a in range(len(agents))] for ch in range(3)]
        tbufs = [[torch.zeros((max(1, total), sizes[ch]), dtype=torch.uint8, device="cuda")
                  for _ in range(max(1, len(trainers)))] for ch in range(3)]
        aptr = [t.data_ptr() for ch in range(3) for t in abufs[ch]]
        tptr = [t.data_ptr() for ch in range(3) for t in tbufs[ch]]

        def go():
            return G.run_channels_device(w, plan, topo, cfg, rq["duration"], aptr, tptr, total)
        got = run(rs, go)
        torch.cuda.synchronize()
        if got is None:
            continue
        n += 1
        for k in ("pps", "ttop", "records_produced", "records_delivered", "units_sent", "batches_emitted",
                  "bytes_moved", "transfer_busy_time", "delivery_makespan", "training_makespan"):
            assert getattr(got, k) == rs[k], (k, rq)
        assert [[t, v] for t, v in sorted(got.trainer_records.items())] == rs["trainer_records"]
        assert [[b.trainer_gmi, b.emit_time, [[r.agent_gmi, r.seq] for r in b.records]] for b in got.batches] == \
            rs["batches"]
        # payloads: each trainer's receive buffers hold its batches' records in delivery order
        for ti, t in enumerate(trainers):
            keys = [(r.agent_gmi, r.seq) for b in got.batches if b.trainer_gmi == t for r in b.records]
            if not keys:
                continue
            ai = torch.tensor([agents.index(a) for a, _ in keys], device="cuda")
            sq = torch.tensor([s for _, s in keys], device="cuda")
            for ch in range(3):
                stacked = torch.stack(abufs[ch])  # [agents][cap][bytes]
                want = stacked[ai, sq]
                assert torch.equal(tbufs[ch][ti][:len(keys)], want), (t, ch, rq)
    assert n >= 40, n
