#!/usr/bin/env python3
"""Decoupled layout (serving GMI + trainer GMI) of a config file at several serving-partition sizes,
beside the single context: device-timed env-steps/s.
    python tools/exp_decoupled.py configs/hm_8192env_4gmi.cfg 16 24 32 40"""
import copy
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timed(cfg, iters=10):
    import torch
    from paper_2206_08482_b200.ppo import Trainer
    t = Trainer(cfg)
    for _ in range(3):
        t.iteration()
    upd = torch.cuda.ExternalStream(t.stream(-1))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(upd)
    for _ in range(iters):
        t.iteration_async()
    b.record(upd)
    st = t.synchronize()
    ms = a.elapsed_time(b) / iters
    t.close()
    return st.env_steps / (ms / 1e3), ms


def main():
    from paper_2206_08482_b200.ppo import PpoConfig
    base = PpoConfig.from_config_file(sys.argv[1])
    one = copy.deepcopy(base)
    one.num_envs //= max(1, base.num_gpus)  # one GPU's share of the job
    one.num_gpus, one.rank = 1, 0
    one.gmis_per_gpu, one.gmi_backend, one.sm_per_gmi = 1, 0, 0
    v, ms = timed(one)
    print(json.dumps({"layout": "single context", "value": v, "ms": ms}), flush=True)
    for sms in [int(x) for x in sys.argv[2:]]:
        d = copy.deepcopy(one)
        d.decoupled, d.gmi_backend, d.serving_sms = 1, 1, sms
        v2, ms2 = timed(d)
        print(json.dumps({"layout": f"decoupled serving {sms} SMs", "value": v2, "ms": ms2, "vs_single": v2 / v}),
              flush=True)


if __name__ == "__main__":
    main()
