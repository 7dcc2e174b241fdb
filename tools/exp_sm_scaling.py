#!/usr/bin/env python3
"""How the iteration of one GMI scales with its green-context SM count (decoupled-layout sizing):
for each SM count, device-timed iterations and the rollout / update split from one instrumented
iteration.   python tools/exp_sm_scaling.py configs/hm_8192env_4gmi.cfg 144 128 112 96"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    path = sys.argv[1]
    for sms in [int(x) for x in sys.argv[2:]]:
        cfg = PpoConfig.from_config_file(path)
        cfg.gmis_per_gpu, cfg.gmi_backend, cfg.sm_per_gmi = 1, 1, sms
        t = Trainer(cfg)
        for _ in range(3):
            t.iteration()
        upd = torch.cuda.ExternalStream(t.stream(-1))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(upd)
        for _ in range(10):
            t.iteration_async()
        b.record(upd)
        st = t.synchronize()
        ms = a.elapsed_time(b) / 10
        t.set_instrument(True)
        t.iteration()
        t.iteration()
        prof = t.profile()
        roll = sum(prof[k]["ms"] for k in ("roll_gemm", "roll_head", "act_env", "val_gemm", "val_head", "gae"))
        upd_ms = sum(v["ms"] for k, v in prof.items() if k not in ("roll_gemm", "roll_head", "act_env", "val_gemm",
                                                                      "val_head", "gae"))
        print(json.dumps({"sms": sms, "ms_per_iteration": ms, "env_steps_per_s": st.env_steps / (ms / 1e3),
                          "instrumented_rollout_ms": roll, "instrumented_update_ms": upd_ms}), flush=True)
        t.close()


if __name__ == "__main__":
    main()
