"""Experiment: how rollout and full-iteration times scale with the SMs of a green-context GMI
(premise check for the decoupled sim/agent + trainer layout)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_08482_b200.ppo import PpoConfig, Trainer

def timeit(fn, n=10):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
    res = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); res.append(time.perf_counter() - t0)
    res.sort(); return res[len(res)//2] * 1e3

out = {}
for sms in [int(x) for x in sys.argv[1].split(",")]:
    for nocl in ["0", "1"]:
        os.environ["GMI_ROLLOUT_NOCLUSTER"] = nocl
        kw = dict(gmi_backend=1, sm_per_gmi=sms) if sms < 148 else {}
        t = Trainer(PpoConfig(num_envs=4096, **kw))
        r = timeit(t.rollout)
        it = timeit(t.iteration, 6) if nocl == "0" else None
        out[f"{sms}sm_nocl{nocl}"] = dict(rollout_plus_value_ms=r, iteration_ms=it)
        print(sms, nocl, r, it, flush=True)
        t.close()
print(json.dumps(out))
