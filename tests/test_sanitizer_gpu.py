"""compute-sanitizer over small PPO iterations (tools/sanitize_run.py: SMALL 12:64:64:3 with 2
GMIs, the 3x256 bench shape at 128 envs, the single-rank peer exchange; eager + graph replay).

memcheck and synccheck must report 0 errors. racecheck must report no hazard outside one
documented pattern: the shared-memory operand tiles of rollout_kernel (cuda/rollout.cu) are
rewritten by the epilogue threads (next layer's activations, the head's mu staging, the next
observation) after the tile's last reader -- a tcgen05.mma -- has completed. That ordering runs
writer -> mbarrier arrive -> MMA issuer's wait -> tcgen05.mma -> tcgen05.commit (a hardware
mbarrier arrive) -> the next writer's wait, which racecheck cannot see (it tracks thread-issued
barriers only), so it reports the two generic-proxy writes as a WAW hazard.
"""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tool):
    cmd = ["compute-sanitizer", "--tool", tool, "--print-limit", "200", sys.executable,
           os.path.join(ROOT, "tools", "sanitize_run.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    for name in ("small ok", "at ok", "xchg ok"):
        assert name in out, out[-3000:]
    return out


@pytest.mark.parametrize("tool", ["memcheck", "synccheck"])
def test_sanitizer_clean(cuda, tool):
    out = _run(tool)
    assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]


def test_racecheck_only_documented_mma_ordered_tile_reuse(cuda):
    out = _run("racecheck")
    sites = re.findall(r"(?:Race reported between|and) (Write|Read) access at (.*?)\+0x", out)
    for kind, fn in sites:
        assert kind == "Write" and "rollout_kernel" in fn and "rollout_cluster" not in fn, (kind, fn)
