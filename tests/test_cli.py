"""`gmux` CLI (paper_2206_08482_b200/bin/gmux, csrc/cli/gmux_cli.cpp) vs the reference CLI.

SURVEY §8f row 3: the reference's own proj/tools/gmux.cpp, compiled unmodified against a
CLI11 shim (oracle/shim/CLI11.hpp, oracle/Makefile), produced tests/golden/cli_golden.json
(tests/golden/gen_cli_golden.py): stdout and exit code for 56 command lines -- every
subcommand in text and structured (nlohmann JSON, key order of std::map) form, strategy
overrides, bandwidth overrides, config-file workloads, and the error paths of the exit-code
split (G:389-411). Ours must reproduce stdout byte for byte and the exit code exactly.
Host-only: runs on CPU."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2206_08482_b200", "bin", "gmux")
CASES = json.load(open(os.path.join(ROOT, "tests", "golden", "cli_golden.json")))


@pytest.mark.parametrize("case", CASES, ids=[" ".join(c["args"])[:80] for c in CASES])
def test_cli_matches_reference(case):
    assert os.path.exists(CLI), "build the CLI first (python -c 'import __graft_entry__ as g; g.build()')"
    p = subprocess.run([CLI] + case["args"], cwd=ROOT, capture_output=True, text=True, timeout=60)
    assert p.returncode == case["rc"], (p.returncode, p.stderr)
    assert p.stdout == case["stdout"]


def test_cli_reduce_on_device_flag_is_scoped():
    # B200 extension flags exist only on their subcommand, like the reference's options
    p = subprocess.run([CLI, "validate", "--device"], cwd=ROOT, capture_output=True, text=True, timeout=60)
    assert p.returncode == 2


@pytest.mark.gpu
def test_cli_reduce_on_device_matches_simulator(cuda):
    """`reduce --device`: the reduction data path (K1 fold) runs on the B200; the verified
    sum, the strategy and the trace are those of the host simulator."""
    args = ["reduce", "--layout", "[[0,1],[2,3]]", "--format", "structured"]
    host = json.loads(subprocess.run([CLI] + args, cwd=ROOT, capture_output=True, text=True).stdout)
    dev = json.loads(subprocess.run([CLI] + args + ["--device"], cwd=ROOT, capture_output=True, text=True).stdout)
    assert dev.pop("device") is True
    assert dev == host
