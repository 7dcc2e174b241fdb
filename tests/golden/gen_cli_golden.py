#!/usr/bin/env python3
"""Generates tests/golden/cli_golden.json: stdout and exit code of the REFERENCE CLI
(proj/tools/gmux.cpp compiled unmodified by oracle/Makefile against oracle/shim/CLI11.hpp,
binary oracle/_ref/gmux_ref_cli) for every command line in CASES. tests/test_cli.py replays
the same command lines against paper_2206_08482_b200/bin/gmux and requires identical bytes.
Config files are the repo's own (configs/, tests/golden/cli/), relative to the repo root."""
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(ROOT, "oracle", "_ref", "gmux_ref_cli")

C = "configs/"
G = "tests/golden/cli/"
CASES = []
for fmt in ("text", "structured"):
    f = ["--format", fmt]
    CASES += [
        ["validate", "--topology", C + "sh_sweep_8gpu.cfg"] + f,
        ["validate", "--topology", C + "mig_serving.cfg"] + f,
        ["validate", "--topology", G + "invalid_shares.cfg"] + f,
        ["validate", "--topology", G + "mig.cfg"] + f,
        ["plan", "--topology", C + "sh_sweep_8gpu.cfg", "--mode", "sync_train"] + f,
        ["plan", "--topology", C + "sh_sweep_8gpu.cfg", "--mode", "serving"] + f,
        ["plan", "--topology", C + "decoupled_8gpu.cfg", "--mode", "async_train"] + f,
        ["plan", "--topology", G + "mig.cfg", "--mode", "serving"] + f,
        ["plan", "--mode", "serving", "--workload", "HM"] + f,
        ["plan", "--mode", "sync_train", "--workload", "FC", "--b1", "2.5"] + f,
        ["reduce", "--layout", "[[0,1],[2,3]]"] + f,
        ["reduce", "--layout", "[[0,1],[2,3]]", "--force-strategy", "har"] + f,
        ["reduce", "--layout", "[[0, 1, 2], [3]]"] + f,
        ["reduce", "--layout", "[[0,1],[2,3],[4,5],[6,7]]", "--topology", C + "sh_sweep_8gpu.cfg"] + f,
        ["reduce", "--layout", "[[0,1,2,3]]", "--payload", "1000", "--b1", "3"] + f,
        ["reduce", "--layout", "[[0,4],[1,5],[2,6],[3,7]]", "--workload", "SH", "--b2", "45"] + f,
        ["pipeline", "--topology", C + "decoupled_8gpu.cfg"] + f,
        ["pipeline", "--topology", C + "sh_sweep_8gpu.cfg", "--duration", "500"] + f,
        ["search"] + f,
        ["search", "--topology", C + "sh_sweep_8gpu.cfg"] + f,
        ["search", "--workload", "HM", "--sat-threshold", "0.5"] + f,
        ["search", "--topology", C + "mig_serving.cfg"] + f,
    ]
CASES += [
    ["reduce", "--layout", "[[0,1],[2,3]]", "--full-trace"],
    ["reduce", "--layout", "[[0,1,2],[3]]", "--force-strategy", "mrr"],  # MultiStreamError -> 1
    ["reduce", "--layout", "[[0,1],[1,2]]"],                             # duplicate id -> 2
    ["reduce", "--layout", "[[0,1]"],                                    # bad layout -> 2
    ["reduce"],                                                          # missing --layout -> 2
    ["validate"],                                                        # --topology required -> 2
    ["plan", "--mode", "bogus"],                                         # -> 2
    ["plan", "--topology", "no/such/file.cfg"],                          # -> 2
    ["plan", "--workload", "NOPE"],                                      # unknown benchmark -> 2
    ["plan", "--topology", C + "mig_serving.cfg", "--mode", "async_train"],  # 1 GPU: PlanError -> 1
    ["frobnicate"],                                                      # -> 2
    ["validate", "--format", "xml", "--topology", C + "mig_serving.cfg"],   # -> 2
]


def main():
    out = []
    for args in CASES:
        p = subprocess.run([REF] + args, cwd=ROOT, capture_output=True, text=True)
        out.append({"args": args, "rc": p.returncode, "stdout": p.stdout})
    path = os.path.join(ROOT, "tests", "golden", "cli_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"{len(out)} cases -> {path}")


if __name__ == "__main__":
    main()
