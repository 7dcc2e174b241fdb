"""the topology extension for B200 (reference enum stops at sm80,
topology.hpp:20). MPS shares on an sm100 GPU are realised as SM-partitioned green contexts in
whole 8-SM groups (cuDevSmResourceSplitByCount granularity, cuda.h:25262); validate_layout
flags shares below one group. MIG partitions on sm100 are checked against NVIDIA's published
B200 180 GB profile table (MIG mode is disabled on the pool's B200s, so the table cannot be
probed with `nvidia-smi mig -lgip` there). The sm70 / sm80 rules stay the reference's
(tests/test_planner_golden.py)."""
import os

from paper_2206_08482_b200 import gmux
from paper_2206_08482_b200.ppo import PpoConfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_green_context_sizes():
    assert gmux.green_sms(1.0) == 144
    assert gmux.green_sms(0.125) == 16
    assert gmux.green_sms(0.875) == 128
    assert gmux.green_sms(0.25) == 32
    assert gmux.green_sms(0.05) == 0
    assert gmux.green_sms(0.5, sm_units=132) == 64


def _b200(parts):
    t = gmux.Topology([gmux.GpuSpec(0, gmux.GpuArch.SM100, 8, 180.0)])
    t.partitions = parts
    return t


def test_sm100_share_below_one_group_is_a_violation():
    ok = _b200([gmux.mps_partition(0, 0, 0.125, 22.5), gmux.mps_partition(1, 0, 0.875, 157.5)])
    assert gmux.validate_layout(ok) == []
    bad = _b200([gmux.mps_partition(0, 0, 0.05, 9.0), gmux.mps_partition(1, 0, 0.95, 171.0)])
    v = gmux.validate_layout(bad)
    assert len(v) == 1 and v[0].gpu_id == 0 and "8-SM green-context group" in v[0].rule


def test_sm100_mig_profiles():
    """B200 MIG table (NVIDIA's 180 GB profiles): 7 usable compute slices, 8 memory slices;
    A100 profiles are not B200 profiles; sm80 keeps the reference table."""
    ok = [gmux.mig_partition(0, 0, "3g.90gb"), gmux.mig_partition(1, 0, "3g.90gb")]
    assert gmux.validate_layout(_b200(ok)) == []
    seven = [gmux.mig_partition(i, 0, "1g.23gb") for i in range(7)]
    assert gmux.validate_layout(_b200(seven)) == []
    v = gmux.validate_layout(_b200(seven + [gmux.mig_partition(7, 0, "1g.23gb")]))
    assert len(v) == 1 and "exceeds 7 usable units" in v[0].rule
    mem = [gmux.mig_partition(0, 0, "4g.90gb"), gmux.mig_partition(1, 0, "1g.45gb"),
           gmux.mig_partition(2, 0, "1g.45gb"), gmux.mig_partition(3, 0, "1g.23gb")]
    v = gmux.validate_layout(_b200(mem))
    assert len(v) == 1 and "exceeds 8 memory slices" in v[0].rule
    v = gmux.validate_layout(_b200([gmux.mig_partition(0, 0, "3g.20gb")]))
    assert len(v) == 1 and "not an allowed MIG profile" in v[0].rule
    a100 = gmux.Topology([gmux.GpuSpec(0, gmux.GpuArch.SM80, 8, 40.0)], [gmux.mig_partition(0, 0, "3g.20gb")])
    assert gmux.validate_layout(a100) == []


def test_decoupled_config_serving_share_matches_green_context():
    cfg = gmux.load_config(os.path.join(ROOT, "configs", "at_4096env_decoupled.cfg"))
    topo = gmux.topology_from_config(cfg)
    share = topo.partitions[0].sm_share
    assert gmux.green_sms(share) == PpoConfig.from_config_file(
        os.path.join(ROOT, "configs", "at_4096env_decoupled.cfg")).serving_sms == 16
