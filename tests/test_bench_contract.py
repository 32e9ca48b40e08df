"""CPU: the host-side pieces of bench.py the driver's contract rests on (no GPU, no timing):
workload shapes per BASELINE config and rank count, the shift sharding under torchrun, the
right-hand sides, and the guard on roofline.traffic."""
import argparse
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("name,ne,m,per,pattern", [("config0", 1000, 1, 1, 0), ("config1", 10000, 1, 8, 0),
                                                     ("config2", 50000, 1, 8, 0), ("config3", 500000, 4, 16, 0x11),
                                                     ("config4", 5000000, 4, 8, 0x10)])
@pytest.mark.parametrize("world", [1, 2, 8])
def test_workload_is_weakly_scaled_and_sharded_by_shift(name, ne, m, per, pattern, world):
    seen = []
    for rank in range(world):
        got_ne, got_m, mine, all_shifts, got_pattern = bench.workload(name, world, rank)
        assert (got_ne, got_m, got_pattern) == (ne, m, pattern)
        assert len(mine) == per and len(all_shifts) == per * world  # fixed work per GPU
        seen += mine
    assert sorted(seen) == sorted(all_shifts)  # every shift solved exactly once
    if name != "config0":
        assert min(all_shifts) == pytest.approx(10.0) and max(all_shifts) == pytest.approx(1e4)
        assert all(a < b for a, b in zip(all_shifts, all_shifts[1:]))


def test_default_workload_is_the_largest_single_gpu_config():
    sys_argv, sys.argv = sys.argv, ["bench.py"]
    try:
        args = bench.parse()
    finally:
        sys.argv = sys_argv
    assert args.workload == "config3" and args.gpus == 1 and args.warmup >= 3
    ne, m, mine, all_shifts, pattern = bench.workload(args.workload, 1, 0)
    cfg = bench.config_dict(args, ne, m, all_shifts, pattern, 1)
    assert "configs[3]" in cfg["workload"] and cfg["n"] == 1000000 and cfg["rhs"] == 4 and cfg["shifts_total"] == 16
    assert cfg["spai"] == "ls-A2-colscale" and "model" not in cfg


def test_rhs_blocks_are_unit_loads():
    B = bench.rhs_block(2000, 1)
    assert B.shape == (2000, 1) and B.sum() == 1.0 and B[1998, 0] == 1.0  # tip deflection dof
    B = bench.rhs_block(2000, 4)
    assert B.shape == (2000, 4) and np.all(B.sum(axis=0) == 1.0)
    assert [int(np.argmax(B[:, c])) for c in range(4)] == [498, 998, 1498, 1998]  # w at 25/50/75/100 % of L


def test_traffic_is_reported_only_for_the_captured_kernel_source(tmp_path, monkeypatch):
    got, note = bench.ncu_traffic("config1", 1000)
    assert got is None and "no ncu capture" in note
    summ = json.load(open(os.path.join(ROOT, "profiles", "r02_ncu_summary.json")))
    ent = summ["r02_cg_stream_config3"]
    got, note = bench.ncu_traffic("config3", 1000)
    if got is not None:  # the committed capture belongs to this tree's kernel
        assert got == pytest.approx(ent["dram_bytes_per_cg_iteration"] * 1000)
        assert got > 16 * (8 * 5e6 + 8 * 1e7 + 48 * 4e6) * 1000  # real traffic is above the algorithmic bytes
    else:
        assert "older kernel source" in note
    # a different kernel source must turn the number off, not leave it stale
    fake = tmp_path / "repo"
    (fake / "profiles").mkdir(parents=True)
    (fake / "paper_1606_01216_b200" / "csrc").mkdir(parents=True)
    for rel in ent["source_files"]:
        (fake / rel).write_text("// edited kernel\n")
    json.dump(summ, open(fake / "profiles" / "r02_ncu_summary.json", "w"))
    monkeypatch.setattr(bench, "ROOT", str(fake))
    got, note = bench.ncu_traffic("config3", 1000)
    assert got is None and "older kernel source" in note
