"""bench.py on CPU: the module imports, its defaults follow the contract (C5, the largest
single-GPU BASELINE configuration; W >= 3), and the sync interval default is per config."""
import sys

import bench


def test_bench_defaults(monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse()
    assert a.config == "c5" and a.gpus == 1 and a.warmup >= 3 and a.impl == "ours"
    assert a.sync_mode == "delta"


def test_cpu_topology_reports_cores():
    t = bench.cpu_topology()
    assert t["threads_available"] >= 1 and t["logical_cpus"] >= 1
