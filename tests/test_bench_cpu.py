"""The bench's reference arm (the driver runs `bench.py --impl reference`) on the CPU: it must
print one JSON line with the reference's own run_algorithm throughput and exit 0."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    from oracle.oracle import Ref
    if not Ref.available():
        pytest.skip("oracle/_ref/libdmm_ref.so not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                        "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference" and line["metric"] == "keys/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and "correct" in line["cpu_baseline"]["sample"]


def test_reference_arm_names_the_b200_config():
    # the default (cfg3) reference arm times the same 32 x 128 tiles and prints the B200 arm's
    # config object; cfg2's arm names the 32 x 16 shape it actually times
    import bench
    assert bench.workload_config("cfg3")["m"] == 128 and bench.workload_config("cfg3")["w"] == 32
    assert bench.workload_config("cfg3")["keys_per_gpu"] == 1 << 32
    assert bench.workload_config("cfg2")["workload"].endswith("DMM_FLAG_EXT_PARTIAL_GROUPS]")


def test_verify_sort_full_on_host_tensors():
    # the bench's full-size check (per-tile sum / sum of squares / XOR, ascending, sampled exact
    # tiles) and its negative controls, on CPU tensors
    import numpy as np
    import torch

    import bench
    rng = np.random.default_rng(0)
    g = torch.from_numpy(rng.integers(0, 2 ** 32, size=(64, 32, 128), dtype=np.uint64).astype(np.uint32)
                         .view(np.int32))
    s = torch.from_numpy(np.sort(g.numpy().view(np.uint32).reshape(64, -1), axis=1).astype(np.uint32)
                         .view(np.int32).reshape(64, 32, 128))
    assert bench.verify_sort_full(g, s, 64)["ok"]
    assert not bench.verify_sort_full(g, torch.zeros_like(s), 64)["ok"]
    bad = s.clone()
    bad[3, 0, 0] = bad[3, 0, 1]  # a duplicated key replaces another: multiset broken
    r = bench.verify_sort_full(g, bad, 64)
    assert not (r["sum_sumsq"] and r["xor"])
    bad = s.clone()
    bad.view(64, -1)[7, :2] = bad.view(64, -1)[7, :2].flip(0)  # same multiset, out of order
    if int(s.view(64, -1)[7, 0]) != int(s.view(64, -1)[7, 1]):
        r = bench.verify_sort_full(g, bad, 64)
        assert r["sum_sumsq"] and r["xor"] and not r["ascending"]


def test_ncu_unit_normalisation():
    # ncu prints durations in whatever unit fits; traffic.json is always in microseconds
    import importlib.util
    spec = importlib.util.spec_from_file_location("ncs", os.path.join(ROOT, "profiles", "ncu_summarize.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    assert m.to_us("23.418048", "msecond") == pytest.approx(23418.048)
    assert m.to_us("193.248", "usecond") == pytest.approx(193.248)
    assert m.to_us("1,024", "nsecond") == pytest.approx(1.024)
    assert m.to_ghz("1.96", "Ghz") == pytest.approx(1.96)
    assert m.to_bytes("17.18", "Gbyte") == pytest.approx(17.18e9)
