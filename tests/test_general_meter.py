"""The recursion's step meter (csrc/general_meter.cuh, dmm_general_steps): Machine::steps() and
GeneralStats::cleanup_retries of partition_general / integer_sort_general (partition.hpp:363-449),
w > m included, against the reference.

CPU: the meter's source compiled for the host (the same header the device kernel runs) against
the committed fixtures (tests/golden/make_general_steps.py) and, where oracle/_ref exists,
against fresh reference runs.  GPU: dmm_general_steps through the C ABI and run_algorithm's
report against the same fixtures.
"""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = os.path.join(ROOT, "tests", "golden", "general_steps.npz")
HOST_SRC = r"""
#include "general_meter.cuh"
#include <algorithm>
#include <vector>
extern "C" uint64_t gm_steps(uint32_t* g, uint32_t W, uint32_t M, uint64_t domain, uint32_t* retries) {
    std::vector<uint32_t> ws(dmmmeter::workspace_words(W, M));
    return dmmmeter::general_steps(g, W, M, domain, ws.data(), retries);
}
"""


def _fixture():
    z = np.load(FIX)
    keys = sorted({k.rsplit("_", 1)[0] for k in z.files})
    return {k: {f: z[f"{k}_{f}"] for f in ("in", "domain", "steps", "retries", "out")} for k in keys}


@pytest.fixture(scope="module")
def host_meter(tmp_path_factory):
    d = tmp_path_factory.mktemp("gm")
    src, so = d / "gm.cpp", d / "gm.so"
    src.write_text(HOST_SRC)
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I",
                    os.path.join(ROOT, "paper_1507_01391_b200", "csrc"), str(src), "-o", str(so)], check=True)
    lib = C.CDLL(str(so))
    lib.gm_steps.restype = C.c_uint64
    lib.gm_steps.argtypes = [C.POINTER(C.c_uint32), C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32)]

    def run(grid, domain):
        g = np.ascontiguousarray(grid, dtype=np.uint32).copy()
        rt = C.c_uint32()
        s = lib.gm_steps(g.ctypes.data_as(C.POINTER(C.c_uint32)), g.shape[0], g.shape[1], int(domain), C.byref(rt))
        return int(s), int(rt.value), g
    return run


def test_host_meter_matches_fixtures(host_meter):
    n = 0
    for shape, f in _fixture().items():
        for k in range(len(f["steps"])):
            s, rt, g = host_meter(f["in"][k], f["domain"][k])
            assert (s, rt) == (int(f["steps"][k]), int(f["retries"][k])), (shape, k)
            assert np.array_equal(g, f["out"][k]), (shape, k)
            n += 1
    assert n > 200


def test_fixture_covers_retries_and_data_dependence():
    fx = _fixture()
    assert sum(int((f["retries"] > 0).sum()) for f in fx.values()) >= 50
    assert len(set(fx["128x32"]["steps"].tolist())) > 3  # shearsort leaves: data-dependent


def test_host_meter_vs_reference_fresh(host_meter, ref):
    from oracle.oracle import ALGORITHMS
    rng = np.random.default_rng(7)
    for (w, m) in [(32, 16), (16, 8), (64, 8), (64, 32), (32, 4), (16, 2)]:
        for seed in range(100, 106):
            if m >= 8:
                g = ref.gen_instance(1, w, m, seed)
                _, _, rep = ref.run_algorithm(ALGORITHMS["partition_general"], g, seed)
                s, rt, _ = host_meter(g, w)
                assert (s, rt) == (rep["steps"], rep["cleanup_retries"]), (w, m, seed)
            domain = int(rng.choice([2, w, w * m]))
            g = rng.integers(0, domain, size=(w, m))
            st, out, rep = ref.integer_sort_general_steps(g, domain)
            assert st == 0
            s, rt, got = host_meter(g, domain)
            assert (s, rt) == (rep["steps"], rep["cleanup_retries"]), (w, m, seed, domain)
            assert np.array_equal(got, out.astype(np.uint32))


@pytest.mark.gpu
def test_device_meter_matches_fixtures():
    import torch
    from paper_1507_01391_b200 import instance
    for shape, f in _fixture().items():
        for dom in sorted(set(f["domain"].tolist())):
            sel = f["domain"] == dom
            grid = torch.from_numpy(f["in"][sel].astype(np.int64)).to(torch.int32).cuda()
            steps, retries = instance.general_steps(grid, int(dom))
            assert steps.cpu().numpy().astype(np.uint64).tolist() == f["steps"][sel].tolist(), (shape, dom)
            assert retries.cpu().numpy().astype(np.uint32).tolist() == f["retries"][sel].tolist(), (shape, dom)


@pytest.mark.gpu
def test_run_algorithm_reports_recursion_steps():
    from paper_1507_01391_b200 import instance
    fx = _fixture()
    for shape in ("32x16", "64x8", "128x32"):
        f = fx[shape]
        w, m = map(int, shape.split("x"))
        for k in range(len(f["steps"])):
            if int(f["domain"][k]) != w:
                continue
            inst = instance.Instance(kind="partition", w=w, m=m, seed=k,
                                     grid=f["in"][k].astype(np.uint64))
            o = instance.run_algorithm("partition_general", inst, seed=k)
            assert o.report.correct
            assert o.report.steps == int(f["steps"][k]) and o.report.work == int(f["steps"][k]) * w, (shape, k)
            assert o.report.cleanup_retries == int(f["retries"][k])


@pytest.mark.gpu
def test_device_meter_rejects_shapes():
    import torch
    from paper_1507_01391_b200 import dmm
    g = torch.zeros(1, 32, 8, dtype=torch.int32, device="cuda")
    steps = torch.empty(1, dtype=torch.int64, device="cuda")
    # 32 x 8: the leftover balancing group of 4 fails g^2 <= m (reference: ShapeViolation)
    assert dmm.lib().dmm_general_steps(g.data_ptr(), 32, 8, 1, 32, steps.data_ptr(), None, None) != 0
