"""ctypes bindings for the parity checker (TEST INFRASTRUCTURE ONLY).

Two libraries:
  * ``Port`` -- the C restatement ``oracle/_build/libdmm_oracle.so`` (dmm_oracle.c);
  * ``Ref``  -- the unmodified reference compiled in place, ``oracle/_ref/libdmm_ref.so``.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl
reference`` legs import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libdmm_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdmm_ref.so")

# Algorithm enum, instance.hpp:148-157 (same order in dmm_oracle.h)
SORT_SHORT_WIDE, SORT_SQUARE, SORT_TALL = 0, 1, 2
PARTITION_SHORT_WIDE, PARTITION_SQUARE, PARTITION_GENERAL = 3, 4, 5
INTEGER_SORT_GENERAL, PERMUTE = 6, 7
ALGORITHMS = {
    "sort_short_wide": 0, "sort_square": 1, "sort_tall": 2, "partition_short_wide": 3,
    "partition_square": 4, "partition_general": 5, "integer_sort_general": 6, "permute": 7,
}
KIND_SORT, KIND_PARTITION, KIND_PERMUTE = 0, 1, 2

FLAG_EXT_PARTIAL_GROUPS = 1
FLAG_NONSTRICT = 2
FLAG_NO_ENFORCE_PRE = 4

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)


class GeneralStats(C.Structure):
    _fields_ = [("cleanup_retries", C.c_uint32), ("sorted", C.c_uint32)]


class PermuteReport(C.Structure):
    _fields_ = [
        ("iterations", C.c_uint32), ("fallback", C.c_uint32), ("used_packing", C.c_uint32),
        ("packed_width", C.c_uint32), ("threshold", C.c_uint64), ("random_words", C.c_uint64),
        ("cleanup_retries", C.c_uint32), ("n_hist", C.c_uint32), ("leftover_history", C.c_uint64 * 64),
    ]

    def as_dict(self):
        return {
            "iterations": self.iterations, "fallback": bool(self.fallback),
            "used_packing": bool(self.used_packing), "packed_width": self.packed_width,
            "threshold": self.threshold, "random_words": self.random_words,
            "cleanup_retries": self.cleanup_retries,
            "leftover_history": [int(self.leftover_history[i]) for i in range(self.n_hist)],
        }


class PortRunReport(C.Structure):
    _fields_ = [("correct", C.c_uint32), ("iterations", C.c_uint32), ("fallback", C.c_uint32),
                ("cleanup_retries", C.c_uint32)]


class RefRunReport(C.Structure):
    _fields_ = [("steps", C.c_uint64), ("work", C.c_uint64), ("conflicts", C.c_uint64),
                ("correct", C.c_uint32), ("iterations", C.c_uint32), ("fallback", C.c_uint32),
                ("cleanup_retries", C.c_uint32)]


def build(quiet: bool = True) -> None:
    """Build the checker libraries (oracle/Makefile); _ref only where /root/reference exists."""
    out = subprocess.run(["make", "-C", HERE, "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def _ptr(a, t=u64p):
    return a.ctypes.data_as(t)


class Port:
    """The C restatement (dmm_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.dmmo_gen_instance.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, u64p]
        L.dmmo_gen_sort_u32.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, u64p]
        L.dmmo_partition_general.argtypes = [C.c_uint32, C.c_uint32, u64p, C.c_uint32, C.POINTER(GeneralStats)]
        L.dmmo_integer_sort_general.argtypes = [C.c_uint32, C.c_uint32, u64p, C.c_uint64, C.c_uint32,
                                                C.POINTER(GeneralStats)]
        for f in ("dmmo_partition_square", "dmmo_partition_short_wide", "dmmo_sort_tall",
                  "dmmo_to_column_major", "dmmo_to_row_major"):
            getattr(L, f).argtypes = [C.c_uint32, C.c_uint32, u64p]
        L.dmmo_transpose_square.argtypes = [C.c_uint32, u64p]
        L.dmmo_sort_short_wide.argtypes = [C.c_uint32, C.c_uint32, u64p, C.c_int]
        L.dmmo_sort_square.argtypes = [C.c_uint32, C.c_uint32, u64p, C.c_int]
        L.dmmo_sort_wide_any.argtypes = [C.c_uint32, C.c_uint32, u64p, C.c_int]
        L.dmmo_permute.argtypes = [C.c_uint32, C.c_uint32, u64p, C.c_uint64, C.c_uint32, C.c_uint32, u64p,
                                   C.POINTER(PermuteReport), u32p]
        L.dmmo_general_sort_shape_ok.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32]
        L.dmmo_permute_threshold.argtypes = [C.c_uint32, C.c_uint32]
        L.dmmo_permute_threshold.restype = C.c_uint64
        L.dmmo_partition_params.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, u32p, u32p, u32p]
        L.dmmo_run_algorithm.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, u64p, C.c_uint32, u64p,
                                         C.POINTER(PortRunReport), C.POINTER(PermuteReport), u32p]
        L.dmmo_partition_general_batch.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, u32p, u32p, C.c_uint32,
                                                   C.POINTER(GeneralStats)]
        L.dmmo_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.dmmo_rng_next.argtypes = [C.c_void_p]
        L.dmmo_rng_next.restype = C.c_uint64
        L.dmmo_splitmix64.argtypes = [C.c_uint64]
        L.dmmo_splitmix64.restype = C.c_uint64

    # --- generators -----------------------------------------------------
    def gen_instance(self, kind: int, w: int, m: int, seed: int) -> np.ndarray:
        g = np.zeros(w * m, dtype=np.uint64)
        self.lib.dmmo_gen_instance(kind, w, m, seed, _ptr(g))
        return g.reshape(w, m)

    def gen_sort_u32(self, w: int, m: int, seed: int) -> np.ndarray:
        g = np.zeros(w * m, dtype=np.uint64)
        self.lib.dmmo_gen_sort_u32(w, m, seed, _ptr(g))
        return g.reshape(w, m)

    def mt19937_64(self, seed: int, n: int) -> list[int]:
        buf = C.create_string_buffer(312 * 8 + 16)
        self.lib.dmmo_rng_seed(buf, seed)
        return [self.lib.dmmo_rng_next(buf) for _ in range(n)]

    # --- algorithms -----------------------------------------------------
    def partition_general(self, grid, flags: int = 0):
        g = _u64(grid).copy()
        w, m = g.shape
        st = GeneralStats()
        s = self.lib.dmmo_partition_general(w, m, _ptr(g), flags, C.byref(st))
        return s, g, {"cleanup_retries": st.cleanup_retries, "sorted": bool(st.sorted)}

    def integer_sort_general(self, grid, domain: int, flags: int = 0):
        g = _u64(grid).copy()
        w, m = g.shape
        st = GeneralStats()
        s = self.lib.dmmo_integer_sort_general(w, m, _ptr(g), domain, flags, C.byref(st))
        return s, g, {"cleanup_retries": st.cleanup_retries, "sorted": bool(st.sorted)}

    def simple(self, name: str, grid, *extra):
        g = _u64(grid).copy()
        w, m = g.shape
        fn = getattr(self.lib, "dmmo_" + name)
        if name == "transpose_square":
            s = fn(w, _ptr(g))
        else:
            s = fn(w, m, _ptr(g), *extra)
        return s, g

    def permute(self, grid, seed: int, alpha: int = 4, iter_cap: int = 64):
        g = _u64(grid)
        w, m = g.shape
        out = np.zeros_like(g)
        rep = PermuteReport()
        shifts = np.zeros(w, dtype=np.uint32)
        s = self.lib.dmmo_permute(w, m, _ptr(g), seed, alpha, iter_cap, _ptr(out), C.byref(rep), _ptr(shifts, u32p))
        d = rep.as_dict()
        d["shifts"] = shifts.tolist()
        return s, out, d

    def general_sort_shape_ok(self, W: int, M: int, flags: int = 0) -> bool:
        return bool(self.lib.dmmo_general_sort_shape_ok(W, M, flags))

    def permute_threshold(self, w: int, m: int) -> int:
        return int(self.lib.dmmo_permute_threshold(w, m))

    def partition_params(self, W: int, M: int, flags: int = 0):
        r, d, s = C.c_uint32(), C.c_uint32(), C.c_uint32()
        st = self.lib.dmmo_partition_params(W, M, flags, C.byref(r), C.byref(d), C.byref(s))
        return st, (r.value, d.value, s.value)

    def partition_general_batch(self, inst: np.ndarray, flags: int = 0):
        inst = np.ascontiguousarray(inst, dtype=np.uint32)
        count, w, m = inst.shape
        out = np.empty_like(inst)
        st = (GeneralStats * count)()
        s = self.lib.dmmo_partition_general_batch(w, m, count, _ptr(inst, u32p), _ptr(out, u32p), flags, st)
        return s, out, np.array([[x.cleanup_retries, x.sorted] for x in st], dtype=np.uint32)


class Ref:
    """The unmodified reference, compiled in place (oracle/_ref/libdmm_ref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path + " (build with `make -C oracle ref` where /root/reference exists)")
        self.lib = C.CDLL(path)
        L = self.lib
        L.dmmr_gen_instance.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, u64p]
        L.dmmr_run_algorithm.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, u64p, C.c_int, u64p,
                                         C.POINTER(RefRunReport), C.POINTER(PermuteReport), u32p]
        L.dmmr_integer_sort_general.argtypes = [C.c_uint32, C.c_uint32, u64p, C.c_uint64, C.c_int, C.c_int, u32p,
                                                u32p, u64p, C.c_uint32, u32p]
        L.dmmr_partition_general.argtypes = [C.c_uint32, C.c_uint32, u64p, C.c_int, u32p, u32p]
        L.dmmr_integer_sort_general_steps.argtypes = [C.c_uint32, C.c_uint32, u64p, C.c_uint64, C.c_int, C.c_int,
                                                      u32p, u32p, u64p]
        L.dmmr_permute.argtypes = [C.c_uint32, C.c_uint32, u64p, C.c_uint64, C.c_uint32, C.c_uint32, u64p,
                                   C.POINTER(PermuteReport), u32p]
        L.dmmr_layout.argtypes = [C.c_int, C.c_uint32, C.c_uint32, u64p]
        L.dmmr_general_sort_shape_ok.argtypes = [C.c_uint64, C.c_uint64]
        L.dmmr_permute_threshold.argtypes = [C.c_uint32, C.c_uint32]
        L.dmmr_instance_to_text.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, u64p, C.c_char_p,
                                            C.c_uint64]
        L.dmmr_instance_to_text.restype = C.c_uint64
        L.dmmr_instance_from_text.argtypes = [C.c_char_p, u64p, u64p, C.c_uint64]
        L.dmmr_trace_text.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.c_char_p, C.c_uint64]
        L.dmmr_trace_text.restype = C.c_uint64
        L.dmmr_verify_trace_text.argtypes = [C.c_char_p]
        L.dmmr_verify_trace_text.restype = C.c_int64
        L.dmmr_offline_schedule.argtypes = [C.c_uint32, C.c_uint32, u32p, u32p, u32p, u32p]
        L.dmmr_schedule_to_text.argtypes = [u32p, u32p, C.c_uint32, C.c_char_p, C.c_uint64]
        L.dmmr_schedule_to_text.restype = C.c_uint64
        L.dmmr_permute_threshold.restype = C.c_uint64
        L.dmmr_cpu_baseline.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, u32p, u64p, C.c_uint64,
                                        C.c_uint32, C.POINTER(C.c_double), u64p]

    def gen_instance(self, kind: int, w: int, m: int, seed: int) -> np.ndarray:
        g = np.zeros(w * m, dtype=np.uint64)
        self.lib.dmmr_gen_instance(kind, w, m, seed, _ptr(g))
        return g.reshape(w, m)

    def instance_to_text(self, kind: int, w: int, m: int, seed: int, grid) -> str:
        g = np.ascontiguousarray(grid, dtype=np.uint64).reshape(-1)
        n = self.lib.dmmr_instance_to_text(kind, w, m, seed, _ptr(g), None, 0)
        buf = C.create_string_buffer(n)
        self.lib.dmmr_instance_to_text(kind, w, m, seed, _ptr(g), buf, n)
        return buf.raw[:n].decode()

    def offline_schedule(self, w: int, m: int, perm):
        """-> (status, rounds: list of lists of (src_bank, src_off, dst_bank, dst_off))"""
        p = np.ascontiguousarray(perm, dtype=np.uint32).reshape(-1)
        n = w * m
        moves = np.zeros(max(4 * n, 4), dtype=np.uint32)
        lens = np.zeros(max(n, 1), dtype=np.uint32)
        nr = C.c_uint32()
        s = self.lib.dmmr_offline_schedule(w, m, _ptr(p, u32p), _ptr(moves, u32p), _ptr(lens, u32p), C.byref(nr))
        rounds, k = [], 0
        for r in range(nr.value if s == 0 else 0):
            rounds.append([tuple(int(x) for x in moves[4 * j: 4 * j + 4]) for j in range(k, k + int(lens[r]))])
            k += int(lens[r])
        return s, rounds

    def trace_text(self, alg: int, w: int, m: int, seed: int) -> str:
        n = self.lib.dmmr_trace_text(alg, w, m, seed, None, 0)
        buf = C.create_string_buffer(max(n, 1))
        self.lib.dmmr_trace_text(alg, w, m, seed, buf, n)
        return buf.raw[:n].decode()

    def verify_trace_text(self, text: str) -> int:
        return int(self.lib.dmmr_verify_trace_text(text.encode()))

    def schedule_to_text(self, rounds) -> str:
        mv = np.array([x for r in rounds for x in r], dtype=np.uint32).reshape(-1)
        if mv.size == 0:
            mv = np.zeros(4, dtype=np.uint32)
        lens = np.array([len(r) for r in rounds] or [0], dtype=np.uint32)
        n = self.lib.dmmr_schedule_to_text(_ptr(mv, u32p), _ptr(lens, u32p), len(rounds), None, 0)
        buf = C.create_string_buffer(max(n, 1))
        self.lib.dmmr_schedule_to_text(_ptr(mv, u32p), _ptr(lens, u32p), len(rounds), buf, n)
        return buf.raw[:n].decode()

    def instance_from_text(self, text: str, cap: int = 1 << 16):
        """-> (status, (kind, w, m, seed), grid[:w*m])"""
        hdr = np.zeros(4, dtype=np.uint64)
        g = np.zeros(cap, dtype=np.uint64)
        s = self.lib.dmmr_instance_from_text(text.encode(), _ptr(hdr), _ptr(g), cap)
        k, w, m, sd = (int(x) for x in hdr)
        return s, (k, w, m, sd), g[: w * m] if s == 0 else None

    def run_algorithm(self, alg: int, grid, seed: int, strict: bool = True):
        g = _u64(grid)
        w, m = g.shape
        out = np.zeros_like(g)
        rep = RefRunReport()
        prep = PermuteReport()
        shifts = np.zeros(w, dtype=np.uint32)
        s = self.lib.dmmr_run_algorithm(alg, w, m, seed, _ptr(g), int(strict), _ptr(out), C.byref(rep),
                                        C.byref(prep), _ptr(shifts, u32p))
        r = {"steps": rep.steps, "conflicts": rep.conflicts, "correct": bool(rep.correct),
             "iterations": rep.iterations, "fallback": bool(rep.fallback), "cleanup_retries": rep.cleanup_retries}
        if alg == PERMUTE:
            r["pipeline"] = prep.as_dict()
            r["pipeline"]["shifts"] = shifts.tolist()
        return s, out, r

    def integer_sort_general(self, grid, domain: int, enforce_pre: bool = True, strict: bool = True,
                             probe_snaps: int = 0):
        g = _u64(grid).copy()
        w, m = g.shape
        cr, so, ns = C.c_uint32(), C.c_uint32(), C.c_uint32()
        snaps = np.zeros((max(probe_snaps, 1), w, m), dtype=np.uint64)
        s = self.lib.dmmr_integer_sort_general(w, m, _ptr(g), domain, int(enforce_pre), int(strict), C.byref(cr),
                                               C.byref(so), _ptr(snaps) if probe_snaps else None, probe_snaps,
                                               C.byref(ns))
        res = {"cleanup_retries": cr.value, "sorted": bool(so.value)}
        if probe_snaps:
            res["snapshots"] = snaps[: min(ns.value, probe_snaps)]
        return s, g, res

    def integer_sort_general_steps(self, grid, domain: int, enforce_pre: bool = False, strict: bool = False):
        """integer_sort_general on any keys < domain: (status, final grid, {steps, cleanup_retries, sorted})."""
        g = _u64(grid).copy()
        w, m = g.shape
        cr, so, st = C.c_uint32(), C.c_uint32(), C.c_uint64()
        s = self.lib.dmmr_integer_sort_general_steps(w, m, _ptr(g), domain, int(enforce_pre), int(strict),
                                                     C.byref(cr), C.byref(so), C.byref(st))
        return s, g, {"steps": st.value, "cleanup_retries": cr.value, "sorted": bool(so.value)}

    def partition_general(self, grid, strict: bool = True):
        g = _u64(grid).copy()
        w, m = g.shape
        cr, so = C.c_uint32(), C.c_uint32()
        s = self.lib.dmmr_partition_general(w, m, _ptr(g), int(strict), C.byref(cr), C.byref(so))
        return s, g, {"cleanup_retries": cr.value, "sorted": bool(so.value)}

    def permute(self, grid, seed: int, alpha: int = 4, iter_cap: int = 64):
        g = _u64(grid)
        w, m = g.shape
        out = np.zeros_like(g)
        rep = PermuteReport()
        shifts = np.zeros(w, dtype=np.uint32)
        s = self.lib.dmmr_permute(w, m, _ptr(g), seed, alpha, iter_cap, _ptr(out), C.byref(rep), _ptr(shifts, u32p))
        d = rep.as_dict()
        d["shifts"] = shifts.tolist()
        return s, out, d

    def layout(self, op: str, grid):
        g = _u64(grid).copy()
        w, m = g.shape
        s = self.lib.dmmr_layout({"transpose_square": 0, "to_column_major": 1, "to_row_major": 2}[op], w, m, _ptr(g))
        return s, g

    def general_sort_shape_ok(self, W: int, M: int) -> bool:
        return bool(self.lib.dmmr_general_sort_shape_ok(W, M))

    def permute_threshold(self, w: int, m: int) -> int:
        return int(self.lib.dmmr_permute_threshold(w, m))

    def cpu_baseline(self, alg: int, inst: np.ndarray, seeds=None, domain: int = 0, nthreads: int = 0):
        """Time the reference's run_algorithm over `inst` (count x w x m, u32) on nthreads host threads."""
        inst = np.ascontiguousarray(inst, dtype=np.uint32)
        count, w, m = inst.shape
        if nthreads <= 0:
            nthreads = os.cpu_count() or 1
        sd = None if seeds is None else np.ascontiguousarray(seeds, dtype=np.uint64)
        secs = C.c_double()
        good = C.c_uint64()
        s = self.lib.dmmr_cpu_baseline(alg, w, m, count, _ptr(inst, u32p), _ptr(sd) if sd is not None else None,
                                       domain, nthreads, C.byref(secs), C.byref(good))
        return s, secs.value, good.value
